// Three-stage FP64 FFT L = E * E * F held by G = E F threads (one pencil pair per CTA), E complex
// values per thread, two XOR-swizzled shared-memory exchanges, __syncthreads as the group barrier.
// Instances: E = 32, F = 2 / 4 (L = 2048 / 4096, the long pencils of BASELINE C3: throughput form),
// E = 16, F = 8 / 16 (L = 2048 / 4096 with 2-4x the threads per pair and half the registers: lower
// latency per pair) and E = 8, F = 8 (L = 512: the latency form for small grids such as C2, where a
// pass has fewer pencil pairs than the GPU has warps).  Requires F <= E, E % F == 0.
//
// Forward, natural input x_j (column layout: thread t holds x[t + G m], m < E):
//   j = t + G m,  t = a + F b,  k = k1 + E c + E^2 e
//   X_k = sum_{a} W_F^{a e} W_G^{a c} sum_{b} W_E^{b c} [ W_L^{t k1} sum_m W_E^{m k1} x_{t+Gm} ]
//   stage A: DFT-E over m, twiddle W_L^{t k1}         (thread t)
//   stage B: DFT-E over b, twiddle W_G^{a c}          (thread (k1, a) = (t/F, t%F))
//   stage C: DFT-F over a                              (thread (k1, a0): c = a0 (E/F) + s)
// Row layout: register r = s F + e holds X[k1 + E (a0 (E/F) + s) + E^2 e].
// The inverse (row -> column) runs the transposed pipeline on conjugated data.
#pragma once
#include "fft.cuh"

namespace rsfde {

template <int E_, int F>
struct Fft3 {
  static constexpr int E = E_, G = E * F, L = E * G, N = L / 2, CS = E / F;
  static_assert(F <= E && E % F == 0, "Fft3: F <= E, F | E");
  static constexpr int SWA = (8 / F > 1) ? (8 / F - 1) : 0;
  __device__ static __forceinline__ int ia(int k1, int tt) { return k1 * G + (tt ^ (F * (k1 & SWA))); }
  __device__ static __forceinline__ int ib(int k1, int a, int c) {
    const int row = k1 * F + a;
    return row * E + (c ^ ((row + (c >> 3)) & 7));
  }

  // twiddles W_L^{g k1}: E <= 16 forms read their seed from the table's second half (coalesced)
  __device__ static __forceinline__ void twid(double2 (&v)[E], const double2* __restrict__ tw, int g) {
    if constexpr (E <= 16) twiddle_col_x<E, false>(v, tw, g, L);
    else twiddle_col<E, false>(v, tw, g, L);
  }

  __device__ static __forceinline__ void fwd(double2 (&v)[E], double2* buf, int t, const double2* __restrict__ tw) {
    const int k1 = t / F, a = t % F;
    dft<E>(v);
    twid(v, tw, t);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < E; ++q) buf[ia(q, t)] = v[q];
    __syncthreads();
#pragma unroll
    for (int b = 0; b < E; ++b) v[b] = buf[ia(k1, a + F * b)];
    dft<E>(v);
    twid(v, tw, E * a);  // W_G^{a c} = W_L^{E a c}
    __syncthreads();
#pragma unroll
    for (int c = 0; c < E; ++c) buf[ib(k1, a, c)] = v[c];
    __syncthreads();
#pragma unroll
    for (int s = 0; s < CS; ++s)
#pragma unroll
      for (int a2 = 0; a2 < F; ++a2) v[s * F + a2] = buf[ib(k1, a2, a * CS + s)];
#pragma unroll
    for (int s = 0; s < CS; ++s) dft<F>(v + s * F);
  }

  __device__ static __forceinline__ void inv(double2 (&v)[E], double2* buf, int t, const double2* __restrict__ tw) {
    const int k1 = t / F, a = t % F;
#pragma unroll
    for (int i = 0; i < E; ++i) v[i].y = -v[i].y;
#pragma unroll
    for (int s = 0; s < CS; ++s) dft<F>(v + s * F);  // over e -> index a2
    __syncthreads();
#pragma unroll
    for (int s = 0; s < CS; ++s)
#pragma unroll
      for (int a2 = 0; a2 < F; ++a2) buf[ib(k1, a2, a * CS + s)] = v[s * F + a2];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < E; ++c) v[c] = buf[ib(k1, a, c)];
    twid(v, tw, E * a);
    dft<E>(v);  // over c -> index b (t' = a + F b)
    __syncthreads();
#pragma unroll
    for (int b = 0; b < E; ++b) buf[ia(k1, a + F * b)] = v[b];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < E; ++q) v[q] = buf[ia(q, t)];
    twid(v, tw, t);
    dft<E>(v);  // over k1 -> index m
#pragma unroll
    for (int i = 0; i < E; ++i) v[i].y = -v[i].y;
  }

  __host__ __device__ static __forceinline__ int rowk(int t, int r) {
    const int s = r / F, e = r % F;
    return (t / F) + E * ((t % F) * CS + s) + E * E * e;
  }
  // row register r holds an index k < N  <=>  e < F/2 (compile-time after unrolling)
  __host__ __device__ static constexpr bool lower(int r) { return (r % F) < F / 2; }
};

}  // namespace rsfde
