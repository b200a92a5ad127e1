// FP64 FFT building blocks for sm_100a: in-register radix-2 DFTs and a two-stage
// warp-group FFT of length L = E*G (E complex values per thread, G threads per
// transform, G | 32, G <= E) with exactly one shared-memory exchange.
//
// Layouts of one length-L transform held by a group of G threads (thread g):
//   column layout : v[m]          = x[g + G*m],            m  = 0..E-1
//   row layout    : v[ri*G + k2]  = X[(g*R + ri) + E*k2],  ri = 0..R-1, k2 = 0..G-1, R = E/G
// fft_fwd maps column -> row layout (X_k = sum_j x_j W_L^{jk}, W_L = exp(-2 pi i/L));
// fft_inv maps row -> column layout (x_j = sum_k X_k W_L^{-jk}, unnormalised).
//
// Derivation (four-step / Cooley-Tukey with L = E*G): j = g + G m, k = k1 + E k2,
//   X_{k1+E k2} = sum_g W_G^{g k2} [ W_L^{g k1} sum_m x_{g+G m} W_E^{m k1} ].
#pragma once
#include <cuda_runtime.h>

#include "dft_consts.cuh"

namespace rsfde {

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 c_conj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 c_mulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}

// v * W_n^e with W_n = exp(-2 pi i / n), n | 64, e and n compile-time after unrolling
__device__ __forceinline__ double2 c_twc(double2 v, int e, int n) {
  e &= (n - 1);
  if (e == 0) return v;
  if (4 * e == n) return make_double2(v.y, -v.x);          // * (-i)
  if (2 * e == n) return make_double2(-v.x, -v.y);         // * (-1)
  if (4 * e == 3 * n) return make_double2(-v.y, v.x);      // * (+i)
  const int k = e * (64 / n);
  const double c = dftc::C64(k);
  const double s = -dftc::S64(k);
  return make_double2(fma(v.x, c, -v.y * s), fma(v.x, s, v.y * c));
}

__host__ __device__ __forceinline__ constexpr int ilog2c(int n) {
  int r = 0;
  while ((1 << r) < n) ++r;
  return r;
}
__host__ __device__ __forceinline__ constexpr int brevc(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}

// In-register forward DFT of N points a[0], a[S], ..., a[(N-1)S]; natural order in and out.
// Radix-2 decimation in time: the (free) bit-reversal renaming first, then log2 N butterfly stages
// a' = u + W w, b' = u - W w.  For a non-trivial twiddle the product is folded into FMAs:
// a' = fma(W, w, u) in 4 FMAs and b' = 2u - a' in 2, i.e. 6 FP64 operations per butterfly instead of
// 8 for a twiddle product followed by an add and a subtract (the FFT is FP64-pipe bound).
template <int N, int S = 1>
__device__ __forceinline__ void dft(double2* a) {
  if (N == 1) return;
  constexpr int BITS = ilog2c(N);
  {
    double2 t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] = a[brevc(i, BITS) * S];
#pragma unroll
    for (int i = 0; i < N; ++i) a[i * S] = t[i];
  }
#pragma unroll
  for (int h = 1; h < N; h <<= 1) {
#pragma unroll
    for (int i0 = 0; i0 < N; i0 += 2 * h) {
#pragma unroll
      for (int k = 0; k < h; ++k) {
        const double2 u = a[(i0 + k) * S];
        const double2 w = a[(i0 + k + h) * S];
        const int n2 = 2 * h;
        if (k == 0) {                       // W = 1
          a[(i0 + k) * S] = c_add(u, w);
          a[(i0 + k + h) * S] = c_sub(u, w);
        } else if (4 * k == n2) {           // W = -i: W w = (w.y, -w.x)
          a[(i0 + k) * S] = make_double2(u.x + w.y, u.y - w.x);
          a[(i0 + k + h) * S] = make_double2(u.x - w.y, u.y + w.x);
        } else {
          const int kk = k * (64 / n2);
          const double c = dftc::C64(kk), sn = -dftc::S64(kk);  // W = c + i sn = exp(-2 pi i k / n2)
          const double ax = fma(c, w.x, fma(-sn, w.y, u.x));
          const double ay = fma(c, w.y, fma(sn, w.x, u.y));
          a[(i0 + k) * S] = make_double2(ax, ay);
          a[(i0 + k + h) * S] = make_double2(fma(2.0, u.x, -ax), fma(2.0, u.y, -ay));
        }
      }
    }
  }
}

// inverse (unnormalised) in-register DFT: conj(DFT(conj(a)))
template <int N, int S = 1>
__device__ __forceinline__ void idft(double2* a) {
#pragma unroll
  for (int i = 0; i < N; ++i) a[i * S].y = -a[i * S].y;
  dft<N, S>(a);
#pragma unroll
  for (int i = 0; i < N; ++i) a[i * S].y = -a[i * S].y;
}

// v[k1] *= W_L^{+-g k1}, k1 = 0..E-1.  tw[k] = W_L^k (exact, host long double).
// W_L^{8 a g} is loaded exactly for every group of 8; inside a group the powers follow by
// recurrence (<= 7 complex products, relative error <= ~2e-15), keeping only 3 complex
// values live.
template <int E, bool INV>
__device__ __forceinline__ void twiddle_col(double2 (&v)[E], const double2* __restrict__ tw, int g, int L) {
  const double2 w1 = __ldg(tw + g);
  double2 w = w1;
  // (one flat loop: the nested group loop with a `break` made nvcc keep v[] in local memory for E = 16)
#pragma unroll
  for (int k1 = 1; k1 < E; ++k1) {
    if ((k1 & 7) == 0) w = __ldg(tw + ((k1 * g) & (L - 1)));
    else if (k1 > 1) w = c_mul(w, w1);
    v[k1] = INV ? c_mulc(v[k1], w) : c_mul(v[k1], w);
  }
}

// The same for E <= 16 with the seed W_L^{8 g} read from the second half of the table (tw[L + g] =
// W_L^{8 g}): consecutive g read consecutive addresses instead of one 128-byte line per lane
// (ncu, three-stage L = 4096 kernels: the seed loads were 20 % of the global L1 tag requests).
template <int E, bool INV>
__device__ __forceinline__ void twiddle_col_x(double2 (&v)[E], const double2* __restrict__ tw, int g, int L) {
  static_assert(E <= 16, "twiddle_col_x: one seed (k1 = 8)");
  const double2 w1 = __ldg(tw + g);
  double2 w = w1;
#pragma unroll
  for (int k1 = 1; k1 < E; ++k1) {
    if (k1 == 8) w = __ldg(tw + L + g);
    else if (k1 > 1) w = c_mul(w, w1);
    v[k1] = INV ? c_mulc(v[k1], w) : c_mul(v[k1], w);
  }
}

// The same with the exactly loaded powers W_L^{8 a g} (a = 0: W_L^g itself) taken from a small shared
// table tws[a * G + g] filled once per CTA (they depend on g only): a global load here sits at the head
// of the recurrence chain of every FFT of every tile.
template <int E, int G, bool INV>
__device__ __forceinline__ void twiddle_col_s(double2 (&v)[E], const double2* tws, int g) {
  const double2 w1 = tws[g];
  double2 w = w1;
#pragma unroll
  for (int k1 = 1; k1 < E; ++k1) {
    if ((k1 & 7) == 0) w = tws[(k1 >> 3) * G + g];
    else if (k1 > 1) w = c_mul(w, w1);
    v[k1] = INV ? c_mulc(v[k1], w) : c_mul(v[k1], w);
  }
}
// fill: tws[a * G + g] = W_L^{8 a g} (a >= 1), tws[g] = W_L^g
template <int E, int G>
__device__ __forceinline__ void twiddle_table_fill(double2* tws, const double2* __restrict__ tw, int tid, int nthreads) {
  constexpr int L = E * G;
  for (int i = tid; i < (E / 8) * G; i += nthreads) {
    const int a = i / G, g = i % G;
    tws[i] = __ldg(tw + (a == 0 ? g : ((8 * a * g) & (L - 1))));
  }
}

// XOR swizzle of the exchange buffer (row k1, column t) -> conflict-free 16-byte accesses
template <int E, int G>
__device__ __forceinline__ int xidx(int k1, int t) {
  constexpr int R = E / G;
  return (G >= 8) ? (k1 * G + (t ^ ((k1 / R) & 7))) : (k1 * G + t);
}

// Forward FFT, column layout in -> row layout out.  buf: L double2 of shared memory owned
// by this group.  Caller guarantees nobody else is reading buf (a __syncwarp precedes).
// (split in two halves so that a caller can wait for its exchange buffer between them: the first
// half touches registers only)
template <int E, int G>
__device__ __forceinline__ void fft_fwd_pre(double2 (&v)[E], int g, const double2* __restrict__ tw) {
  dft<E>(v);
  twiddle_col<E, false>(v, tw, g, E * G);
}
template <int E, int G>
__device__ __forceinline__ void fft_fwd_pre_s(double2 (&v)[E], int g, const double2* tws) {
  dft<E>(v);
  twiddle_col_s<E, G, false>(v, tws, g);
}
// the exchange alone (E == G: one row per thread), for callers that schedule the second DFT themselves
template <int E, int G>
__device__ __forceinline__ void fft_exchange(double2 (&v)[E], double2* buf, int g) {
  static_assert(E == G, "fft_exchange: square split");
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < E; ++k1) buf[xidx<E, G>(k1, g)] = v[k1];
  __syncwarp();
#pragma unroll
  for (int t = 0; t < G; ++t) v[t] = buf[xidx<E, G>(g, t)];
}
template <int E, int G>
__device__ __forceinline__ void fft_fwd_post(double2 (&v)[E], double2* buf, int g) {
  constexpr int R = E / G;
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < E; ++k1) buf[xidx<E, G>(k1, g)] = v[k1];
  __syncwarp();
#pragma unroll
  for (int ri = 0; ri < R; ++ri)
#pragma unroll
    for (int t = 0; t < G; ++t) v[ri * G + t] = buf[xidx<E, G>(g * R + ri, t)];
#pragma unroll
  for (int ri = 0; ri < R; ++ri) dft<G>(v + ri * G);
}
template <int E, int G>
__device__ __forceinline__ void fft_fwd(double2 (&v)[E], double2* buf, int g, const double2* __restrict__ tw) {
  constexpr int R = E / G;
  constexpr int L = E * G;
  dft<E>(v);
  twiddle_col<E, false>(v, tw, g, L);
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < E; ++k1) buf[xidx<E, G>(k1, g)] = v[k1];
  __syncwarp();
#pragma unroll
  for (int ri = 0; ri < R; ++ri)
#pragma unroll
    for (int t = 0; t < G; ++t) v[ri * G + t] = buf[xidx<E, G>(g * R + ri, t)];
#pragma unroll
  for (int ri = 0; ri < R; ++ri) dft<G>(v + ri * G);
}

// Inverse (unnormalised) FFT, row layout in -> column layout out.
template <int E, int G>
__device__ __forceinline__ void fft_inv(double2 (&v)[E], double2* buf, int g, const double2* __restrict__ tw) {
  constexpr int R = E / G;
  constexpr int L = E * G;
#pragma unroll
  for (int ri = 0; ri < R; ++ri) idft<G>(v + ri * G);
  __syncwarp();
#pragma unroll
  for (int ri = 0; ri < R; ++ri)
#pragma unroll
    for (int t = 0; t < G; ++t) buf[xidx<E, G>(g * R + ri, t)] = v[ri * G + t];
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < E; ++k1) v[k1] = buf[xidx<E, G>(k1, g)];
  twiddle_col<E, true>(v, tw, g, L);
  idft<E>(v);
}

}  // namespace rsfde
