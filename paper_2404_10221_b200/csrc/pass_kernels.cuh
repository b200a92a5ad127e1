// Per-axis pencil-pass kernels of the tau-preconditioned operator (FP64, sm_100a).
//
// One pass walks every pencil (line) of the grid along one axis.  Two pencils are packed
// into one complex sequence (real part = pencil p, imaginary part = pencil q) so that one
// complex FFT of length L = 2(n+1) serves both:
//
//  * Toeplitz product T x: circulant embedding of order L, zero-padded pair,
//    FFT -> multiply by the real even spectrum c^ (host, long double) -> inverse FFT.
//    Because c^ is real and even, IFFT(c^ FFT(x_p + i x_q)) = T x_p + i T x_q.
//  * DST-I S x: odd extension of the pair, one FFT, S x_p = -s Im Z / 2,
//    S x_q = s Re Z / 2 with s = sqrt(2/(n+1)) -- no partner exchange needed.
//  * DST of a zero-padded pair (needed for S H r = lambda^H S r, Lemma 3.5): from the
//    conv's forward FFT, D_p[k] = -(Im Z_k - Im Z_{L-k})/2, D_q[k] = (Re Z_k - Re Z_{L-k})/2.
//
// Operator pass ("oper"): inputs X, R -> outputs
//     Y = [S](H X + eta T R),  C = [S] H R           (SPECTRAL selects the [S])
// and on the last axis (LAST) only Y; with SPECTRAL the last pass also applies the
// d-level spectrum (Lambda^-1 of P_hat, P_alpha, P_alpha^{1/2} or H) and the inverse DST
// along the axis (DST . Lambda^-1 . DST fused).  Chained over the axes this computes
//     A v = H E v + S_alpha v                            (physical)
//     P_hat^{-1} A v = S Lambda_hat^{-1} S A v           (spectral; + inverse DSTs)
// using  S_d..S_1 (H_d..H_1 E v + sum_i eta_i prod_{l!=i} H_l T_i v)  =  the chain
//   a_1 = S_1(H_1 E v + eta_1 T_1 v), c_1 = S_1 H_1 v,
//   a_i = S_i(H_i a_{i-1} + eta_i T_i c_{i-1}), c_i = S_i H_i c_{i-1},
// which is exact because operators on different axes commute (Eq.(Salpha)).
#pragma once
#include <cuda_runtime.h>

#include "fft.cuh"
#include "kernels.cuh"

namespace rsfde {

constexpr int kThreads = 128;

struct PairInfo {
  long long base_p, base_q;  // offset of axis position j = 1 (memory index 0) of pencils p, q
  bool vp, vq;               // pencil exists and is not the zero pad column
  int cp[3], cq[3];          // 0-based coordinates of the pencils (entry [axis] unused)
};

__device__ __forceinline__ void coords_of(const PassParams& p, long long row_or_pencil, int* c) {
  const Geom& G = p.geo;
  c[0] = c[1] = c[2] = 0;
  if (p.contiguous) {
    // row o over axes 0..d-2
    long long o = row_or_pencil;
    if (G.d == 3) { c[0] = (int)(o / G.n[1]); c[1] = (int)(o % G.n[1]); }
    else if (G.d == 2) { c[0] = (int)o; }
  } else {
    const long long o = row_or_pencil / p.inner;
    const long long i = row_or_pencil % p.inner;
    if (G.d == 3) {
      if (p.axis == 0) { c[1] = (int)(i / G.P); c[2] = (int)(i % G.P); }
      else { c[0] = (int)o; c[2] = (int)i; }
    } else {  // d == 2, axis 0
      c[1] = (int)i;
    }
  }
}

__device__ __forceinline__ PairInfo pair_info(const PassParams& p, long long pair, bool active) {
  PairInfo pi;
  const Geom& G = p.geo;
  if (p.contiguous) {
    const long long rows = G.NP / G.P;
    const long long r0 = 2 * pair, r1 = 2 * pair + 1;
    pi.base_p = r0 * G.P;
    pi.base_q = r1 * G.P;
    pi.vp = active && r0 < rows;
    pi.vq = active && r1 < rows;
    coords_of(p, r0, pi.cp);
    coords_of(p, r1 < rows ? r1 : r0, pi.cq);
  } else {
    const long long pen = 2 * pair;  // even pencil index, inner is even
    const long long o = pen / p.inner, i = pen % p.inner;
    pi.base_p = o * (long long)p.n * p.inner + i;
    pi.base_q = pi.base_p + 1;
    coords_of(p, pen, pi.cp);
    coords_of(p, pen + 1, pi.cq);
    const int dl = G.d - 1;
    pi.vp = active && pi.cp[dl] < G.n[dl];
    pi.vq = active && pi.cq[dl] < G.n[dl];
  }
  if (!pi.vp) pi.base_p = 0;
  if (!pi.vq) pi.base_q = 0;
  return pi;
}

// value pair at axis position j (1..n); zero outside or for invalid pencils
__device__ __forceinline__ double2 ld_pair(const PassParams& p, const double* __restrict__ X, const PairInfo& pi,
                                           int j) {
  double2 r = make_double2(0.0, 0.0);
  if (j < 1 || j > p.n) return r;
  const long long off = (long long)(j - 1) * p.stride;
  if (!p.contiguous && pi.vq) {
    r = __ldg(reinterpret_cast<const double2*>(X + pi.base_p + off));
  } else {
    if (pi.vp) r.x = __ldg(X + pi.base_p + off);
    if (pi.vq) r.y = __ldg(X + pi.base_q + off);
  }
  return r;
}

__device__ __forceinline__ void st_pair(const PassParams& p, double* X, const PairInfo& pi, int j, double2 v) {
  if (j < 1 || j > p.n) return;
  const long long off = (long long)(j - 1) * p.stride;
  if (!p.contiguous && pi.vp && pi.vq) {
    *reinterpret_cast<double2*>(X + pi.base_p + off) = v;
  } else {
    if (pi.vp) X[pi.base_p + off] = v.x;
    if (pi.vq) X[pi.base_q + off] = v.y;
  }
}

// e(x_J, t) for the pencil with coordinates c (entry [axis] replaced by j-1)
__device__ __forceinline__ double e_at(const PassParams& p, const int* c, int j) {
  const ECoef& E = p.e;
  int cc[3] = {c[0], c[1], c[2]};
  cc[p.axis] = j - 1;
  const Geom& G = p.geo;
  if (E.kind == 2) {
    long long off = cc[0];
    if (G.d >= 2) off = off * G.n[1] + cc[1];
    if (G.d >= 3) off = off * G.n[2] + cc[2];
    return __ldg(E.grid + off);
  }
  double prod = 1.0, sum = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (i < G.d) {
      if (E.g[i]) prod *= __ldg(E.g[i] + cc[i]);
      if (E.k[i]) sum += __ldg(E.k[i] + cc[i]);
    }
  }
  return E.a + E.b * prod + sum;
}

// X channel at position j: input X, or (E o R) (scaled), or 0
__device__ __forceinline__ double2 xval(const PassParams& p, const PairInfo& pi, int j, double rs) {
  if (j < 1 || j > p.n) return make_double2(0.0, 0.0);
  if (p.xmode == X_INPUT) return ld_pair(p, p.X, pi, j);
  if (p.xmode == X_ZERO) return make_double2(0.0, 0.0);
  const double2 r = ld_pair(p, p.R, pi, j);
  return make_double2(pi.vp ? rs * r.x * e_at(p, pi.cp, j) : 0.0, pi.vq ? rs * r.y * e_at(p, pi.cq, j) : 0.0);
}

// Lambda of the preconditioner at spectral multi-index (c with [axis] = k-1)
__device__ __forceinline__ double spec_at(const PassParams& p, const int* c, int k) {
  const Spec& S = p.spec;
  const int d = p.geo.d;
  int kk[3] = {c[0], c[1], c[2]};
  kk[p.axis] = k - 1;
  double lamH = 1.0, lamP = S.ebar;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (i < d) {
      const double lh = __ldg(S.lamH[i] + kk[i]);
      lamH *= lh;
      lamP += S.eta[i] * __ldg(S.q[i] + kk[i]) / lh;
    }
  }
  switch (S.kind) {
    case SPEC_PHAT: return lamP * lamH;
    case SPEC_PALPHA: return lamP;
    case SPEC_PALPHA_SQRT: return sqrt(lamP);
    default: return lamH;
  }
}

// --- odd extension: v[m] (m < E/2) holds x at j = g + G m (< N); fill m >= E/2 with -x[L-j]
template <int E, int G>
__device__ __forceinline__ void odd_extend(double2 (&v)[E], double2* buf, int g) {
  constexpr int L = E * G, N = L / 2;
  __syncwarp();
#pragma unroll
  for (int m = 0; m < E / 2; ++m) buf[g + G * m] = v[m];
  __syncwarp();
#pragma unroll
  for (int m = E / 2; m < E; ++m) {
    const int j = g + G * m;
    const double2 t = (j == N) ? make_double2(0.0, 0.0) : buf[L - j];
    v[m] = make_double2(-t.x, -t.y);
  }
}

// row-layout index helper: k of register r = ri*G + k2
template <int E, int G>
__device__ __forceinline__ int row_k(int g, int r) {
  constexpr int R = E / G;
  return (g * R + r / G) + E * (r % G);
}

// DST . Lambda^{-1} . DST on the last axis, given the first FFT's row-layout output Z of the
// odd-extended pair.  Result (the second DST, scaled) left in row layout in v.
template <int E, int G>
__device__ __forceinline__ void scale_and_second_dst(const PassParams& p, const PairInfo& pi, double2 (&v)[E],
                                                     double2* buf, int g) {
  constexpr int L = E * G;
  const double hs = 0.5 * p.dst_scale;
  __syncwarp();
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int k = row_k<E, G>(g, r);
    double2 w = make_double2(0.0, 0.0);
    if (k >= 1 && k <= p.n) {
      const double yp = -v[r].y * hs, yq = v[r].x * hs;
      w.x = pi.vp ? yp / spec_at(p, pi.cp, k) : 0.0;
      w.y = pi.vq ? yq / spec_at(p, pi.cq, k) : 0.0;
    }
    buf[k] = w;
  }
  __syncwarp();
  constexpr int N = L / 2;
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int j = g + G * m;
    if (m < E / 2) {
      v[m] = buf[j];
    } else {
      const double2 t = (j == N) ? make_double2(0.0, 0.0) : buf[L - j];
      v[m] = make_double2(-t.x, -t.y);
    }
  }
  fft_fwd<E, G>(v, buf, g, p.tw);
}

// store the DST result held in row layout: S x_p = -s Im Z/2, S x_q = s Re Z/2
template <int E, int G>
__device__ __forceinline__ void store_dst_rows(const PassParams& p, double* out, const PairInfo& pi,
                                               const double2 (&v)[E], int g) {
  const double hs = 0.5 * p.dst_scale;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int k = row_k<E, G>(g, r);
    st_pair(p, out, pi, k, make_double2(-v[r].y * hs, v[r].x * hs));
  }
}

template <int E, int G, bool SPECTRAL, bool LAST>
__global__ void __launch_bounds__(kThreads) oper_pass_kernel(const PassParams p) {
  extern __shared__ double2 smem[];
  constexpr int L = E * G;
  constexpr int GROUPS = kThreads / G;
  const int grp = threadIdx.x / G;
  const int g = threadIdx.x % G;
  double2* buf = smem + grp * L;
  const long long pair = (long long)blockIdx.x * GROUPS + grp;
  const bool active = pair < p.npairs;
  const PairInfo pi = pair_info(p, active ? pair : 0, active);
  const double rs = p.rscale ? __ldg(p.rscale) : 1.0;

  double2 v[E];
  // 1. zero-padded R pair, column layout
#pragma unroll
  for (int m = 0; m < E; ++m) {
    if (m < E / 2) {
      const double2 r = ld_pair(p, p.R, pi, g + G * m);
      v[m] = make_double2(rs * r.x, rs * r.y);
    } else {
      v[m] = make_double2(0.0, 0.0);
    }
  }
  // 2. forward FFT (conv), row layout
  fft_fwd<E, G>(v, buf, g, p.tw);
  // 3. C = S H R = lambda^H . S R from the zero-padded spectrum (spectral, non-last)
  if (SPECTRAL && !LAST) {
    __syncwarp();
#pragma unroll
    for (int r = 0; r < E; ++r) buf[row_k<E, G>(g, r)] = v[r];
    __syncwarp();
    const double hs = 0.5 * p.dst_scale;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int k = row_k<E, G>(g, r);
      if (k >= 1 && k <= p.n) {
        const double2 zk = v[r], zm = buf[L - k];
        const double f = hs * __ldg(p.lamH + k - 1);
        st_pair(p, p.C, pi, k, make_double2(-(zk.y - zm.y) * f, (zk.x - zm.x) * f));
      }
    }
  }
  // 4. spectral multiply by c^/L and inverse FFT -> T R in column layout
#pragma unroll
  for (int r = 0; r < E; ++r) v[r] = c_scale(v[r], __ldg(p.chat + row_k<E, G>(g, r)));
  fft_inv<E, G>(v, buf, g, p.tw);
  // 5. y = H X + eta T R on positions j = g + G m, m < E/2 (physical C = H R here too)
#pragma unroll
  for (int m = 0; m < E / 2; ++m) {
    const int j = g + G * m;
    double2 y = make_double2(0.0, 0.0);
    if (j >= 1 && j <= p.n) {
      const double2 x0 = xval(p, pi, j, rs), xl = xval(p, pi, j - 1, rs), xr = xval(p, pi, j + 1, rs);
      y.x = fma(p.hc0, x0.x, fma(p.hc1, xl.x + xr.x, p.eta * v[m].x));
      y.y = fma(p.hc0, x0.y, fma(p.hc1, xl.y + xr.y, p.eta * v[m].y));
      if (!SPECTRAL) {
        if (LAST) {
          if (p.B) {
            const double2 b = ld_pair(p, p.B, pi, j);
            y.x = fma(p.ycoef, y.x, p.bcoef * b.x);
            y.y = fma(p.ycoef, y.y, p.bcoef * b.y);
          } else {
            y.x *= p.ycoef;
            y.y *= p.ycoef;
          }
        } else {
          const double2 r0 = ld_pair(p, p.R, pi, j), rl = ld_pair(p, p.R, pi, j - 1), rr = ld_pair(p, p.R, pi, j + 1);
          const double2 c = make_double2(rs * fma(p.hc0, r0.x, p.hc1 * (rl.x + rr.x)),
                                         rs * fma(p.hc0, r0.y, p.hc1 * (rl.y + rr.y)));
          st_pair(p, p.C, pi, j, c);
        }
        st_pair(p, p.Y, pi, j, y);
      }
    }
    v[m] = y;
  }
  if (!SPECTRAL) return;
  // 6. DST of y (odd extension), optionally Lambda^{-1} and the second DST
  odd_extend<E, G>(v, buf, g);
  fft_fwd<E, G>(v, buf, g, p.tw);
  if (LAST) scale_and_second_dst<E, G>(p, pi, v, buf, g);
  store_dst_rows<E, G>(p, p.Y, pi, v, g);
}

template <int E, int G, bool LAST>
__global__ void __launch_bounds__(kThreads) dst_pass_kernel(const PassParams p) {
  extern __shared__ double2 smem[];
  constexpr int L = E * G;
  constexpr int GROUPS = kThreads / G;
  const int grp = threadIdx.x / G;
  const int g = threadIdx.x % G;
  double2* buf = smem + grp * L;
  const long long pair = (long long)blockIdx.x * GROUPS + grp;
  const bool active = pair < p.npairs;
  const PairInfo pi = pair_info(p, active ? pair : 0, active);
  double2 v[E];
#pragma unroll
  for (int m = 0; m < E / 2; ++m) v[m] = ld_pair(p, p.X, pi, g + G * m);
  odd_extend<E, G>(v, buf, g);
  fft_fwd<E, G>(v, buf, g, p.tw);
  if (LAST) scale_and_second_dst<E, G>(p, pi, v, buf, g);
  store_dst_rows<E, G>(p, p.Y, pi, v, g);
}

// ----------------------------------------------------------------------------- launchers
template <int E, int G>
cudaError_t launch_oper_eg(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  constexpr int GROUPS = kThreads / G;
  const size_t smem = (size_t)GROUPS * E * G * sizeof(double2);
  const long long blocks = (p.npairs + GROUPS - 1) / GROUPS;
  void (*k)(PassParams);
  if (spectral) k = last ? oper_pass_kernel<E, G, true, true> : oper_pass_kernel<E, G, true, false>;
  else k = last ? oper_pass_kernel<E, G, false, true> : oper_pass_kernel<E, G, false, false>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  k<<<(unsigned)blocks, kThreads, smem, s>>>(p);
  return cudaGetLastError();
}

template <int E, int G>
cudaError_t launch_dst_eg(const PassParams& p, bool last, cudaStream_t s) {
  constexpr int GROUPS = kThreads / G;
  const size_t smem = (size_t)GROUPS * E * G * sizeof(double2);
  const long long blocks = (p.npairs + GROUPS - 1) / GROUPS;
  void (*k)(PassParams) = last ? dst_pass_kernel<E, G, true> : dst_pass_kernel<E, G, false>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  k<<<(unsigned)blocks, kThreads, smem, s>>>(p);
  return cudaGetLastError();
}

#define RSFDE_INSTANTIATE_L(E, G)                                                                      \
  template cudaError_t launch_oper_eg<E, G>(const PassParams&, bool, bool, cudaStream_t);             \
  template cudaError_t launch_dst_eg<E, G>(const PassParams&, bool, cudaStream_t);

}  // namespace rsfde
