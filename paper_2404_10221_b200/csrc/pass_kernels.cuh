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
//
// Kernel structure (v2): every kernel is a loop over FFT *phases* with ONE FFT code body
// (small code -> no I-cache starvation, fewer live registers); per-pencil constants of
// e(x,t) and of the spectrum are computed once per pair; stencil neighbours come from the
// pair's shared-memory buffer instead of extra global loads.
#pragma once
#include <cuda_runtime.h>

#include "fft.cuh"
#include "fft3.cuh"
#include "kernels.cuh"

namespace rsfde {

constexpr int kThreads = 128;

enum PassMode { MODE_OPER_PHYS = 0, MODE_OPER_PHYS_LAST = 1, MODE_OPER_SPEC = 2, MODE_OPER_SPEC_LAST = 3,
                MODE_DST = 4, MODE_DST_LAST = 5 };

struct PairCtx {
  long long off_p, off_q;  // element offset of axis position j = 1 of pencils p, q
  long long pen_p, pen_q;  // pencil (row) index of p and q (for the per-pencil constants)
  bool vp, vq;             // pencil exists and is not the zero pad column
  bool vec2;               // strided axis with both pencils valid: one 16-byte access per position
};

// per-pencil constants of e(x,t) (separable / grid) and of the last-axis spectrum
struct PencilConsts {
  double eP_p, eP_q;       // prod_{i != axis} g_i(x_i) of each pencil (separable e)
  double eK_p, eK_q;       // sum_{i != axis} k_i(x_i)
  long long eoff_p, eoff_q;  // dense offset of position j = 1 (grid e)
  double cH_p, cH_q;       // prod_{i != axis} lambda^H_i(k_i)      (last-axis spectrum)
  double cP_p, cP_q;       // sum_{i != axis} eta_i q_i / lambda^H_i
};

// coordinates (0-based) of a pencil; entry [axis] = 0.  Pencil indices stay below 2^23 (every
// n_i + 1 <= 2048), so the index arithmetic is 32-bit (a 64-bit division costs ~10x more).
__device__ __forceinline__ void pencil_coords(const PassParams& p, long long idx, int& c0, int& c1, int& c2) {
  const Geom& G = p.geo;
  const unsigned u = (unsigned)idx;
  c0 = c1 = c2 = 0;
  if (p.contiguous) {
    if (G.d == 3) { c0 = (int)(u / (unsigned)G.n[1]); c1 = (int)(u % (unsigned)G.n[1]); }
    else if (G.d == 2) { c0 = (int)u; }
  } else {
    const unsigned inner = (unsigned)p.inner;
    const unsigned o = u / inner;
    const unsigned i = u - o * inner;
    if (G.d == 3) {
      if (p.axis == 0) { c1 = (int)(i / (unsigned)G.P); c2 = (int)(i % (unsigned)G.P); }
      else { c0 = (int)o; c2 = (int)i; }
    } else {
      c1 = (int)i;
    }
  }
}

__device__ __forceinline__ void pencil_consts(const PassParams& p, int c0, int c1, int c2, double& eP, double& eK,
                                              long long& eoff, double& cH, double& cP, bool want_e = true,
                                              bool want_spec = true) {
  const int c[3] = {c0 + p.coff[0], c1 + p.coff[1], c2 + p.coff[2]};  // global coordinates
  const Geom& G = p.geo;
  eP = 1.0; eK = 0.0; cH = 1.0; cP = 0.0; eoff = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (i < G.d && i != p.axis) {
      if (want_e && p.e.g[i]) eP *= __ldg(p.e.g[i] + c[i]);
      if (want_e && p.e.k[i]) eK += __ldg(p.e.k[i] + c[i]);
      if (want_spec && p.spec.lamH[i]) {
        cH *= __ldg(p.spec.lamH[i] + c[i]);
        cP += __ldg(p.spec.tq[i] + c[i]);
      }
    }
  }
  // dense offset of (c with c[axis] = 0) for a grid coefficient (unsharded grids only)
  long long off = c0;
  if (G.d >= 2) off = off * G.n[1] + c1;
  if (G.d >= 3) off = off * G.n[2] + c2;
  eoff = off;
}

// pencil inside the global grid on every non-pass axis?
__device__ __forceinline__ bool pencil_inside(const PassParams& p, int c0, int c1, int c2) {
  const int c[3] = {c0, c1, c2};
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (i < p.geo.d && i != p.axis) ok = ok && (c[i] + p.coff[i] < p.cext[i]);
  return ok;
}

__device__ __forceinline__ PairCtx make_pair(const PassParams& p, long long pair, bool active) {
  PairCtx pc;
  const Geom& G = p.geo;
  int a0, a1, a2, b0, b1, b2;
  if (p.contiguous) {
    const long long rows = G.NP / G.P;
    const long long r0 = 2 * pair, r1 = 2 * pair + 1;
    const long long rl = p.seg_lg ? (1ll << p.seg_lg) : (long long)G.P;  // pencil (row) length in memory
    pc.off_p = r0 * rl;
    pc.off_q = r1 * rl;
    pc.pen_p = r0;
    pc.pen_q = r1 < rows ? r1 : r0;
    pencil_coords(p, pc.pen_p, a0, a1, a2);
    pencil_coords(p, pc.pen_q, b0, b1, b2);
    pc.vp = active && r0 < rows && pencil_inside(p, a0, a1, a2);
    pc.vq = active && r1 < rows && pencil_inside(p, b0, b1, b2);
  } else {
    const long long pen = 2 * pair;  // even pencil index; inner is even
    const unsigned inner = (unsigned)p.inner;
    const unsigned o = (unsigned)pen / inner, i = (unsigned)pen - o * inner;
    pc.off_p = (long long)o * p.n * p.inner + i;
    pc.off_q = pc.off_p + 1;
    pc.pen_p = pen;
    pc.pen_q = pen + 1;
    pencil_coords(p, pen, a0, a1, a2);
    pencil_coords(p, pen + 1, b0, b1, b2);
    pc.vp = active && pencil_inside(p, a0, a1, a2);
    pc.vq = active && pencil_inside(p, b0, b1, b2);
  }
  if (!pc.vp) { pc.off_p = 0; pc.pen_p = 0; }
  if (!pc.vq) { pc.off_q = 0; pc.pen_q = 0; }
  pc.vec2 = !p.contiguous && pc.vp && pc.vq;
  return pc;
}

__device__ __forceinline__ PencilConsts make_consts(const PassParams& p, const PairCtx& pc, bool want_e = true,
                                                    bool want_spec = true) {
  PencilConsts k;
  int a0, a1, a2, b0, b1, b2;
  pencil_coords(p, pc.pen_p, a0, a1, a2);
  pencil_coords(p, pc.pen_q, b0, b1, b2);
  pencil_consts(p, a0, a1, a2, k.eP_p, k.eK_p, k.eoff_p, k.cH_p, k.cP_p, want_e, want_spec);
  pencil_consts(p, b0, b1, b2, k.eP_q, k.eK_q, k.eoff_q, k.cH_q, k.cP_q, want_e, want_spec);
  return k;
}

// offset of axis position j (1..n) from the pencil base: (j-1) stride, or the segmented contiguous layout
__device__ __forceinline__ long long pos_off(const PassParams& p, int j) {
  const int x = j - 1;
  if (p.seg_lg) return (long long)(x >> p.seg_lg) * p.seg_stride + (x & ((1 << p.seg_lg) - 1));
  return (long long)x * p.stride;
}

// value pair at axis position j (1..n); zero outside or for invalid pencils
__device__ __forceinline__ double2 ld_pair(const PassParams& p, const double* __restrict__ X, const PairCtx& pc,
                                           int j) {
  double2 r = make_double2(0.0, 0.0);
  if (j < 1 || j > p.n) return r;
  const long long off = pos_off(p, j);
  if (pc.vec2) {
    r = __ldg(reinterpret_cast<const double2*>(X + pc.off_p + off));
  } else {
    if (pc.vp) r.x = __ldg(X + pc.off_p + off);
    if (pc.vq) r.y = __ldg(X + pc.off_q + off);
  }
  return r;
}

__device__ __forceinline__ void st_pair(const PassParams& p, double* X, const PairCtx& pc, int j, double2 v) {
  if (j < 1 || j > p.n) return;
  const long long off = pos_off(p, j);
  if (pc.vec2) {
    *reinterpret_cast<double2*>(X + pc.off_p + off) = v;
  } else {
    if (pc.vp) X[pc.off_p + off] = v.x;
    if (pc.vq) X[pc.off_q + off] = v.y;
  }
}

// e(x, t) of both pencils at axis position j (1..n)
__device__ __forceinline__ double2 e_pair(const PassParams& p, const PairCtx& pc, const PencilConsts& kc, int j,
                                          double2 eab) {
  const ECoef& E = p.e;
  if (E.kind == 2) {
    // dense stride of the axis (d <= 3: at most two later axes)
    const long long st = (p.axis + 1 < p.geo.d ? (long long)p.geo.n[p.axis + 1] : 1ll) *
                         (p.axis + 2 < p.geo.d ? (long long)p.geo.n[p.axis + 2] : 1ll);
    const long long o = (long long)(j - 1) * st;
    return make_double2(pc.vp ? __ldg(E.grid + kc.eoff_p + o) : 0.0, pc.vq ? __ldg(E.grid + kc.eoff_q + o) : 0.0);
  }
  const double ga = E.g[p.axis] ? __ldg(E.g[p.axis] + j - 1) : 1.0;
  const double ka = E.k[p.axis] ? __ldg(E.k[p.axis] + j - 1) : 0.0;
  return make_double2(fma(eab.y * kc.eP_p, ga, eab.x) + (kc.eK_p + ka), fma(eab.y * kc.eP_q, ga, eab.x) + (kc.eK_q + ka));
}

// Lambda of both pencils at last-axis spectral index k (1..n)
__device__ __forceinline__ double2 spec_pair_v(const PassParams& p, const PencilConsts& kc, double lh, double tq);
__device__ __forceinline__ double2 spec_pair(const PassParams& p, const PencilConsts& kc, int k) {
  const Spec& S = p.spec;
  return spec_pair_v(p, kc, __ldg(S.lamH[p.axis] + k - 1), __ldg(S.tq[p.axis] + k - 1));
}
// the same from the table values lambda^H_k and eta q_k / lambda^H_k of the pass axis
__device__ __forceinline__ double2 spec_pair_v(const PassParams& p, const PencilConsts& kc, double lh, double tq) {
  const Spec& S = p.spec;
  const double lPp = S.ebar + kc.cP_p + tq, lPq = S.ebar + kc.cP_q + tq;
  switch (S.kind) {
    case SPEC_PHAT: return make_double2(lPp * (kc.cH_p * lh), lPq * (kc.cH_q * lh));
    case SPEC_PALPHA: return make_double2(lPp, lPq);
    case SPEC_PALPHA_SQRT: return make_double2(sqrt(lPp), sqrt(lPq));
    case SPEC_PALPHA_RSQRT: return make_double2(1.0 / sqrt(lPp), 1.0 / sqrt(lPq));
    case SPEC_HP_SQRT: return make_double2(kc.cH_p * lh * sqrt(lPp), kc.cH_q * lh * sqrt(lPq));
    default: return make_double2(kc.cH_p * lh, kc.cH_q * lh);
  }
}

// row-layout index k of register r = ri*G + k2
template <int E, int G>
__device__ __forceinline__ int row_k(int g, int r) {
  constexpr int R = E / G;
  return (g * R + r / G) + E * (r % G);
}

// ---------------------------------------------------------------------------------- FFT core
// flip the sign of x when msk has the sign bit set (integer XOR: no FP64 pipe use)
__device__ __forceinline__ double sgnx(double x, unsigned long long msk) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)msk);
}

// Forward (column -> row layout) or inverse (row -> column layout) FFT, E == G.
template <int E, int G>
__device__ __forceinline__ void fft_core(double2 (&v)[E], double2* buf, int g, const double2* __restrict__ tw,
                                         bool inv) {
  static_assert(E == G, "fft_core: square split only (E == G)");
  if (inv) fft_inv<E, G>(v, buf, g, tw);
  else fft_fwd<E, G>(v, buf, g, tw);
}

// general split (E = R G, R > 1): two DFT bodies (stage sizes differ)
template <int E, int G>
__device__ __forceinline__ void fft_core_rect(double2 (&v)[E], double2* buf, int g, const double2* __restrict__ tw,
                                              bool inv) {
  constexpr int R = E / G;
  constexpr int L = E * G;
  const unsigned long long msk = inv ? 0x8000000000000000ull : 0ull;
#pragma unroll
  for (int i = 0; i < E; ++i) v[i].y = sgnx(v[i].y, msk);
  if (inv) {
#pragma unroll
    for (int ri = 0; ri < R; ++ri) dft<G>(v + ri * G);
  } else {
    dft<E>(v);
  }
  // (conj of the intermediate cancels: keep the conjugated values through the exchange and
  //  use the forward twiddle on them, which equals conj(inverse twiddle of the true values))
  if (!inv) twiddle_col<E, false>(v, tw, g, L);
  __syncwarp();
  if (!inv) {
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) buf[xidx<E, G>(k1, g)] = v[k1];
    __syncwarp();
#pragma unroll
    for (int ri = 0; ri < R; ++ri)
#pragma unroll
      for (int t = 0; t < G; ++t) v[ri * G + t] = buf[xidx<E, G>(g * R + ri, t)];
  } else {
#pragma unroll
    for (int ri = 0; ri < R; ++ri)
#pragma unroll
      for (int t = 0; t < G; ++t) buf[xidx<E, G>(g * R + ri, t)] = v[ri * G + t];
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) v[k1] = buf[xidx<E, G>(k1, g)];
    twiddle_col<E, false>(v, tw, g, L);
  }
  if (inv) {
    dft<E>(v);
  } else {
#pragma unroll
    for (int ri = 0; ri < R; ++ri) dft<G>(v + ri * G);
  }
#pragma unroll
  for (int i = 0; i < E; ++i) v[i].y = sgnx(v[i].y, msk);
}

template <int E, int G>
__device__ __forceinline__ void fft_any(double2 (&v)[E], double2* buf, int g, const double2* __restrict__ tw,
                                        bool inv) {
  if constexpr (E == G) fft_core<E, G>(v, buf, g, tw, inv);
  else fft_core_rect<E, G>(v, buf, g, tw, inv);
}

// ---------------------------------------------------------------------------------- layouts
// Lay2: two-stage FFT, G <= 32 threads per pair, several pairs per CTA, warp-level sync.
template <int E_, int G_>
struct Lay2 {
  static constexpr int E = E_, G = G_, L = E * G, N = L / 2, GROUPS = kThreads / G, THREADS = kThreads;
  static constexpr int MINB = E >= 32 ? 3 : 4;
  __device__ static __forceinline__ void sync() { __syncwarp(); }
  __device__ static __forceinline__ int rowk(int g, int r) { return row_k<E, G>(g, r); }
  __host__ __device__ static constexpr bool lower(int r) { return (r % G) < G / 2; }
  __device__ static __forceinline__ int sw(int k) { return k; }  // row-layout staging index (see Lay3)
  static constexpr bool ROWTAB = false;
  __device__ static __forceinline__ void fft(double2 (&v)[E], double2* buf, int g, const double2* __restrict__ tw,
                                             bool inv) {
    fft_any<E, G>(v, buf, g, tw, inv);
  }
};
// Lay3: three-stage FFT (fft3.cuh), one pair per CTA of E F threads, CTA-level sync.
template <int E_, int F>
struct Lay3 {
  using FT = Fft3<E_, F>;
  static constexpr int E = FT::E, G = FT::G, L = FT::L, N = FT::N, GROUPS = 1, THREADS = FT::G;
  // E = 32: 3 / 6 CTAs per SM (L = 4096 / 2048, as measured in round 1); E <= 16: 128 registers
  // 256-thread form (L = 4096): 3 CTAs per SM at 85 registers (small spills) beat 2 at 128: C3 5.02 -> 4.86 ms
  // per CN step same-box (profiles/r02_c3_experiments.txt)
  static constexpr int MINB = E == 32 ? (F == 2 ? 6 : 3) : (THREADS == 256 ? 3 : (65536 / 128) / THREADS);
  __device__ static __forceinline__ void sync() { __syncthreads(); }
  __device__ static __forceinline__ int rowk(int t, int r) { return FT::rowk(t, r); }
  __host__ __device__ static constexpr bool lower(int r) { return FT::lower(r); }
  // Row-layout staging index.  The 8 lanes of a quarter-warp hold k = k1 + (E CS) a + ... with the same
  // k1 and consecutive a: unswizzled, their 16-byte values fall into one bank group (ncu: 32 wavefronts
  // per request against 4 ideal).  XOR the bank-group bits with a's low bits; column-order readers
  // (8 consecutive j) see a permutation inside their aligned group of 8.
  static constexpr int SWSH = ilog2c(E * (E / F));
  static constexpr bool ROWTAB = E == 16 && F == 16;  // PassParams::chat_rl / lamH_rl / tq_rl are in this layout
  __device__ static __forceinline__ int sw(int k) { return F >= 8 ? (k ^ ((k >> SWSH) & 7)) : k; }
  __device__ static __forceinline__ void fft(double2 (&v)[E], double2* buf, int t, const double2* __restrict__ tw,
                                             bool inv) {
    if (inv) FT::inv(v, buf, t, tw);
    else FT::fwd(v, buf, t, tw);
  }
};

// column layout v[m] (m < E/2) holds x at j = g + G m (< N): fill the odd extension m >= E/2
template <class T>
__device__ __forceinline__ void odd_extend(double2 (&v)[T::E], double2* buf, int g) {
  constexpr int E = T::E, G = T::G, L = T::L, N = T::N;
  T::sync();
#pragma unroll
  for (int m = 0; m < E / 2; ++m) buf[g + G * m] = v[m];
  T::sync();
#pragma unroll
  for (int m = E / 2; m < E; ++m) {
    const int j = g + G * m;
    const double2 t = (j == N) ? make_double2(0.0, 0.0) : buf[L - j];
    v[m] = make_double2(-t.x, -t.y);
  }
}

// The same odd extension through warp shuffles (groups of G <= 32 lanes, Lay2 layouts): the mirror
// L - j of j = g + G m is (G - g) + G (E - 1 - m) for g > 0 -- lane G - g of the group, register
// E - 1 - m -- and G (E - m) for g = 0 (the lane's own register E - m; j = N is the zero).  No pair
// buffer, so a tile whose staged outputs are still being copied out by the store warps does not wait
// here, and half the shared-memory traffic of the buffer version (64 SHFL vs 32 16-byte accesses).
template <class T>
__device__ __forceinline__ void odd_extend_shfl(double2 (&v)[T::E], int g) {
  constexpr int E = T::E, G = T::G;
  static_assert(G <= 32, "odd_extend_shfl: one FFT group per (part of a) warp");
  const int src = (G - g) & (G - 1);
#pragma unroll
  for (int m = E / 2; m < E; ++m) {
    const double2 a = v[E - 1 - m];
    double2 t;
    t.x = __shfl_sync(0xffffffffu, a.x, src, G);
    t.y = __shfl_sync(0xffffffffu, a.y, src, G);
    if (g == 0) t = (m == E / 2) ? make_double2(0.0, 0.0) : v[E - m];
    v[m] = make_double2(-t.x, -t.y);
  }
}

// ---------------------------------------------------------------------------------- the kernel
// Each group of G threads processes one pencil pair; the grid covers all pairs.  (A persistent
// grid -- with L2 prefetch, or with cp.async double buffering of the next pair -- was measured
// slower on B200: groups drift apart, the 16-byte row pieces of neighbouring pairs stop sharing
// L2 sectors in time and DRAM reads grow 2.7x.)
template <class T, int MODE>
__global__ void __launch_bounds__(T::THREADS, T::MINB) pass_kernel(const PassParams p) {
  extern __shared__ double2 smem[];
  if (skip_launch(p.skip)) return;  // speculative launch after convergence (uniform over the grid)
  constexpr int E = T::E, G = T::G, L = T::L, N = T::N, GROUPS = T::GROUPS;
  constexpr bool OPER = MODE <= MODE_OPER_SPEC_LAST;
  constexpr bool SPECTRAL = MODE == MODE_OPER_SPEC || MODE == MODE_OPER_SPEC_LAST || MODE >= MODE_DST;
  constexpr bool LAST = MODE == MODE_OPER_PHYS_LAST || MODE == MODE_OPER_SPEC_LAST || MODE == MODE_DST_LAST;
  const int grp = threadIdx.x / G;
  const int g = threadIdx.x % G;
  double2* buf = smem + grp * L;
  const double rs = p.rscale ? __ldg(p.rscale) : 1.0;  // lazy basis normalisation of the input
  const double hs = 0.5 * p.dst_scale;
  const bool rl = T::ROWTAB && p.chat_rl != nullptr;  // spectral tables read in row layout (coalesced)
  {
    const long long pair = (long long)blockIdx.x * GROUPS + grp;
    const bool active = pair < p.npairs;
    const PairCtx pc = make_pair(p, active ? pair : 0, active);

    double2 v[E];
    // ---- phase-0 input
    if (OPER) {
      // zero-padded R pair (the Toeplitz convolution input)
#pragma unroll
      for (int m = 0; m < E; ++m) {
        if (m < E / 2) {
          const double2 r = ld_pair(p, p.R, pc, g + G * m);
          v[m] = make_double2(rs * r.x, rs * r.y);
        } else {
          v[m] = make_double2(0.0, 0.0);
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < E / 2; ++m) v[m] = c_scale(ld_pair(p, p.X, pc, g + G * m), rs);
      odd_extend<T>(v, buf, g);
    }

    // phases: OPER: 0 conv-fwd, 1 conv-inv, 2 dst(y) [, 3 second dst]; DST: 2 dst [, 3 second dst]
    constexpr int first = OPER ? 0 : 2;
    constexpr int last_phase = OPER && !SPECTRAL ? 1 : (LAST ? 3 : 2);
    // one rolled phase loop: one copy of each FFT body (smaller code, fewer live registers)
#pragma unroll 1
    for (int ph = first; ph <= last_phase; ++ph) {
      T::fft(v, buf, g, p.tw, ph == 1);
      if (ph == 0) {
        // conv forward done (row layout).  C = S H R = s lambda^H D(R) (spectral, non-last)
        if (SPECTRAL && !LAST) {
          T::sync();
#pragma unroll
          for (int r = 0; r < E; ++r) buf[T::sw(T::rowk(g, r))] = v[r];
          T::sync();
#pragma unroll
          for (int r = 0; r < E; ++r) {
            if (!T::lower(r)) continue;  // k >= N (compile-time in row layout)
            const int k = T::rowk(g, r);
            if (k >= 1) {
              const double2 zk = v[r], zm = buf[T::sw(L - k)];
              const double f = hs * (rl ? __ldg(p.lamH_rl + r * G + g) : __ldg(p.lamH + k - 1));
              st_pair(p, p.C, pc, k, make_double2(-(zk.y - zm.y) * f, (zk.x - zm.x) * f));
            }
          }
        }
#pragma unroll
        for (int r = 0; r < E; ++r)
          v[r] = c_scale(v[r], rl ? __ldg(p.chat_rl + r * G + g) : __ldg(p.chat + T::rowk(g, r)));
      } else if (ph == 1) {
        // conv inverse done: column layout, T R at j = g + G m (m < E/2).
        // X channel at j, neighbours through the shared buffer
        const PencilConsts kc = (p.xmode == X_E_TIMES_R) ? make_consts(p, pc) : PencilConsts{};
        const double2 eab = e_ab(p.e);
        T::sync();
#pragma unroll
        for (int m = 0; m < E / 2; ++m) {
          const int j = g + G * m;
          double2 x = make_double2(0.0, 0.0);
          if (j >= 1 && j <= p.n) {
            if (p.xmode == X_INPUT) {
              x = ld_pair(p, p.X, pc, j);
            } else if (p.xmode == X_E_TIMES_R) {
              const double2 r = ld_pair(p, p.R, pc, j);
              const double2 e = e_pair(p, pc, kc, j, eab);
              x = make_double2(rs * r.x * e.x, rs * r.y * e.y);
            }
          }
          buf[j] = x;
        }
        if (g == 0) buf[N] = make_double2(0.0, 0.0);
        T::sync();
#pragma unroll
        for (int m = 0; m < E / 2; ++m) {
          const int j = g + G * m;
          double2 y = make_double2(0.0, 0.0);
          if (j >= 1 && j <= p.n) {
            const double2 xl = buf[j - 1], x0 = buf[j], xn = buf[j + 1];
            y.x = fma(p.hc0, x0.x, fma(p.hc1, xl.x + xn.x, p.eta * v[m].x));
            y.y = fma(p.hc0, x0.y, fma(p.hc1, xl.y + xn.y, p.eta * v[m].y));
          }
          v[m] = y;
        }
        if (!SPECTRAL) {
          // physical outputs: Y (+ B on the last axis), C = H R (non-last)
#pragma unroll
          for (int m = 0; m < E / 2; ++m) {
            const int j = g + G * m;
            if (j >= 1 && j <= p.n) {
              double2 y = v[m];
              if (LAST) {
                if (p.B) {
                  const double2 b = ld_pair(p, p.B, pc, j);
                  y = make_double2(fma(p.ycoef, y.x, p.bcoef * b.x), fma(p.ycoef, y.y, p.bcoef * b.y));
                } else {
                  y = c_scale(y, p.ycoef);
                }
              }
              st_pair(p, p.Y, pc, j, y);
            }
          }
          if (!LAST) {
            // C = H R: stage R through the buffer for the neighbours
            T::sync();
#pragma unroll
            for (int m = 0; m < E / 2; ++m) {
              const double2 r = ld_pair(p, p.R, pc, g + G * m);
              buf[g + G * m] = make_double2(rs * r.x, rs * r.y);
            }
            T::sync();
#pragma unroll
            for (int m = 0; m < E / 2; ++m) {
              const int j = g + G * m;
              if (j >= 1 && j <= p.n) {
                const double2 rl = buf[j - 1], r0 = buf[j], rn = buf[j + 1];
                st_pair(p, p.C, pc, j, make_double2(fma(p.hc0, r0.x, p.hc1 * (rl.x + rn.x)),
                                                    fma(p.hc0, r0.y, p.hc1 * (rl.y + rn.y))));
              }
            }
          }
        } else {
          odd_extend<T>(v, buf, g);
        }
      } else if (ph == 2) {
        // first DST done (row layout): S y_p = -s Im Z/2, S y_q = s Re Z/2
        if (!LAST) {
#pragma unroll
          for (int r = 0; r < E; ++r) {
            if (!T::lower(r)) continue;
            st_pair(p, p.Y, pc, T::rowk(g, r), make_double2(-v[r].y * hs, v[r].x * hs));
          }
        } else {
          // Lambda^{-1} scaling, then odd extension for the second DST
          const PencilConsts kc = make_consts(p, pc);
          T::sync();
#pragma unroll
          for (int r = 0; r < E; ++r) {
            if (!T::lower(r)) continue;  // only k < N feeds the odd extension
            const int k = T::rowk(g, r);
            double2 w = make_double2(0.0, 0.0);
            if (k >= 1) {
              const double2 lam = rl ? spec_pair_v(p, kc, __ldg(p.lamH_rl + r * G + g), __ldg(p.tq_rl + r * G + g))
                                     : spec_pair(p, kc, k);
              w.x = pc.vp ? (-v[r].y * hs) / lam.x : 0.0;
              w.y = pc.vq ? (v[r].x * hs) / lam.y : 0.0;
            }
            buf[T::sw(k)] = w;
          }
          T::sync();
#pragma unroll
          for (int m = 0; m < E; ++m) {
            const int j = g + G * m;
            if (m < E / 2) {
              v[m] = buf[T::sw(j)];
            } else {
              const double2 t = (j == N) ? make_double2(0.0, 0.0) : buf[T::sw(L - j)];
              v[m] = make_double2(-t.x, -t.y);
            }
          }
        }
      } else {
        // second DST done
#pragma unroll
        for (int r = 0; r < E; ++r) {
          if (!T::lower(r)) continue;
          st_pair(p, p.Y, pc, T::rowk(g, r), make_double2(-v[r].y * hs, v[r].x * hs));
        }
      }
    }
  }
}

// ----------------------------------------------------------------------------- launchers
template <class T, int MODE>
cudaError_t launch_mode(const PassParams& p, cudaStream_t s) {
  const size_t smem = (size_t)T::GROUPS * T::L * sizeof(double2);
  // once per device (thread-safe: batched solves drive several streams and devices)
  struct Tag {};
  const int attr = per_device_once<Tag>([smem](int) -> int {
    return (int)cudaFuncSetAttribute(pass_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr != (int)cudaSuccess) return attr < 0 ? cudaErrorInvalidDevice : (cudaError_t)attr;
  const long long blocks = (p.npairs + T::GROUPS - 1) / T::GROUPS;
  pass_kernel<T, MODE><<<(unsigned)blocks, T::THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_oper_t(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  if (spectral) return last ? launch_mode<T, MODE_OPER_SPEC_LAST>(p, s) : launch_mode<T, MODE_OPER_SPEC>(p, s);
  return last ? launch_mode<T, MODE_OPER_PHYS_LAST>(p, s) : launch_mode<T, MODE_OPER_PHYS>(p, s);
}

template <class T>
cudaError_t launch_dst_t(const PassParams& p, bool last, cudaStream_t s) {
  return last ? launch_mode<T, MODE_DST_LAST>(p, s) : launch_mode<T, MODE_DST>(p, s);
}

#define RSFDE_INSTANTIATE_T(T)                                                             \
  template cudaError_t launch_oper_t<T>(const PassParams&, bool, bool, cudaStream_t);     \
  template cudaError_t launch_dst_t<T>(const PassParams&, bool, cudaStream_t);

}  // namespace rsfde
