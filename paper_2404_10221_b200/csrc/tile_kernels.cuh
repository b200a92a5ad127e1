// Warp-specialised tile pipeline for the spectral operator and DST pencil passes at L = 1024 (n = 511,
// C5) and L = 512 (n = 255, C4).
//
// A persistent CTA = CW compute warps + one producer warpgroup (setmaxnreg moves its registers to the
// compute warps).  A tile = TP adjacent pencil pairs, one FFT group (G threads) per pair: on a strided
// axis 2 TP adjacent pencils = 16 TP contiguous bytes of every row, on the contiguous axis 2 TP
// adjacent rows.  The producer streams each tile input into a shared stage with cp.async.bulk.tensor
// box loads (tensor maps built per launch on the host) tracked by an mbarrier transaction count; the
// compute warps read their pair's column out of the swizzled stage, release it (the next input
// streams in while they compute) and run the FFT phases with per-pair shared exchange buffers.
// Strided outputs leave as row pieces stored cooperatively by the compute warps; neighbouring pairs
// are processed in lockstep, so every DRAM sector is read and written once (ncu:
// profiles/r01_ncu_traffic.json).
//
// Job sequence per tile (consumed in the same order by producer and compute warps):
//   spectral operator pass:  [R_t] [X_t (X_INPUT) | R_t again (X = E o R)]      (X_ZERO: [R_t])
//   DST pass:                [X_t]
#pragma once
#include "pass_kernels.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>

namespace rsfde {

// experiments only (tools/tile_variants.sh): bit 1 = skip the FFTs, bit 2 = skip the global stores
#ifndef RSFDE_TILE_SKIP
#define RSFDE_TILE_SKIP 0
#endif
#ifndef RSFDE_TILE_COOP_STORES  // strided axes: stage outputs in shared memory, store whole tile rows cooperatively
#define RSFDE_TILE_COOP_STORES 1   // (0: 16-byte pieces straight from registers -- measured 17 % slower at 511^3)
#endif
#ifndef RSFDE_TILE_PINGPONG  // CW = 8: the two compute warps of a sub-partition take turns on the FP64 pipe
#define RSFDE_TILE_PINGPONG 0
#endif
#ifndef RSFDE_TILE_TABS_SMEM  // c^ and lambda^H of the operator passes in shared memory (L = 1024 path)
#define RSFDE_TILE_TABS_SMEM 1
#endif
#ifndef RSFDE_TILE_TRACE  // experiments only: per-tile clock64 stamps of warp 0 of every CTA
#define RSFDE_TILE_TRACE 0
#endif
#if RSFDE_TILE_TRACE
__device__ unsigned long long g_tile_trace[512][32][12];
__device__ int g_trace_launch = 0, g_trace_target = -1;  // launch counter / launch to record (-1: every one)
#define TTRACE(slot)                                                                                   \
  if (threadIdx.x == 0 && blockIdx.x < 512 && tcount < 32 &&                                           \
      (g_trace_target < 0 || g_trace_target == trace_launch)) {                                        \
    unsigned smid;                                                                                     \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                                                \
    g_tile_trace[blockIdx.x][tcount][slot] = clock64();                                                \
    g_tile_trace[blockIdx.x][tcount][7] = smid;                                                        \
  }
#else
#define TTRACE(slot)
#endif

// Tile width TP pencil pairs.  A pair is one FFT group of T::G threads (32 at L = 1024, 16 at
// L = 512), so a compute warp holds 32 / G pairs and a tile CW = TP G / 32 compute warps.  CW = 8: one
// CTA of 12 warps per SM (compute warps at 232 registers); CW = 4: two CTAs of 8 warps per SM (216).
// 128-byte rows (TP = 8) are needed on axes whose rows are >= 1 MB apart (every row piece is then its
// own 2 MB page, and TMA throughput is set by the number of row pieces: tools/micro/tma_micro.cu,
// 3.0 vs 5.9 TB/s).
template <int CW>
struct TileCfg {
  static constexpr int kTileThreads = CW == 8 ? 384 : 256;
  static constexpr int kCtasPerSm = CW == 8 ? 1 : 2;
  static constexpr int kComputeRegs = CW == 8 ? 232 : 216;
};
constexpr int kProducerRegs = 40;
constexpr int kBoxRows = 256;
#define RSFDE_TILE_CONSTS                                                        \
  constexpr int kTilePairs = TP;                                                 \
  constexpr int kTilePencils = 2 * TP;                   /* adjacent pencils */  \
  constexpr int kRowBytes = 8 * kTilePencils;            /* bytes of a row */    \
  constexpr int kNBox = NH / kBoxRows;                   /* boxes per job */     \
  constexpr size_t kStageBytes = (size_t)kNBox * kBoxRows * kRowBytes;           \
  (void)kTilePairs; (void)kTilePencils; (void)kRowBytes; (void)kStageBytes;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// The suspend-time hint lets a waiting warp sleep in the barrier unit until the phase completes
// instead of re-issuing try_wait: the spinning producer warp otherwise took ~7 % of the issue slots
// of its sub-partition from the compute warp beside it (ncu, profiles/r01_ncu_tile_final_summary.txt).
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
}
template <int CW>
__device__ __forceinline__ void compute_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(32 * CW) : "memory"); }
// Strided tiles hand their staged outputs to the three spare warps of the producer warpgroup (the
// "store warps"): named barrier 2 = outputs staged (compute warps arrive, store warps wait), 3 = pair
// buffers free again (store warps arrive, compute warps wait right before their next buffer write).
constexpr int kStoreWarps = 3;
template <int CW>
__device__ __forceinline__ void named_sync(int id) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(32 * (CW + kStoreWarps)) : "memory");
}
template <int CW>
__device__ __forceinline__ void named_arrive(int id) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "n"(32 * (CW + kStoreWarps)) : "memory");
}

// FP64 ping-pong (CW = 8, one CTA per SM): compute warps w and w + 4 share a scheduler / FP64 pipe.
// Left alone they fall into lockstep (both in an FFT's register phase, then both in the shared-memory
// plumbing: the pass time is the SUM of its FP64 and shared-memory times, profiles/r02_tile_experiments.txt).
// A token per sub-partition (named barriers 4 + s for warps 0-3, 8 + s for warps 4-7, 64 threads each)
// is held during the register DFT bursts, so one warp's burst runs against the other's exchange, stage
// reads and stores.  Strict alternation: warp w + 4 primes the token of warp w at kernel start; every
// warp runs the same number of bursts (all warps of a CTA process the same tiles).
template <int CW>
struct PingPong {
  static constexpr bool on = RSFDE_TILE_PINGPONG && CW == 8;
  int mine, other;
  __device__ __forceinline__ PingPong(int warp) : mine(4 + (warp & 3) + 4 * (warp >> 2)), other(4 + (warp & 3) + 4 * (1 - (warp >> 2))) {
    if (on && warp >= 4) asm volatile("bar.arrive %0, 64;\n" ::"r"(other) : "memory");
  }
  __device__ __forceinline__ void acquire() const {
    if (on) asm volatile("bar.sync %0, 64;\n" ::"r"(mine) : "memory");
  }
  __device__ __forceinline__ void release() const {
    if (on) asm volatile("bar.arrive %0, 64;\n" ::"r"(other) : "memory");
  }
  // warps 0-3 absorb the last (unmatched) release of their partner
  __device__ __forceinline__ void finish(int warp) const {
    if (on && warp < 4) asm volatile("bar.sync %0, 64;\n" ::"r"(mine) : "memory");
  }
};

// element offset of the first pencil of tile t (strided: pencil 16t; contiguous: row 16t)
template <int TP, int NH, bool CT>
__device__ __forceinline__ long long tile_base(const PassParams& p, long long t) {
  RSFDE_TILE_CONSTS
  if (CT) return kTilePencils * t * p.geo.P;
  const unsigned pen = (unsigned)(kTilePencils * t), inner = (unsigned)p.inner;
  const unsigned o = pen / inner, i = pen - o * inner;
  return (long long)o * p.n * p.inner + i;
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Stage layout.  Strided axis: tensor map {inner, n, outer} (pencil, axis position, outer block),
// box {16, 256, 1} with the 128-byte swizzle -> stage row r (axis position r + 1) holds the 16
// pencils of the tile as 8 chunks of 16 bytes (one per pair), chunk w stored at w ^ (r & 7).
// Contiguous axis: tensor map {P, rows}, box {256, 16} -> stage[half][row][256].

// producer: one lane streams one tile input into the stage (two box copies)
template <int TP, int NH, bool CT>
__device__ __forceinline__ void produce(const PassParams& p, const CUtensorMap* tm, long long t, char* stage,
                                        unsigned long long* full) {
  RSFDE_TILE_CONSTS
  mbar_expect_tx(full, (unsigned)kStageBytes);
  if (CT && p.seg_lg) {
    // segmented rows (all-to-all blocks): one box {2^seg_lg, pencils, segments} -> stage [seg][pencil][x_l]
    tma_load_3d(stage, tm, 0, (int)(kTilePencils * t), 0, full);
  } else if (CT) {
#pragma unroll
    for (int b = 0; b < kNBox; ++b)
      tma_load_3d(stage + (size_t)b * (kStageBytes / kNBox), tm, b * kBoxRows, (int)(kTilePencils * t), 0, full);
  } else {
    const unsigned pen = (unsigned)(kTilePencils * t), inner = (unsigned)p.inner;
    const int o = (int)(pen / inner), i = (int)(pen - (unsigned)o * inner);
#pragma unroll
    for (int b = 0; b < kNBox; ++b) tma_load_3d(stage + (size_t)b * (kStageBytes / kNBox), tm, i, b * kBoxRows, o, full);
  }
}

// 1/x to ~1 ulp: hardware approximation + two Newton steps (instead of a full IEEE division)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// value pair (p, q) of compute warp w at axis position j (1..n) from the stage
template <int TP, int NH, bool CT>
__device__ __forceinline__ double2 stage_pair(const PassParams& p, const char* stage, int w, int j) {
  RSFDE_TILE_CONSTS
  const int r = j - 1;
  if (CT) {  // stage [r >> lg][pencil][r & (2^lg - 1)], lg = 8 (two 256-row boxes) or the segment length
    const int lg = p.seg_lg ? p.seg_lg : 8;
    const double* s = reinterpret_cast<const double*>(stage) + (r >> lg) * (kTilePencils << lg) + (r & ((1 << lg) - 1));
    return make_double2(s[(2 * w) << lg], s[(2 * w + 1) << lg]);
  }
  // 128-byte swizzle: 16-byte chunk c of row r at c ^ (r & 7); 64-byte swizzle: c ^ ((r >> 1) & 3)
  const int sw = kTilePairs == 8 ? (r & 7) : ((r >> 1) & 3);
  return *reinterpret_cast<const double2*>(stage + (size_t)r * kRowBytes + ((w ^ sw) << 4));
}

// Stage column of pair w for the axis positions j = j0 + G m (m = 0, 1, ...): the swizzle chunk of a
// strided stage row r depends on r mod 8 only (r & 7, or (r >> 1) & 3), which G m (G = 16, 32) does not
// change, so one base pointer per thread serves every m (constant offsets m G kRowBytes); contiguous
// stage: element (r & 255) of box (r >> 8) of pencil 2w / 2w + 1.  Valid for j0 - 1 + G m in 0..NH-1.
template <int TP, int NH, bool CT, int G>
struct StageCol {
  const char* base;
  __device__ __forceinline__ StageCol(const PassParams& p, const char* stage, int w, int j0) {
    RSFDE_TILE_CONSTS
    const int r = j0 - 1;
    if (CT) {
      lg = p.seg_lg ? p.seg_lg : 8;
      base = stage + (size_t)((2 * w) << lg) * 8;  // (r handled in at())
      r0 = r;
    } else {
      const int sw = kTilePairs == 8 ? (r & 7) : ((r >> 1) & 3);
      base = stage + (ptrdiff_t)r * kRowBytes + ((w ^ sw) << 4);
      r0 = 0;
    }
  }
  int r0, lg;
  __device__ __forceinline__ double2 at(int m) const {
    RSFDE_TILE_CONSTS
    if (CT) {
      const int r = r0 + G * m;
      const double* s = reinterpret_cast<const double*>(base) + (r >> lg) * (kTilePencils << lg) + (r & ((1 << lg) - 1));
      return make_double2(s[0], s[1 << lg]);
    }
    return *reinterpret_cast<const double2*>(base + (ptrdiff_t)m * G * kRowBytes);
  }
};

// XOR swizzle of the per-pair output buffers so that the cooperative row stores read
// conflict-free across the 8 buffers
__device__ __forceinline__ int oswz(int k, int w) { return k ^ (w & 7); }

// Strided axes: the staged outputs of the tile's pairs (pair buffers, k = 1..n at oswz(k, q)) leave as
// whole tile rows.  The compute thread count is a multiple of TP, so a thread always serves the same
// pair column q and rows row0, row0 + RSTEP, ...: no index division, one validity load, one pointer
// increment per row.
template <int TP, int NT, int L, int kN>
__device__ __forceinline__ void coop_store_rows(const double2* bufs, const int* tvalid, double* out, long long base,
                                                long long stride, int tid) {
  constexpr int RSTEP = NT / TP;
  static_assert(NT % TP == 0, "store threads must be a multiple of the tile width");
  const int q = tid % TP, row0 = tid / TP;
  const int vm = tvalid[q];
  if (!(vm & 1) || (RSFDE_TILE_SKIP & 2)) return;
  const double2* src = bufs + q * L;
  double* dst = out + base + (long long)row0 * stride + 2 * q;
  const long long dstep = (long long)RSTEP * stride;
#pragma unroll 4
  for (int row = row0; row < kN; row += RSTEP, dst += dstep) {
    const double2 c = src[oswz(row + 1, q)];
    if (vm & 2) *reinterpret_cast<double2*>(dst) = c;
    else *dst = c.x;
  }
}

template <int MODE, class T, int TP, bool CT>
__global__ void __launch_bounds__(TileCfg<TP * T::G / 32>::kTileThreads, TileCfg<TP * T::G / 32>::kCtasPerSm)
    tile_kernel(const PassParams p, const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmX) {
  constexpr int E = T::E, G = T::G, L = T::L, N = T::N, NH = T::N;
  // the pencil length along the pass axis is fixed by the FFT length (p.n == N - 1, checked by the
  // launcher): compile-time bounds turn the per-element range tests into predicates and let the
  // compiler schedule the unrolled plumbing loops freely
  constexpr int kN = N - 1;
  constexpr int PPW = 32 / G;           // pencil pairs per compute warp
  constexpr int CW = TP / PPW;          // compute warps
  constexpr int kComputeThreads = 32 * CW;
  RSFDE_TILE_CONSTS
  constexpr bool OPER = MODE == MODE_OPER_SPEC || MODE == MODE_OPER_SPEC_LAST;
  constexpr bool LAST = MODE == MODE_OPER_SPEC_LAST || MODE == MODE_DST_LAST;
  extern __shared__ __align__(128) char tsm_raw[];
  char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);  // TMA swizzle needs 1 KB alignment
  double2* bufs = reinterpret_cast<double2*>(tsm);                        // TP x L x 16 bytes
  char* stage = tsm + (size_t)kTilePairs * L * sizeof(double2);           // 1024-aligned
  __shared__ __align__(8) unsigned long long full_bar, empty_bar;
  __shared__ int tvalid[2][kTilePairs];  // validity bits (p, q) of each pair, by tile parity (store warps)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long ntiles = CT ? ((p.geo.NP / p.geo.P) + kTilePencils - 1) / kTilePencils : (p.npairs + kTilePairs - 1) / kTilePairs;
  // e(x, t) constant along the pass axis (no axis factor g_a, k_a: e.g. C5's e(x1, t) on the x3 pass):
  // X = E o R is R times a per-pencil constant, so the stencil reads R from the stage of job 0, which
  // stays resident until then (one load of R per tile instead of two)
  const bool single_R = OPER && p.xmode == X_E_TIMES_R && p.e.kind != 2 && !p.e.g[p.axis] && !p.e.k[p.axis];
  const int jobs_per_tile = OPER ? ((p.xmode == X_ZERO || single_R) ? 1 : 2) : 1;
  if (skip_launch(p.skip)) return;  // speculative launch after convergence (uniform over the grid)
  if (threadIdx.x == 0) {
    mbar_init(&full_bar, 1);
    mbar_init(&empty_bar, CW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= CW) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    if (warp != CW) {
      if (CT || warp > CW + kStoreWarps) return;
      // -------------------------------------------------------------- store warps (strided tiles)
      const int sid = threadIdx.x - 32 * (CW + 1);
      int tc = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++tc) {
        const long long base = tile_base<TP, NH, CT>(p, t);
        if (OPER && !LAST) {
          named_sync<CW>(2);
          coop_store_rows<TP, 32 * kStoreWarps, L, kN>(bufs, tvalid[tc & 1], p.C, base, p.stride, sid);
          named_arrive<CW>(3);
        }
        named_sync<CW>(2);
        coop_store_rows<TP, 32 * kStoreWarps, L, kN>(bufs, tvalid[tc & 1], p.Y, base, p.stride, sid);
        named_arrive<CW>(3);
      }
      return;
    }
    // ------------------------------------------------------------------ producer warp
    long long job = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int k = 0; k < jobs_per_tile; ++k, ++job) {
        if (job > 0) mbar_wait(&empty_bar, (unsigned)((job - 1) & 1));
        const CUtensorMap* src = OPER ? ((k == 0 || p.xmode == X_E_TIMES_R) ? &tmR : &tmX) : &tmX;
        if (lane == 0) produce<TP, NH, CT>(p, src, t, stage, &full_bar);
        __syncwarp();
      }
    }
    return;
  }

  // -------------------------------------------------------------------- compute warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(TileCfg<CW>::kComputeRegs));
  // separable e(x, t) along the pass axis (X = E o R): the axis factors g_a, k_a in shared memory
  // (last axis: the same arrays hold the spectrum tables lambda^H_k and tq_k of the axis)
  __shared__ double e_ga[N], e_ka[N];
  const bool e_tab = OPER && p.xmode == X_E_TIMES_R && p.e.kind != 2;
  const bool e_const = single_R;
  if (e_tab) {
    const double* ga = p.e.g[p.axis];
    const double* ka = p.e.k[p.axis];
    for (int j = threadIdx.x; j < N; j += kComputeThreads) {
      e_ga[j] = (ga && j < kN) ? __ldg(ga + j) : 1.0;
      e_ka[j] = (ka && j < kN) ? __ldg(ka + j) : 0.0;
    }
    compute_bar<CW>();
  }
  if (LAST && !e_tab) {
    const double* lh = p.spec.lamH[p.axis];
    const double* tq = p.spec.tq[p.axis];
    for (int j = threadIdx.x; j < N; j += kComputeThreads) {
      e_ga[j] = (lh && j < kN) ? __ldg(lh + j) : 1.0;
      e_ka[j] = (tq && j < kN) ? __ldg(tq + j) : 0.0;
    }
    compute_bar<CW>();
  }
  // The axis tables c^ (even: c^_k = c^_{L-k}, so N + 1 values) and lambda^H of the operator passes in
  // shared memory: every tile reads them right where they are used, and a global load there is an exposed
  // L1/L2 latency on each warp's dependency chain.  Only where the 8 KB fit beside two resident CTAs
  // (same-box A/B: x3 pass 1616 -> 1575 us, last pass 1902 -> 1862 us, C4 chain -3 %; the 4-pair L = 1024
  // kernels would drop to a smaller L1 carve-out and ran 22 % slower, so they keep the global loads).
  // (E == G DST passes: the four exactly loaded twiddle powers per lane of the FFT's twiddle stage, 2 KB;
  // same-box A/B: inverse DST x2 538 -> 523 us, DST x3 477 -> 471 us; no gain in the operator passes)
  constexpr bool TWS = RSFDE_TILE_TABS_SMEM && E == G && !OPER;
  __shared__ double2 tw_s[TWS ? (E / 8) * G : 1];
  if constexpr (TWS) {
    twiddle_table_fill<E, G>(tw_s, p.tw, threadIdx.x, kComputeThreads);
    compute_bar<CW>();
  }
  constexpr bool TABS = RSFDE_TILE_TABS_SMEM && OPER && (CW == 8 || L <= 512);
  __shared__ double chat_s[TABS ? N + 1 : 1], lamH_s[(TABS && !LAST) ? N : 1];
  if constexpr (TABS) {
    for (int j = threadIdx.x; j <= N; j += kComputeThreads) chat_s[j] = __ldg(p.chat + j);
    if (!LAST)
      for (int j = threadIdx.x; j < kN; j += kComputeThreads) lamH_s[j] = __ldg(p.lamH + j);
    compute_bar<CW>();
  }
  const int g = lane % G, w = warp * PPW + lane / G;  // FFT-group thread index, pencil pair in the tile
  double2* buf = bufs + w * L;
  const PingPong<CW> pp(warp);
  const double rs = p.rscale ? __ldg(p.rscale) : 1.0;
  // The DST scale hs is applied once, early: to the input of a DST pass, to y = H X + eta T R in an
  // operator pass and to Lambda^-1 before the last inverse DST -- never to the row-layout outputs.
  const double hs = 0.5 * p.dst_scale;
  const double rsh = rs * hs;
  // the lazy basis scale rs of R folds into eta (T R enters y only as eta T R) and into the C factor
  const double hc0s = p.hc0 * hs, hc1s = p.hc1 * hs, etas = p.eta * rsh, crs = OPER ? rsh : hs;
  const double etas_y = (E == G) ? -etas : etas;
  long long job = 0;
  int tcount = 0;
  bool pend_free = false;  // staged outputs handed to the store warps, pair buffers not yet released
#if RSFDE_TILE_TRACE
  const int trace_launch = *(volatile int*)&g_trace_launch;
#endif
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++tcount) {
    const long long pair = (long long)kTilePairs * t + w;
    const bool active = pair < p.npairs;
    const PairCtx pc = make_pair(p, active ? pair : 0, active);
    if (g == 0) tvalid[tcount & 1][w] = (pc.vp ? 1 : 0) | (pc.vq ? 2 : 0);
    // per-pencil constants of e(x,t): their table loads are issued here, at the tile start, so that
    // their latency hides behind the first FFT (not in the last-axis kernel, where the live
    // registers would spill; the last-axis spectrum constants are loaded where they are used)
    const PencilConsts kc0 = (OPER && !LAST && p.xmode == X_E_TIMES_R) ? make_consts(p, pc, true, false) : PencilConsts{};
    double2 v[E];
    TTRACE(0)
    // ---- job 0: primary input
    mbar_wait(&full_bar, (unsigned)(job & 1));
    TTRACE(1)
    if (OPER) {
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const int j = g + G * m;
        double2 r = make_double2(0.0, 0.0);
        if (m < E / 2 && j >= 1 && j <= kN) {
          r = stage_pair<TP, NH, CT>(p, stage, w, j);  // raw R (rs folded into eta and the C factor)
          r = make_double2(pc.vp ? r.x : 0.0, pc.vq ? r.y : 0.0);
        }
        v[m] = r;
      }
    } else {
#pragma unroll
      for (int m = 0; m < E / 2; ++m) {
        const int j = g + G * m;
        double2 r = make_double2(0.0, 0.0);
        if (j >= 1 && j <= kN) {
          r = stage_pair<TP, NH, CT>(p, stage, w, j);
          r = make_double2(pc.vp ? rsh * r.x : 0.0, pc.vq ? rsh * r.y : 0.0);
        }
        v[m] = r;
      }
    }
    if (!single_R) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar);
      ++job;
    }
    // (shuffle form: no pair-buffer write, so the previous tile's staged outputs, which the store warps
    // may still be copying out, are waited for only at the exchange of the FFT below)
    // Strided tiles only (same-box A/B at 511^3: inverse DST x2 557 -> 540 us, last pass 1915 -> 1896 us;
    // the contiguous-axis passes were 4 % slower with shuffles and keep the buffer form).
    if (!OPER) {
      if (CT) odd_extend<T>(v, buf, g);
      else odd_extend_shfl<T>(v, g);
    }

    const int first = OPER ? 0 : 2;
    const int last_phase = LAST ? 3 : 2;
#pragma unroll 1
    for (int ph0 = first; ph0 <= last_phase; ++ph0) {
      // One FFT body per kernel: the phase index is made opaque to the compiler (otherwise it clones
      // the loop body per phase, 4 FFT bodies = 270 KB of SASS and instruction-cache stalls), and the
      // inverse transform is conj(FFT(conj(.))), which for E == G maps the row layout to the column
      // layout exactly like fft_inv.
      int ph;
      asm volatile("mov.b32 %0, %1;" : "=r"(ph) : "r"(ph0));
      if (!(RSFDE_TILE_SKIP & 1)) {
        if constexpr (E == G) {
          // phase 1 (the convolution's inverse FFT) is conj(FFT(conj(.))): the input conj is folded
          // into the spectrum scaling of phase 0 and the output conj into the stencil of phase 1
          pp.acquire();
          if constexpr (TWS) fft_fwd_pre_s<E, G>(v, g, tw_s);
          else fft_fwd_pre<E, G>(v, g, p.tw);
          pp.release();
          if (!CT && pend_free) {  // the register-only first half overlaps the store warps' copy
            named_sync<CW>(3);
            pend_free = false;
          }
          fft_exchange<E, G>(v, buf, g);
          pp.acquire();
          dft<G>(v);
          pp.release();
        } else {
          if (!CT && pend_free) {
            named_sync<CW>(3);
            pend_free = false;
          }
          T::fft(v, buf, g, p.tw, ph == 1);  // E = R G: forward and inverse differ in layout
        }
      }
      TTRACE(2 + ph)
      if (OPER && ph == 0) {
        // C = S H R = s lambda^H D(R) (non-last spectral pass), via the partner spectrum
        if (!LAST) {
          // only the upper half is read back (the partner L - k of a lower k >= 1 is >= N + 1)
          __syncwarp();
#pragma unroll
          for (int r = 0; r < E; ++r)
            if (!T::lower(r)) buf[T::rowk(g, r)] = v[r];
          __syncwarp();
          double2 cv[E / 2];
#pragma unroll
          for (int r = 0, i = 0; r < E; ++r) {
            if (!T::lower(r)) continue;
            const int k = T::rowk(g, r);
            const double2 zm = (k >= 1) ? buf[L - k] : make_double2(0.0, 0.0);
            const double f = (k >= 1) ? crs * (TABS ? lamH_s[k - 1] : __ldg(p.lamH + k - 1)) : 0.0;
            cv[i++] = make_double2(-(v[r].y - zm.y) * f, (v[r].x - zm.x) * f);
          }
          if (CT && E == G) {
            // contiguous axis: row register r holds k = g + G r, so a warp's stores of one r are 32
            // consecutive doubles of each pencil -- coalesced straight from registers, no staging
            double* cp = p.C + pc.off_p + (g - 1);  // k - 1 = (g - 1) + G r: constant offsets per r
            double* cq = p.C + pc.off_q + (g - 1);
#pragma unroll
            for (int r = 0, i = 0; r < E; ++r) {
              if (!T::lower(r)) continue;
              if ((r > 0 || g > 0) && !(RSFDE_TILE_SKIP & 2)) {
                if (p.seg_lg) {
                  const long long o = pos_off(p, g + G * r);
                  if (pc.vp) p.C[pc.off_p + o] = cv[i].x;
                  if (pc.vq) p.C[pc.off_q + o] = cv[i].y;
                } else {
                  if (pc.vp) cp[G * r] = cv[i].x;
                  if (pc.vq) cq[G * r] = cv[i].y;
                }
              }
              ++i;
            }
          } else if (!RSFDE_TILE_COOP_STORES) {
            // store C straight from registers: 16-byte (pencil pair) pieces per row on strided axes
            // (the neighbouring pairs' warps fill the rest of each row piece at the same time; L2
            // merges the sectors), coalesced 8-byte elements on the contiguous axis
#pragma unroll
            for (int r = 0, i = 0; r < E; ++r) {
              if (!T::lower(r)) continue;
              if (!(RSFDE_TILE_SKIP & 2)) st_pair(p, p.C, pc, T::rowk(g, r), cv[i]);
              ++i;
            }
          } else {
          __syncwarp();
#pragma unroll
          for (int r = 0, i = 0; r < E; ++r) {
            if (!T::lower(r)) continue;
            buf[oswz(T::rowk(g, r), w)] = cv[i++];
          }
          // store C
          if (CT) {
            __syncwarp();
            for (int j = g + 1; j <= kN; j += G) {
              const double2 c = buf[oswz(j, w)];
              if (RSFDE_TILE_SKIP & 2) continue;
              const long long o = pos_off(p, j);
              if (pc.vp) p.C[pc.off_p + o] = c.x;
              if (pc.vq) p.C[pc.off_q + o] = c.y;
            }
            __syncwarp();
          } else {
            named_arrive<CW>(2);  // the store warps write C out while the next FFT starts
            pend_free = true;
          }
          }  // RSFDE_TILE_COOP_STORES
        }
        TTRACE(9)
        if constexpr (E == G) {
          // scaled conj spectrum: the inverse FFT of phase 1 runs as a forward FFT (see above)
#pragma unroll
          for (int r = 0; r < E; ++r) {
            const int kk = T::rowk(g, r);
            const double ch = TABS ? chat_s[T::lower(r) ? kk : L - kk] : __ldg(p.chat + kk);
            v[r] = make_double2(v[r].x * ch, -v[r].y * ch);
          }
        } else {
#pragma unroll
          for (int r = 0; r < E; ++r) {
            const int kk = T::rowk(g, r);
            v[r] = c_scale(v[r], TABS ? chat_s[T::lower(r) ? kk : L - kk] : __ldg(p.chat + kk));
          }
        }
      } else if (OPER && ph == 1) {
        // X channel from the stage (job 1) into the pair buffer (x = X, or e o R), then
        // y = H X + eta T R on j = g + G m with the stencil neighbours from the buffer
        const PencilConsts kc = (LAST && p.xmode == X_E_TIMES_R) ? make_consts(p, pc, true, false) : kc0;
        const double2 eab = e_ab(p.e);
        if (p.xmode != X_ZERO && !single_R) mbar_wait(&full_bar, (unsigned)(job & 1));
        TTRACE(11)
        if (p.xmode == X_INPUT || e_const) {
          // X is an input vector (or R times a pencil constant): the stencil neighbours come straight
          // from the stage (3 shared loads per value instead of a load, a store to the pair buffer and
          // 3 loads); invalid pencils are masked on y (their stage values are finite: zero pads or TMA
          // zero fill)
          if (p.xmode == X_INPUT) {
            const StageCol<TP, NH, CT, G> c0(p, stage, w, g), cl(p, stage, w, g - 1), cn(p, stage, w, g + 1);
#pragma unroll
            for (int m = 0; m < E / 2; ++m) {
              const int j = g + G * m;
              double2 y = make_double2(0.0, 0.0);
              if (j >= 1 && j <= kN) {
                const double2 x0 = c0.at(m);
                const double2 xl = (j > 1) ? cl.at(m) : make_double2(0.0, 0.0);
                const double2 xn = (j < kN) ? cn.at(m) : make_double2(0.0, 0.0);
                y.x = pc.vp ? fma(hc0s, x0.x, fma(hc1s, xl.x + xn.x, etas * v[m].x)) : 0.0;
                y.y = pc.vq ? fma(hc0s, x0.y, fma(hc1s, xl.y + xn.y, etas_y * v[m].y)) : 0.0;
              }
              v[m] = y;
            }
          } else {
            // e = a + b eP + eK on the whole pencil (the axis factors are 1 and 0)
            const double sp = rs * (fma(eab.y * kc.eP_p, 1.0, eab.x) + kc.eK_p);
            const double sq = rs * (fma(eab.y * kc.eP_q, 1.0, eab.x) + kc.eK_q);
            const StageCol<TP, NH, CT, G> c0(p, stage, w, g), cl(p, stage, w, g - 1), cn(p, stage, w, g + 1);
#pragma unroll
            for (int m = 0; m < E / 2; ++m) {
              const int j = g + G * m;
              double2 y = make_double2(0.0, 0.0);
              if (j >= 1 && j <= kN) {
                const double2 x0 = c0.at(m);
                const double2 xl = (j > 1) ? cl.at(m) : make_double2(0.0, 0.0);
                const double2 xn = (j < kN) ? cn.at(m) : make_double2(0.0, 0.0);
                y.x = pc.vp ? fma(sp, fma(hc0s, x0.x, hc1s * (xl.x + xn.x)), etas * v[m].x) : 0.0;
                y.y = pc.vq ? fma(sq, fma(hc0s, x0.y, hc1s * (xl.y + xn.y)), etas_y * v[m].y) : 0.0;
              }
              v[m] = y;
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar);
          ++job;
        } else {
        __syncwarp();
#pragma unroll
        for (int m = 0; m < E / 2; ++m) {
          const int j = g + G * m;
          double2 x = make_double2(0.0, 0.0);
          if (p.xmode != X_ZERO && j >= 1 && j <= kN) {
            x = stage_pair<TP, NH, CT>(p, stage, w, j);
            if (p.xmode == X_E_TIMES_R) {
              double2 e;
              if (e_tab) {
                const double ga = e_ga[j - 1], ka = e_ka[j - 1];
                e = make_double2(fma(eab.y * kc.eP_p, ga, eab.x) + (kc.eK_p + ka),
                                 fma(eab.y * kc.eP_q, ga, eab.x) + (kc.eK_q + ka));
              } else {
                e = e_pair(p, pc, kc, j, eab);
              }
              x = make_double2(rs * x.x * e.x, rs * x.y * e.y);
            }
            if (!pc.vp) x.x = 0.0;
            if (!pc.vq) x.y = 0.0;
          }
          buf[j] = x;
        }
        if (g == 0) buf[N] = make_double2(0.0, 0.0);
        if (p.xmode != X_ZERO) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar);
          ++job;
        }
        __syncwarp();
#pragma unroll
        for (int m = 0; m < E / 2; ++m) {
          const int j = g + G * m;
          double2 y = make_double2(0.0, 0.0);
          if (j >= 1 && j <= kN) {
            const double2 xl = buf[j - 1], x0 = buf[j], xn = buf[j + 1];
            // (E == G: phase 1 returned conj(T R), so the imaginary part enters with -eta)
            y.x = fma(hc0s, x0.x, fma(hc1s, xl.x + xn.x, etas * v[m].x));
            y.y = fma(hc0s, x0.y, fma(hc1s, xl.y + xn.y, etas_y * v[m].y));
          }
          v[m] = y;
        }
        }  // X_INPUT
        TTRACE(10)
        if (CT) odd_extend<T>(v, buf, g);
        else odd_extend_shfl<T>(v, g);
      } else if (ph == 2 && LAST) {
        // S y (row layout, k = g + G r for r < E/2) into the pair buffer, then Lambda^{-1} in a rolled
        // loop over the same k (small code: the spectrum kinds are a runtime switch)
        const PencilConsts ks = make_consts(p, pc, false, true);
        const Spec& S = p.spec;
        const bool fast = S.kind == SPEC_PHAT || S.kind == SPEC_PALPHA || S.kind == SPEC_HINV;
        const double icHp = ((S.kind == SPEC_PALPHA) ? 1.0 : 1.0 / ks.cH_p) * hs;  // (hs of the inverse DST)
        const double icHq = ((S.kind == SPEC_PALPHA) ? 1.0 : 1.0 / ks.cH_q) * hs;
        bool done = false;
        if constexpr (E == G) {
          if (fast && !e_tab) {
            // row register m holds k = g + G m, which is also column index j = g + G m of this thread:
            // the scaled values stay in registers and the mirror half of the odd extension of the
            // second DST comes from the partner lanes by shuffle
#pragma unroll
            for (int m = 0; m < E / 2; ++m) {
              const int k = g + G * m;
              double2 wv = make_double2(0.0, 0.0);
              if (k >= 1) {
                const double lh = (S.kind == SPEC_PALPHA) ? 1.0 : e_ga[k - 1];
                double lp = 1.0, lq = 1.0;
                if (S.kind != SPEC_HINV) {
                  const double tq = e_ka[k - 1];
                  lp = S.ebar + ks.cP_p + tq;
                  lq = S.ebar + ks.cP_q + tq;
                }
                wv.x = pc.vp ? -v[m].y * (rcp_nr(lp * lh) * icHp) : 0.0;
                wv.y = pc.vq ? v[m].x * (rcp_nr(lq * lh) * icHq) : 0.0;
              }
              v[m] = wv;
            }
            odd_extend_shfl<T>(v, g);
            done = true;
          }
        }
        if (!done) {
        __syncwarp();
#pragma unroll
        for (int r = 0; r < E; ++r) {
          if (!T::lower(r)) continue;
          buf[T::rowk(g, r)] = make_double2(-v[r].y, v[r].x);
        }
        __syncwarp();  // (E > G: the loop below reads k values written by other threads of the group)
        // Lambda = (ebar + cP + tq_k) cH lh_k (P_hat) | (ebar + cP + tq_k) (P_alpha) | cH lh_k (H):
        // one fast reciprocal per value instead of an IEEE division
        if (fast && !e_tab) {
          // unrolled: the 16 values are independent (a rolled loop serialises the latencies)
#pragma unroll
          for (int m = 0; m < E / 2; ++m) {
            const int k = g + G * m;
            double2 wv = make_double2(0.0, 0.0);
            if (k >= 1) {
              const double2 z = buf[k];
              const double lh = (S.kind == SPEC_PALPHA) ? 1.0 : e_ga[k - 1];
              double lp = 1.0, lq = 1.0;
              if (S.kind != SPEC_HINV) {
                const double tq = e_ka[k - 1];
                lp = S.ebar + ks.cP_p + tq;
                lq = S.ebar + ks.cP_q + tq;
              }
              wv.x = pc.vp ? z.x * (rcp_nr(lp * lh) * icHp) : 0.0;
              wv.y = pc.vq ? z.y * (rcp_nr(lq * lh) * icHq) : 0.0;
            }
            buf[k] = wv;
          }
        } else {
#pragma unroll 1
          for (int m = 0; m < E / 2; ++m) {
            const int k = g + G * m;
            double2 wv = make_double2(0.0, 0.0);
            if (k >= 1) {
              const double2 z = buf[k];
              const double2 lam = spec_pair(p, ks, k);
              wv.x = pc.vp ? (z.x * hs) / lam.x : 0.0;
              wv.y = pc.vq ? (z.y * hs) / lam.y : 0.0;
            }
            buf[k] = wv;
          }
        }
        TTRACE(8)
        __syncwarp();
#pragma unroll
        for (int m = 0; m < E; ++m) {
          const int j = g + G * m;
          if (m < E / 2) {
            v[m] = buf[j];
          } else {
            const double2 tt = (j == N) ? make_double2(0.0, 0.0) : buf[L - j];
            v[m] = make_double2(-tt.x, -tt.y);
          }
        }
        }  // !done
      } else {
        // final DST (row layout) -> Y
        if (CT && E == G) {
          // contiguous axis: coalesced stores straight from the row registers (see the C output)
          double* yp = p.Y + pc.off_p + (g - 1);
          double* yq = p.Y + pc.off_q + (g - 1);
#pragma unroll
          for (int r = 0; r < E; ++r) {
            if (!T::lower(r)) continue;
            if ((r > 0 || g > 0) && !(RSFDE_TILE_SKIP & 2)) {
              if (p.seg_lg) {  // (the send blocks of the next all-to-all)
                const long long o = pos_off(p, g + G * r);
                if (pc.vp) p.Y[pc.off_p + o] = -v[r].y;
                if (pc.vq) p.Y[pc.off_q + o] = v[r].x;
              } else {
                if (pc.vp) yp[G * r] = -v[r].y;
                if (pc.vq) yq[G * r] = v[r].x;
              }
            }
          }
        } else if (!RSFDE_TILE_COOP_STORES) {
#pragma unroll
          for (int r = 0; r < E; ++r) {
            if (!T::lower(r)) continue;
            if (!(RSFDE_TILE_SKIP & 2)) st_pair(p, p.Y, pc, T::rowk(g, r), make_double2(-v[r].y, v[r].x));
          }
        } else {
        __syncwarp();
#pragma unroll
        for (int r = 0; r < E; ++r) {
          if (!T::lower(r)) continue;
          buf[oswz(T::rowk(g, r), w)] = make_double2(-v[r].y, v[r].x);
        }
        if (CT) {
          __syncwarp();
          for (int j = g + 1; j <= kN; j += G) {
            const double2 yv = buf[oswz(j, w)];
            if (RSFDE_TILE_SKIP & 2) continue;
            const long long o = pos_off(p, j);
            if (pc.vp) p.Y[pc.off_p + o] = yv.x;
            if (pc.vq) p.Y[pc.off_q + o] = yv.y;
          }
          __syncwarp();
        } else {
          named_arrive<CW>(2);  // the store warps write Y out during the next tile's first FFT
          pend_free = true;
        }
        }  // RSFDE_TILE_COOP_STORES
      }
    }
    TTRACE(6)
  }
  pp.finish(warp);
#if RSFDE_TILE_TRACE
  // count launches (the last compute thread to finish bumps the counter once per launch)
  __shared__ int done_warps;
  if (threadIdx.x == 0) done_warps = 0;
  compute_bar<CW>();
  if (lane == 0 && atomicAdd(&done_warps, 1) == 0 && blockIdx.x == 0) atomicAdd(&g_trace_launch, 1);
#endif
}

// host: tensor map of one input vector for this pass (see the stage layout above)
template <int TP, int NH>
static cudaError_t tile_tensor_map(const PassParams& p, const double* X, CUtensorMap* tm) {
  RSFDE_TILE_CONSTS
  // driver entry point, fetched once (thread-safe static initialisation)
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return cudaErrorNotSupported;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], es[3] = {1, 1, 1};
  CUtensorMapSwizzle swz;
  if (p.contiguous && p.seg_lg) {
    // segmented rows: {x_l < 2^seg_lg, pencil, segment}, segment stride seg_stride; one box per tile
    const long long S = 1ll << p.seg_lg;
    dims[0] = (cuuint64_t)S; dims[1] = (cuuint64_t)(p.geo.NP / p.geo.P); dims[2] = (cuuint64_t)(NH / S);
    strides[0] = (cuuint64_t)S * 8; strides[1] = (cuuint64_t)p.seg_stride * 8;
    box[0] = (cuuint32_t)S; box[1] = kTilePencils; box[2] = (cuuint32_t)(NH / S);
    if (S > 256 || NH % S) return cudaErrorInvalidValue;
    swz = CU_TENSOR_MAP_SWIZZLE_NONE;
  } else if (p.contiguous) {
    dims[0] = (cuuint64_t)p.geo.P; dims[1] = (cuuint64_t)(p.geo.NP / p.geo.P); dims[2] = 1;
    strides[0] = dims[0] * 8; strides[1] = dims[0] * dims[1] * 8;
    box[0] = kBoxRows; box[1] = kTilePencils; box[2] = 1;
    swz = CU_TENSOR_MAP_SWIZZLE_NONE;
  } else {
    dims[0] = (cuuint64_t)p.inner; dims[1] = (cuuint64_t)p.n; dims[2] = (cuuint64_t)(p.geo.NP / ((long long)p.n * p.inner));
    strides[0] = dims[0] * 8; strides[1] = dims[0] * dims[1] * 8;
    box[0] = kTilePencils; box[1] = kBoxRows; box[2] = 1;
    swz = kTilePairs == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  }
  const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int MODE, class T, int TP, bool CT>
cudaError_t launch_tile_ct(const PassParams& p, cudaStream_t s) {
  constexpr int NH = T::N, CW = TP * T::G / 32;
  RSFDE_TILE_CONSTS
  if (p.n != T::N - 1) return cudaErrorInvalidValue;
  constexpr int kTileThreads = TileCfg<CW>::kTileThreads, kCtasPerSm = TileCfg<CW>::kCtasPerSm;
  constexpr bool OPER = MODE == MODE_OPER_SPEC || MODE == MODE_OPER_SPEC_LAST;
  const size_t smem = (size_t)kTilePairs * T::L * sizeof(double2) + kStageBytes + 1024;  // + alignment slack
  // kernel attribute and SM count, once per device (thread-safe)
  struct Tag {};
  const int sms = per_device_once<Tag>([smem](int dev) -> int {
    if (cudaFuncSetAttribute(tile_kernel<MODE, T, TP, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return -1;
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  });
  if (sms <= 0) return cudaErrorInvalidValue;
  alignas(64) CUtensorMap tmR, tmX;
  memset(&tmR, 0, sizeof(tmR));
  memset(&tmX, 0, sizeof(tmX));
  cudaError_t err = cudaSuccess;
  if (OPER) err = tile_tensor_map<TP, NH>(p, p.R, &tmR);
  if (err == cudaSuccess && (!OPER || p.xmode == X_INPUT)) err = tile_tensor_map<TP, NH>(p, p.X, &tmX);
  if (err != cudaSuccess) return err;
  const long long ntiles = p.contiguous ? ((p.geo.NP / p.geo.P) + kTilePencils - 1) / kTilePencils : (p.npairs + kTilePairs - 1) / kTilePairs;
  // (experiments: RSFDE_TILE_CTAS overrides the resident CTAs per SM of the persistent grid)
  static const int ctas_env = getenv("RSFDE_TILE_CTAS") ? atoi(getenv("RSFDE_TILE_CTAS")) : 0;
  const int cps = ctas_env > 0 ? ctas_env : kCtasPerSm;
  const long long blocks = ntiles < (long long)cps * sms ? ntiles : (long long)cps * sms;
  tile_kernel<MODE, T, TP, CT><<<(unsigned)blocks, kTileThreads, smem, s>>>(p, tmR, tmX);
  err = cudaGetLastError();
  if (err != cudaSuccess && getenv("RSFDE_DEBUG")) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, tile_kernel<MODE, T, TP, CT>);
    fprintf(stderr, "tile_kernel<%d>: regs %d maxthreads %d static %zu maxdyn %d local %zu smem %zu blocks %lld\n", MODE,
            a.numRegs, a.maxThreadsPerBlock, a.sharedSizeBytes, a.maxDynamicSharedSizeBytes, a.localSizeBytes, smem,
            blocks);
  }
  return err;
}

// contiguous (last-axis) and strided tiles are separate kernels (smaller code, fewer branches)
template <int MODE, class T, int TP>
cudaError_t launch_tile(const PassParams& p, cudaStream_t s) {
  return p.contiguous ? launch_tile_ct<MODE, T, TP, true>(p, s) : launch_tile_ct<MODE, T, TP, false>(p, s);
}

}  // namespace rsfde
