// instantiation of the pencil-pass kernels for FFT length L = 1024 (n = 511, the C5 grid), with the
// warp-specialised tile pipeline (tile_kernels.cuh) for the spectral operator and DST passes
#include "tile_kernels.cuh"
#include <cstdlib>
#include <cstring>
namespace rsfde {
using T1024 = Lay2<32, 32>;
RSFDE_INSTANTIATE_T(T1024)

// tile width in pencil pairs: 8 (one CTA of 8 compute warps per SM; 128-byte row pieces on a strided
// axis, 16 rows on the contiguous axis) wherever the geometry allows it, else 4 = 64-byte row pieces (two
// CTAs of 4 compute warps per SM), 0 = no tile pipeline (a strided tile must be adjacent pencils of one
// block).  With the axis tables in shared memory (8-warp kernels only: tile_kernels.cuh) the 8-pair tiles
// are the faster ones on every axis of the 511^3 grid (same-box A/B, last session of round 2: x2 operator
// pass 1517 -> 1462 us, inverse DST x2 524 -> 493 us; on x1, whose rows are 2 MB apart, 128-byte pieces were
// already needed for the TMA rate).  RSFDE_TILE128=0 / RSFDE_TILE_CT8=0 select the 4-pair tiles on the
// strided / contiguous axes (tests and experiments).
static int tile_pairs(const PassParams& p) {
  if (p.flags & PASS_FLAG_NO_PIPE) return 0;
  const char* ct8 = getenv("RSFDE_TILE_CT8");
  if (p.contiguous) return (ct8 && !strcmp(ct8, "0")) ? 4 : 8;
  const char* f128 = getenv("RSFDE_TILE128");
  const bool force64 = f128 && !strcmp(f128, "0");
  if (p.inner % 16 == 0 && !force64) return 8;
  return p.inner % 8 == 0 ? 4 : 0;
}

template <int MODE>
static cudaError_t launch_tile_any(const PassParams& p, int tp, cudaStream_t s) {
  return tp == 8 ? launch_tile<MODE, T1024, 8>(p, s) : launch_tile<MODE, T1024, 4>(p, s);
}

cudaError_t launch_oper_1024(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  const int tp = tile_pairs(p);
  if (spectral && tp) return last ? launch_tile_any<MODE_OPER_SPEC_LAST>(p, tp, s) : launch_tile_any<MODE_OPER_SPEC>(p, tp, s);
  return launch_oper_t<T1024>(p, spectral, last, s);
}

cudaError_t launch_dst_1024(const PassParams& p, bool last, cudaStream_t s) {
  const int tp = tile_pairs(p);
  if (tp) return last ? launch_tile_any<MODE_DST_LAST>(p, tp, s) : launch_tile_any<MODE_DST>(p, tp, s);
  return launch_dst_t<T1024>(p, last, s);
}
}  // namespace rsfde

#if RSFDE_TILE_TRACE
extern "C" int rsfde_debug_tile_trace_select(int launch) {
  int zero = 0;
  cudaMemcpyToSymbol(rsfde::g_trace_launch, &zero, sizeof(int));
  return (int)cudaMemcpyToSymbol(rsfde::g_trace_target, &launch, sizeof(int));
}
extern "C" int rsfde_debug_tile_trace(void* host) {
  return (int)cudaMemcpyFromSymbol(host, rsfde::g_tile_trace, sizeof(rsfde::g_tile_trace));
}
#endif
