// instantiation of the pencil-pass kernels for FFT length L = 1024 (n = 511, the C5 grid), with the
// warp-specialised tile pipeline (tile_kernels.cuh) for the spectral operator and DST passes
#include "tile_kernels.cuh"
#include <cstdlib>
#include <cstring>
namespace rsfde {
using T1024 = Lay2<32, 32>;
RSFDE_INSTANTIATE_T(T1024)

// tile width in pencil pairs: 8 = 128-byte rows (one CTA of 8 compute warps per SM), 4 = 64-byte rows
// (two CTAs of 4 compute warps per SM), 0 = no tile pipeline (a strided tile must be adjacent pencils
// of one block)
static int tile_pairs(const PassParams& p) {
  if (p.flags & PASS_FLAG_NO_PIPE) return 0;
  const char* ct8 = getenv("RSFDE_TILE_CT8");  // contiguous axis: 8-pair tiles (x3 oper pass 1.82 -> 1.62 ms same-box; RSFDE_TILE_CT8=0: 4-pair tiles)
  if (p.contiguous) return (ct8 && !strcmp(ct8, "0")) ? 4 : 8;
  // 128-byte rows where rows are >= 1 MB apart (x1 of the C5 grid: every row piece is its own 2 MB
  // page and the TMA rate follows the row-piece count; measured 2 % faster K chain).
  // RSFDE_TILE128=1 forces them on every eligible strided pass (test coverage at small sizes).
  const char* f128 = getenv("RSFDE_TILE128");
  const bool force128 = f128 && strcmp(f128, "0");
  const bool force64 = f128 && !strcmp(f128, "0");  // (experiments: 64-byte tiles everywhere)
  if (p.inner % 16 == 0 && !force64 && (force128 || p.stride * 8 >= (1ll << 20))) return 8;
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
