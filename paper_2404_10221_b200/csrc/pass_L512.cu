// instantiation of the pencil-pass kernels for FFT length L = 512 (n = 255: the C4 grid), with the
// warp-specialised tile pipeline (tile_kernels.cuh) for the spectral operator and DST passes: an FFT
// group is 16 threads, so a compute warp holds two pencil pairs and a 16-pencil tile (128-byte rows)
// four compute warps (two CTAs per SM)
#include <cstdlib>

#include "tile_kernels.cuh"
namespace rsfde {
using T512 = Lay2<32, 16>;
using T512s = Lay3<8, 8>;
RSFDE_INSTANTIATE_T(T512)
RSFDE_INSTANTIATE_T(T512s)

// Small grids (fewer pencil pairs than ~4 per SM, e.g. C2's 128 pairs per pass): the latency form,
// one pair per 64-thread CTA with E = 8 values per thread (three-stage 8 x 8 x 8 FFT, fft3.cuh),
// about 1/4 of the per-thread FP64 chain of the E = 32 tile FFT.  RSFDE_SMALL_PAIRS overrides the
// threshold (0 disables the latency form).
static bool small_512(const PassParams& p) {
  const char* v = getenv("RSFDE_SMALL_PAIRS");
  const long long lim = v ? atoll(v) : 4ll * device_sm_count();
  return p.npairs <= lim;
}

// 8 pairs per tile (a strided tile must be 16 adjacent pencils of one block); 0 = no tile pipeline
static int tile_pairs_512(const PassParams& p) {
  if (p.flags & PASS_FLAG_NO_PIPE) return 0;
  if (p.contiguous) return 8;
  return p.inner % 16 == 0 ? 8 : 0;
}

cudaError_t launch_oper_512(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  if (small_512(p)) return launch_oper_t<T512s>(p, spectral, last, s);
  if (spectral && tile_pairs_512(p))
    return last ? launch_tile<MODE_OPER_SPEC_LAST, T512, 8>(p, s) : launch_tile<MODE_OPER_SPEC, T512, 8>(p, s);
  return launch_oper_t<T512>(p, spectral, last, s);
}

cudaError_t launch_dst_512(const PassParams& p, bool last, cudaStream_t s) {
  if (small_512(p)) return launch_dst_t<T512s>(p, last, s);
  if (tile_pairs_512(p)) return last ? launch_tile<MODE_DST_LAST, T512, 8>(p, s) : launch_tile<MODE_DST, T512, 8>(p, s);
  return launch_dst_t<T512>(p, last, s);
}
}  // namespace rsfde
