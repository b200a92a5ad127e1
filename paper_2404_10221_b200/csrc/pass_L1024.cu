// instantiation of the pencil-pass kernels for FFT length L = 1024 (n = 511, the C5 grid), with the
// warp-specialised tile pipeline (tile_kernels.cuh) for the spectral operator and DST passes
#include "tile_kernels.cuh"
namespace rsfde {
using T1024 = Lay2<32, 32>;
RSFDE_INSTANTIATE_T(T1024)

static bool tile_ok(const PassParams& p) {
  if (p.flags & PASS_FLAG_NO_PIPE) return false;
  return p.contiguous || (p.inner % kTilePencils == 0);  // a strided tile = adjacent pencils of one block
}

cudaError_t launch_oper_1024(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  if (spectral && tile_ok(p)) return last ? launch_tile<MODE_OPER_SPEC_LAST>(p, s) : launch_tile<MODE_OPER_SPEC>(p, s);
  return launch_oper_t<T1024>(p, spectral, last, s);
}

cudaError_t launch_dst_1024(const PassParams& p, bool last, cudaStream_t s) {
  if (tile_ok(p)) return last ? launch_tile<MODE_DST_LAST>(p, s) : launch_tile<MODE_DST>(p, s);
  return launch_dst_t<T1024>(p, last, s);
}
}  // namespace rsfde
