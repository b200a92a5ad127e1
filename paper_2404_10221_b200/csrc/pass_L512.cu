// instantiation of the pencil-pass kernels for FFT length L = 512 (n = 255: the C4 grid), with the
// warp-specialised tile pipeline (tile_kernels.cuh) for the spectral operator and DST passes: an FFT
// group is 16 threads, so a compute warp holds two pencil pairs and a 16-pencil tile (128-byte rows)
// four compute warps (two CTAs per SM)
#include "tile_kernels.cuh"
namespace rsfde {
using T512 = Lay2<32, 16>;
RSFDE_INSTANTIATE_T(T512)

// 8 pairs per tile (a strided tile must be 16 adjacent pencils of one block); 0 = no tile pipeline
static int tile_pairs_512(const PassParams& p) {
  if (p.flags & PASS_FLAG_NO_PIPE) return 0;
  if (p.contiguous) return 8;
  return p.inner % 16 == 0 ? 8 : 0;
}

cudaError_t launch_oper_512(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  if (spectral && tile_pairs_512(p))
    return last ? launch_tile<MODE_OPER_SPEC_LAST, T512, 8>(p, s) : launch_tile<MODE_OPER_SPEC, T512, 8>(p, s);
  return launch_oper_t<T512>(p, spectral, last, s);
}

cudaError_t launch_dst_512(const PassParams& p, bool last, cudaStream_t s) {
  if (tile_pairs_512(p)) return last ? launch_tile<MODE_DST_LAST, T512, 8>(p, s) : launch_tile<MODE_DST, T512, 8>(p, s);
  return launch_dst_t<T512>(p, last, s);
}
}  // namespace rsfde
