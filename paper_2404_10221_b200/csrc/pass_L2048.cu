// instantiation of the pencil-pass kernels for FFT length L = 2048 (n = 1023): three-stage FFT with
// E = 16 over 128 threads per pair (default) or E = 32 over 64 threads (RSFDE_FFT3_E=32)
#include "pass_kernels.cuh"
namespace rsfde {
using T2048 = Lay3<32, 2>;
using T2048h = Lay3<16, 8>;
RSFDE_INSTANTIATE_T(T2048)
RSFDE_INSTANTIATE_T(T2048h)

bool fft3_e32();

cudaError_t launch_oper_2048(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  return fft3_e32() ? launch_oper_t<T2048>(p, spectral, last, s) : launch_oper_t<T2048h>(p, spectral, last, s);
}
cudaError_t launch_dst_2048(const PassParams& p, bool last, cudaStream_t s) {
  return fft3_e32() ? launch_dst_t<T2048>(p, last, s) : launch_dst_t<T2048h>(p, last, s);
}
}  // namespace rsfde
