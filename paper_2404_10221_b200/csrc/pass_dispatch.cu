// FFT-length dispatch of the pencil-pass launchers (instantiations live in pass_L*.cu)
#include "pass_kernels.cuh"

namespace rsfde {

cudaError_t launch_oper_1024(const PassParams& p, bool spectral, bool last, cudaStream_t s);
cudaError_t launch_dst_1024(const PassParams& p, bool last, cudaStream_t s);
cudaError_t launch_oper_512(const PassParams& p, bool spectral, bool last, cudaStream_t s);
cudaError_t launch_dst_512(const PassParams& p, bool last, cudaStream_t s);
cudaError_t launch_oper_2048(const PassParams& p, bool spectral, bool last, cudaStream_t s);
cudaError_t launch_dst_2048(const PassParams& p, bool last, cudaStream_t s);
cudaError_t launch_oper_4096(const PassParams& p, bool spectral, bool last, cudaStream_t s);
cudaError_t launch_dst_4096(const PassParams& p, bool last, cudaStream_t s);
extern template cudaError_t launch_oper_t<Lay2<2, 2>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<2, 2>>(const PassParams&, bool, cudaStream_t);
extern template cudaError_t launch_oper_t<Lay2<4, 2>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<4, 2>>(const PassParams&, bool, cudaStream_t);
extern template cudaError_t launch_oper_t<Lay2<8, 2>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<8, 2>>(const PassParams&, bool, cudaStream_t);
extern template cudaError_t launch_oper_t<Lay2<16, 2>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<16, 2>>(const PassParams&, bool, cudaStream_t);
extern template cudaError_t launch_oper_t<Lay2<32, 2>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<32, 2>>(const PassParams&, bool, cudaStream_t);
extern template cudaError_t launch_oper_t<Lay2<32, 4>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<32, 4>>(const PassParams&, bool, cudaStream_t);
extern template cudaError_t launch_oper_t<Lay2<32, 8>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<32, 8>>(const PassParams&, bool, cudaStream_t);
extern template cudaError_t launch_oper_t<Lay2<32, 16>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<32, 16>>(const PassParams&, bool, cudaStream_t);
extern template cudaError_t launch_oper_t<Lay2<32, 32>>(const PassParams&, bool, bool, cudaStream_t);
extern template cudaError_t launch_dst_t<Lay2<32, 32>>(const PassParams&, bool, cudaStream_t);

cudaError_t launch_oper_pass(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  switch (p.L) {
    case 4: return launch_oper_t<Lay2<2, 2>>(p, spectral, last, s);
    case 8: return launch_oper_t<Lay2<4, 2>>(p, spectral, last, s);
    case 16: return launch_oper_t<Lay2<8, 2>>(p, spectral, last, s);
    case 32: return launch_oper_t<Lay2<16, 2>>(p, spectral, last, s);
    case 64: return launch_oper_t<Lay2<32, 2>>(p, spectral, last, s);
    case 128: return launch_oper_t<Lay2<32, 4>>(p, spectral, last, s);
    case 256: return launch_oper_t<Lay2<32, 8>>(p, spectral, last, s);
    case 512: return launch_oper_512(p, spectral, last, s);
    case 1024: return launch_oper_1024(p, spectral, last, s);
    case 2048: return launch_oper_2048(p, spectral, last, s);
    case 4096: return launch_oper_4096(p, spectral, last, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_dst_pass(const PassParams& p, bool last, cudaStream_t s) {
  switch (p.L) {
    case 4: return launch_dst_t<Lay2<2, 2>>(p, last, s);
    case 8: return launch_dst_t<Lay2<4, 2>>(p, last, s);
    case 16: return launch_dst_t<Lay2<8, 2>>(p, last, s);
    case 32: return launch_dst_t<Lay2<16, 2>>(p, last, s);
    case 64: return launch_dst_t<Lay2<32, 2>>(p, last, s);
    case 128: return launch_dst_t<Lay2<32, 4>>(p, last, s);
    case 256: return launch_dst_t<Lay2<32, 8>>(p, last, s);
    case 512: return launch_dst_512(p, last, s);
    case 1024: return launch_dst_1024(p, last, s);
    case 2048: return launch_dst_2048(p, last, s);
    case 4096: return launch_dst_4096(p, last, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rsfde
