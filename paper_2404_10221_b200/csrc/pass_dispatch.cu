// FFT-length dispatch of the pencil-pass launchers (instantiations live in pass_L*.cu)
#include "pass_kernels.cuh"

namespace rsfde {

#define RSFDE_DECL_L(E, G)                                                                   \
  extern template cudaError_t launch_oper_eg<E, G>(const PassParams&, bool, bool, cudaStream_t); \
  extern template cudaError_t launch_dst_eg<E, G>(const PassParams&, bool, cudaStream_t);
RSFDE_DECL_L(2, 2)
RSFDE_DECL_L(4, 2)
RSFDE_DECL_L(8, 2)
RSFDE_DECL_L(16, 2)
RSFDE_DECL_L(32, 2)
RSFDE_DECL_L(32, 4)
RSFDE_DECL_L(32, 8)
RSFDE_DECL_L(32, 16)
RSFDE_DECL_L(32, 32)

#define RSFDE_L_CASES(M, ...)                \
  switch (p.L) {                             \
    case 4: return M<2, 2>(__VA_ARGS__); \
    case 8: return M<4, 2>(__VA_ARGS__); \
    case 16: return M<8, 2>(__VA_ARGS__); \
    case 32: return M<16, 2>(__VA_ARGS__); \
    case 64: return M<32, 2>(__VA_ARGS__); \
    case 128: return M<32, 4>(__VA_ARGS__); \
    case 256: return M<32, 8>(__VA_ARGS__); \
    case 512: return M<32, 16>(__VA_ARGS__); \
    case 1024: return M<32, 32>(__VA_ARGS__); \
    default: return cudaErrorInvalidValue;   \
  }

cudaError_t launch_oper_pass(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  RSFDE_L_CASES(launch_oper_eg, p, spectral, last, s)
}

cudaError_t launch_dst_pass(const PassParams& p, bool last, cudaStream_t s) {
  RSFDE_L_CASES(launch_dst_eg, p, last, s)
}

}  // namespace rsfde
