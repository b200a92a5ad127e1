// instantiation of the pencil-pass kernels for FFT length L = 256
#include "pass_kernels.cuh"
namespace rsfde {
RSFDE_INSTANTIATE_L(32, 8)
}
