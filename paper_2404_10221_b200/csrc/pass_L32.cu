// instantiation of the pencil-pass kernels for FFT length L = 32
#include "pass_kernels.cuh"
namespace rsfde {
RSFDE_INSTANTIATE_L(16, 2)
}
