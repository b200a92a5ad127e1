// instantiation of the pencil-pass kernels for FFT length L = 128
#include "pass_kernels.cuh"
namespace rsfde {
using T128 = Lay2<32, 4>;
RSFDE_INSTANTIATE_T(T128)
}
