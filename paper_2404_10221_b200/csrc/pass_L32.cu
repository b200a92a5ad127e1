// instantiation of the pencil-pass kernels for FFT length L = 32
#include "pass_kernels.cuh"
namespace rsfde {
using T32 = Lay2<16, 2>;
RSFDE_INSTANTIATE_T(T32)
}
