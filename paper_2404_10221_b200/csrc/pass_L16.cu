// instantiation of the pencil-pass kernels for FFT length L = 16
#include "pass_kernels.cuh"
namespace rsfde {
using T16 = Lay2<8, 2>;
RSFDE_INSTANTIATE_T(T16)
}
