// instantiation of the pencil-pass kernels for FFT length L = 8
#include "pass_kernels.cuh"
namespace rsfde {
using T8 = Lay2<4, 2>;
RSFDE_INSTANTIATE_T(T8)
}
