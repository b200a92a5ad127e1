// instantiation of the pencil-pass kernels for FFT length L = 4
#include "pass_kernels.cuh"
namespace rsfde {
using T4 = Lay2<2, 2>;
RSFDE_INSTANTIATE_T(T4)
}
