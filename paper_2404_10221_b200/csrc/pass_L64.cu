// instantiation of the pencil-pass kernels for FFT length L = 64
#include "pass_kernels.cuh"
namespace rsfde {
using T64 = Lay2<32, 2>;
RSFDE_INSTANTIATE_T(T64)
}
