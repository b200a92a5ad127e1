// instantiation of the pencil-pass kernels for FFT length L = 1024
#include "pass_kernels.cuh"
namespace rsfde {
using T1024 = Lay2<32, 32>;
RSFDE_INSTANTIATE_T(T1024)
}
