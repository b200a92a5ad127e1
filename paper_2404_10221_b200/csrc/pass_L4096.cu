// instantiation of the pencil-pass kernels for FFT length L = 4096
#include "pass_kernels.cuh"
namespace rsfde {
using T4096 = Lay3<4>;
RSFDE_INSTANTIATE_T(T4096)
}
