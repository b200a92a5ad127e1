// instantiation of the pencil-pass kernels for FFT length L = 2048
#include "pass_kernels.cuh"
namespace rsfde {
using T2048 = Lay3<2>;
RSFDE_INSTANTIATE_T(T2048)
}
