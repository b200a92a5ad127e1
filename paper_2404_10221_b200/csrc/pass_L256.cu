// instantiation of the pencil-pass kernels for FFT length L = 256
#include "pass_kernels.cuh"
namespace rsfde {
using T256 = Lay2<32, 8>;
RSFDE_INSTANTIATE_T(T256)
}
