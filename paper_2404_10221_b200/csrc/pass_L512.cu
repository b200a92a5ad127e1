// instantiation of the pencil-pass kernels for FFT length L = 512
#include "pass_kernels.cuh"
namespace rsfde {
using T512 = Lay2<32, 16>;
RSFDE_INSTANTIATE_T(T512)
}
