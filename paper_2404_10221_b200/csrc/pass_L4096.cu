// instantiation of the pencil-pass kernels for FFT length L = 4096 (n = 2047: BASELINE C3).
// Two three-stage FFT forms (fft3.cuh): E = 16 values per thread over 256 threads per pencil pair
// (default: half the per-pair latency and registers of the E = 32 form, so more pairs in flight),
// and E = 32 over 128 threads (RSFDE_FFT3_E=32, the round-1 form).
#include <cstdlib>
#include <cstring>

#include "pass_kernels.cuh"
namespace rsfde {
using T4096 = Lay3<32, 4>;
using T4096h = Lay3<16, 16>;
RSFDE_INSTANTIATE_T(T4096)
RSFDE_INSTANTIATE_T(T4096h)

void row_layout_4096(int* idx) {
  for (int r = 0; r < T4096h::E; ++r)
    for (int t = 0; t < T4096h::G; ++t) idx[r * T4096h::G + t] = T4096h::FT::rowk(t, r);
}

bool fft3_e32() {
  const char* v = getenv("RSFDE_FFT3_E");  // (read per call: tests toggle it)
  return v && !strcmp(v, "32");
}

cudaError_t launch_oper_4096(const PassParams& p, bool spectral, bool last, cudaStream_t s) {
  return fft3_e32() ? launch_oper_t<T4096>(p, spectral, last, s) : launch_oper_t<T4096h>(p, spectral, last, s);
}
cudaError_t launch_dst_4096(const PassParams& p, bool last, cudaStream_t s) {
  return fft3_e32() ? launch_dst_t<T4096>(p, last, s) : launch_dst_t<T4096h>(p, last, s);
}
}  // namespace rsfde
