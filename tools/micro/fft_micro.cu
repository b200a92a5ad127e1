// Micro-benchmark: throughput of the in-register two-stage FFT (L = 1024, E = G = 32) without
// global memory traffic, at the production launch shape (128 threads, 4 pairs/CTA, 3 CTAs/SM).
#include <cstdio>
#include <vector>
#include "fft.cuh"
using namespace rsfde;

__global__ void __launch_bounds__(128, 3) fft_only(double2* out, const double2* tw, int reps) {
  extern __shared__ double2 smem[];
  const int g = threadIdx.x & 31, grp = threadIdx.x >> 5;
  double2* buf = smem + grp * 1024;
  double2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = make_double2(1e-3 * (g + m), 1e-3 * (blockIdx.x + m));
#pragma unroll 1
  for (int r = 0; r < reps; ++r) {
    fft_fwd<32, 32>(v, buf, g, tw);
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = c_scale(v[m], 1.0 / 1024.0);
  }
  double2 acc = make_double2(0, 0);
#pragma unroll
  for (int m = 0; m < 32; ++m) acc = c_add(acc, v[m]);
  if (acc.x == 12345.0) out[0] = acc;
}

// 8 warps per CTA, 1 CTA per SM (the tile-pipeline shape)
__global__ void __launch_bounds__(256, 1) fft_only8(double2* out, const double2* tw, int reps) {
  extern __shared__ double2 smem[];
  const int g = threadIdx.x & 31, grp = threadIdx.x >> 5;
  double2* buf = smem + grp * 1024;
  double2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = make_double2(1e-3 * (g + m), 1e-3 * (blockIdx.x + m));
#pragma unroll 1
  for (int r = 0; r < reps; ++r) {
    fft_fwd<32, 32>(v, buf, g, tw);
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = c_scale(v[m], 1.0 / 1024.0);
  }
  double2 acc = make_double2(0, 0);
#pragma unroll
  for (int m = 0; m < 32; ++m) acc = c_add(acc, v[m]);
  if (acc.x == 12345.0) out[0] = acc;
}

int main() {
  const int L = 1024;
  std::vector<double2> tw(L);
  for (int k = 0; k < L; ++k) tw[k] = make_double2(cos(2 * M_PI * k / L), -sin(2 * M_PI * k / L));
  double2 *dtw, *dout;
  cudaMalloc(&dtw, L * 16);
  cudaMalloc(&dout, 16);
  cudaMemcpy(dtw, tw.data(), L * 16, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(fft_only, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int pairs = 130816, blocks = pairs / 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fft_only<<<blocks, 128, 65536>>>(dout, dtw, 1);
  for (int reps : {1, 4}) {
    cudaEventRecord(a);
    fft_only<<<blocks, 128, 65536>>>(dout, dtw, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("reps %d: %.3f ms total, %.3f ms per full-grid FFT pass (C5: %d pairs)\n", reps, ms, ms / reps, pairs);
  }
  cudaFuncSetAttribute(fft_only8, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int reps : {1, 4}) {
    // persistent-style: 148 CTAs x 8 pairs, each CTA repeats (pairs / (148*8)) tiles via reps scaling
    const int tiles = (pairs + 148 * 8 - 1) / (148 * 8);
    cudaEventRecord(a);
    fft_only8<<<148, 256, 131072>>>(dout, dtw, reps * tiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("8 warps/SM: reps %d: %.3f ms per full-grid FFT pass\n", reps, ms / reps);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
