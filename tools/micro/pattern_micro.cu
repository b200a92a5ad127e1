// Micro-benchmark: the global access pattern of a pencil pass along the strided axis x1 of the
// C5 grid (511 x 511 x 512 doubles), no arithmetic.  Variants:
//  A: production pattern -- one 16-byte (p,q) pair per row, lane g loads rows g + 32 m
//  B/C/D: tiles of 4/8/16 pairs (64/128/256 B per row per CTA), coalesced through shared memory
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N1 = 511, N2 = 511, P = 512;
constexpr long long STRIDE = (long long)N2 * P;
constexpr long long NP = (long long)N1 * STRIDE;

__global__ void __launch_bounds__(128) pattA(const double* __restrict__ x, double* __restrict__ y) {
  const int g = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long pair = (long long)blockIdx.x * 4 + w;
  const long long off = 2 * pair;
  double2 v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = g + 32 * m;
    v[m] = (j >= 1 && j <= N1) ? __ldg(reinterpret_cast<const double2*>(x + off + (j - 1) * STRIDE)) : make_double2(0, 0);
  }
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = g + 32 * m;
    if (j >= 1 && j <= N1) *reinterpret_cast<double2*>(y + off + (j - 1) * STRIDE) = v[m];
  }
}

// A32: each warp owns 2 adjacent pairs (32 B = one sector per row); lane g loads/stores rows
// g + 32 m with two adjacent 16-byte accesses (CTA = 4 warps = 128 B per row)
__global__ void __launch_bounds__(128) pattA32(const double* __restrict__ x, double* __restrict__ y) {
  const int g = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long off = 16LL * blockIdx.x + 4 * w;
  double2 v[16], u[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = g + 32 * m;
    if (j >= 1 && j <= N1) {
      const double2* q = reinterpret_cast<const double2*>(x + off + (j - 1) * STRIDE);
      v[m] = __ldg(q);
      u[m] = __ldg(q + 1);
    }
  }
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = g + 32 * m;
    if (j >= 1 && j <= N1) {
      double2* q = reinterpret_cast<double2*>(y + off + (j - 1) * STRIDE);
      q[0] = v[m];
      q[1] = u[m];
    }
  }
}
// E: per-lane row loads (as A), stores staged through smem and written coalesced (64 B/row)
__global__ void __launch_bounds__(128) pattE(const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ double2 tile_raw[];
  double2 (*tile)[4] = reinterpret_cast<double2 (*)[4]>(tile_raw);
  const int g = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long off0 = 8LL * blockIdx.x;
  const long long off = off0 + 2 * w;
  double2 v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = g + 32 * m;
    v[m] = (j >= 1 && j <= N1) ? __ldg(reinterpret_cast<const double2*>(x + off + (j - 1) * STRIDE)) : make_double2(0, 0);
  }
#pragma unroll
  for (int m = 0; m < 16; ++m) tile[g + 32 * m][w] = v[m];
  __syncthreads();
  for (int e = threadIdx.x; e < N1 * 4; e += 128) {
    const int row = e / 4, q = e % 4;
    reinterpret_cast<double2*>(y + off0 + row * STRIDE)[q] = tile[row + 1][q];
  }
}
// F: coalesced loads through smem, per-lane row stores (as A)
__global__ void __launch_bounds__(128) pattF(const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ double2 tile_raw[];
  double2 (*tile)[4] = reinterpret_cast<double2 (*)[4]>(tile_raw);
  const int g = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long off0 = 8LL * blockIdx.x;
  for (int e = threadIdx.x; e < N1 * 4; e += 128) {
    const int row = e / 4, q = e % 4;
    tile[row + 1][q] = __ldg(reinterpret_cast<const double2*>(x + off0 + row * STRIDE) + q);
  }
  __syncthreads();
  const long long off = off0 + 2 * w;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = g + 32 * m;
    if (j >= 1 && j <= N1) *reinterpret_cast<double2*>(y + off + (j - 1) * STRIDE) = tile[j][w];
  }
}

template <int PAIRS>
__global__ void __launch_bounds__(32 * PAIRS) pattTile(const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ double2 tile_raw[];
  double2 (*tile)[PAIRS] = reinterpret_cast<double2 (*)[PAIRS]>(tile_raw);
  const long long off = 2LL * PAIRS * blockIdx.x;
  for (int e = threadIdx.x; e < N1 * PAIRS; e += blockDim.x) {
    const int row = e / PAIRS, q = e % PAIRS;
    tile[row + 1][q] = __ldg(reinterpret_cast<const double2*>(x + off + row * STRIDE) + q);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < N1 * PAIRS; e += blockDim.x) {
    const int row = e / PAIRS, q = e % PAIRS;
    reinterpret_cast<double2*>(y + off + row * STRIDE)[q] = tile[row + 1][q];
  }
}

int main() {
  double *x, *y;
  cudaMalloc(&x, NP * 8);
  cudaMalloc(&y, NP * 8);
  cudaMemset(x, 0, NP * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long long pairs = STRIDE / 2;
  float ms;
  cudaFuncSetAttribute(pattE, cudaFuncAttributeMaxDynamicSharedMemorySize, 512*4*16);
  cudaFuncSetAttribute(pattF, cudaFuncAttributeMaxDynamicSharedMemorySize, 512*4*16);
  cudaFuncSetAttribute(pattTile<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512*4*16);
  cudaFuncSetAttribute(pattTile<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512*8*16);
  cudaFuncSetAttribute(pattTile<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 512*16*16);
  const double bytes = 2.0 * 8 * N1 * STRIDE;
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(a); pattA<<<pairs / 4, 128>>>(x, y); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("A  lane-per-row, 64 B/CTA/row        %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a); pattA32<<<pairs / 8, 128>>>(x, y); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("A32 lane-per-row, 32 B/warp, 128 B/CTA %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a); pattE<<<pairs / 4, 128, 512 * 4 * 16>>>(x, y); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("E  row-per-lane loads, coalesced stores %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a); pattF<<<pairs / 4, 128, 512 * 4 * 16>>>(x, y); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("F  coalesced loads, row-per-lane stores %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a); pattTile<4><<<pairs / 4, 128, 512 * 4 * 16>>>(x, y); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("B  coalesced, 64 B/CTA/row, smem     %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a); pattTile<8><<<pairs / 8, 256, 512 * 8 * 16>>>(x, y); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("C  coalesced, 128 B/CTA/row, smem    %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a); pattTile<16><<<pairs / 16, 512, 512 * 16 * 16>>>(x, y); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("D  coalesced, 256 B/CTA/row, smem    %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a); cudaMemcpyAsync(y, x, NP * 8, cudaMemcpyDeviceToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("memcpy                                %.3f ms  %.0f GB/s\n", ms, 2.0 * 8 * NP / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
