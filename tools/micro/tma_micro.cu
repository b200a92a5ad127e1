// Micro-benchmark: TMA (cp.async.bulk.tensor) read throughput for the strided-axis tile pattern of
// the C5 grid (511 x 511 x 512 doubles, pass along x1 = stride 2 MB): boxes {P pencils, 256 rows}
// streamed into a ring of S shared stages by one thread per CTA, no consumers (each stage is
// re-armed as soon as it lands).  Prints GB/s per (pencils per box, stages, CTAs per SM).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void tma_read(const __grid_constant__ CUtensorMap tm, int inner, int n, int outer, int pencils,
                         int stages, long long ntiles, unsigned box_bytes, double* sink) {
  extern __shared__ __align__(1024) char sm_raw[];
  char* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) unsigned long long bar[8];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const unsigned stage_bytes = 2 * box_bytes;
  long long it = 0;
  unsigned phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double acc = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = (int)(it % stages);
    if (it >= stages) {
      asm volatile(
          "{.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}" ::"r"(
              su32(&bar[s])),
          "r"(phase[s])
          : "memory");
      phase[s] ^= 1;
      acc += *reinterpret_cast<const double*>(sm + (size_t)s * stage_bytes);
    }
    const long long pen = (long long)pencils * t;
    const int o = (int)(pen / inner), i = (int)(pen % inner);
    char* dst = sm + (size_t)s * stage_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(stage_bytes)
                 : "memory");
    for (int b = 0; b < 2; ++b)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4}], [%5];" ::"r"(su32(dst + b * box_bytes)),
          "l"(&tm), "r"(i), "r"(b * 256), "r"(o), "r"(su32(&bar[s]))
          : "memory");
  }
  // drain
  for (long long k = (it > stages ? it - stages : 0); k < it; ++k) {
    const int s = (int)(k % stages);
    asm volatile(
        "{.reg .pred P1;\nW2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W2;\n}" ::"r"(
            su32(&bar[s])),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const int n = 511, P = 512;
  const long long NP = (long long)n * n * P;
  double* X;
  double* sink;
  cudaMalloc(&X, NP * 8);
  cudaMalloc(&sink, 8);
  cudaMemset(X, 0, NP * 8);
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int axis = 0; axis < 0; ++axis) {
    // axis 0: inner = n*P (stride 2 MB), outer 1; axis 1: inner = P (stride 4 KB), outer n
    const long long inner = axis == 0 ? (long long)n * P : P, outer = axis == 0 ? 1 : n;
    for (int pencils : {4, 8, 16, 32}) {
      CUtensorMap tm;
      cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)n, (cuuint64_t)outer};
      cuuint64_t strides[2] = {(cuuint64_t)inner * 8, (cuuint64_t)inner * n * 8};
      cuuint32_t box[3] = {(cuuint32_t)pencils, 256, 1}, es[3] = {1, 1, 1};
      CUtensorMapSwizzle swz = pencils == 4 ? CU_TENSOR_MAP_SWIZZLE_32B
                               : pencils == 8 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_128B;
      if (pencils == 32) swz = CU_TENSOR_MAP_SWIZZLE_NONE;
      CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d (pencils %d)\n", (int)r, pencils); continue; }
      const unsigned box_bytes = pencils * 8 * 256;
      const long long ntiles = inner * outer / pencils;
      for (int stages : {1, 2, 3, 4}) {
        for (int cps : {1, 2, 4}) {
          const size_t smem = (size_t)stages * 2 * box_bytes + 1024;
          if (smem * cps > 220 * 1024) continue;
          tma_read<<<sms * cps, 32, smem>>>(tm, (int)inner, n, (int)outer, pencils, stages, ntiles, box_bytes, sink);
          cudaEventRecord(a);
          tma_read<<<sms * cps, 32, smem>>>(tm, (int)inner, n, (int)outer, pencils, stages, ntiles, box_bytes, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          printf("axis %d pencils %2d (%3d B rows) stages %d ctas/SM %d: %.3f ms  %.0f GB/s\n", axis, pencils,
                 pencils * 8, stages, cps, ms, NP * 8 / (ms * 1e-3) / 1e9);
        }
      }
    }
  }
  // axis 0 (plane stride n*P + pad doubles): does breaking the power-of-two plane stride help?
  for (int pad : {0, 16, 32, 64, 128, 256, 512}) {
    const long long inner = (long long)n * P, outer = 1, pitch = inner + pad;
    if (pitch * n > NP + 0) {
      // reuse X: the last rows fall outside the allocation for pad > 0 -> use fewer rows
    }
    const int rows = (int)((NP) / pitch);
    for (int pencils : {8, 16}) {
      CUtensorMap tm;
      cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)outer};
      cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * rows * 8};
      cuuint32_t box[3] = {(cuuint32_t)pencils, 256, 1}, es[3] = {1, 1, 1};
      CUtensorMapSwizzle swz = pencils == 8 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
      CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
      const unsigned box_bytes = pencils * 8 * 256;
      const long long ntiles = inner / pencils;
      for (int stages : {1, 2}) {
        for (int cps : {2, 4}) {
          const size_t smem = (size_t)stages * 2 * box_bytes + 1024;
          if (smem * cps > 220 * 1024) continue;
          tma_read<<<sms * cps, 32, smem>>>(tm, (int)inner, rows, (int)outer, pencils, stages, ntiles, box_bytes, sink);
          cudaEventRecord(a);
          tma_read<<<sms * cps, 32, smem>>>(tm, (int)inner, rows, (int)outer, pencils, stages, ntiles, box_bytes, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double bytes = (double)inner * 512 * 8;  // two boxes of 256 rows per tile
          printf("axis 0 pad %4d pencils %2d stages %d ctas/SM %d: %.3f ms  %.0f GB/s\n", pad, pencils, stages, cps, ms,
                 bytes / (ms * 1e-3) / 1e9);
        }
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
