// Can the kernels read pageable host memory directly (HMM / ATS)?  Prints the
// device attributes and, if pageable access is reported, times a streaming
// copy kernel from malloc'd memory to device memory (first touch and warm).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmm_probe hmm_probe.cu
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__global__ void stream_copy(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

int main() {
  int pma = 0, pmauhpt = 0, hnpma = 0, cma = 0;
  cudaDeviceGetAttribute(&pma, cudaDevAttrPageableMemoryAccess, 0);
  cudaDeviceGetAttribute(&pmauhpt, cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0);
  cudaDeviceGetAttribute(&hnpma, cudaDevAttrHostNativeAtomicSupported, 0);
  cudaDeviceGetAttribute(&cma, cudaDevAttrConcurrentManagedAccess, 0);
  printf("pageableMemoryAccess=%d usesHostPageTables=%d hostNativeAtomics=%d concurrentManagedAccess=%d\n", pma,
         pmauhpt, hnpma, cma);
  if (!pma) return 0;
  const size_t bytes = size_t(256) << 20;
  float4* h = static_cast<float4*>(malloc(bytes));
  memset(h, 1, bytes);
  float4* d;
  cudaMalloc(&d, bytes);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    stream_copy<<<148 * 8, 256>>>(h, d, bytes / 16);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("rep %d: %s, %.2f ms, %.1f GB/s\n", rep, cudaGetErrorString(e), ms, bytes / ms / 1e6);
  }
  return 0;
}
