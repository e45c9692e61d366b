// Copy-ceiling probe for bulk (TMA) copies (development tool, not product
// code): does moving a tile HBM -> smem -> HBM with cp.async.bulk in both
// directions beat per-thread 16-byte LDG/STG streaming?  1 GiB in + 1 GiB out.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_copy_probe tma_copy_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <typename F>
float time_it(F f, int iters = 20) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / iters;
}

// LOAD 0: per-thread 16 B LDG.cs into registers, then STS into the tile
// LOAD 1: one bulk G2S copy (mbarrier)
// STORE 0: per-thread LDS + 16 B STG.cs
// STORE 1: one bulk S2G copy (bulk_group), waited on before exit
template <int LOAD, int STORE>
__global__ void tile_copy(const char* __restrict__ in, char* __restrict__ out, int tile) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  const size_t base = size_t(blockIdx.x) * tile;
  if constexpr (LOAD == 1) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(tile) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       s32(sm)),
                   "l"(in + base), "r"(tile), "r"(s32(&bar))
                   : "memory");
    }
    __syncthreads();
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done)
                   : "r"(s32(&bar))
                   : "memory");
    }
  } else {
    const float4* src = reinterpret_cast<const float4*>(in + base);
    float4* dst = reinterpret_cast<float4*>(sm);
    const int n = tile / 16;
    float4 r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = threadIdx.x + i * blockDim.x;
      if (k < n) r[i] = __ldcs(src + k);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = threadIdx.x + i * blockDim.x;
      if (k < n) dst[k] = r[i];
    }
    __syncthreads();
  }
  if constexpr (STORE == 1) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + base), "r"(s32(sm)),
                   "r"(tile)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  } else {
    const float4* src = reinterpret_cast<const float4*>(sm);
    float4* dst = reinterpret_cast<float4*>(out + base);
    const int n = tile / 16;
    for (int k = threadIdx.x; k < n; k += blockDim.x) __stcs(dst + k, src[k]);
  }
}

int main() {
  const size_t bytes = size_t(1) << 30;
  char *in, *out;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMemset(in, 1, bytes);
  auto rep = [&](const char* name, int tile, int threads, float ms) {
    printf("%-34s tile=%6d thr=%4d %8.1f us %7.1f GB/s\n", name, tile, threads, ms * 1e3, 2.0 * bytes / (ms * 1e-3) / 1e9);
  };
  for (int tile : {8192, 16384, 32768}) {
    for (int threads : {64, 128, 256}) {
      if (tile / 16 > threads * 16) continue;  // LOAD 0 holds 16 float4 per thread
      const unsigned grid = unsigned(bytes / tile);
      cudaFuncSetAttribute(tile_copy<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile);
      cudaFuncSetAttribute(tile_copy<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile);
      cudaFuncSetAttribute(tile_copy<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile);
      cudaFuncSetAttribute(tile_copy<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile);
      rep("LDG->smem->STG", tile, threads, time_it([&] { tile_copy<0, 0><<<grid, threads, tile>>>(in, out, tile); }));
      rep("bulk G2S->smem->STG", tile, threads, time_it([&] { tile_copy<1, 0><<<grid, threads, tile>>>(in, out, tile); }));
      rep("LDG->smem->bulk S2G", tile, threads, time_it([&] { tile_copy<0, 1><<<grid, threads, tile>>>(in, out, tile); }));
      rep("bulk G2S->smem->bulk S2G", tile, threads, time_it([&] { tile_copy<1, 1><<<grid, threads, tile>>>(in, out, tile); }));
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
