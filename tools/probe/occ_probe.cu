// Occupancy probe (development tool, not product code): times stockham_kernel
// variants on a 1 GiB -> 1 GiB batch while capping the resident CTAs per SM
// with extra dynamic shared memory, to find how many bytes in flight per SM
// the kernels want.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o occ_probe occ_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2203_09384_b200/csrc/sfft_kernels.cuh"

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

template <typename T, int N, int R, int SEQ, int LAYOUT, int TWP, int LOADER>
void run(const char* name, void* in, void* out, void* tw, size_t bytes) {
  using C = sfft::cx_t<T>;
  auto k = sfft::stockham_kernel<T, N, R, SEQ, false, LAYOUT, TWP, LOADER>;
  constexpr int threads = (N / R) * SEQ;
  const int base = SEQ * sfft::Smem<T, LAYOUT, R>::size(N) * int(sizeof(C));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const long long batch = (long long)(bytes / (N * sizeof(C)));
  const unsigned grid = unsigned((batch + SEQ - 1) / SEQ);
  int maxb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, k, threads, base);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  printf("%s regs=%d smem=%d max_ctas_per_sm=%d\n", name, fa.numRegs, base, maxb);
  for (int cap = 2; cap <= maxb + 1; cap += (cap < 8 ? 1 : 2)) {
    const int c = cap > maxb ? maxb : cap;
    int smem = base;
    if (c < maxb) smem = (220 * 1024) / c - 1024;  // 228 KB per SM, ~1 KB reserved per CTA
    if (smem < base) smem = base;
    int got = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&got, k, threads, smem);
    const float ms = time_it([&] {
      k<<<grid, threads, smem>>>(static_cast<const C*>(in), static_cast<C*>(out), static_cast<const C*>(tw),
                                 batch, nullptr);
    });
    printf("  ctas/sm=%2d (%3d warps) inflight/SM=%6.1f KB  %.1f us  %.1f GB/s\n", got, got * threads / 32,
           got * SEQ * N * sizeof(C) / 1024.0, ms * 1e3, 2.0 * bytes / (ms * 1e-3) / 1e9);
    if (c == maxb) break;
  }
}

// Same kernel at its own smem size, with the L1/shared carveout preference
// swept (percent of the max shared memory); reports resident CTAs per SM.
template <typename T, int N, int R, int SEQ, int LAYOUT, int TWP, int LOADER>
void carve(const char* name, void* in, void* out, void* tw, size_t bytes) {
  using C = sfft::cx_t<T>;
  auto k = sfft::stockham_kernel<T, N, R, SEQ, false, LAYOUT, TWP, LOADER>;
  constexpr int threads = (N / R) * SEQ;
  const int smem = SEQ * sfft::Smem<T, LAYOUT, R>::size(N) * int(sizeof(C));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const long long batch = (long long)(bytes / (N * sizeof(C)));
  const unsigned grid = unsigned((batch + SEQ - 1) / SEQ);
  printf("%s carveout sweep (smem/CTA %d B)\n", name, smem);
  for (int pct : {-1, 25, 40, 50, 60, 70, 80, 100}) {
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    int got = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&got, k, threads, smem);
    const float ms = time_it([&] {
      k<<<grid, threads, smem>>>(static_cast<const C*>(in), static_cast<C*>(out), static_cast<const C*>(tw),
                                 batch, nullptr);
    });
    printf("  carveout=%4d%% occ_api=%2d  %.1f us  %.1f GB/s\n", pct, got, ms * 1e3,
           2.0 * bytes / (ms * 1e-3) / 1e9);
  }
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, -1);
}

int main() {
  const size_t bytes = size_t(1) << 30;
  void *in, *out, *tw;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMalloc(&tw, 1 << 20);
  cudaMemset(in, 0, bytes);
  cudaMemset(tw, 0, 1 << 20);
  run<float, 1024, 32, 2, 1, 1, 1>("f32 N1024 R32 S2 TMA", in, out, tw, bytes);
  run<float, 1024, 32, 2, 1, 1, 0>("f32 N1024 R32 S2", in, out, tw, bytes);
  run<float, 1024, 32, 4, 1, 1, 0>("f32 N1024 R32 S4", in, out, tw, bytes);
  run<float, 1024, 16, 1, 1, 1, 1>("f32 N1024 R16 S1 TMA", in, out, tw, bytes);
  run<float, 1024, 16, 1, 1, 1, 0>("f32 N1024 R16 S1", in, out, tw, bytes);
  run<float, 2048, 16, 1, 1, 1, 0>("f32 N2048 R16 S1", in, out, tw, bytes);
  run<float, 2048, 16, 1, 1, 1, 1>("f32 N2048 R16 S1 TMA", in, out, tw, bytes);
  run<float, 512, 16, 4, 1, 1, 0>("f32 N512 R16 S4", in, out, tw, bytes);
  run<double, 2048, 16, 1, 0, 1, 0>("f64 N2048 R16 S1", in, out, tw, bytes);
  run<double, 1024, 16, 2, 0, 1, 0>("f64 N1024 R16 S2", in, out, tw, bytes);
  carve<float, 1024, 32, 2, 1, 1, 0>("f32 N1024 R32 S2", in, out, tw, bytes);
  carve<float, 1024, 32, 2, 1, 1, 1>("f32 N1024 R32 S2 TMA", in, out, tw, bytes);
  carve<float, 1024, 16, 1, 1, 1, 1>("f32 N1024 R16 S1 TMA", in, out, tw, bytes);
  carve<float, 1024, 16, 1, 1, 1, 0>("f32 N1024 R16 S1", in, out, tw, bytes);
  carve<float, 2048, 16, 1, 1, 1, 0>("f32 N2048 R16 S1", in, out, tw, bytes);
  carve<float, 2048, 16, 1, 1, 1, 1>("f32 N2048 R16 S1 TMA", in, out, tw, bytes);
  carve<double, 2048, 16, 1, 0, 1, 0>("f64 N2048 R16 S1", in, out, tw, bytes);
  carve<double, 2048, 16, 1, 0, 1, 1>("f64 N2048 R16 S1 TMA", in, out, tw, bytes);
  carve<double, 1024, 16, 2, 0, 1, 0>("f64 N1024 R16 S2", in, out, tw, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
