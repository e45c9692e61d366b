// HBM ceiling probe (development tool, not product code): streaming kernels
// with different access shapes, to learn what read+write bandwidth a B200
// sustains for a 1 GiB -> 1 GiB pass.
#include <cstdio>
#include <cuda_runtime.h>

template <int VEC, int UNROLL, bool CS>
__global__ void copy_k(const char* __restrict__ in, char* __restrict__ out, size_t n_vec) {
  using V = typename std::conditional<VEC == 16, float4, typename std::conditional<VEC == 8, float2, float>::type>::type;
  const V* a = reinterpret_cast<const V*>(in);
  V* b = reinterpret_cast<V*>(out);
  size_t i = (size_t)blockIdx.x * blockDim.x * UNROLL + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x * UNROLL;
  for (; i < n_vec; i += stride) {
    V r[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      size_t k = i + (size_t)u * blockDim.x;
      if (k < n_vec) r[u] = CS ? __ldcs(a + k) : a[k];
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      size_t k = i + (size_t)u * blockDim.x;
      if (k < n_vec) { if (CS) __stcs(b + k, r[u]); else b[k] = r[u]; }
    }
  }
}

__global__ void read_k(const float4* __restrict__ a, size_t n, float* sink) {
  float acc = 0.f;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(a + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 123.456f) *sink = acc;
}
__global__ void write_k(float4* __restrict__ a, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(a + i, make_float4(1.f, 2.f, 3.f, 4.f));
}

template <typename F>
float time_it(F f, int iters = 20) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / iters;
}

int main() {
  const size_t bytes = size_t(1) << 30;
  char *in, *out; float* sink;
  cudaMalloc(&in, bytes); cudaMalloc(&out, bytes); cudaMalloc(&sink, 4);
  cudaMemset(in, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char* name, float ms, double traffic) { printf("%-40s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, traffic / (ms * 1e-3) / 1e9); };
  for (int blocks_per_sm : {4, 8, 16, 32}) {
    for (int threads : {256, 512}) {
      int grid = sms * blocks_per_sm;
      char name[128];
      sprintf(name, "copy16 u4 cs grid=%dx%d t=%d", sms, blocks_per_sm, threads);
      rep(name, time_it([&] { copy_k<16, 4, true><<<grid, threads>>>(in, out, bytes / 16); }), 2.0 * bytes);
    }
  }
  int grid = sms * 16;
  rep("copy16 u1 cs", time_it([&] { copy_k<16, 1, true><<<grid, 256>>>(in, out, bytes / 16); }), 2.0 * bytes);
  rep("copy16 u8 cs", time_it([&] { copy_k<16, 8, true><<<grid, 256>>>(in, out, bytes / 16); }), 2.0 * bytes);
  rep("copy16 u4 default cache", time_it([&] { copy_k<16, 4, false><<<grid, 256>>>(in, out, bytes / 16); }), 2.0 * bytes);
  rep("copy8 u8 cs", time_it([&] { copy_k<8, 8, true><<<grid, 256>>>(in, out, bytes / 8); }), 2.0 * bytes);
  rep("copy4 u8 cs", time_it([&] { copy_k<4, 8, true><<<grid, 256>>>(in, out, bytes / 4); }), 2.0 * bytes);
  rep("copy16 one-shot grid (no loop)", time_it([&] { copy_k<16, 4, true><<<unsigned(bytes / 16 / 1024), 256>>>(in, out, bytes / 16); }), 2.0 * bytes);
  rep("read-only 16B", time_it([&] { read_k<<<grid, 256>>>(reinterpret_cast<const float4*>(in), bytes / 16, sink); }), 1.0 * bytes);
  rep("write-only 16B", time_it([&] { write_k<<<grid, 256>>>(reinterpret_cast<float4*>(out), bytes / 16); }), 1.0 * bytes);
  rep("cudaMemcpyD2D", time_it([&] { cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice); }), 2.0 * bytes);
  return 0;
}
