// Do warp shuffles share the L1 data pipe with shared-memory accesses?
// Three loops per thread -- SHFL only, LDS.128 only, both interleaved -- timed
// with clock64() on a full SM (1024 threads).  If the mixed loop takes about
// max(shfl, lds) cycles the two use separate datapaths; about the sum, the
// same one.  (Decides whether an in-warp exchange by shuffles could relieve
// the data pipe that limits the fp64 N=2048 kernel, profiles/r02_fp64_2048_datapipe.txt.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl_probe shfl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int MODE>  // 0 shfl, 1 lds, 2 both
__global__ void probe(float* out, long long* cycles) {
  __shared__ float4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x;
  const long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    if (MODE != 1) {
      // 4 independent 32-bit shuffles = one 16-byte value per lane
      a0 = __shfl_xor_sync(0xffffffffu, a0, 1);
      a1 = __shfl_xor_sync(0xffffffffu, a1, 2);
      a2 = __shfl_xor_sync(0xffffffffu, a2, 4);
      a3 = __shfl_xor_sync(0xffffffffu, a3, 8);
    }
    if (MODE != 0) {
      // one conflict-free 16-byte shared load per lane (4 wavefronts per warp)
      const float4 v = buf[(idx + i * 32) & 2047];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + acc.x + acc.y + acc.z + acc.w;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
double run(int sms) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * 1024);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  probe<MODE><<<sms, 1024>>>(out, cyc);
  probe<MODE><<<sms, 1024>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  cudaFree(out);
  cudaFree(cyc);
  return double(mx);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double warp_iters = 32.0 * ITERS;  // 32 warps per SM
  const double s = run<0>(sms), l = run<1>(sms), b = run<2>(sms);
  printf("shfl only: %.0f cycles (%.2f SHFL.32 warp-instr/clk/SM)\n", s, 4 * warp_iters / s);
  printf("lds only : %.0f cycles (%.2f LDS.128 warp-instr/clk/SM = %.2f wavefronts/clk)\n", l, warp_iters / l,
         4 * warp_iters / l);
  printf("both     : %.0f cycles (sum %.0f, max %.0f)\n", b, s + l, s > l ? s : l);
  return 0;
}
