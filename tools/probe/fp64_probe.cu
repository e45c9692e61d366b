// FP64 pipe throughput on this part: DFMA / DADD / DMUL warp-instructions per
// SM per clock, measured with clock64() inside the kernel (independent of the
// SM clock the power state picks).  Used to decide whether the fp64 N=2048
// FFT kernel (640 FP64 instructions per thread) is FP64-pipe bound.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;     // independent dependency chains per thread
constexpr int ITERS = 4096;   // loop trips; each trip issues CHAINS ops

template <int OP>
__global__ void fp64_loop(double* out, long long* cycles, double a, double b) {
  double v[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) v[c] = __fma_rn(v[c], a, b);
      if (OP == 1) v[c] = __dadd_rn(v[c], b);
      if (OP == 2) v[c] = __dmul_rn(v[c], a);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int sms, int threads) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * sms * threads);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  fp64_loop<OP><<<sms, threads>>>(out, cyc, 1.0000001, 1e-9);  // warm
  fp64_loop<OP><<<sms, threads>>>(out, cyc, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double lane_ops = double(threads) * ITERS * CHAINS;  // per CTA (one CTA per SM)
  printf("%s threads/SM=%d: %.1f lane-ops/clk/SM (%.2f warp-instr/clk/SM)\n", name, threads, lane_ops / mx,
         lane_ops / mx / 32.0);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {256, 512, 1024}) {
    run<0>("DFMA", sms, t);
    run<1>("DADD", sms, t);
    run<2>("DMUL", sms, t);
  }
  return 0;
}
