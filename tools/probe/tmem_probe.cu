// Could tensor memory carry the FFT's exchanges?  Throughput of the tcgen05
// paths that move data between shared memory, TMEM and registers, and
// whether they contend with LDS for the L1 data pipe that limits the fp64
// N=2048 kernel (profiles/r02_fp64_2048_datapipe.txt):
//   mode 0: LDS.128 loop, 4 warps                       (the LSU data pipe alone)
//   mode 1: tcgen05.cp 128x256b smem -> TMEM, one thread (the tensor-core smem read path)
//   mode 2: modes 0 and 1 together (warps 1-3 LDS, warp 0 lane 0 cp)
//   mode 3: tcgen05.ld 32x32b.x16 TMEM -> registers, 4 warps
//   mode 4: modes 0 (warps 0-3 LDS) and 3 interleaved per warp
//   mode 5: mode 1's copies issued by lane 0 of all four warps (a quarter each)
// One CTA of 128 threads per SM, 64 KB of shared memory, all 512 TMEM columns.
// Cycles from clock64() of the slowest CTA; run under ncu for the pipe counters.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// SM100 shared-memory matrix descriptor (cute::UMMA::SmemDescriptor layout):
// start >> 4 in [0,14), LBO >> 4 in [16,30), SBO >> 4 in [32,46), version 1 in [46,48), no swizzle.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3fff) | (uint64_t((lbo >> 4) & 0x3fff) << 16) |
         (uint64_t((sbo >> 4) & 0x3fff) << 32) | (uint64_t(1) << 46);
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(float* out, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) unsigned long long bar;
  float4* buf = reinterpret_cast<float4*>(smem);  // 64 KB = 4096 float4
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4096; i += 128) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(MODE == 5 ? 4 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  float4 acc = make_float4(0, 0, 0, 0);
  uint32_t r[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = 0;

  const long long t0 = clock64();
  const bool do_lds = MODE == 0 || MODE == 4 || (MODE == 2 && warp > 0);
  const bool do_cp = ((MODE == 1 || MODE == 2) && tid == 0) || (MODE == 5 && (tid & 31) == 0);
  const int cp_iters = MODE == 5 ? ITERS / 4 : ITERS;
  const bool do_ld = MODE == 3 || MODE == 4;
  if (do_cp) {
    const uint32_t s0 = smem_u32(smem);
    for (int i = warp * cp_iters; i < (warp + 1) * cp_iters; ++i) {
      // 128 rows x 32 B = 4 KB per copy, rotating over the 64 KB buffer and 8 column groups
      const uint64_t d = smem_desc(s0 + (i & 15) * 4096, 128, 256);
      const uint32_t dst = tmem + ((i & 7) * 8);  // 8 columns (32 B) per lane
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(dst), "l"(d));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done)
                   : "r"(smem_u32(&bar)));
    }
  }
  if (do_lds || do_ld) {
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i) {
      if (do_lds) {
        const float4 v = buf[(tid + i * 128) & 4095];  // conflict-free, 4 wavefronts per warp
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      if (do_ld) {
        const uint32_t src = tmem + (uint32_t(warp * 32) << 16) + uint32_t((i & 31) * 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(src));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc.x += __uint_as_float(r[0] ^ r[5] ^ r[10] ^ r[15]);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  out[blockIdx.x * 128 + tid] = acc.x + acc.y + acc.z + acc.w;
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
double run(int sms) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * 128);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  probe<MODE><<<sms, 128, 65536>>>(out, cyc);
  probe<MODE><<<sms, 128, 65536>>>(out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("mode %d: %s\n", MODE, cudaGetErrorString(e));
    return -1;
  }
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
  const double lds_bytes = 128.0 * 16 * ITERS;        // per SM
  const double cp_bytes = 4096.0 * ITERS;              // per SM
  const double ld_bytes = 128.0 * 16 * 4 * ITERS;      // 4 warps x 32 lanes x 16 words
  const double c0 = run<0>(sms), c1 = run<1>(sms), c2 = run<2>(sms), c3 = run<3>(sms), c4 = run<4>(sms),
               c5 = run<5>(sms);
  printf("mode 0 LDS only      : %9.0f cycles, %6.1f B/clk/SM\n", c0, lds_bytes / c0);
  printf("mode 1 tcgen05.cp    : %9.0f cycles, %6.1f B/clk/SM\n", c1, cp_bytes / c1);
  printf("mode 2 cp + LDS(3w)  : %9.0f cycles (LDS alone 3 warps ~ %.0f, cp alone %.0f)\n", c2, c0 * 0.75, c1);
  printf("mode 3 tcgen05.ld    : %9.0f cycles, %6.1f B/clk/SM\n", c3, ld_bytes / c3);
  printf("mode 4 ld + LDS      : %9.0f cycles (sum %.0f, max %.0f)\n", c4, c0 + c3, c0 > c3 ? c0 : c3);
  printf("mode 5 cp, 4 issuers : %9.0f cycles, %6.1f B/clk/SM\n", c5, cp_bytes / c5);
  return 0;
}
