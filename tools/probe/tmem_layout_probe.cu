// Layout check for the staging gather through tensor memory: a row of 2048
// complex doubles sits linearly in shared memory; eight tcgen05.cp 128x256b
// copies (no-swizzle descriptor: SBO = 128 B between 8-row core matrices,
// LBO = 2048 B between the two 16-byte K chunks, start advancing 4096 B)
// should give TMEM lane t the elements x[t + 128 m], m = 0..15, and one
// tcgen05.ld 32x32b.x64 per warp should put them in registers in m order.
// Prints the number of mismatching (thread, m) pairs and a few samples.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_layout_probe tmem_layout_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3fff) | (uint64_t((lbo >> 4) & 0x3fff) << 16) |
         (uint64_t((sbo >> 4) & 0x3fff) << 32) | (uint64_t(1) << 46);
}

__global__ void __launch_bounds__(128, 1) layout(int* bad, double2* sample) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) unsigned long long bar;
  double2* row = reinterpret_cast<double2*>(smem);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 2048; i += 128) row[i] = make_double2(i, -i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t s0 = smem_u32(smem);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t d = smem_desc(s0 + k * 4096, 2048, 128);
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + k * 8), "l"(d));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[64];
  const uint32_t src = tmem + (uint32_t(warp * 32) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(src));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(src + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  int nbad = 0;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const double re = __hiloint2double(int(r[4 * m + 1]), int(r[4 * m + 0]));
    const double im = __hiloint2double(int(r[4 * m + 3]), int(r[4 * m + 2]));
    const int want = tid + 128 * m;
    if (re != double(want) || im != -double(want)) ++nbad;
    if (tid < 4 || tid == 37 || tid == 127) sample[tid * 16 + m] = make_double2(re, im);
  }
  atomicAdd(bad, nbad);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  int* bad;
  double2* sample;
  cudaMalloc(&bad, sizeof(int));
  cudaMalloc(&sample, sizeof(double2) * 128 * 16);
  cudaMemset(bad, 0, sizeof(int));
  cudaMemset(sample, 0, sizeof(double2) * 128 * 16);
  cudaFuncSetAttribute(layout, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  layout<<<1, 128, 32768>>>(bad, sample);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  int h = 0;
  double2 s[128 * 16];
  cudaMemcpy(&h, bad, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(s, sample, sizeof(s), cudaMemcpyDeviceToHost);
  printf("mismatches: %d of %d\n", h, 128 * 16);
  for (int t : {0, 1, 2, 3, 37, 127}) {
    printf("thread %3d:", t);
    for (int m = 0; m < 16; ++m) printf(" %g", s[t * 16 + m].x);
    printf("\n");
  }
  return 0;
}
