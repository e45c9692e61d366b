// Stage-level entry points: the reference's per-stage API on the GPU.
//
// The hot path is the fused kernel in sfft_kernels.cuh (all log2 N stages in
// one HBM pass).  These two small kernels exist so the reference's stage-level
// interface -- digit-reversal gather + one radix-2/4/8 DIT stage at a time
// (planner.py:62-89, kernels.py:28-151) -- is available on device buffers with
// the same semantics, e.g. to compose custom stage lists as the reference's
// tests do (tests/test_kernels.py:25-36).
#include <cuda_runtime.h>

#include <string>

#include "../../include/sfft.h"
#include "sfft_device.cuh"
#include "sfft_internal.h"

namespace {

int stage_fail(int code, const std::string& msg) { return sfft_internal_fail(code, msg); }

template <typename C>
__device__ __forceinline__ C c_add(C a, C b) { return C{a.x + b.x, a.y + b.y}; }
template <typename C>
__device__ __forceinline__ C c_sub(C a, C b) { return C{a.x - b.x, a.y - b.y}; }
template <typename C>
__device__ __forceinline__ C c_mul(C a, C b) { return C{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
// rot * a with rot = -i (forward) or +i (inverse)  (kernels.py:116)
template <typename C>
__device__ __forceinline__ C c_rot(C a, bool inverse) { return inverse ? C{-a.y, a.x} : C{a.y, -a.x}; }

template <typename C>
__device__ __forceinline__ void dft4(C v0, C v1, C v2, C v3, bool inv, C* y) {
  // kernels.py:98-104
  const C t0 = c_add(v0, v2), t1 = c_sub(v0, v2), t2 = c_add(v1, v3), t3 = c_rot(c_sub(v1, v3), inv);
  y[0] = c_add(t0, t2);
  y[1] = c_add(t1, t3);
  y[2] = c_sub(t0, t2);
  y[3] = c_sub(t1, t3);
}

// One radix-R DIT stage over rows of n elements with sub-spectrum length m.
// Thread = (row, group g, position j); operand q of the group is multiplied
// by table[(n/span)*q*j mod n] (conjugated for the inverse) -- kernels.py:41-72.
template <typename T, int R>
__global__ void dit_stage_kernel(const sfft::cx_t<T>* __restrict__ in, sfft::cx_t<T>* __restrict__ out,
                                 const sfft::cx_t<T>* __restrict__ table, int n, int m, bool inverse,
                                 long long total) {
  using C = sfft::cx_t<T>;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  const int per_row = n / R;
  const long long row = tid / per_row;
  const int rem = int(tid - row * per_row);
  const int g = rem / m;
  const int j = rem - g * m;
  const int span = R * m;
  const C* src = in + row * n + g * span + j;
  C* dst = out + row * n + g * span + j;
  C v[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    C w = table[((long long)(n / span) * q * j) % n];
    if (inverse) w.y = -w.y;
    v[q] = c_mul(src[q * m], w);
  }
  if constexpr (R == 2) {
    dst[0] = c_add(v[0], v[1]);
    dst[m] = c_sub(v[0], v[1]);
  } else if constexpr (R == 4) {
    C y[4];
    dft4(v[0], v[1], v[2], v[3], inverse, y);
#pragma unroll
    for (int s = 0; s < 4; ++s) dst[s * m] = y[s];
  } else {
    // kernels.py:126-151: two DFT-4s, eighth-root constants on the odd half
    C e[4], o[4];
    dft4(v[0], v[2], v[4], v[6], inverse, e);
    dft4(v[1], v[3], v[5], v[7], inverse, o);
    const T h = T(0.7071067811865476);
    const C w1 = inverse ? C{h, h} : C{h, -h};    // sqrt(1/2) * (1 + rot)
    const C w3 = inverse ? C{-h, h} : C{-h, -h};  // sqrt(1/2) * (rot - 1)
    o[1] = c_mul(o[1], w1);
    o[2] = c_rot(o[2], inverse);
    o[3] = c_mul(o[3], w3);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      dst[s * m] = c_add(e[s], o[s]);
      dst[(s + 4) * m] = c_sub(e[s], o[s]);
    }
  }
}

template <typename T>
__global__ void gather_kernel(const sfft::cx_t<T>* __restrict__ in, sfft::cx_t<T>* __restrict__ out,
                              const long long* __restrict__ perm, int n, long long total) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  const long long row = tid / n;
  const int p = int(tid - row * n);
  const long long q = perm[p];
  // an out-of-range entry never reads outside its row: it yields NaN (sfft.h)
  out[tid] = (unsigned long long)q < (unsigned long long)n
                 ? in[row * n + q]
                 : sfft::cx_t<T>{T(__int_as_float(0x7fc00000)), T(__int_as_float(0x7fc00000))};
}

template <typename T>
cudaError_t launch_stage(int radix, const void* in, void* out, const void* table, int n, int m, bool inv,
                         long long batch, cudaStream_t st) {
  using C = sfft::cx_t<T>;
  const long long total = batch * (n / radix);
  const unsigned blocks = unsigned((total + 255) / 256);
  auto i = static_cast<const C*>(in);
  auto o = static_cast<C*>(out);
  auto t = static_cast<const C*>(table);
  if (radix == 2) dit_stage_kernel<T, 2><<<blocks, 256, 0, st>>>(i, o, t, n, m, inv, total);
  if (radix == 4) dit_stage_kernel<T, 4><<<blocks, 256, 0, st>>>(i, o, t, n, m, inv, total);
  if (radix == 8) dit_stage_kernel<T, 8><<<blocks, 256, 0, st>>>(i, o, t, n, m, inv, total);
  return cudaGetLastError();
}

}  // namespace

extern "C" {

int sfft_stage(int32_t n, int32_t precision, int32_t radix, int32_t stride, int32_t direction,
               const void* d_table, const void* d_in, void* d_out, int64_t batch, void* stream) {
  if (radix != 2 && radix != 4 && radix != 8)
    return stage_fail(SFFT_ERR_PLAN, "unsupported radix " + std::to_string(radix));
  if (n < 1 || stride < 1 || n % (radix * stride) != 0)
    return stage_fail(SFFT_ERR_PLAN, "radix-" + std::to_string(radix) + " stage needs stride dividing " +
                                         std::to_string(n) + "//" + std::to_string(radix) + ", got stride " +
                                         std::to_string(stride));
  if (precision != SFFT_SINGLE && precision != SFFT_DOUBLE)
    return stage_fail(SFFT_ERR_ARGUMENT, "precision must be SFFT_SINGLE or SFFT_DOUBLE");
  if (batch < 0) return stage_fail(SFFT_ERR_SHAPE, "batch must be >= 0");
  if (batch == 0) return SFFT_OK;
  if (!d_table || !d_in || !d_out) return stage_fail(SFFT_ERR_ARGUMENT, "NULL pointer");
  if (d_in == d_out) return stage_fail(SFFT_ERR_ARGUMENT, "stages are out-of-place (kernels.py:75-80)");
  const bool inv = direction == SFFT_INVERSE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const cudaError_t e = precision == SFFT_SINGLE
                            ? launch_stage<float>(radix, d_in, d_out, d_table, n, stride, inv, batch, st)
                            : launch_stage<double>(radix, d_in, d_out, d_table, n, stride, inv, batch, st);
  if (e != cudaSuccess) return stage_fail(SFFT_ERR_CUDA, std::string("stage launch: ") + cudaGetErrorString(e));
  return SFFT_OK;
}

int sfft_permute(int32_t n, int32_t precision, const int64_t* d_perm, const void* d_in, void* d_out,
                 int64_t batch, void* stream) {
  if (n < 1) return stage_fail(SFFT_ERR_INVALID_LENGTH, "length must be >= 1");
  if (precision != SFFT_SINGLE && precision != SFFT_DOUBLE)
    return stage_fail(SFFT_ERR_ARGUMENT, "precision must be SFFT_SINGLE or SFFT_DOUBLE");
  if (batch < 0) return stage_fail(SFFT_ERR_SHAPE, "batch must be >= 0");
  if (batch == 0) return SFFT_OK;
  if (!d_perm || !d_in || !d_out || d_in == d_out)
    return stage_fail(SFFT_ERR_ARGUMENT, "NULL or aliased pointer");
  const long long total = batch * n;
  const unsigned blocks = unsigned((total + 255) / 256);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (precision == SFFT_SINGLE)
    gather_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float2*>(d_in), static_cast<float2*>(d_out),
                                                 reinterpret_cast<const long long*>(d_perm), n, total);
  else
    gather_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double2*>(d_in), static_cast<double2*>(d_out),
                                                  reinterpret_cast<const long long*>(d_perm), n, total);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stage_fail(SFFT_ERR_CUDA, std::string("permute launch: ") + cudaGetErrorString(e));
  return SFFT_OK;
}

}  // extern "C"
