// C-ABI implementation: plan construction, twiddle tables, kernel dispatch,
// and the host-buffer pipeline.  See include/sfft.h for the contract and the
// reference interfaces each entry point replaces.
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/sfft.h"
#include "host_copy.h"
#include "sfft_internal.h"
#include "sfft_variants.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace

int sfft_internal_fail(int code, const std::string& msg) { return fail(code, msg); }

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  return fail(SFFT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

using sfft_impl::LaunchFn;
using sfft_impl::Variant;

// Variant table, [precision][log2 n]; entry 0 is the planner's default.
// Chosen so every CTA has 128-256 threads, every sequence is touched with
// >= 32-byte contiguous segments per warp instruction, and the swizzled
// exchanges are conflict-free (tests/test_bank_model.py).  The entries are
// instantiated by the sfft_table_*.cu translation units.
const std::vector<Variant>& variants(int precision, int log2n) {
  using namespace sfft_impl;
  static const auto table = [] {
    std::vector<std::vector<Variant>> t(2 * 12);
    for (int l = 1; l <= 11; ++l) {
      t[l] = l <= 8 ? table_f32_small(l) : l == 9 ? table_f32_512(l) : l == 10 ? table_f32_1024(l) : table_f32_2048(l);
      t[12 + l] = l <= 8    ? table_f64_small(l)
                  : l == 9  ? table_f64_512(l)
                  : l == 10 ? table_f64_1024(l)
                            : table_f64_2048(l);
    }
    return t;
  }();
  return table[precision * 12 + log2n];
}

bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }
int log2i(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// numerics.py:55-71: angle = (-2*pi/n)*k in double, cos + i*sin, factors[0] = 1.
void base_table(int n, std::vector<double>& re, std::vector<double>& im) {
  re.resize(n);
  im.resize(n);
  const double step = -2.0 * M_PI / double(n);
  for (int k = 0; k < n; ++k) {
    const double a = step * double(k);
    re[k] = std::cos(a);
    im[k] = std::sin(a);
  }
  re[0] = 1.0;
  im[0] = 0.0;
}

void write_table(int precision, const std::vector<double>& re, const std::vector<double>& im,
                 const std::vector<int>& idx, std::vector<unsigned char>& bytes) {
  const size_t e = precision == SFFT_SINGLE ? 8 : 16;
  bytes.resize(idx.size() * e);
  for (size_t i = 0; i < idx.size(); ++i) {
    if (precision == SFFT_SINGLE) {
      const float v[2] = {float(re[idx[i]]), float(im[idx[i]])};  // rounded once
      std::memcpy(bytes.data() + i * e, v, e);
    } else {
      const double v[2] = {re[idx[i]], im[idx[i]]};
      std::memcpy(bytes.data() + i * e, v, e);
    }
  }
}

int check_length(int32_t n) {
  if (!is_pow2(n))
    return fail(SFFT_ERR_INVALID_LENGTH,
                "transform length must be a power of two, got " + std::to_string(n));
  if (n < SFFT_MIN_LENGTH || n > SFFT_MAX_LENGTH)
    return fail(SFFT_ERR_UNSUPPORTED_LENGTH, "length " + std::to_string(n) +
                                                 " outside supported range [2, 2048]");
  return SFFT_OK;
}

struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) {
      err = cudaSetDevice(dev);
      changed = err == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
};

constexpr int kMaxHostStreams = 8;

// SFFT_SMEM_CARVEOUT (-1..100) overrides every variant's carveout (tuning).
int carveout_override() {
  static const int v = [] {
    const char* e = std::getenv("SFFT_SMEM_CARVEOUT");
    if (e == nullptr || *e == 0) return -2;
    const int c = std::atoi(e);
    return c >= -1 && c <= 100 ? c : -2;
  }();
  return v;
}

// Host pipeline shape: device buffer slots and chunk size (env
// SFFT_HOST_SLOTS / SFFT_HOST_CHUNK_MB override the defaults, read once).
struct HostPipelineShape {
  // measured on the B200 host link (profiles/r01_e2e_sweep.jsonl,
  // r01_e2e_link.jsonl): 32 MiB chunks, 3 slots in flight
  int slots = 3;
  int64_t chunk_bytes = int64_t(32) << 20;
  // Mid-size calls are cut into several chunks (>= min_chunk bytes) so
  // their copies overlap instead of running H2D, kernel and D2H back to
  // back: pinned calls into 4 (<= 32 MiB) or 8 chunks, pageable ones into 4
  // (their host copies want >= 4 MiB pieces).  Measured 2-512 MiB
  // (tools/e2e_size_probe.py, profiles/r02_host_split.txt); SFFT_HOST_SPLIT=1
  // restores one chunk per 32 MiB.
  int split = 0;  // 0: the rule above; else that many chunks for every call
  int64_t min_chunk = int64_t(2) << 20;
  HostPipelineShape() {
    if (const char* e = std::getenv("SFFT_HOST_SPLIT")) {
      const int v = std::atoi(e);
      if (v >= 1 && v <= 64) split = v;
    }
    if (const char* e = std::getenv("SFFT_HOST_MIN_CHUNK_KB")) {
      const long v = std::atol(e);
      if (v >= 64 && v <= (long(1) << 20)) min_chunk = int64_t(v) << 10;
    }
    if (const char* e = std::getenv("SFFT_HOST_SLOTS")) {
      const int v = std::atoi(e);
      if (v >= 2 && v <= kMaxHostStreams) slots = v;
    }
    if (const char* e = std::getenv("SFFT_HOST_CHUNK_MB")) {
      const long v = std::atol(e);
      if (v >= 1 && v <= 1024) chunk_bytes = int64_t(v) << 20;
    }
  }
};
const HostPipelineShape& host_shape() {
  static const HostPipelineShape shape;
  return shape;
}
constexpr int64_t kSmallCallBytes = int64_t(1) << 20;  // single-stream fast path
// Zero-copy latency path: calls whose output is at most this many bytes run
// the kernel straight on pinned, mapped host staging (env
// SFFT_ZERO_COPY_BYTES overrides, 0 disables, capped at kSmallCallBytes).
// Not for large calls: one kernel over 512 MiB of mapped pinned rows moves
// 39 GB/s each way against the copy engines' 45 (c2 e2e 13.8 vs 11.9 ms,
// tools/gpu_zc_pinned_r02.sh) -- SM-initiated PCIe traffic is the slower path.
int64_t zero_copy_bytes() {
  static const int64_t v = [] {
    int64_t b = kSmallCallBytes;  // faster than the copy engines at every size up to 1 MiB
    if (const char* e = std::getenv("SFFT_ZERO_COPY_BYTES")) b = std::atoll(e);
    return b < 0 ? 0 : (b > kSmallCallBytes ? kSmallCallBytes : b);
  }();
  return v;
}

// Per-thread resources of the synchronous entry points: a pinned, mapped
// non-finite flag (no memset kernel, no D2H copy to read it) and a pair of
// timing events per device.
struct ThreadSync {
  int32_t* h_flag = nullptr;
  int32_t* d_flag = nullptr;
  // one pair of timing events per device this thread has timed on, created
  // on first use and kept (indexed by device ordinal, grown on demand)
  std::vector<std::array<cudaEvent_t, 2>> ev;
  ~ThreadSync() {
    if (h_flag) cudaFreeHost(h_flag);
  }
  cudaError_t flag() {
    if (h_flag) return cudaSuccess;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&h_flag), sizeof(int32_t),
                                  cudaHostAllocMapped | cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_flag), h_flag, 0);
    return e;
  }
  cudaError_t events(int device, cudaEvent_t** out) {
    if (device < 0) return cudaErrorInvalidDevice;
    if (size_t(device) >= ev.size()) ev.resize(size_t(device) + 1, {nullptr, nullptr});
    auto& pair = ev[size_t(device)];
    if (pair[0] == nullptr) {
      cudaError_t e = cudaEventCreate(&pair[0]);
      if (e == cudaSuccess) e = cudaEventCreate(&pair[1]);
      if (e != cudaSuccess) {
        if (pair[0]) cudaEventDestroy(pair[0]);
        pair = {nullptr, nullptr};
        return e;
      }
    }
    *out = pair.data();
    return cudaSuccess;
  }
};
thread_local ThreadSync t_sync;

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Device alias of page-locked host memory the kernels can address directly
// (16-byte aligned; with unified addressing every cudaHostAlloc / registered
// buffer is mapped), else nullptr.
void* mapped_alias(const void* p) {
  if (reinterpret_cast<uintptr_t>(p) % 16) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Host-buffer pipeline of one device (sfft_execute_host*), shared by every
// plan on that device and kept for the life of the process: one stream per
// engine (H2D copies, kernels, D2H copies), `nslots` device chunk buffers
// cycled through them and ordered by per-slot events, and the pinned
// staging for pageable user memory.  Sharing it means a new plan's first
// host call reuses the ~200 MB of pinned staging and device slots instead
// of allocating its own (pinning costs ~1 ms per MiB on the B200 host:
// tools/first_call_probe.py); calls on one device serialise on `mu`, which
// costs nothing -- they would contend for the same host link anyway.
struct HostPipeline {
  std::mutex mu;
  bool ready = false;
  int nslots = 0;
  int64_t slot_bytes = 0;  // capacity of each device slot buffer
  cudaStream_t st_h2d = nullptr, st_kernel = nullptr, st_d2h = nullptr;
  cudaEvent_t ev_h2d[kMaxHostStreams] = {};  // slot's H2D done (kernel may read d_in)
  cudaEvent_t ev_k[kMaxHostStreams] = {};    // slot's kernel done (d_in free, D2H may read d_out)
  cudaEvent_t ev_d2h[kMaxHostStreams] = {};  // slot's D2H done (d_out and host staging free)
  void* d_in[kMaxHostStreams] = {};
  void* d_out[kMaxHostStreams] = {};
  int32_t* h_flag = nullptr;  // pinned + mapped: kernels OR into it, host reads it
  int32_t* d_flag = nullptr;  // device alias of h_flag
  unsigned char* h_stage = nullptr;  // pinned bounce buffer for small pageable calls
  unsigned char* h_zc = nullptr;     // pinned + mapped staging of the zero-copy path (in | out)
  unsigned char* d_zc = nullptr;     // its device alias
  // pinned per-slot chunk staging for large pageable calls
  unsigned char* h_chunk_in[kMaxHostStreams] = {};
  unsigned char* h_chunk_out[kMaxHostStreams] = {};
  int64_t h_chunk_bytes = 0;
};

// process-lifetime registry (never torn down: static destruction may run
// after the CUDA runtime has unloaded)
HostPipeline& host_pipeline(int device) {
  static std::mutex registry_mu;
  static std::vector<HostPipeline*> registry;
  std::lock_guard<std::mutex> lock(registry_mu);
  if (size_t(device) >= registry.size()) registry.resize(size_t(device) + 1, nullptr);
  if (registry[size_t(device)] == nullptr) registry[size_t(device)] = new HostPipeline();
  return *registry[size_t(device)];
}

}  // namespace

struct sfft_plan {
  int32_t n = 0, precision = 0, direction = 0, device = 0, variant = 0;
  int64_t batch = 0;
  const Variant* v = nullptr;
  void* d_tw = nullptr;
  std::vector<unsigned char> host_base;  // base table in plan precision
};

extern "C" {

int sfft_version(void) { return 100; /* 0.1.0 */ }

const char* sfft_last_error(void) { return g_last_error.c_str(); }

int sfft_num_variants(int32_t n, int32_t precision) {
  if (!is_pow2(n) || n < SFFT_MIN_LENGTH || n > SFFT_MAX_LENGTH) return 0;
  if (precision != SFFT_SINGLE && precision != SFFT_DOUBLE) return 0;
  return int(variants(precision, log2i(n)).size());
}

int sfft_build_twiddle_table(int32_t n, int32_t precision, void* host_out, int64_t capacity) {
  if (!is_pow2(n) || n > 4096)
    return fail(SFFT_ERR_INVALID_LENGTH, "table length must be a power of two <= 4096");
  if (precision != SFFT_SINGLE && precision != SFFT_DOUBLE)
    return fail(SFFT_ERR_ARGUMENT, "precision must be SFFT_SINGLE or SFFT_DOUBLE");
  const int64_t need = int64_t(n) * (precision == SFFT_SINGLE ? 8 : 16);
  if (host_out == nullptr || capacity < need)
    return fail(SFFT_ERR_ARGUMENT, "output buffer too small for twiddle table");
  std::vector<double> re, im;
  base_table(n, re, im);
  std::vector<int> idx(n);
  for (int k = 0; k < n; ++k) idx[k] = k;
  std::vector<unsigned char> bytes;
  write_table(precision, re, im, idx, bytes);
  std::memcpy(host_out, bytes.data(), bytes.size());
  return SFFT_OK;
}

int sfft_plan_create_variant(sfft_plan_t* out, int32_t n, int32_t precision, int32_t direction,
                             int64_t batch, int32_t device, int32_t variant) {
  if (out == nullptr) return fail(SFFT_ERR_ARGUMENT, "plan out-pointer is NULL");
  *out = nullptr;
  if (int rc = check_length(n)) return rc;
  if (precision != SFFT_SINGLE && precision != SFFT_DOUBLE)
    return fail(SFFT_ERR_ARGUMENT, "precision must be SFFT_SINGLE or SFFT_DOUBLE");
  if (direction != SFFT_FORWARD && direction != SFFT_INVERSE)
    return fail(SFFT_ERR_ARGUMENT, "direction must be SFFT_FORWARD or SFFT_INVERSE");
  if (batch < 0) return fail(SFFT_ERR_SHAPE, "batch must be >= 0");
  const auto& vs = variants(precision, log2i(n));
  if (variant < 0 || variant >= int(vs.size()))
    return fail(SFFT_ERR_PLAN, "kernel variant " + std::to_string(variant) + " does not exist");
  if (device < 0) return fail(SFFT_ERR_ARGUMENT, "device must be >= 0");

  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device >= ndev)
    return fail(SFFT_ERR_CUDA, "device " + std::to_string(device) + " not present (" +
                                   std::to_string(ndev) + " visible)");

  sfft_plan* p = new (std::nothrow) sfft_plan();
  if (p == nullptr) return fail(SFFT_ERR_ARGUMENT, "out of host memory");
  p->n = n;
  p->precision = precision;
  p->direction = direction;
  p->batch = batch;
  p->device = device;
  p->variant = variant;
  p->v = &vs[variant];

  std::vector<double> re, im;
  base_table(n, re, im);
  std::vector<int> idx(n);
  for (int k = 0; k < n; ++k) idx[k] = k;
  write_table(precision, re, im, idx, p->host_base);

  // per-pass table: pass p >= 1, entry [(q-1)*L + k] = w_{L r}^{q k} = base[(n/(L r)) q k]
  std::vector<int> tidx;
  if (p->v->kernel == SFFT_KERNEL_FOURSTEP) {
    // fourstep_kernel's table: tw[c * 32 + n1] = W_n^(n1 * pw[c])
    static constexpr int pw[12] = {1, 2, 3, 4, 0, 8, 16, 24, 32, 40, 48, 56};
    for (int c = 0; c < 12; ++c)
      for (int n1 = 0; n1 < 32; ++n1) tidx.push_back((n1 * pw[c]) % n);
  } else if (p->v->kernel != SFFT_KERNEL_TILE) {  // stockham and split2: per-pass tables
    int L = p->v->radices[0];
    for (int pass = 1; pass < p->v->passes; ++pass) {
      const int r = p->v->radices[pass];
      const int step = n / (L * r);
      for (int q = 1; q < r; ++q)
        for (int k = 0; k < L; ++k) tidx.push_back(step * q * k);
      L *= r;
    }
  }

  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) {
    delete p;
    return cuda_fail(guard.err, "cudaSetDevice");
  }
  if (!tidx.empty()) {
    std::vector<unsigned char> bytes;
    write_table(precision, re, im, tidx, bytes);
    e = cudaMalloc(&p->d_tw, bytes.size());
    if (e == cudaSuccess) e = cudaMemcpy(p->d_tw, bytes.data(), bytes.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(p->d_tw);
      delete p;
      return cuda_fail(e, "twiddle upload");
    }
  }
  e = p->v->prepare[direction](carveout_override() >= -1 ? carveout_override() : p->v->carveout);
  if (e == cudaSuccess && p->v->prepare_real[direction])  // the real loader's own carveout rule
    e = p->v->prepare_real[direction](carveout_override() >= -1 ? carveout_override() : p->v->real_carveout);
  if (e != cudaSuccess) {
    cudaFree(p->d_tw);
    delete p;
    return cuda_fail(e, "cudaFuncSetAttribute");
  }
  *out = p;
  return SFFT_OK;
}

int sfft_plan_create(sfft_plan_t* out, int32_t n, int32_t precision, int32_t direction,
                     int64_t batch, int32_t device) {
  return sfft_plan_create_variant(out, n, precision, direction, batch, device, 0);
}

int sfft_plan_destroy(sfft_plan_t p) {
  if (p == nullptr) return SFFT_OK;
  {
    DeviceGuard guard(p->device);
    if (p->d_tw) cudaFree(p->d_tw);
  }
  delete p;
  return SFFT_OK;
}

int sfft_plan_info(sfft_plan_t p, sfft_plan_info_t* info) {
  if (p == nullptr || info == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL plan or info");
  std::memset(info, 0, sizeof(*info));
  info->n = p->n;
  info->precision = p->precision;
  info->direction = p->direction;
  info->device = p->device;
  info->batch = p->batch;
  info->kernel = p->v->kernel;
  info->elems_per_thread = p->v->r;
  info->seqs_per_cta = p->v->seq;
  info->threads_per_cta = p->v->threads;
  info->smem_bytes = p->v->smem;
  info->num_passes = p->v->passes;
  for (int i = 0; i < 8; ++i) info->radices[i] = p->v->radices[i];
  info->twiddle_elems = p->v->tw_len;
  info->variant = p->variant;
  info->layout = p->v->layout;
  info->twiddle_policy = p->v->twp;
  info->loader = p->v->loader;
  info->smem_carveout = carveout_override() >= -1 ? carveout_override() : p->v->carveout;
  info->pipeline_stages = p->v->stages;
  info->real_input = p->v->launch_real[0] != nullptr;
  info->real_loader = p->v->real_loader;
  return SFFT_OK;
}

int sfft_variant_info(int32_t n, int32_t precision, int32_t variant, sfft_plan_info_t* info) {
  if (info == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL info");
  if (int rc = check_length(n)) return rc;
  if (precision != SFFT_SINGLE && precision != SFFT_DOUBLE)
    return fail(SFFT_ERR_ARGUMENT, "precision must be SFFT_SINGLE or SFFT_DOUBLE");
  const auto& vs = variants(precision, log2i(n));
  if (variant < 0 || variant >= int(vs.size()))
    return fail(SFFT_ERR_PLAN, "kernel variant " + std::to_string(variant) + " does not exist");
  const Variant& v = vs[variant];
  std::memset(info, 0, sizeof(*info));
  info->n = n;
  info->precision = precision;
  info->kernel = v.kernel;
  info->elems_per_thread = v.r;
  info->seqs_per_cta = v.seq;
  info->threads_per_cta = v.threads;
  info->smem_bytes = v.smem;
  info->num_passes = v.passes;
  for (int i = 0; i < 8; ++i) info->radices[i] = v.radices[i];
  info->twiddle_elems = v.tw_len;
  info->variant = variant;
  info->layout = v.layout;
  info->twiddle_policy = v.twp;
  info->loader = v.loader;
  info->smem_carveout = v.carveout;
  info->pipeline_stages = v.stages;
  info->real_input = v.launch_real[0] != nullptr;
  info->real_loader = v.real_loader;
  return SFFT_OK;
}

int sfft_plan_twiddles(sfft_plan_t p, void* host_out, int64_t capacity) {
  if (p == nullptr || host_out == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL argument");
  if (capacity < int64_t(p->host_base.size()))
    return fail(SFFT_ERR_ARGUMENT, "output buffer too small for twiddle table");
  std::memcpy(host_out, p->host_base.data(), p->host_base.size());
  return SFFT_OK;
}

namespace {
// Input and output may be the same buffer (complex input, in place: every
// kernel reads its rows before writing them) or disjoint.  Any other overlap
// -- a shifted view, or real input under its complex output (output row r
// covers real rows 2r and 2r+1, which other CTAs / later pipeline chunks have
// not read yet) -- would race, so it is refused.
bool overlap_refused(const sfft_plan* p, const void* in, const void* out, int64_t batch, int32_t input_kind) {
  const int64_t row = int64_t(p->n) * (p->precision == SFFT_SINGLE ? 8 : 16);
  const int64_t in_row = input_kind == SFFT_INPUT_REAL ? row / 2 : row;
  const uintptr_t i0 = reinterpret_cast<uintptr_t>(in), o0 = reinterpret_cast<uintptr_t>(out);
  const bool overlap = i0 < o0 + uintptr_t(batch * row) && o0 < i0 + uintptr_t(batch * in_row);
  if (!overlap) return false;
  if (i0 == o0 && input_kind == SFFT_INPUT_COMPLEX) return false;
  fail(SFFT_ERR_ARGUMENT,
       "input and output overlap: only an identical complex input/output buffer runs in place");
  return true;
}

// the kernel for (plan, input kind), or nullptr with the error recorded
LaunchFn pick_launch(sfft_plan_t p, int32_t input_kind, const void* d_in, const void* d_out, int* rc) {
  *rc = SFFT_OK;
  if (input_kind != SFFT_INPUT_COMPLEX && input_kind != SFFT_INPUT_REAL) {
    *rc = fail(SFFT_ERR_ARGUMENT, "input_kind must be SFFT_INPUT_COMPLEX or SFFT_INPUT_REAL");
    return nullptr;
  }
  // Both input kinds need 16-byte alignment: the complex loaders move 8- or
  // 16-byte elements, and the real loaders read 16-byte chunks of reals
  // (tile kernels: cp.async 16; fp32 N = 2: 8-byte pairs; bulk TMA: 16-byte
  // source alignment).  A real row view at a 4- or 8-byte offset is refused
  // here instead of faulting in the kernel (the Python layer re-copies it).
  if ((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out)) & 15u) {
    *rc = fail(SFFT_ERR_ARGUMENT, "data pointers must be 16-byte aligned (input and output)");
    return nullptr;
  }
  if (input_kind == SFFT_INPUT_COMPLEX) return p->v->launch[p->direction];
  if (p->v->launch_real[p->direction] == nullptr) {
    *rc = fail(SFFT_ERR_ARGUMENT, "this plan's kernel has no real-input path (see sfft_plan_info.real_input)");
    return nullptr;
  }
  return p->v->launch_real[p->direction];
}
}  // namespace

int sfft_execute_ex(sfft_plan_t p, const void* d_in, void* d_out, int64_t batch, void* stream,
                    int32_t* d_nonfinite, int32_t input_kind) {
  if (p == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL plan");
  if (batch < 0) return fail(SFFT_ERR_SHAPE, "batch must be >= 0");
  if (batch == 0) return SFFT_OK;
  if (d_in == nullptr || d_out == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL data pointer");
  int rc = SFFT_OK;
  const LaunchFn launch = pick_launch(p, input_kind, d_in, d_out, &rc);
  if (launch == nullptr) return rc;
  if (overlap_refused(p, d_in, d_out, batch, input_kind)) return SFFT_ERR_ARGUMENT;
  DeviceGuard guard(p->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  // Programmatic dependent launch overlaps back-to-back eager launches, but
  // inside a captured CUDA graph its programmatic edges cost more than they
  // save (fp64 N=2048 x 64 rows: 6.4 vs 3.5 us per replayed call;
  // tools/graph_probe.py, profiles/r02_graph_probe.txt), so captured
  // launches use plain stream order.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &cap) != cudaSuccess) {
    cudaGetLastError();
    cap = cudaStreamCaptureStatusNone;
  }
  const cudaError_t e = launch(d_in, d_out, p->d_tw, batch, reinterpret_cast<int*>(d_nonfinite),
                               static_cast<cudaStream_t>(stream), cap == cudaStreamCaptureStatusNone);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return SFFT_OK;
}

int sfft_execute(sfft_plan_t p, const void* d_in, void* d_out, int64_t batch, void* stream,
                 int32_t* d_nonfinite) {
  return sfft_execute_ex(p, d_in, d_out, batch, stream, d_nonfinite, SFFT_INPUT_COMPLEX);
}

int sfft_execute_sync_ex(sfft_plan_t p, const void* d_in, void* d_out, int64_t batch, void* stream,
                         float* kernel_ms, int32_t input_kind) {
  if (p == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL plan");
  if (batch < 0) return fail(SFFT_ERR_SHAPE, "batch must be >= 0");
  if (kernel_ms) *kernel_ms = 0.f;
  if (batch == 0) return SFFT_OK;
  if (d_in == nullptr || d_out == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL data pointer");
  int rc = SFFT_OK;
  const LaunchFn launch = pick_launch(p, input_kind, d_in, d_out, &rc);
  if (launch == nullptr) return rc;
  if (overlap_refused(p, d_in, d_out, batch, input_kind)) return SFFT_ERR_ARGUMENT;
  DeviceGuard guard(p->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  cudaError_t e = t_sync.flag();
  if (e != cudaSuccess) return cuda_fail(e, "flag allocation");
  *t_sync.h_flag = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t* ev = nullptr;
  if (kernel_ms) {
    e = t_sync.events(p->device, &ev);
    if (e == cudaSuccess) e = cudaEventRecord(ev[0], st);
    if (e != cudaSuccess) return cuda_fail(e, "event record");
  }
  e = launch(d_in, d_out, p->d_tw, batch, t_sync.d_flag, st, true);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  if (kernel_ms) {
    e = cudaEventRecord(ev[1], st);
    if (e != cudaSuccess) return cuda_fail(e, "event record");
  }
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "stream sync");
  if (kernel_ms) cudaEventElapsedTime(kernel_ms, ev[0], ev[1]);
  if (*reinterpret_cast<volatile int32_t*>(t_sync.h_flag))
    return fail(SFFT_ERR_DOMAIN, "signal contains NaN or Inf values");
  return SFFT_OK;
}

int sfft_execute_sync(sfft_plan_t p, const void* d_in, void* d_out, int64_t batch, void* stream,
                      float* kernel_ms) {
  return sfft_execute_sync_ex(p, d_in, d_out, batch, stream, kernel_ms, SFFT_INPUT_COMPLEX);
}

int sfft_execute_host_ex(sfft_plan_t p, const void* h_in, void* h_out, int64_t batch, int32_t input_kind) {
  if (p == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL plan");
  if (batch < 0) return fail(SFFT_ERR_SHAPE, "batch must be >= 0");
  if (batch == 0) return SFFT_OK;
  if (h_in == nullptr || h_out == nullptr) return fail(SFFT_ERR_ARGUMENT, "NULL data pointer");
  if (input_kind != SFFT_INPUT_COMPLEX && input_kind != SFFT_INPUT_REAL)
    return fail(SFFT_ERR_ARGUMENT, "input_kind must be SFFT_INPUT_COMPLEX or SFFT_INPUT_REAL");
  const bool real = input_kind == SFFT_INPUT_REAL;
  const LaunchFn launch = real ? p->v->launch_real[p->direction] : p->v->launch[p->direction];
  if (launch == nullptr)
    return fail(SFFT_ERR_ARGUMENT, "this plan's kernel has no real-input path (see sfft_plan_info.real_input)");
  if (overlap_refused(p, h_in, h_out, batch, input_kind)) return SFFT_ERR_ARGUMENT;
  HostPipeline& hp = host_pipeline(p->device);
  std::lock_guard<std::mutex> lock(hp.mu);
  DeviceGuard guard(p->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
  // output rows are complex; real input rows carry half the bytes (H2D only)
  const int64_t row_bytes = int64_t(p->n) * (p->precision == SFFT_SINGLE ? 8 : 16);
  const int64_t in_row_bytes = real ? row_bytes / 2 : row_bytes;
  cudaError_t e = cudaSuccess;
  if (!hp.ready) {
    hp.nslots = host_shape().slots;
    for (cudaStream_t* st : {&hp.st_h2d, &hp.st_kernel, &hp.st_d2h})
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(st, cudaStreamNonBlocking);
    for (int i = 0; i < hp.nslots && e == cudaSuccess; ++i)
      for (cudaEvent_t* ev : {&hp.ev_h2d[i], &hp.ev_k[i], &hp.ev_d2h[i]})
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e == cudaSuccess)
      e = cudaHostAlloc(reinterpret_cast<void**>(&hp.h_flag), sizeof(int32_t) * kMaxHostStreams,
                        cudaHostAllocMapped | cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&hp.d_flag), hp.h_flag, 0);
    if (e != cudaSuccess) return cuda_fail(e, "host pipeline setup");
    hp.ready = true;
  }
  const int64_t total = batch * row_bytes;
  const int64_t total_in = batch * in_row_bytes;
  // chunks large enough for full-rate DMA, small enough to overlap copies in
  // both directions with the kernels of neighbouring chunks.
  // Staging buffers grow on demand, so small calls stay small (and
  // zero-copy calls allocate none).
  // Full 32 MiB chunks for long calls; mid-size calls in several chunks
  // (HostPipelineShape).  The pinned check only matters for copy-engine calls.
  const bool pinned = total > kSmallCallBytes && is_pinned(h_in) && is_pinned(h_out);
  int64_t chunk_bytes = host_shape().chunk_bytes;
  {
    const int split = host_shape().split ? host_shape().split : (pinned && total > (int64_t(32) << 20) ? 8 : 4);
    const int64_t per = (total + split - 1) / split;
    const int64_t want = per < host_shape().min_chunk ? host_shape().min_chunk : per;
    if (want < chunk_bytes) chunk_bytes = want;
  }
  const int64_t max_chunk_rows = chunk_bytes / row_bytes > 0 ? chunk_bytes / row_bytes : 1;
  const int64_t want_rows = batch < max_chunk_rows ? batch : max_chunk_rows;
  const int64_t chunk_rows = want_rows;  // rows per pipeline chunk of this call
  auto ensure_slots = [&]() -> cudaError_t {
    if (chunk_rows * row_bytes > hp.slot_bytes) {  // capacity in bytes: plans of any N share the slots
      for (cudaStream_t st : {hp.st_h2d, hp.st_kernel, hp.st_d2h}) cudaStreamSynchronize(st);
      for (int i = 0; i < hp.nslots; ++i) {
        cudaFree(hp.d_in[i]);
        cudaFree(hp.d_out[i]);
        hp.d_in[i] = hp.d_out[i] = nullptr;
      }
      hp.slot_bytes = 0;
      cudaError_t err = cudaSuccess;
      for (int i = 0; i < hp.nslots && err == cudaSuccess; ++i) {
        err = cudaMalloc(&hp.d_in[i], chunk_rows * row_bytes);
        if (err == cudaSuccess) err = cudaMalloc(&hp.d_out[i], chunk_rows * row_bytes);
      }
      if (err != cudaSuccess) return err;
      hp.slot_bytes = chunk_rows * row_bytes;
    }
    return cudaSuccess;
  };
  for (int i = 0; i < kMaxHostStreams; ++i) hp.h_flag[i] = 0;

  if (total <= zero_copy_bytes()) {
    // zero-copy latency path: the kernel reads its input from and writes its
    // output to pinned, host-mapped staging over PCIe -- one launch and one
    // sync, no copy-engine round trips (tools/zero_copy_probe.py)
    if (hp.h_zc == nullptr) {
      e = cudaHostAlloc(reinterpret_cast<void**>(&hp.h_zc), 2 * kSmallCallBytes,
                        cudaHostAllocMapped | cudaHostAllocPortable);
      if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&hp.d_zc), hp.h_zc, 0);
      if (e != cudaSuccess) {
        if (hp.h_zc) cudaFreeHost(hp.h_zc);
        hp.h_zc = hp.d_zc = nullptr;
        return cuda_fail(e, "zero-copy staging allocation");
      }
    }
    // page-locked user buffers are addressed in place; pageable ones go
    // through the staging (a host memcpy each way)
    const auto* ib = static_cast<const unsigned char*>(h_in);
    const auto* ob = static_cast<const unsigned char*>(h_out);
    const bool overlap = ib < ob + total && ob < ib + total_in;  // e.g. in place: stage the input
    const void* k_in = overlap ? nullptr : mapped_alias(h_in);
    void* k_out = mapped_alias(h_out);
    if (k_in == nullptr) {
      std::memcpy(hp.h_zc, h_in, size_t(total_in));
      k_in = hp.d_zc;
    }
    e = launch(k_in, k_out ? k_out : hp.d_zc + kSmallCallBytes, p->d_tw, batch, hp.d_flag, hp.st_kernel, false);
    if (e == cudaSuccess) e = cudaStreamSynchronize(hp.st_kernel);
    if (e != cudaSuccess) return cuda_fail(e, "zero-copy call");
    if (k_out == nullptr) std::memcpy(h_out, hp.h_zc + kSmallCallBytes, size_t(total));
  } else if (total <= kSmallCallBytes) {
    // latency path: one stream; pageable user memory goes through a pinned
    // bounce buffer (a host memcpy is cheaper than the driver's staging)
    e = ensure_slots();
    if (e != cudaSuccess) return cuda_fail(e, "host staging allocation");
    const bool small_pinned = is_pinned(h_in) && is_pinned(h_out);
    if (!small_pinned && hp.h_stage == nullptr) {
      e = cudaHostAlloc(reinterpret_cast<void**>(&hp.h_stage), 2 * kSmallCallBytes, cudaHostAllocPortable);
      if (e != cudaSuccess) return cuda_fail(e, "pinned staging allocation");
    }
    const void* src = h_in;
    void* dst = h_out;
    if (!small_pinned) {
      std::memcpy(hp.h_stage, h_in, size_t(total_in));
      src = hp.h_stage;
      dst = hp.h_stage + kSmallCallBytes;
    }
    cudaStream_t st = hp.st_h2d;
    e = cudaMemcpyAsync(hp.d_in[0], src, size_t(total_in), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = launch(hp.d_in[0], hp.d_out[0], p->d_tw, batch, hp.d_flag, st, false);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dst, hp.d_out[0], size_t(total), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "small-call pipeline");
    if (!small_pinned) std::memcpy(h_out, dst, size_t(total));
  } else {
    e = ensure_slots();
    if (e != cudaSuccess) return cuda_fail(e, "host staging allocation");
    // Three engines, one stream each -- H2D copies, kernels, D2H copies --
    // with chunk k in device slot k % S.  Per slot:
    //   H2D(k)    waits kernel(k-S)  (d_in free)
    //   kernel(k) waits H2D(k) and D2H(k-S)  (d_out free)
    //   D2H(k)    waits kernel(k)
    // so each copy engine sees an uninterrupted queue in its own direction.
    // Measured (tools/e2e_link_probe.py, profiles/r01_e2e_link.jsonl): 97-99 %
    // of two free-running full-size concurrent copies on the same box; the
    // link, not the pipeline, is the bound.  (Geometric ramp-in/ramp-out
    // chunk sizes against fill/drain measured no gain:
    // profiles/r02_host_ramp_negative.txt.)
    const unsigned char* src = static_cast<const unsigned char*>(h_in);
    unsigned char* dst = static_cast<unsigned char*>(h_out);
    const int S = hp.nslots;
    const int64_t stage_bytes = chunk_rows * row_bytes;
    if (!pinned && hp.h_chunk_bytes < stage_bytes) {
      for (cudaStream_t st : {hp.st_h2d, hp.st_kernel, hp.st_d2h}) cudaStreamSynchronize(st);
      for (int i = 0; i < S; ++i) {
        if (hp.h_chunk_in[i]) cudaFreeHost(hp.h_chunk_in[i]);
        if (hp.h_chunk_out[i]) cudaFreeHost(hp.h_chunk_out[i]);
        hp.h_chunk_in[i] = hp.h_chunk_out[i] = nullptr;
      }
      hp.h_chunk_bytes = 0;
      for (int i = 0; i < S && e == cudaSuccess; ++i) {
        e = cudaHostAlloc(reinterpret_cast<void**>(&hp.h_chunk_in[i]), stage_bytes, cudaHostAllocPortable);
        if (e == cudaSuccess)
          e = cudaHostAlloc(reinterpret_cast<void**>(&hp.h_chunk_out[i]), stage_bytes, cudaHostAllocPortable);
      }
      if (e != cudaSuccess) return cuda_fail(e, "pinned chunk staging allocation");
      hp.h_chunk_bytes = stage_bytes;
    }
    auto& pool = sfft_host::CopyPool::instance();
    // a failure mid-pipeline drains the streams before returning, so the next
    // call never races leftover copies on the slot buffers
    auto fail_sync = [&](cudaError_t err, const char* what) {
      for (cudaStream_t st : {hp.st_h2d, hp.st_kernel, hp.st_d2h}) cudaStreamSynchronize(st);
      return cuda_fail(err, what);
    };
    // staged (pageable) path: which rows each slot's host staging holds
    int64_t slot_row[kMaxHostStreams] = {}, slot_rows[kMaxHostStreams] = {};
    auto drain_slot = [&](int s) -> cudaError_t {
      if (slot_rows[s] == 0) return cudaSuccess;
      const cudaError_t err = cudaEventSynchronize(hp.ev_d2h[s]);
      if (err != cudaSuccess) return err;
      pool.memcpy(dst + slot_row[s] * row_bytes, hp.h_chunk_out[s], size_t(slot_rows[s] * row_bytes));
      slot_rows[s] = 0;
      return cudaSuccess;
    };
    int chunk = 0;
    for (int64_t row = 0; row < batch; row += chunk_rows, ++chunk) {
      const int s = chunk % S;
      const bool reuse = chunk >= S;  // the slot's previous chunk is in flight
      const int64_t rows = batch - row < chunk_rows ? batch - row : chunk_rows;
      const size_t bytes = size_t(rows * row_bytes);
      const size_t in_bytes = size_t(rows * in_row_bytes);
      const void* h2d_src = src + row * in_row_bytes;
      void* d2h_dst = dst + row * row_bytes;
      if (!pinned) {
        // the slot's previous chunk must have left the host staging (its D2H
        // done implies its H2D done)
        e = drain_slot(s);
        if (e != cudaSuccess) return fail_sync(e, "staging drain");
        pool.memcpy(hp.h_chunk_in[s], src + row * in_row_bytes, in_bytes);
        h2d_src = hp.h_chunk_in[s];
        d2h_dst = hp.h_chunk_out[s];
      }
      if (reuse) e = cudaStreamWaitEvent(hp.st_h2d, hp.ev_k[s], 0);
      if (e == cudaSuccess) e = cudaMemcpyAsync(hp.d_in[s], h2d_src, in_bytes, cudaMemcpyHostToDevice, hp.st_h2d);
      if (e == cudaSuccess) e = cudaEventRecord(hp.ev_h2d[s], hp.st_h2d);
      if (e != cudaSuccess) return fail_sync(e, "H2D copy");
      e = cudaStreamWaitEvent(hp.st_kernel, hp.ev_h2d[s], 0);
      if (e == cudaSuccess && reuse) e = cudaStreamWaitEvent(hp.st_kernel, hp.ev_d2h[s], 0);
      if (e == cudaSuccess)
        e = launch(hp.d_in[s], hp.d_out[s], p->d_tw, rows, hp.d_flag + s, hp.st_kernel, false);
      if (e == cudaSuccess) e = cudaEventRecord(hp.ev_k[s], hp.st_kernel);
      if (e != cudaSuccess) return fail_sync(e, "kernel launch");
      e = cudaStreamWaitEvent(hp.st_d2h, hp.ev_k[s], 0);
      if (e == cudaSuccess) e = cudaMemcpyAsync(d2h_dst, hp.d_out[s], bytes, cudaMemcpyDeviceToHost, hp.st_d2h);
      if (e == cudaSuccess) e = cudaEventRecord(hp.ev_d2h[s], hp.st_d2h);
      if (e != cudaSuccess) return fail_sync(e, "D2H copy");
      if (!pinned) {
        slot_row[s] = row;
        slot_rows[s] = rows;
      }
    }
    if (!pinned) {
      // drain in chunk order (oldest first)
      for (int k = 0; k < S; ++k) {
        e = drain_slot((chunk + k) % S);
        if (e != cudaSuccess) return fail_sync(e, "staging drain");
      }
    }
    for (cudaStream_t st : {hp.st_h2d, hp.st_kernel, hp.st_d2h}) {
      e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return cuda_fail(e, "stream sync");
    }
  }
  for (int i = 0; i < kMaxHostStreams; ++i)
    if (reinterpret_cast<volatile int32_t*>(hp.h_flag)[i])
      return fail(SFFT_ERR_DOMAIN, "signal contains NaN or Inf values");
  return SFFT_OK;
}

int sfft_execute_host(sfft_plan_t p, const void* h_in, void* h_out, int64_t batch) {
  return sfft_execute_host_ex(p, h_in, h_out, batch, SFFT_INPUT_COMPLEX);
}

}  // extern "C"
