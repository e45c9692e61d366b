// Kernel variants: the launch/prepare entry points of every compiled
// instantiation and the Variant records the planner picks from.  Included by
// sfft_api.cu and by the per-(precision, N) table translation units
// (sfft_table_*.cu), which instantiate the kernels in parallel builds.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "../../include/sfft.h"
#include "sfft_kernels.cuh"

namespace sfft_impl {

// pdl: launch with programmatic stream serialization (see launch_pdl)
using LaunchFn = cudaError_t (*)(const void* in, void* out, const void* tw, long long batch,
                                 int* flag, cudaStream_t st, bool pdl);
using PrepareFn = cudaError_t (*)(int carveout);

struct Variant {
  int kernel;      // SFFT_KERNEL_*
  int r;           // elements per thread (stockham R; tile: n)
  int seq;         // sequences per CTA
  int layout;      // smem layout (stockham): 1 padded, 2 row swizzle, 3 split re/im exchange (fp64)
  int twp;         // twiddle policy (stockham): 0 all loaded, 1 powers of two + products,
                   // 2 two-level split, 3 one load + squarings (sfft_kernels.cuh)
  int loader;      // input path (stockham): 0 per-thread LDG, 1 one bulk TMA copy per CTA,
                   // 2 persistent CTAs with a `stages`-deep bulk TMA pipeline,
                   // 3 bulk TMA + gathers through tensor memory (fp64 N=2048),
                   // 4 as 3 but only the staging gather through tensor memory
  int stages;      // loader 2: shared-memory stage buffers per CTA
  int carveout;    // preferred shared-memory carveout, % of max (-1: driver default)
  int threads;     // threads per CTA
  int smem;        // dynamic smem bytes
  int passes;
  int radices[8];
  int tw_len;      // per-pass twiddle elements
  LaunchFn launch[2];    // [direction]
  PrepareFn prepare[2];  // [direction]
  // real-valued input rows (imaginary parts zero), default variants only.
  // Same passes (hence the same arithmetic: bit-identical to widening); the
  // loader may differ (real_loader), with its own carveout rule.
  LaunchFn launch_real[2];
  PrepareFn prepare_real[2];
  int real_loader;
  int real_carveout;
};

// ---------------------------------------------------------------- launchers
template <typename T, int N, int R, int SEQ, int LAYOUT>
constexpr int stockham_smem() {
  return SEQ * sfft::Smem<T, LAYOUT, R>::size(N) * int(sizeof(sfft::cx_t<T>));
}

// SFFT_PDL=0 disables programmatic dependent launch (A/B and debugging).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SFFT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute
// (the kernels call griddepcontrol.wait before any global access).
// Used for launches on the caller's stream; the host pipeline, whose kernels
// follow cross-stream event waits, launches with pdl = false.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), long long grid, int threads, int smem, cudaStream_t st,
                       Args... args) {
  if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(threads));
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl && pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...);
}

// the Stockham kernel, or its register-capped twin when MINB > 1
template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int LOADER, bool RIN, int MINB>
auto stockham_kernel_ptr() {
  if constexpr (MINB > 1)
    return sfft::stockham_kernel_capped<T, N, R, SEQ, INV, LAYOUT, TWP, LOADER, RIN, MINB>;
  else
    return sfft::stockham_kernel<T, N, R, SEQ, INV, LAYOUT, TWP, LOADER, RIN>;
}

template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int LOADER, bool RIN = false, int MINB = 1>
cudaError_t launch_stockham(const void* in, void* out, const void* tw, long long batch, int* flag,
                            cudaStream_t st, bool pdl) {
  using C = sfft::cx_t<T>;
  using In = std::conditional_t<RIN, T, C>;
  constexpr int threads = (N / R) * SEQ;
  constexpr int smem = stockham_smem<T, N, R, SEQ, LAYOUT>();
  const long long grid = (batch + SEQ - 1) / SEQ;
  return launch_pdl(pdl, stockham_kernel_ptr<T, N, R, SEQ, INV, LAYOUT, TWP, LOADER, RIN, MINB>(), grid, threads, smem,
                    st, static_cast<const In*>(in), static_cast<C*>(out), static_cast<const C*>(tw), batch, flag);
}
template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int LOADER, bool RIN = false, int MINB = 1>
cudaError_t prepare_stockham(int carveout) {
  const auto k = stockham_kernel_ptr<T, N, R, SEQ, INV, LAYOUT, TWP, LOADER, RIN, MINB>();
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       stockham_smem<T, N, R, SEQ, LAYOUT>());
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  return e;
}

// ------------------------------------------------- persistent pipeline
template <typename T, int N, int R, int SEQ, int LAYOUT, int STAGES>
constexpr int pipe_smem() {
  return STAGES * stockham_smem<T, N, R, SEQ, LAYOUT>();
}

// Resident CTAs of `kernel` on the current device, times its SM count: the
// persistent grid.  `cache` belongs to one kernel instantiation (a static of
// the launcher template below), so two pipelined kernels of the same
// signature never share a grid size.
template <typename K>
int persistent_grid(K kernel, int threads, int smem, std::atomic<int> (&cache)[16]) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return 0;
  if (const int c = cache[dev].load(std::memory_order_relaxed); c > 0) return c;
  int sms = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess) return 0;
  if (per_sm < 1) per_sm = 1;
  cache[dev].store(sms * per_sm, std::memory_order_relaxed);  // racing writers store the same value
  return sms * per_sm;
}

template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int STAGES>
cudaError_t launch_stockham_pipe(const void* in, void* out, const void* tw, long long batch, int* flag,
                                 cudaStream_t st, bool pdl) {
  using C = sfft::cx_t<T>;
  constexpr int threads = (N / R) * SEQ;
  constexpr int smem = pipe_smem<T, N, R, SEQ, LAYOUT, STAGES>();
  const auto k = sfft::stockham_pipe_kernel<T, N, R, SEQ, INV, LAYOUT, TWP, STAGES>;
  const long long tiles = (batch + SEQ - 1) / SEQ;
  static std::atomic<int> grid_cache[16] = {};  // per instantiation
  const int full = persistent_grid(k, threads, smem, grid_cache);
  if (full <= 0) return cudaErrorInvalidConfiguration;
  const long long grid = tiles < full ? tiles : full;
  return launch_pdl(pdl, k, grid, threads, smem, st, static_cast<const C*>(in), static_cast<C*>(out),
                    static_cast<const C*>(tw), batch, flag);
}
template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int STAGES>
cudaError_t prepare_stockham_pipe(int carveout) {
  const auto k = sfft::stockham_pipe_kernel<T, N, R, SEQ, INV, LAYOUT, TWP, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       pipe_smem<T, N, R, SEQ, LAYOUT, STAGES>());
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  return e;
}

template <typename T, int N, int SPT, int W, bool RIN = false>
constexpr int tile_smem() {
  return W * sfft::tile_chunks<T, N, SPT, RIN>() * 16;
}

template <typename T, int N, int SPT, int W, bool INV, bool RIN = false>
cudaError_t launch_tile(const void* in, void* out, const void*, long long batch, int* flag,
                        cudaStream_t st, bool pdl) {
  using C = sfft::cx_t<T>;
  using In = std::conditional_t<RIN, T, C>;
  constexpr int smem = tile_smem<T, N, SPT, W, RIN>();
  constexpr long long per_cta = 32LL * SPT * W;
  const long long grid = (batch + per_cta - 1) / per_cta;
  return launch_pdl(pdl, sfft::tile_kernel<T, N, SPT, W, INV, RIN>, grid, 32 * W, smem, st,
                    static_cast<const In*>(in), static_cast<C*>(out), batch, flag);
}
template <typename T, int N, int SPT, int W, bool INV, bool RIN = false>
cudaError_t prepare_tile(int carveout) {
  constexpr int smem = tile_smem<T, N, SPT, W, RIN>();
  const auto k = sfft::tile_kernel<T, N, SPT, W, INV, RIN>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  return e;
}

// RMINB: min-blocks (register cap) of the real-input instantiations only;
// RLOADER: their loader (the passes, hence the results, are the complex
// kernel's whatever the loader)
template <typename T, int N, int R, int SEQ, int LAYOUT = 2, int TWP = 0, int LOADER = 0, bool REAL = false,
          int RMINB = 1, int RLOADER = LOADER>
Variant stockham_variant() {
  Variant v{};
  v.kernel = SFFT_KERNEL_STOCKHAM;
  v.r = R;
  v.seq = SEQ;
  v.layout = LAYOUT;
  v.threads = (N / R) * SEQ;
  v.smem = stockham_smem<T, N, R, SEQ, LAYOUT>();
  v.passes = sfft::num_passes(N, R);
  for (int p = 0; p < v.passes && p < 8; ++p) v.radices[p] = sfft::pass_radix(N, R, p);
  v.tw_len = sfft::twiddle_table_len(N, R);
  v.twp = TWP;
  v.loader = LOADER;
  // Per-thread global loads land in L1 before they reach registers, so every
  // LDG line in flight holds L1 capacity.  Left to the driver, a variant
  // whose resident CTAs fill the smem carveout (e.g. 12 x 16.9 KB -> 228 KB,
  // 28 KB of L1) starves its own loads: 5.6 instead of 6.9-7.0 TB/s
  // (tools/probe/occ_probe.cu, profiles/r01_occ_probe.txt).  Capping shared
  // memory at half the unified 256 KB keeps >= 124 KB of L1.  Bulk (TMA)
  // copies land in shared memory directly and keep the driver default.
  v.carveout = LOADER == 0 ? 50 : -1;
  v.real_loader = LOADER;
  v.real_carveout = v.carveout;
  v.launch[0] = &launch_stockham<T, N, R, SEQ, false, LAYOUT, TWP, LOADER>;
  v.launch[1] = &launch_stockham<T, N, R, SEQ, true, LAYOUT, TWP, LOADER>;
  v.prepare[0] = &prepare_stockham<T, N, R, SEQ, false, LAYOUT, TWP, LOADER>;
  v.prepare[1] = &prepare_stockham<T, N, R, SEQ, true, LAYOUT, TWP, LOADER>;
  if constexpr (REAL) {
    v.launch_real[0] = &launch_stockham<T, N, R, SEQ, false, LAYOUT, TWP, RLOADER, true, RMINB>;
    v.launch_real[1] = &launch_stockham<T, N, R, SEQ, true, LAYOUT, TWP, RLOADER, true, RMINB>;
    v.prepare_real[0] = &prepare_stockham<T, N, R, SEQ, false, LAYOUT, TWP, RLOADER, true, RMINB>;
    v.prepare_real[1] = &prepare_stockham<T, N, R, SEQ, true, LAYOUT, TWP, RLOADER, true, RMINB>;
    v.real_loader = RLOADER;
    v.real_carveout = RLOADER == 0 ? 50 : -1;
  }
  return v;
}

// persistent pipelined Stockham (loader 2)
template <typename T, int N, int R, int SEQ, int LAYOUT, int TWP, int STAGES>
Variant pipe_variant() {
  Variant v = stockham_variant<T, N, R, SEQ, LAYOUT, TWP, 1>();
  v.loader = 2;
  v.stages = STAGES;
  v.smem = pipe_smem<T, N, R, SEQ, LAYOUT, STAGES>();
  v.carveout = -1;  // bulk copies land in shared memory; the driver sizes it
  v.real_loader = v.loader;
  v.real_carveout = v.carveout;
  v.launch[0] = &launch_stockham_pipe<T, N, R, SEQ, false, LAYOUT, TWP, STAGES>;
  v.launch[1] = &launch_stockham_pipe<T, N, R, SEQ, true, LAYOUT, TWP, STAGES>;
  v.prepare[0] = &prepare_stockham_pipe<T, N, R, SEQ, false, LAYOUT, TWP, STAGES>;
  v.prepare[1] = &prepare_stockham_pipe<T, N, R, SEQ, true, LAYOUT, TWP, STAGES>;
  return v;
}

// bulk TMA + tensor-memory gathers (sfft_kernels.cuh: stockham_tmem_kernel, loader 3)
template <typename T, int N, int R, bool INV, int TWP, bool RIN, int MINB, bool XCH>
cudaError_t launch_stockham_tmem(const void* in, void* out, const void* tw, long long batch, int* flag,
                                 cudaStream_t st, bool pdl) {
  using C = sfft::cx_t<T>;
  using In = std::conditional_t<RIN, T, C>;
  return launch_pdl(pdl, sfft::stockham_tmem_kernel<T, N, R, INV, TWP, RIN, MINB, XCH>, batch, N / R,
                    N * int(sizeof(C)), st, static_cast<const In*>(in), static_cast<C*>(out),
                    static_cast<const C*>(tw), batch, flag);
}
template <typename T, int N, int R, bool INV, int TWP, bool RIN, int MINB, bool XCH>
cudaError_t prepare_stockham_tmem(int carveout) {
  const auto k = sfft::stockham_tmem_kernel<T, N, R, INV, TWP, RIN, MINB, XCH>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, N * int(sizeof(sfft::cx_t<T>)));
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  return e;
}
template <typename T, int N, int R, int TWP, bool REAL = false, int MINB = 1, bool XCH = true>
Variant tmem_variant() {
  Variant v = stockham_variant<T, N, R, 1, 2, TWP, 1>();
  v.loader = XCH ? 3 : 4;
  v.carveout = -1;  // the bulk copy lands in shared memory
  v.real_loader = v.loader;
  v.real_carveout = v.carveout;
  v.launch[0] = &launch_stockham_tmem<T, N, R, false, TWP, false, MINB, XCH>;
  v.launch[1] = &launch_stockham_tmem<T, N, R, true, TWP, false, MINB, XCH>;
  v.prepare[0] = &prepare_stockham_tmem<T, N, R, false, TWP, false, MINB, XCH>;
  v.prepare[1] = &prepare_stockham_tmem<T, N, R, true, TWP, false, MINB, XCH>;
  v.launch_real[0] = v.launch_real[1] = nullptr;
  v.prepare_real[0] = v.prepare_real[1] = nullptr;
  if constexpr (REAL) {
    v.launch_real[0] = &launch_stockham_tmem<T, N, R, false, TWP, true, MINB, XCH>;
    v.launch_real[1] = &launch_stockham_tmem<T, N, R, true, TWP, true, MINB, XCH>;
    v.prepare_real[0] = &prepare_stockham_tmem<T, N, R, false, TWP, true, MINB, XCH>;
    v.prepare_real[1] = &prepare_stockham_tmem<T, N, R, true, TWP, true, MINB, XCH>;
  }
  return v;
}

// two-warp split-radix-2 kernel (sfft_kernels.cuh: split2_kernel)
template <typename T, int N, int R, int LAYOUT>
constexpr int split2_smem() {
  return 2 * sfft::Smem<T, LAYOUT, R>::size(N / 2) * int(sizeof(sfft::cx_t<T>));
}
template <typename T, int N, int R, bool INV, int LAYOUT, int TWP, bool RIN = false>
cudaError_t launch_split2(const void* in, void* out, const void* tw, long long batch, int* flag,
                          cudaStream_t st, bool pdl) {
  using C = sfft::cx_t<T>;
  using In = std::conditional_t<RIN, T, C>;
  return launch_pdl(pdl, sfft::split2_kernel<T, N, R, INV, LAYOUT, TWP, RIN>, batch, 64,
                    split2_smem<T, N, R, LAYOUT>(), st, static_cast<const In*>(in), static_cast<C*>(out),
                    static_cast<const C*>(tw), batch, flag);
}
template <typename T, int N, int R, bool INV, int LAYOUT, int TWP, bool RIN = false>
cudaError_t prepare_split2(int carveout) {
  const auto k = sfft::split2_kernel<T, N, R, INV, LAYOUT, TWP, RIN>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, split2_smem<T, N, R, LAYOUT>());
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  return e;
}
// Pass list and twiddle table are the generic Stockham ones for (N, R) --
// [R, ..., 2] with the radix-2 level last -- so only the launch changes.
template <typename T, int N, int R, int LAYOUT, int TWP, bool REAL = false>
Variant split2_variant() {
  static_assert(sfft::pass_radix(N, R, sfft::num_passes(N, R) - 1) == 2 && N / 2 / R == 32, "split2 geometry");
  Variant v = stockham_variant<T, N, R, 1, LAYOUT, TWP, 1>();
  v.kernel = SFFT_KERNEL_SPLIT2;
  v.threads = 64;
  v.seq = 1;
  v.smem = split2_smem<T, N, R, LAYOUT>();
  v.carveout = -1;  // the bulk copy lands in shared memory
  v.real_loader = v.loader;
  v.real_carveout = v.carveout;
  v.launch[0] = &launch_split2<T, N, R, false, LAYOUT, TWP>;
  v.launch[1] = &launch_split2<T, N, R, true, LAYOUT, TWP>;
  v.prepare[0] = &prepare_split2<T, N, R, false, LAYOUT, TWP>;
  v.prepare[1] = &prepare_split2<T, N, R, true, LAYOUT, TWP>;
  v.launch_real[0] = v.launch_real[1] = nullptr;
  v.prepare_real[0] = v.prepare_real[1] = nullptr;
  if constexpr (REAL) {
    v.launch_real[0] = &launch_split2<T, N, R, false, LAYOUT, TWP, true>;
    v.launch_real[1] = &launch_split2<T, N, R, true, LAYOUT, TWP, true>;
    v.prepare_real[0] = &prepare_split2<T, N, R, false, LAYOUT, TWP, true>;
    v.prepare_real[1] = &prepare_split2<T, N, R, true, LAYOUT, TWP, true>;
  }
  return v;
}

// fp64 N = 2048 four-step kernel (sfft_kernels.cuh: fourstep_kernel): four
// warps per sequence, one exchange, three radix-2 levels through warp shuffles
template <typename T, bool INV, bool RIN, int MINB>
cudaError_t launch_fourstep(const void* in, void* out, const void* tw, long long batch, int* flag,
                            cudaStream_t st, bool pdl) {
  using C = sfft::cx_t<T>;
  using In = std::conditional_t<RIN, T, C>;
  return launch_pdl(pdl, sfft::fourstep_kernel<T, INV, RIN, MINB>, batch, 128, 2048 * int(sizeof(C)), st,
                    static_cast<const In*>(in), static_cast<C*>(out), static_cast<const C*>(tw), batch, flag);
}
template <typename T, bool INV, bool RIN, int MINB>
cudaError_t prepare_fourstep(int carveout) {
  const auto k = sfft::fourstep_kernel<T, INV, RIN, MINB>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * int(sizeof(sfft::cx_t<T>)));
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  return e;
}
// Steps: radix 64 (over n2) then radix 32 (over n1); the twiddle table is the
// kernel's own (12 powers of W2048^n1 per n1, built by sfft_plan_create).
constexpr int kFourstepTwiddleElems = 12 * 32;
template <typename T, bool REAL = false, int MINB = 5>
Variant fourstep_variant() {
  Variant v{};
  v.kernel = SFFT_KERNEL_FOURSTEP;
  v.r = 16;
  v.seq = 1;
  v.layout = 0;
  v.twp = 2;
  v.loader = 1;
  v.carveout = -1;  // the bulk copy lands in shared memory
  v.real_loader = v.loader;
  v.real_carveout = v.carveout;
  v.threads = 128;
  v.smem = 2048 * int(sizeof(sfft::cx_t<T>));
  v.passes = 2;
  v.radices[0] = 64;
  v.radices[1] = 32;
  v.tw_len = kFourstepTwiddleElems;
  v.launch[0] = &launch_fourstep<T, false, false, MINB>;
  v.launch[1] = &launch_fourstep<T, true, false, MINB>;
  v.prepare[0] = &prepare_fourstep<T, false, false, MINB>;
  v.prepare[1] = &prepare_fourstep<T, true, false, MINB>;
  if constexpr (REAL) {
    v.launch_real[0] = &launch_fourstep<T, false, true, MINB>;
    v.launch_real[1] = &launch_fourstep<T, true, true, MINB>;
    v.prepare_real[0] = &prepare_fourstep<T, false, true, MINB>;
    v.prepare_real[1] = &prepare_fourstep<T, true, true, MINB>;
  }
  return v;
}

template <typename T, int N, int SPT, int W, bool REAL = false>
Variant tile_variant() {
  Variant v{};
  v.kernel = SFFT_KERNEL_TILE;
  v.r = N;
  v.seq = 32 * SPT * W;
  v.threads = 32 * W;
  v.smem = tile_smem<T, N, SPT, W>();
  v.passes = 1;
  v.radices[0] = N;
  v.tw_len = 0;
  v.carveout = -1;  // cp.async stages through shared memory, not L1 lines
  v.real_loader = v.loader;
  v.real_carveout = v.carveout;
  v.launch[0] = &launch_tile<T, N, SPT, W, false>;
  v.launch[1] = &launch_tile<T, N, SPT, W, true>;
  v.prepare[0] = &prepare_tile<T, N, SPT, W, false>;
  v.prepare[1] = &prepare_tile<T, N, SPT, W, true>;
  if constexpr (REAL) {
    v.launch_real[0] = &launch_tile<T, N, SPT, W, false, true>;
    v.launch_real[1] = &launch_tile<T, N, SPT, W, true, true>;
    v.prepare_real[0] = &prepare_tile<T, N, SPT, W, false, true>;
    v.prepare_real[1] = &prepare_tile<T, N, SPT, W, true, true>;
  }
  return v;
}

// Variant tables of one (precision, log2 n) group; entry 0 is the planner's
// default.  Defined by the sfft_table_*.cu translation units.
std::vector<Variant> table_f32_small(int log2n);  // N = 2 .. 256
std::vector<Variant> table_f32_512(int log2n);
std::vector<Variant> table_f32_1024(int log2n);
std::vector<Variant> table_f32_2048(int log2n);
std::vector<Variant> table_f64_small(int log2n);  // N = 2 .. 256
std::vector<Variant> table_f64_512(int log2n);
std::vector<Variant> table_f64_1024(int log2n);
std::vector<Variant> table_f64_2048(int log2n);

}  // namespace sfft_impl
