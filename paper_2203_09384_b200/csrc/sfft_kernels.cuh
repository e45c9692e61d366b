// Batched C2C FFT kernels for sm_100a.
//
// Kernel families covering N = 2 .. 2048 in fp32 and fp64:
//
// * stockham_kernel  (N >= 64 fp32, N >= 32 fp64)
//   G = N/R threads own one sequence; each thread keeps R elements in
//   registers.  Pass 0 loads straight from HBM (lane j reads x[j + m*G]:
//   consecutive lanes, consecutive addresses), every pass is a radix-r DFT in
//   registers with per-pass twiddles from the plan's table, the exchange
//   between passes goes through padded or row-swizzled (bank-conflict-free)
//   shared memory, and the last pass writes straight to HBM in natural order
//   (Stockham autosort: no digit-reversal gather, cf. executor.py:77).
//   One HBM read + one HBM write per element.  With R = 32 / 64 a sequence
//   is one warp (two passes, __syncwarp only) -- the round-2 defaults for
//   fp32 N = 2048 and fp64 N = 512, 1024.
//
// * split2_kernel    (tested variant, fp64 N = 2048): two one-warp N/2
//   transforms of the polyphase halves plus a radix-2 combine.
//
// * fourstep_kernel  (tested variant, fp64 N = 2048): 32 x 64 four-step with
//   one shared-memory exchange and three radix-2 levels through warp shuffles.
//
// * stockham_tmem_kernel (tested variant, fp64 N = 2048): the bulk-TMA
//   Stockham kernel with shared-memory gathers routed through tensor memory
//   (tcgen05.cp + tcgen05.ld) to take them off the L1 data pipe.
//
// * tile_kernel      (N <= 32 fp32, N <= 16 fp64)
//   One thread owns whole sequences.  A warp stages a contiguous tile of
//   32*SPT sequences into swizzled shared memory with 16-byte cp.async
//   (fully coalesced, asynchronous), each thread runs its length-N DFT in
//   registers with compile-time twiddles, and the warp streams the tile back
//   with 16-byte coalesced stores.  fp32 N = 2 (one 16-byte chunk per
//   sequence) skips the staging altogether.
//
// All fuse: the inverse direction (swap trick), the 1/N inverse scale
// (executor.py:93-94; exact for powers of two) and the non-finite input
// check (executor.py:72-73) into the single pass over HBM.
#pragma once

#include "sfft_device.cuh"

namespace sfft {

// ------------------------------------------------------------ pass schedule
// N = R^(P-1) * r_last with the (smaller) remainder radix LAST: pass 0 has
// stride 1 (no twiddles) and every exchange written before the last pass has
// stride L >= R, which keeps the swizzled scatters conflict-free per
// quarter/half-warp phase (tests/test_bank_model.py).
__host__ __device__ constexpr int remainder_radix(int n, int r) {
  while (n % r == 0 && n > 1) n /= r;
  return n;
}
__host__ __device__ constexpr int num_passes(int n, int r) {
  int p = 0;
  int m = n;
  while (m % r == 0 && m > 1) { m /= r; ++p; }
  return p + (m > 1 ? 1 : 0);
}
__host__ __device__ constexpr int pass_radix(int n, int r, int p) {
  return (remainder_radix(n, r) > 1 && p == num_passes(n, r) - 1) ? remainder_radix(n, r) : r;
}
__host__ __device__ constexpr int pass_stride(int n, int r, int p) {
  int l = 1;
  for (int i = 0; i < p; ++i) l *= pass_radix(n, r, i);
  return l;
}
// offset (in elements) of pass p's twiddles in the per-pass table:
// pass p >= 1 stores (r_p - 1) * L_p entries, [(q-1)*L + k] = w_{L r}^{q k}.
__host__ __device__ constexpr int pass_twiddle_offset(int n, int r, int p) {
  int off = 0;
  for (int i = 1; i < p; ++i) off += (pass_radix(n, r, i) - 1) * pass_stride(n, r, i);
  return off;
}
__host__ __device__ constexpr int twiddle_table_len(int n, int r) {
  return pass_twiddle_offset(n, r, num_passes(n, r));
}

// ------------------------------------------------------- smem layouts
// Bank rows are 128 bytes = 16 fp32 / 8 fp64 complex; a warp access is served
// per phase of 16 (8-byte) or 8 (16-byte) lanes.
// LAYOUT 1: per-sequence region with one pad element after every R elements.
//           Stride-R scatters become stride R+1 (odd), and addresses factor:
//           map(base + c) = map(base) + c + c/R for c a multiple of R, so a
//           pass's gathers are one base register plus immediate offsets.
// LAYOUT 2: row swizzle over the CTA-wide index, e ^ ((e / R) & (W - 1)) with
//           W = elements per bank row (needs R >= W).  The XOR only touches
//           bits below log2 R, so for an offset c that is a multiple of R,
//           map(base + c) = map'(base, (c / R) mod W) + c, and for an
//           R-aligned base and c < R, map(base + c) = base + (c ^ term) --
//           every access of a pass is one of <= W precomputed registers plus
//           an immediate (no per-access shift/xor chain, unlike a plain XOR
//           swizzle of e with higher bits of e) and
//           no padding (16-byte accesses stay 128-byte aligned per phase,
//           which LAYOUT 1 breaks).
// LAYOUT 3: fp64 only -- the exchange moves the real parts, then the
//           imaginary parts, through an N-double region (half the bytes of
//           LAYOUT 2) indexed like LAYOUT 2 with 8-byte words (W = 16).  Same
//           wavefronts per exchange, two more barriers, and half the shared
//           memory per sequence: with per-thread loads (LOADER 0) the shared
//           memory holds only the exchange, so the L1 keeps room for the
//           loads in flight and no bulk copy writes + gathers the row through
//           the shared-memory pipe.
// tests/test_bank_model.py replays every access of every variant per phase.
template <typename T, int LAYOUT, int R>
struct Smem {
  static constexpr int W = (sizeof(T) == 4 || LAYOUT == 3) ? 16 : 8;  // words (complex or LAYOUT-3 halves) per 128-byte row
  static constexpr int LGR = ilog2(R);
  static_assert(LAYOUT == 1 || LAYOUT == 2 || LAYOUT == 3, "smem layout");
  static_assert(LAYOUT == 1 || R >= W, "row swizzle needs R >= elements per bank row");
  static_assert(LAYOUT != 3 || sizeof(T) == 8, "split exchange: fp64 only");
  // in complex elements (LAYOUT 3 stores N doubles = N/2 complex)
  __host__ __device__ static constexpr int size(int n) { return LAYOUT == 1 ? n + n / R : (LAYOUT == 3 ? n / 2 : n); }
  __device__ static __forceinline__ int map(int e) {
    if constexpr (LAYOUT == 1) {
      return e + e / R;
    } else {
      return e ^ ((e >> LGR) & (W - 1));
    }
  }
  // map(base + off), off folds to a constant after unrolling; `base_aligned`
  // promises base % R == 0 (so off < R stays inside one padded row).
  __device__ static __forceinline__ int map2(int base, int mapped_base, int off,
                                             bool base_aligned = false) {
    if constexpr (LAYOUT == 1) {
      if (off % R == 0) return mapped_base + off + off / R;
      if (base_aligned && off < R) return mapped_base + off;
    } else {
      // LAYOUT 2 / 3; identical subexpressions per residue are CSE'd across the unrolled pass
      if (off % R == 0) return (base ^ (((base >> LGR) + ((off >> LGR) & (W - 1))) & (W - 1))) + off;
      if (base_aligned && off < R) return base + ((off & (W - 1)) ^ ((base >> LGR) & (W - 1))) + (off & ~(W - 1));
    }
    return map(base + off);
  }
};

// 16-byte-chunk swizzle for the tile kernel (8 chunks per bank row).
__device__ __forceinline__ int swz_chunk(int c) { return c ^ (((c >> 3) ^ (c >> 6)) & 7); }

template <int ID, int COUNT>
__device__ __forceinline__ void named_bar() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");
}

// Barrier over the G threads of one sequence.  Barrier ids are compile-time
// immediates so ptxas reserves only the ids actually used (a register id
// makes it reserve all 16 per CTA).
template <int G, int SEQ>
__device__ __forceinline__ void seq_sync(int s) {
  if constexpr (G <= 32) {
    __syncwarp();
  } else if constexpr (SEQ == 1) {
    __syncthreads();
  } else {
    static_assert(SEQ <= 4, "named barrier ids 1..4");
    switch (s) {  // warp-uniform
      case 0: named_bar<1, G>(); break;
      case 1: named_bar<2, G>(); break;
      case 2: named_bar<3, G>(); break;
      default: named_bar<4, G>(); break;
    }
  }
}

// ---------------------------------------------------------- Stockham kernel
// Non-finite input check, one packed FFMA2 per complex element: Inf/NaN * 0
// = NaN, sticky in `acc`.  fp64 feeds the high words reinterpreted as fp32:
// a non-finite double has all-ones exponent bits 30..20, so its high word is
// an fp32 Inf/NaN too -- as is the high word of a finite |x| >= 2^1017, which
// is why a hit is re-checked exactly (nonfinite_exact) before it is reported.
__device__ __forceinline__ void accumulate_nonfinite(float2& acc, float2 v) {
  acc = fma2(v, make_float2(0.f, 0.f), acc);
}
__device__ __forceinline__ void accumulate_nonfinite(float2& acc, double2 v) {
  const float2 hi = make_float2(__int_as_float(__double2hiint(v.x)), __int_as_float(__double2hiint(v.y)));
  acc = fma2(hi, make_float2(0.f, 0.f), acc);
}
template <int R>
__device__ __forceinline__ bool nonfinite_exact(const float2 (&)[R]) {
  return true;  // the fp32 filter is exact
}
template <int R>
__device__ __forceinline__ bool nonfinite_exact(const double2 (&v)[R]) {
  uint32_t bad = 0;
#pragma unroll
  for (int m = 0; m < R; ++m) bad |= nonfinite_bits(v[m]);
  return bad != 0;
}

__host__ __device__ constexpr int high_pow2(int q) {
  int h = 1;
  while (h * 2 <= q) h *= 2;
  return h;
}

// Apply the pass twiddles w^q, w = w_{L r}^k, to one butterfly's operands.
// TWP 0: every w^q is its own table entry (r-1 loads, exact table values).
// TWP 1: only w^(2^i) are loaded; w^q = w^hi * w^(q-hi) (<= 3 products deep,
//        error <= ~3 ulp) -- trades L1 wavefronts for FMA-pipe work.
// TWP 2: two-level, w^q = w^(q - q mod S) * w^(q mod S) with both factors
//        loaded (S = 4, or 8 for r = 32): one product deep (~1 ulp, against
//        ~3 for TWP 1), fewer products than TWP 1, a few more loads.  At
//        r = 16: 6 loads + 9 products (TWP 1: 4 + 11; TWP 0: 15 + 0).
template <int r>
__host__ __device__ constexpr int twiddle_split() {
  return r >= 32 ? 8 : 4;
}
template <int TWP, int r, int L, int NB, typename C, int R>
__device__ __forceinline__ void apply_pass_twiddles(C (&v)[R], const C* __restrict__ tp, int t) {
  if constexpr (TWP == 0) {
#pragma unroll
    for (int q = 1; q < r; ++q) v[t + q * NB] = cmul(v[t + q * NB], __ldg(tp + (q - 1) * L));
  } else if constexpr (TWP == 2) {
    constexpr int S = twiddle_split<r>();
    C w[r];
    static_for<1, r>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int lo = q % S;
      if constexpr (lo == 0 || q < S) {
        w[q] = __ldg(tp + (q - 1) * L);
      } else {
        w[q] = cmul(w[q - lo], w[lo]);
      }
      v[t + q * NB] = cmul(v[t + q * NB], w[q]);
    });
  } else if constexpr (TWP == 3) {
    // one load per butterfly: w^(2^i) by repeated squaring, the rest as in
    // TWP 1 (<= ~8 ulp; trades L1 data-pipe wavefronts for FP64 products)
    C w[r];
    static_for<1, r>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      if constexpr (q == 1) {
        w[q] = __ldg(tp);
      } else if constexpr ((q & (q - 1)) == 0) {
        w[q] = cmul(w[q / 2], w[q / 2]);
      } else {
        constexpr int hi = high_pow2(q);
        w[q] = cmul(w[hi], w[q - hi]);
      }
      v[t + q * NB] = cmul(v[t + q * NB], w[q]);
    });
  } else {
    C w[r];
    static_for<1, r>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      if constexpr ((q & (q - 1)) == 0) {
        w[q] = __ldg(tp + (q - 1) * L);
      } else {
        constexpr int hi = high_pow2(q);
        w[q] = cmul(w[hi], w[q - hi]);
      }
      v[t + q * NB] = cmul(v[t + q * NB], w[q]);
    });
  }
}

// ------------------------------------------------- TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// one bulk (1-D TMA) copy global -> shared, completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

// ------------------------------------------------ tensor memory (TMEM)
// Shared memory is read through the LSU data pipe -- the unit that limits
// the fp64 N=2048 kernel (profiles/r02_fp64_2048_datapipe.txt).  tcgen05.cp
// reads shared memory through the tensor-core path instead (64 B/clk/SM,
// overlapping LDS) into tensor memory, and tcgen05.ld brings a thread's own
// TMEM lane into registers (252 B/clk/SM) -- neither touches the LSU pipe
// (tools/probe/tmem_probe.cu).  With one thread per TMEM lane (128-thread
// CTAs), a gather v[m] = buf[lane + 128 m] of 16-byte elements from a linear
// buffer is eight 128x256b copies (no-swizzle descriptor: 8-row core matrices
// 128 B apart, the two 16-byte K chunks 2048 B apart; layout pinned by
// tools/probe/tmem_layout_probe.cu) plus two 32-column loads per thread.
struct TmemGather {
  uint32_t tmem;                // this CTA's 64 allocated columns (lane 0)
  unsigned long long* bar;      // completion of the copies (tcgen05.commit)
  uint32_t phase;               // next parity to wait for on `bar`
};

__device__ __forceinline__ uint64_t tmem_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SM100 shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4
  // [16,30), SBO >> 4 [32,46), version 1 [46,48), no swizzle
  return uint64_t((saddr >> 4) & 0x3fff) | (uint64_t((lbo >> 4) & 0x3fff) << 16) |
         (uint64_t((sbo >> 4) & 0x3fff) << 32) | (uint64_t(1) << 46);
}

// v[m] = buf[lane + 128 m], m < 16, for a linear 2048 x 16-byte buffer.  Called
// by all 128 threads after a barrier that orders the buffer's writes (with
// fence.proxy.async by the writers) and every earlier read of the TMEM
// columns (tcgen05.fence::before_thread_sync by the readers).
__device__ __forceinline__ void tmem_gather16(double2 (&v)[16], const void* buf, TmemGather& g) {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t s0 = smem_u32(buf);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t d = tmem_smem_desc(s0 + k * 4096, 2048, 128);
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(g.tmem + k * 8), "l"(d) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(g.bar))
                 : "memory");
  }
  mbar_wait(g.bar, g.phase);
  g.phase ^= 1;
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // two 32-column halves (8 complex doubles each), so only 32 staging
  // registers are live next to v[]
  const uint32_t src = g.tmem + (uint32_t(threadIdx.x & ~31) << 16);  // the warp's 32 lanes
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(src + 32 * h));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int m = 0; m < 8; ++m)
      v[8 * h + m] = double2{__hiloint2double(int(r[4 * m + 1]), int(r[4 * m])),
                             __hiloint2double(int(r[4 * m + 3]), int(r[4 * m + 2]))};
  }
  // the columns may be overwritten by the next gather once every thread has
  // passed a barrier after this point
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// other geometries never take the TMEM path (stockham_passes' static_assert);
// this overload only keeps its discarded branch well-formed for them
template <typename C, int M>
__device__ __forceinline__ void tmem_gather16(C (&)[M], const void*, TmemGather&) {}

// The radix passes of one Stockham sequence, shared by both kernels below.
// On entry v[m] = x[j + m*G] (pass-0 inputs, already validated); the
// exchange region `smq` (per-sequence for LAYOUT 1, CTA-wide for LAYOUT 2
// with `sbase` = s*N) is free; on exit the outputs are stored to `dst_row`
// (nullptr: sequence past the batch, nothing stored) and the region has been
// read for the last time by this thread.
//
// TMEM_LAST (fp64, G = 128, R = 16, one sequence per CTA): the exchange that
// feeds the last pass is scattered to a linear buffer (its Stockham pattern
// writes 8 consecutive 16-byte elements per 8-lane phase: conflict-free
// without a swizzle) and gathered through tensor memory (tmem_gather16)
// instead of LDS.
template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, bool TMEM_LAST = false>
__device__ __forceinline__ void stockham_passes(cx_t<T> (&v)[R], cx_t<T>* __restrict__ smq, int sbase, int j,
                                                int s, cx_t<T>* __restrict__ dst_row,
                                                const cx_t<T>* __restrict__ tw,
                                                TmemGather* tg = nullptr) {
  using C = cx_t<T>;
  using S = Smem<T, LAYOUT, R>;
  constexpr int G = N / R;
  constexpr int NP = num_passes(N, R);
  if constexpr (INV) {
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cswap(v[m]);
  }
  constexpr bool SPLIT = (LAYOUT == 3);  // exchange real parts, then imaginary parts
  static_assert(!TMEM_LAST || (sizeof(T) == 8 && G == 128 && R == 16 && SEQ == 1 && !SPLIT), "TMEM gather geometry");
  T* __restrict__ sq = reinterpret_cast<T*>(smq);
  const int rbase = sbase + j;
  const int rbase_m = S::map(rbase);

  static_for<0, NP>([&](auto P) {
    constexpr int p = decltype(P)::value;
    constexpr int r = pass_radix(N, R, p);
    constexpr int L = pass_stride(N, R, p);
    constexpr int NB = R / r;  // butterflies per thread in this pass
    if constexpr (p > 0) {
      // gather this pass's inputs x[j + m*G] from the exchange buffer (the
      // split exchange and the TMEM gather did it at the end of the previous pass)
      if constexpr (!SPLIT && !(TMEM_LAST && p == NP - 1)) {
#pragma unroll
        for (int m = 0; m < R; ++m) v[m] = smq[S::map2(rbase, rbase_m, m * G)];
      }
      // twiddles w_{L r}^{q k}, k = b mod L  (kernels.py:41-72, gathered
      // from the plan table instead of rebuilt per call)
      const C* twp = tw + pass_twiddle_offset(N, R, p);
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int k = (j + t * G) & (L - 1);
        apply_pass_twiddles<TWP, r, L, NB>(v, twp + k, t);
      }
    }
    // radix-r DFTs in registers
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      C u[r];
#pragma unroll
      for (int q = 0; q < r; ++q) u[q] = v[t + q * NB];
      dft_regs<r>(u);
#pragma unroll
      for (int q = 0; q < r; ++q) v[t + q * NB] = u[q];
    }
    if constexpr (p == NP - 1) {
      // last pass: output index b + q*L == j + m*G -> coalesced store
      if (dst_row != nullptr) {
        C* dst = dst_row + j;
#pragma unroll
        for (int m = 0; m < R; ++m) {
          C y = v[m];
          if constexpr (INV) y = cscale(cswap(y), T(1) / T(N));  // exact: N = 2^k
          st_stream(dst + m * G, y);
        }
      }
    } else {
      if constexpr (p > 0) seq_sync<G, SEQ>(s);  // everyone has read before we overwrite
      constexpr bool aligned = (L == 1 && r == R);  // wbase = b*R
      if constexpr (TMEM_LAST && p == NP - 2) {
        // linear scatter, then the last pass's gather through tensor memory
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          const int b = j + t * G;
          const int k = b & (L - 1);
          const int wbase = sbase + (b - k) * r + k;
#pragma unroll
          for (int q = 0; q < r; ++q) smq[wbase + q * L] = v[t + q * NB];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // STS visible to tcgen05.cp
        seq_sync<G, SEQ>(s);
        tmem_gather16(v, smq, *tg);
      } else if constexpr (SPLIT) {
        // real parts: scatter, barrier, gather the next pass's x[j + m*G];
        // then the imaginary parts the same way (v[.].x already holds new
        // values while v[.].y is still scattered from the old ones)
        static_for<0, 2>([&](auto H) {
          constexpr int h = decltype(H)::value;
          if constexpr (h == 1) seq_sync<G, SEQ>(s);  // real parts read before the buffer is reused
#pragma unroll
          for (int t = 0; t < NB; ++t) {
            const int b = j + t * G;
            const int k = b & (L - 1);
            const int wbase = sbase + (b - k) * r + k;
            const int wbase_m = S::map(wbase);
#pragma unroll
            for (int q = 0; q < r; ++q) {
              const C& y = v[t + q * NB];
              sq[S::map2(wbase, wbase_m, q * L, aligned)] = h == 0 ? y.x : y.y;
            }
          }
          seq_sync<G, SEQ>(s);
#pragma unroll
          for (int m = 0; m < R; ++m) {
            const T x = sq[S::map2(rbase, rbase_m, m * G)];
            if constexpr (h == 0) v[m].x = x; else v[m].y = x;
          }
        });
      } else {
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          const int b = j + t * G;
          const int k = b & (L - 1);
          const int wbase = sbase + (b - k) * r + k;
          const int wbase_m = S::map(wbase);
#pragma unroll
          for (int q = 0; q < r; ++q) smq[S::map2(wbase, wbase_m, q * L, aligned)] = v[t + q * NB];
        }
        seq_sync<G, SEQ>(s);
      }
    }
  });
}

// Output-side NaN/Inf check (the out-of-place default of the Stockham and
// split2 kernels).  X[0] = sum of all N inputs, formed by additions alone
// (every k = 0 twiddle is exactly 1), so a non-finite input always makes
// X[0] non-finite (Inf - Inf = NaN, NaN + x = NaN): one test of X[0] by the
// thread that owns it replaces a test of every input (for fp64 that input
// test costs ~3 instructions per element: packing the high words for FFMA2).
// X[0] can also overflow from finite inputs, so a hit re-reads the row's
// inputs and reports only a truly non-finite one -- the reference's
// input-side semantics (executor.py:72-73).  In-place launches overwrite the
// inputs, so they keep the input-side check at load time.
template <typename C>
__device__ __forceinline__ bool cx_finite(C v) {
  return isfinite(v.x) && isfinite(v.y);
}
template <typename In>
__device__ __noinline__ void recheck_row_inputs(const In* __restrict__ row, int n, int* nonfinite) {
  for (int i = 0; i < n; ++i) {
    bool ok;
    if constexpr (std::is_same_v<In, float> || std::is_same_v<In, double>) {
      ok = isfinite(row[i]);
    } else {
      ok = cx_finite(row[i]);
    }
    if (!ok) {
      atomicOr(nonfinite, 1);
      return;
    }
  }
}

template <typename T, int R>
__device__ __forceinline__ void check_nonfinite(const cx_t<T> (&v)[R], int* nonfinite) {
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int m = 0; m < R; ++m) accumulate_nonfinite(acc, v[m]);
  if ((acc.x != acc.x || acc.y != acc.y) && nonfinite_exact(v)) atomicOr(nonfinite, 1);
}

// Programmatic dependent launch (every kernel here is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): release the next
// kernel in the stream so its CTAs get scheduled while this grid drains, then
// wait for the previous kernel to complete and flush before touching global
// memory -- a chain that reuses buffers stays ordered.  Both are no-ops for
// a launch without the attribute.  Measured: the fixed cost per launch drops
// from 3.9 to 2.0 us (fp32 N=1024) and 8.0 to 5.6 us (fp64 N=2048)
// (tools/batch_scaling.py, profiles/r01_pdl.txt).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// LOADER 0: each thread loads its R elements straight into registers (LDG).
// LOADER 1: one thread issues a single bulk TMA copy of the CTA's SEQ
//           consecutive sequences (one contiguous byte range) into shared
//           memory, the CTA waits on an mbarrier, and pass 0 gathers from
//           shared memory -- no per-thread global loads at all.
// RIN: the input rows are real (N values of T each, imaginary parts zero) --
//      the C2C transform of a real signal reads 4 (8) bytes per element
//      instead of 8 (16) and needs no separate widening pass.
// The body is shared by stockham_kernel and stockham_kernel_capped (below).
template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int LOADER, bool RIN>
__device__ __forceinline__ void stockham_body(const std::conditional_t<RIN, T, cx_t<T>>* __restrict__ in,
                                              cx_t<T>* __restrict__ out, const cx_t<T>* __restrict__ tw,
                                              long long batch, int* __restrict__ nonfinite) {
  using C = cx_t<T>;
  using S = Smem<T, LAYOUT, R>;
  constexpr int G = N / R;
  constexpr int SN = S::size(N);  // smem elements per sequence
  static_assert(G >= 1 && (N % R) == 0, "geometry");
  static_assert(G <= 32 || SEQ <= 4, "named barrier ids");
  static_assert(LOADER == 0 || LAYOUT != 3, "the split exchange region cannot stage a whole row");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sm = reinterpret_cast<C*>(smem_raw);

  const int tid = threadIdx.x;
  const int s = tid / G;
  const int j = tid - s * G;
  const long long seq = (long long)blockIdx.x * SEQ + s;
  const bool valid = seq < batch;
  pdl_enter();

  C v[R];
  if constexpr (LOADER == 1) {
    __shared__ __align__(8) unsigned long long bar;
    const long long seq0 = (long long)blockIdx.x * SEQ;
    const long long nseq = batch - seq0 < SEQ ? batch - seq0 : SEQ;
    if (tid == 0) {
      mbar_init(&bar, 1);
      const uint32_t bytes = uint32_t(nseq * N * int(sizeof(*in)));
      mbar_expect_tx(&bar, bytes);
      bulk_g2s(sm, in + seq0 * N, bytes, &bar);
    }
    __syncthreads();  // barrier initialised before anyone polls it
    mbar_wait(&bar, 0);
    // rows past the batch read stale staging; they are never stored and are
    // excluded from the non-finite check below
    if constexpr (RIN) {
      const T* smr = reinterpret_cast<const T*>(smem_raw);
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = C{smr[s * N + j + m * G], T(0)};
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = sm[s * N + j + m * G];  // linear staging, conflict-free
    }
    __syncthreads();  // staging fully read before the exchange layout reuses it
  } else {
    // rows past the batch (last CTA only) re-read the last row instead of
    // branching around the loads (saves a zero-fill of R registers); they are
    // computed but never stored
    const auto* src = in + (valid ? seq : batch - 1) * N + j;
    if constexpr (RIN) {
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = C{ld_stream(src + m * G), T(0)};
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = ld_stream(src + m * G);
    }
  }
  // NaN/Inf check: on X[0] after the passes (out-of-place), on the loaded
  // inputs when the launch is in place (see recheck_row_inputs)
  const bool in_place = static_cast<const void*>(in) == static_cast<const void*>(out);
  if (nonfinite != nullptr && valid && in_place) check_nonfinite<T, R>(v, nonfinite);
  // LAYOUT 1 keeps each sequence in its own padded region; LAYOUT 2 swizzles
  // the CTA-wide element index (sequences are N apart, N a multiple of R).
  stockham_passes<T, N, R, SEQ, INV, LAYOUT, TWP>(v, LAYOUT == 1 ? sm + s * SN : sm, LAYOUT == 1 ? 0 : s * N, j,
                                                  s, valid ? out + seq * N : nullptr, tw);
  if (nonfinite != nullptr && valid && !in_place && j == 0 && !cx_finite(v[0]))
    recheck_row_inputs(in + seq * N, N, nonfinite);
}

template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int LOADER = 0, bool RIN = false>
__global__ void __launch_bounds__((N / R) * SEQ)
stockham_kernel(const std::conditional_t<RIN, T, cx_t<T>>* __restrict__ in, cx_t<T>* __restrict__ out,
                const cx_t<T>* __restrict__ tw, long long batch, int* __restrict__ nonfinite) {
  stockham_body<T, N, R, SEQ, INV, LAYOUT, TWP, LOADER, RIN>(in, out, tw, batch, nonfinite);
}
// The same kernel with a minimum of MINB resident CTAs per SM requested from
// ptxas (a register cap).  A separate kernel because any explicit min-blocks
// value, 1 included, changes ptxas' allocation (the fp32 N=2048 real-input
// kernel: 214 registers without, 255 + spills with __launch_bounds__(32, 1)).
template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int LOADER, bool RIN, int MINB>
__global__ void __launch_bounds__((N / R) * SEQ, MINB)
stockham_kernel_capped(const std::conditional_t<RIN, T, cx_t<T>>* __restrict__ in, cx_t<T>* __restrict__ out,
                       const cx_t<T>* __restrict__ tw, long long batch, int* __restrict__ nonfinite) {
  stockham_body<T, N, R, SEQ, INV, LAYOUT, TWP, LOADER, RIN>(in, out, tw, batch, nonfinite);
}

// LOADER 3 (fp64 N = 2048, R = 16, 128 threads, one sequence per CTA): the
// LOADER 1 kernel with two of its three shared-memory gathers moved to
// tensor memory -- the row staged by the bulk copy and the exchange that
// feeds the last pass reach registers through tcgen05.cp + tcgen05.ld, so
// the L1 data pipe carries only the bulk-copy writes, two scatters, one
// gather and the stores (~1300 instead of ~1930 wavefront-cycles per row).
// The arithmetic is stockham_passes' unchanged: results are bit-identical
// to LOADER 1's.  Real rows (RIN) are gathered with LDS (8-byte elements
// do not fit the copy's 16-byte rows) and still take the TMEM exchange.
// MINB: minimum resident CTAs per SM requested from ptxas (register cap);
// XCH: also gather the last exchange through TMEM (else LDS, as LOADER 1).
template <typename T, int N, int R, bool INV, int TWP, bool RIN = false, int MINB = 1, bool XCH = true>
__global__ void __launch_bounds__(N / R, MINB)
stockham_tmem_kernel(const std::conditional_t<RIN, T, cx_t<T>>* __restrict__ in, cx_t<T>* __restrict__ out,
                     const cx_t<T>* __restrict__ tw, long long batch, int* __restrict__ nonfinite) {
  using C = cx_t<T>;
  constexpr int G = N / R;
  static_assert(sizeof(T) == 8 && G == 128 && R == 16, "TMEM gather geometry: fp64, 128 lanes, 16 elements");
  constexpr int TMEM_COLS = 64;  // 16 complex doubles per lane

  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sm = reinterpret_cast<C*>(smem_raw);
  __shared__ __align__(8) unsigned long long bar_tma, bar_cp;
  __shared__ uint32_t tmem_base;

  const int j = threadIdx.x;
  const long long seq = blockIdx.x;  // grid = batch: every CTA owns one valid row
  pdl_enter();
  if (j < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (j == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_cp, 1);
    constexpr uint32_t bytes = uint32_t(N * int(sizeof(*in)));
    mbar_expect_tx(&bar_tma, bytes);
    bulk_g2s(sm, in + seq * N, bytes, &bar_tma);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();  // barriers initialised, TMEM address published
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  TmemGather tg{tmem_base, &bar_cp, 0};
  mbar_wait(&bar_tma, 0);
  C v[R];
  if constexpr (RIN) {
    const T* smr = reinterpret_cast<const T*>(smem_raw);
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = C{smr[j + m * G], T(0)};
  } else {
    tmem_gather16(v, sm, tg);  // the bulk copy's writes are async-proxy writes: no proxy fence needed
  }
  __syncthreads();  // staging fully read before the exchange reuses it
  const bool in_place = static_cast<const void*>(in) == static_cast<const void*>(out);
  if (nonfinite != nullptr && in_place) check_nonfinite<T, R>(v, nonfinite);
  stockham_passes<T, N, R, 1, INV, 2, TWP, XCH>(v, sm, 0, j, 0, out + seq * N, tw, &tg);
  if (nonfinite != nullptr && !in_place && j == 0 && !cx_finite(v[0])) recheck_row_inputs(in + seq * N, N, nonfinite);
  __syncthreads();  // every lane's TMEM loads are complete (fenced in tmem_gather16)
  if (j < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tg.tmem), "n"(TMEM_COLS) : "memory");
  }
}

// Two-warp kernel for N = 2 * 32 * R (fp64 N = 2048 with R = 32): one level of
// radix-2 decimation in time around two one-warp Stockham FFTs.
//
// A length-N transform with R elements per thread needs ceil(log_R N) passes,
// i.e. three for fp64 N = 2048 at R <= 32 (R = 64 would need 256 registers
// of data).  Here the CTA (64 threads) takes one sequence with one bulk TMA
// copy; warp w transforms the w-th polyphase half h_w[i] = x[2i + w] (i < N/2)
// with the two-pass, __syncwarp-only passes of the N/2 kernel in its own
// exchange region; then the warps trade half their results through shared
// memory (one 64-thread barrier) and finish with the radix-2 combine
//   X[k] = E[k] + w_N^k O[k],   X[k + N/2] = E[k] - w_N^k O[k]
// -- warp 0 for k < N/4, warp 1 for k >= N/4 -- storing coalesced rows.
// Per element: 1.5 shared-memory exchanges instead of 2 and one CTA barrier
// instead of four.  The gather of the polyphase halves from the linear TMA
// staging reads every other 16-byte element (2-way bank conflict on that
// one access; the exchanges stay conflict-free).
// Twiddles: the N/2 transform's per-pass table, then w_N^k for k < N/2 --
// exactly the generic per-pass table of the pass list [R, ..., 2].
template <typename T, int N, int R, bool INV, int LAYOUT, int TWP, bool RIN = false>
__global__ void __launch_bounds__(64, 6)  // <= 168 registers: 6 CTAs (12 warps) per SM
split2_kernel(const std::conditional_t<RIN, T, cx_t<T>>* __restrict__ in, cx_t<T>* __restrict__ out,
              const cx_t<T>* __restrict__ tw, long long batch, int* __restrict__ nonfinite) {
  using C = cx_t<T>;
  using S = Smem<T, LAYOUT, R>;
  constexpr int H = N / 2;       // half length
  constexpr int G = H / R;       // threads per half transform
  constexpr int SH = S::size(H);  // exchange elements per warp
  constexpr int HR = R / 2;
  static_assert(G == 32, "one warp per half transform");
  static_assert(2 * SH >= N, "staging fits the exchange regions");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sm = reinterpret_cast<C*>(smem_raw);
  __shared__ __align__(8) unsigned long long bar;

  const int tid = threadIdx.x;
  const int w = tid >> 5;
  const int j = tid & 31;
  const long long seq = blockIdx.x;  // one sequence per CTA: every CTA is full
  pdl_enter();

  if (tid == 0) {
    mbar_init(&bar, 1);
    constexpr uint32_t bytes = uint32_t(N * int(sizeof(*in)));
    mbar_expect_tx(&bar, bytes);
    bulk_g2s(sm, in + seq * N, bytes, &bar);
  }
  __syncthreads();  // barrier initialised before anyone polls it
  mbar_wait(&bar, 0);

  // polyphase half w: v[m] = x[2 (j + m G) + w]
  C v[R];
  if constexpr (RIN) {
    const T* smr = reinterpret_cast<const T*>(smem_raw);
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = C{smr[2 * (j + m * G) + w], T(0)};
  } else {
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = sm[2 * (j + m * G) + w];
  }
  __syncthreads();  // staging fully read before the exchange regions reuse it
  const bool in_place = static_cast<const void*>(in) == static_cast<const void*>(out);
  if (nonfinite != nullptr && in_place) check_nonfinite<T, R>(v, nonfinite);
  if constexpr (INV) {
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cswap(v[m]);
  }
  // E (w = 0) or O (w = 1) in natural order: v[m] = F[j + m G]
  stockham_passes<T, H, R, 1, false, LAYOUT, TWP>(v, sm + w * SH, 0, j, 0, nullptr, tw);

  // trade halves: warp 0 keeps k < H/2 and needs O there; warp 1 keeps
  // k >= H/2 and needs E there.  Linear [m][lane] slots: conflict-free.
  __syncthreads();  // both warps done with their exchange regions
  C* xs = sm;
  if (w == 0) {
#pragma unroll
    for (int m = 0; m < HR; ++m) xs[(HR + m) * 32 + j] = v[HR + m];  // E, upper
  } else {
#pragma unroll
    for (int m = 0; m < HR; ++m) xs[m * 32 + j] = v[m];  // O, lower
  }
  __syncthreads();
  const C* twc = tw + twiddle_table_len(H, R);  // w_N^k, k < H
  C* dst = out + seq * N;
  constexpr T scale = T(1) / T(N);  // exact: N = 2^k
  auto combine = [&](C e, C o, int k) {
    const C t = cmul(o, __ldg(twc + k));
    C y0 = cadd(e, t);
    C y1 = csub(e, t);
    if constexpr (INV) {
      y0 = cscale(cswap(y0), scale);
      y1 = cscale(cswap(y1), scale);
    }
    st_stream(dst + k, y0);
    st_stream(dst + k + H, y1);
  };
  if (w == 0) {
    // X[0] = E[0] + O[0]: the out-of-place NaN/Inf check (see recheck_row_inputs)
    if (nonfinite != nullptr && !in_place && j == 0 && !cx_finite(cadd(v[0], xs[j])))
      recheck_row_inputs(in + seq * N, N, nonfinite);
#pragma unroll
    for (int m = 0; m < HR; ++m) combine(v[m], xs[m * 32 + j], j + m * G);
  } else {
#pragma unroll
    for (int m = 0; m < HR; ++m) combine(xs[(HR + m) * 32 + j], v[HR + m], j + (HR + m) * G);
  }
}

// Four-step kernel for fp64 N = 2048 = 32 x 64 with ONE shared-memory
// exchange per row (the R16 default has two): 128 threads, one sequence per
// CTA, 16 complex doubles per thread.  With n = n1 + 32 n2, k = k2 + 64 k1,
//   X[k2 + 64 k1] = sum_n1 W32^(n1 k1) W2048^(n1 k2) sum_n2 x[n1 + 32 n2] W64^(n2 k2).
// Step A, the 32 length-64 DFTs over n2, each on a lane quad (c0, c1) =
//   (lane bit 3, lane bit 4): lane c = c0 + 2 c1 takes n2 = 4a + c, a
//   radix-16 DFT in registers, then two radix-2 levels across the quad
//   (lane ^ 16, then lane ^ 8) through __shfl_xor.
// Step B, the twiddles W2048^(n1 k2): 6 table loads per thread, the other
//   powers by one or two products (as TWP 2).
// Step C, one swizzled shared-memory transpose to (k2, d) per thread, the 32
//   length-32 DFTs over n1 = 2b + d as a radix-16 DFT in registers and one
//   radix-2 level across lane ^ 16, and coalesced stores.
// A shuffle moves each 4-byte word once (one L1 data-pipe cycle per 128 B);
// a shared-memory exchange writes and reads it (two).  L1 data pipe per row:
// gather 256 + exchange 512 + shuffles 384 + stores 256 + twiddles ~48
// wavefronts, against ~1950 for the R16 default (gather, two exchanges,
// stores, twiddles, bulk-copy collisions) -- the unit that bounds that kernel
// under the power cap (profiles/r02_fp64_2048_datapipe.txt).  Conflict-free
// (tests/test_bank_model.py: fourstep_instructions).
// Measured (profiles/r02_fourstep_study.txt): the data pipe drops to 57 %,
// but the operand selects make it issue-heavier (49 vs 33 % issue active)
// and the per-row critical path longer; with 4-5 rows in flight per SM it
// reaches 0.94-0.95x the copy at burst -- a tested variant, not the default.
// Every radix-2 level across a lane pair has both lanes send registers
// 8..15: the upper lane's inputs are pre-modulated by (-1)^(input index)
// (and, for c0 = c1 = 1, negated -- a half-swap of its level-2 operands), which
// rotates its radix-16 outputs by 8, so no lane needs a per-lane register
// choice to send; each lane then picks (z0, z1) from (own, received) with one
// select, and the level's twiddle W^k for its own k.  Table (plan-built,
// tw[c * 32 + n1], w = W2048^n1): c = 0..3 w^1..w^4; c = 4..11 w^(8 j), j = 0..7.
template <typename C>
__device__ __forceinline__ C shfl_xor_c(C v, int m) {
  return C{__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m)};
}
// One radix-2 level across lanes (l, l ^ M) on 2 x 8 registers: on entry
// the lower lane (upper = false) holds A[k] in v[k] and the upper lane holds
// B[(k + 8) mod 16] in v[k] (pre-rotated); the level computes, for its own
// k = i + 8 upper, v[i] = A[k] + w_k B[k] and v[8 + i] = A[k] - w_k B[k] with
// w_k = W_L^(i + J) * (-i)^upper, J = 0 or JSEL (runtime `jsel`).
template <int M, int L, int JSEL, typename C>
__device__ __forceinline__ void pair_level(C (&v)[16], bool upper, bool jsel) {
  using T = decltype(v[0].x);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[8 + i] = shfl_xor_c(v[8 + i], M);
  static_for<0, 8>([&](auto I) {
    constexpr int i = decltype(I)::value;
    const C own = v[i];
    const C got = v[8 + i];
    const C z0 = upper ? got : own;
    const C z1 = upper ? own : got;
    C t;
    if constexpr (JSEL == 0) {
      t = twiddle_const<i, L>(z1);
    } else {
      constexpr int j0 = i * (64 / L), j1 = (i + JSEL) * (64 / L);
      const T c = jsel ? T(cos64(j1)) : T(cos64(j0));
      const T s = jsel ? T(-sin64(j1)) : T(-sin64(j0));
      t = cmul(z1, C{c, s});
    }
    t = upper ? mul_minus_i(t) : t;
    v[i] = cadd(z0, t);
    v[8 + i] = csub(z0, t);
  });
}
__device__ __forceinline__ double flip_sign(double x, int sign_hi) {
  return __hiloint2double(__double2hiint(x) ^ sign_hi, __double2loint(x));
}

template <typename T, bool INV, bool RIN = false, int MINB = 5>
__global__ void __launch_bounds__(128, MINB)
fourstep_kernel(const std::conditional_t<RIN, T, cx_t<T>>* __restrict__ in, cx_t<T>* __restrict__ out,
                const cx_t<T>* __restrict__ tw, long long batch, int* __restrict__ nonfinite) {
  using C = cx_t<T>;
  constexpr int N = 2048;
  constexpr int R = 16;
  static_assert(sizeof(T) == 8, "fp64 geometry (128 threads x 16 complex doubles)");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sm = reinterpret_cast<C*>(smem_raw);
  __shared__ __align__(8) unsigned long long bar;

  const int tid = threadIdx.x;
  const int w = tid >> 5;
  const int lane = tid & 31;
  const bool c0 = (lane >> 3) & 1;
  const bool c1 = (lane >> 4) & 1;
  const int n1 = (lane & 7) + 8 * w;
  const long long seq = blockIdx.x;  // one sequence per CTA: every CTA is full
  pdl_enter();

  if (tid == 0) {
    mbar_init(&bar, 1);
    constexpr uint32_t bytes = uint32_t(N * int(sizeof(*in)));
    mbar_expect_tx(&bar, bytes);
    bulk_g2s(sm, in + seq * N, bytes, &bar);
  }
  __syncthreads();  // barrier initialised before anyone polls it
  mbar_wait(&bar, 0);

  // v[a] = x[n1 + 32 (4 a + c)]: 8-lane phases read 128 contiguous bytes
  C v[R];
  const int g0 = n1 + 32 * (int(c0) + 2 * int(c1));
  if constexpr (RIN) {
    const T* smr = reinterpret_cast<const T*>(smem_raw);
#pragma unroll
    for (int a = 0; a < R; ++a) v[a] = C{smr[g0 + 128 * a], T(0)};
  } else {
#pragma unroll
    for (int a = 0; a < R; ++a) v[a] = sm[g0 + 128 * a];
  }
  __syncthreads();  // staging fully read before the exchange reuses it
  const bool in_place = static_cast<const void*>(in) == static_cast<const void*>(out);
  if (nonfinite != nullptr && in_place) check_nonfinite<T, R>(v, nonfinite);
  if constexpr (INV) {
#pragma unroll
    for (int a = 0; a < R; ++a) v[a] = cswap(v[a]);
  }

  // ---- step A.  Upper lanes of level 1 (c1): (-1)^a rotates their outputs
  // by 8; lane (1, 1) also negates (swaps the halves its level-2 operands
  // land in, so level 2's upper lanes send the right half too).
  {
    const int s_odd = int(c1) << 31;
    const int s_all = int(c0 && c1) << 31;
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const int sg = (a & 1) ? (s_odd ^ s_all) : s_all;
      v[a].x = flip_sign(v[a].x, sg);
      v[a].y = flip_sign(v[a].y, sg);
    }
  }
  dft_regs<R>(v);  // Z_c[k'] (rotated by 8 on c1 lanes)
  // level 1 (n2 bit 1, lanes ^ 16): V_c0[k' + 16 h] at v[8 h + i], k' = i + 8 c1
  pair_level<16, 32, 0>(v, c1, false);
  // level 2 (n2 bit 0, lanes ^ 8): Y[k2] at v[8 h + i], k2 = i + 8 c1 + 16 c0 + 32 h
  pair_level<8, 64, 8>(v, c0, c1);

  // ---- step B.  v[8 h + i] *= w^(8 (c1 + 2 c0) + 32 h) w^i, w = W2048^n1
  {
    const C* tn = tw + n1;
    C wp[8];
#pragma unroll
    for (int i = 1; i <= 4; ++i) wp[i] = __ldg(tn + (i - 1) * 32);
#pragma unroll
    for (int i = 5; i < 8; ++i) wp[i] = cmul(wp[4], wp[i - 4]);
    const int j = int(c1) + 2 * int(c0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const C eh = __ldg(tn + (4 + j + 4 * h) * 32);
      v[8 * h] = cmul(v[8 * h], eh);
#pragma unroll
      for (int i = 1; i < 8; ++i) v[8 * h + i] = cmul(v[8 * h + i], cmul(eh, wp[i]));
    }
  }

  // ---- step C.  Transpose: slot(n1, k2) = 64 n1 + (k2 ^ (n1 & 7)) (8-lane
  // phases: 8 consecutive n1 on write, 8 consecutive k2 on read).
  {
    const int x = n1 & 7;
    C* wrow = sm + 64 * n1 + 8 * int(c1) + 16 * int(c0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      wrow[i ^ x] = v[i];
      wrow[32 + (i ^ x)] = v[8 + i];
    }
  }
  __syncthreads();
  // thread (k2, d): k2 = (lane & 15) + 16 w, d = lane bit 4; v[b] = Y'[2 b + d][k2]
  const int k2 = (lane & 15) + 16 * w;
  const bool d = c1;
  {
    const C* rrow = sm + 64 * int(d);
    int kx[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) kx[q] = k2 ^ (2 * q + int(d));
    const int s_odd = int(d) << 31;  // (-1)^b on the upper lanes: outputs rotated by 8
#pragma unroll
    for (int b = 0; b < R; ++b) {
      C y = rrow[128 * b + kx[b & 3]];
      if (b & 1) y = C{flip_sign(y.x, s_odd), flip_sign(y.y, s_odd)};
      v[b] = y;
    }
  }
  dft_regs<R>(v);
  // n1 bit 0 (lanes ^ 16): X[k2 + 64 (k1' + 16 q)] at v[8 q + i], k1' = i + 8 d
  pair_level<16, 32, 0>(v, d, false);

  C* dst = out + seq * N + k2 + 512 * int(d);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    C y = v[r];
    if constexpr (INV) y = cscale(cswap(y), T(1) / T(N));  // exact: N = 2^k
    st_stream(dst + 64 * (r & 7) + 1024 * (r >> 3), y);
  }
  // X[0] (thread 0, v[0]): the out-of-place NaN/Inf check (see recheck_row_inputs)
  if (nonfinite != nullptr && !in_place && tid == 0 && !cx_finite(v[0]))
    recheck_row_inputs(in + seq * N, N, nonfinite);
}

// Persistent, pipelined variant: a grid of (SMs x resident CTAs) walks the
// batch in tiles of SEQ sequences (tile t, t + grid, ...).  Each CTA owns
// STAGES shared-memory buffers; one thread keeps STAGES - 1 bulk TMA copies
// (cp.async.bulk + mbarrier complete_tx) of the CTA's next tiles in flight
// while every thread computes the current one, whose staging buffer then
// doubles as the exchange buffer of its passes.  Loads stay in flight through
// the compute phases, independent of how fast the SMs clock.
// Measured (profiles/r01_pipe_vs_resident.txt): 5.2-6.3 TB/s against
// 6.9 TB/s for the resident-CTA kernel above, burst and sustained alike.  The
// in-flight tiles must live in shared memory, so at equal on-chip bytes the
// pipeline runs 2-3 CTAs (8-12 warps) per SM where the LDG kernel runs 4-7
// (16-28 warps) with its in-flight lines in L1 -- the extra 100+ KB of L1 is
// what the resident design buys, and the pipeline's compute becomes
// latency-bound.  Kept as a tested variant, not a default.
template <typename T, int N, int R, int SEQ, bool INV, int LAYOUT, int TWP, int STAGES>
__global__ void __launch_bounds__((N / R) * SEQ)
stockham_pipe_kernel(const cx_t<T>* __restrict__ in, cx_t<T>* __restrict__ out,
                     const cx_t<T>* __restrict__ tw, long long batch, int* __restrict__ nonfinite) {
  using C = cx_t<T>;
  using S = Smem<T, LAYOUT, R>;
  constexpr int G = N / R;
  constexpr int SN = S::size(N);
  constexpr int BUF = SEQ * SN;  // elements per stage buffer (>= SEQ*N linear staging)
  static_assert(STAGES >= 2 && STAGES <= 8, "stages");
  static_assert(G >= 1 && (N % R) == 0, "geometry");
  static_assert(G <= 32 || SEQ <= 4, "named barrier ids");

  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sm = reinterpret_cast<C*>(smem_raw);
  __shared__ __align__(8) unsigned long long full[STAGES];

  const int tid = threadIdx.x;
  const int s = tid / G;
  const int j = tid - s * G;
  const long long ntiles = (batch + SEQ - 1) / SEQ;
  const long long step = gridDim.x;
  const bool in_place = static_cast<const void*>(in) == static_cast<const void*>(out);
  pdl_enter();

  auto issue = [&](long long tile, int b) {  // one thread
    const long long seq0 = tile * SEQ;
    const long long nseq = batch - seq0 < SEQ ? batch - seq0 : SEQ;
    const uint32_t bytes = uint32_t(nseq * N * int(sizeof(C)));
    mbar_expect_tx(&full[b], bytes);
    bulk_g2s(sm + b * BUF, in + seq0 * N, bytes, &full[b]);
  };
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < STAGES; ++b) mbar_init(&full[b], 1);
#pragma unroll
    for (int b = 0; b < STAGES - 1; ++b) {
      const long long tile = blockIdx.x + b * step;
      if (tile < ntiles) issue(tile, b);
    }
  }
  __syncthreads();  // barriers initialised before anyone polls them

  int b = 0;
  uint32_t phase = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += step) {
    // refill the buffer freed by the previous tile: STAGES - 1 loads stay in
    // flight while this one is computed
    if (tid == 0) {
      const long long ahead = tile + (STAGES - 1) * step;
      if (ahead < ntiles) issue(ahead, b == 0 ? STAGES - 1 : b - 1);
    }
    C* buf = sm + b * BUF;
    const long long seq = tile * SEQ + s;
    const bool valid = seq < batch;
    mbar_wait(&full[b], phase);
    C v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = buf[s * N + j + m * G];  // linear staging, conflict-free
    if (nonfinite != nullptr && valid && in_place) check_nonfinite<T, R>(v, nonfinite);
    __syncthreads();  // staging fully read before the exchange layout reuses it
    stockham_passes<T, N, R, SEQ, INV, LAYOUT, TWP>(v, LAYOUT == 1 ? buf + s * SN : buf, LAYOUT == 1 ? 0 : s * N,
                                                    j, s, valid ? out + seq * N : nullptr, tw);
    if (nonfinite != nullptr && valid && !in_place && j == 0 && !cx_finite(v[0]))
      recheck_row_inputs(in + seq * N, N, nonfinite);
    // every generic-proxy access to `buf` is done before the async proxy
    // (the refill issued at the top of the next iteration) overwrites it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (++b == STAGES) {
      b = 0;
      phase ^= 1;
    }
  }
}

// -------------------------------------------------------------- tile kernel
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <typename C>
__device__ __forceinline__ void chunk_to_cx(float4 f, C* dst);
template <>
__device__ __forceinline__ void chunk_to_cx<float2>(float4 f, float2* dst) {
  dst[0] = make_float2(f.x, f.y);
  dst[1] = make_float2(f.z, f.w);
}
template <>
__device__ __forceinline__ void chunk_to_cx<double2>(float4 f, double2* dst) {
  dst[0] = *reinterpret_cast<const double2*>(&f);
}
template <typename C>
__device__ __forceinline__ float4 cx_to_chunk(const C* src);
template <>
__device__ __forceinline__ float4 cx_to_chunk<float2>(const float2* src) {
  return make_float4(src[0].x, src[0].y, src[1].x, src[1].y);
}
template <>
__device__ __forceinline__ float4 cx_to_chunk<double2>(const double2* src) {
  return *reinterpret_cast<const float4*>(src);
}

template <typename T, int N, bool INV>
__device__ __forceinline__ void seq_dft(cx_t<T> (&x)[N], uint32_t& bad, bool check) {
  if (check) {
#pragma unroll
    for (int i = 0; i < N; ++i) bad |= nonfinite_bits(x[i]);
  }
  if constexpr (INV) {
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = cswap(x[i]);
  }
  dft_regs<N>(x);
  if constexpr (INV) {
    constexpr T scale = T(1) / T(N);
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = cscale(cswap(x[i]), scale);
  }
}

// 16-byte chunk of real input -> complex elements with zero imaginary parts
template <typename C>
__device__ __forceinline__ void chunk_to_reals(float4 f, C* dst);
template <>
__device__ __forceinline__ void chunk_to_reals<float2>(float4 f, float2* dst) {
  dst[0] = make_float2(f.x, 0.f);
  dst[1] = make_float2(f.y, 0.f);
  dst[2] = make_float2(f.z, 0.f);
  dst[3] = make_float2(f.w, 0.f);
}
template <>
__device__ __forceinline__ void chunk_to_reals<double2>(float4 f, double2* dst) {
  const double2 d = *reinterpret_cast<const double2*>(&f);
  dst[0] = make_double2(d.x, 0.0);
  dst[1] = make_double2(d.y, 0.0);
}

// Shared memory per warp tile, in 16-byte chunks: the complex tile (staged
// input and output in place), plus a separate input tile for real input.
template <typename T, int N, int SPT, bool RIN>
__host__ __device__ constexpr int tile_chunks() {
  constexpr int K = N * int(sizeof(cx_t<T>)) / 16;
  constexpr int KI = RIN ? N * int(sizeof(T)) / 16 : 0;
  return K == 1 ? 0 : 32 * SPT * (K + KI);
}

// RIN: real input rows (see stockham_kernel); fp32 N = 2 reads one 8-byte
// pair per sequence directly, the other sizes stage the real tile in its
// own shared region and write the complex results to the output region.
template <typename T, int N, int SPT, int WARPS, bool INV, bool RIN = false>
__global__ void __launch_bounds__(32 * WARPS)
tile_kernel(const std::conditional_t<RIN, T, cx_t<T>>* __restrict__ in, cx_t<T>* __restrict__ out, long long batch,
            int* __restrict__ nonfinite) {
  using C = cx_t<T>;
  constexpr int E = sizeof(C);
  constexpr int EPC = 16 / E;         // elements per 16-byte chunk
  constexpr int K = N / EPC;          // output (complex) chunks per sequence
  static_assert(K >= 1 && N % EPC == 0, "tile geometry");
  constexpr int RPC = 16 / int(sizeof(T));   // reals per chunk
  constexpr int KI = RIN ? N / RPC : K;      // input chunks per sequence (0: fp32 N=2 real)
  constexpr int TILE_CH = 32 * SPT * K;      // output chunks per warp tile
  constexpr int TILE_IN = 32 * SPT * KI;     // input chunks per warp tile
  constexpr int CPL = SPT * K;               // output chunks per lane

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const long long tile = (long long)blockIdx.x * WARPS + warp;
  const long long total_ch = batch * K;
  const long long ch0 = tile * TILE_CH;
  const float4* gin = reinterpret_cast<const float4*>(in);
  float4* gout = reinterpret_cast<float4*>(out);
  const bool check = nonfinite != nullptr;
  uint32_t bad = 0;
  pdl_enter();

  if constexpr (K == 1) {
    // one chunk == one sequence: no staging
    float4 f[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const long long c = ch0 + lane + 32 * i;
      if constexpr (RIN) {  // fp32 N = 2: one float2 of reals per sequence
        const float2 r = c < total_ch ? ld_stream(reinterpret_cast<const float2*>(in) + c) : make_float2(0.f, 0.f);
        f[i] = make_float4(r.x, 0.f, r.y, 0.f);
      } else {
        f[i] = c < total_ch ? ld_stream(gin + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      C x[N];
      chunk_to_cx<C>(f[i], x);
      seq_dft<T, N, INV>(x, bad, check);
      f[i] = cx_to_chunk<C>(x);
    }
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const long long c = ch0 + lane + 32 * i;
      if (c < total_ch) st_stream(gout + c, f[i]);
    }
  } else {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4* ws = reinterpret_cast<float4*>(smem_raw) + warp * tile_chunks<T, N, SPT, RIN>();
    float4* wi = RIN ? ws + TILE_CH : ws;  // staged input
    const long long total_in = batch * KI;
    const long long ci0 = tile * TILE_IN;
#pragma unroll
    for (int i = 0; i < SPT * KI; ++i) {
      const int c = lane + 32 * i;
      const long long gc = ci0 + c;
      if (gc < total_in) {
        cp_async16(wi + swz_chunk(c), gin + gc);
      } else {
        wi[swz_chunk(c)] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    cp_async_wait_all();
    __syncwarp();
#pragma unroll 1
    for (int u = 0; u < SPT; ++u) {
      const int q = u * 32 + lane;  // sequence within the tile
      C x[N];
      if constexpr (RIN) {
#pragma unroll
        for (int c = 0; c < KI; ++c) chunk_to_reals<C>(wi[swz_chunk(q * KI + c)], x + c * RPC);
      } else {
#pragma unroll
        for (int c = 0; c < K; ++c) chunk_to_cx<C>(ws[swz_chunk(q * K + c)], x + c * EPC);
      }
      seq_dft<T, N, INV>(x, bad, check);
#pragma unroll
      for (int c = 0; c < K; ++c) ws[swz_chunk(q * K + c)] = cx_to_chunk<C>(x + c * EPC);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int c = lane + 32 * i;
      const long long gc = ch0 + c;
      if (gc < total_ch) st_stream(gout + gc, ws[swz_chunk(c)]);
    }
  }
  if (bad) atomicOr(nonfinite, 1);
}

}  // namespace sfft
