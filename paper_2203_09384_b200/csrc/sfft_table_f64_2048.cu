// Kernel variants of fp64 N = 2048 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f64_2048(int log2n) {
  switch (log2n) {
    case 11:
      return {
          stockham_variant<double, 2048, 16, 1, 2, 1, 1, true>(),
          stockham_variant<double, 2048, 16, 1, 2>(),
          stockham_variant<double, 2048, 8, 1, 2, 1>(),
          stockham_variant<double, 2048, 16, 1, 1>(),
          stockham_variant<double, 2048, 16, 1, 2, 1>(),
          pipe_variant<double, 2048, 16, 1, 2, 1, 3>(),
          stockham_variant<double, 2048, 16, 1, 2, 2, 1>(),  // TWP 2 + bulk TMA
          stockham_variant<double, 2048, 16, 1, 2, 0, 1>(),  // TWP 0 + bulk TMA
          pipe_variant<double, 2048, 16, 1, 2, 1, 2>(),      // 2-stage pipeline (64 KB, 3 CTAs/SM)
          // R32 (passes [32, 32, 2], two warps per sequence) + bulk TMA: +1.2 %
          // sustained, -1.2 % burst, +5 % real input against entry 0 -- within
          // box-to-box noise, so entry 0 stays (profiles/r02_wide_radix_study.txt)
          stockham_variant<double, 2048, 32, 1, 2, 1, 1, true>(),
          stockham_variant<double, 2048, 32, 1, 2, 1, 0>(),  // R32, LDG
          // two one-warp N/2 transforms + radix-2 combine (split2_kernel, 6 CTAs
          // per SM).  Against entry 0: sustained +1 to +3 %, real input 6.28 vs
          // 5.67 TB/s, burst -1.9 %, and its polyphase gather reads every other
          // 16-byte element of the linear TMA staging (2-way bank conflict: 25 %
          // excess shared wavefronts); staging with a per-row skew removes the
          // conflict but needs 256 small bulk copies per row, which cut the rate
          // to 5.76 TB/s.  Kept as a tested variant (profiles/r02_wide_radix_study.txt).
          split2_variant<double, 2048, 32, 2, 1, true>(),
          // The two below probe what limits entry 0 under the power cap -- the
          // L1 data pipe (LSU wavefronts), not shared-memory capacity or the
          // FP64 pipe (profiles/r02_fp64_2048_datapipe.txt):
          // split re/im exchange (LAYOUT 3, 16 KB per sequence) + per-thread
          // loads: 28 % fewer shared wavefronts, but the LDG data costs more
          // data-pipe cycles than bulk copy + gather; burst -0.2 %, sustained +0.6 %
          stockham_variant<double, 2048, 16, 1, 3, 1, 0, true>(),
          // TWP 3 (one twiddle load per butterfly, squarings) + bulk TMA: data
          // pipe 75.6 -> 70.4 %, sustained +1.8 %, burst equal, but 19 % more
          // fp64 error (rel-L2 6.6e-16 vs 5.5e-16), so entry 0 stays
          stockham_variant<double, 2048, 16, 1, 2, 3, 1, true>(),
          // bulk TMA + tensor-memory gathers: entry 0's kernel with the staging
          // gather and the last exchange's gather on tcgen05.cp/ld (loader 3),
          // or the staging gather only (loader 4).  The L1 data pipe drops from
          // 75.6 to 43 % of peak, but each 32 KB copy into TMEM takes ~512
          // cycles (64 B/clk) on the CTA's critical path: burst 5.55 / 6.14 vs
          // 6.96 TB/s, sustained 5.20 / 5.41 vs 5.81 (profiles/r02_fp64_2048_datapipe.txt)
          tmem_variant<double, 2048, 16, 1, true>(),
          tmem_variant<double, 2048, 16, 1, true, 1, false>(),
          // four-step 32 x 64 (fourstep_kernel): one shared-memory exchange per
          // row, three radix-2 levels through warp shuffles.  The L1 data pipe
          // drops from 74 to 57 % of peak, but choosing each lane's butterfly
          // operands costs ~300 selects per thread (issue 33 -> 49 %), the row's
          // critical path grows, and with 4-5 rows in flight per SM that is the
          // rate: burst 0.94-0.95x copy, sustained 5.13-5.18 vs 5.73 TB/s for
          // entry 0 (profiles/r02_fourstep_study.txt).  A 64-thread form (32
          // elements per thread, one shuffle level) was latency-bound too (0.94x).
          fourstep_variant<double, true, 4>(),
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
