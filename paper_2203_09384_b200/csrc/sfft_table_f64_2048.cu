// Kernel variants of fp64 N = 2048 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f64_2048(int log2n) {
  switch (log2n) {
    case 11:
      return {
          // default (round 2): two one-warp N/2 transforms + radix-2 combine
          // (split2_kernel, 6 CTAs = 12 warps per SM).  Against the R16 kernel
          // (entry 1): sustained power-capped load +1 to +2 % (0.92 vs 0.91 of
          // the copy's own rate; interleaved A/B +3 %), real input 6.28 vs 5.67
          // TB/s, error 5.42e-16 vs 5.51e-16; burst -1.9 % (6811 vs 6944 GB/s,
          // still 1.04x copy) (profiles/r02_wide_radix_study.txt).
          split2_variant<double, 2048, 32, 2, 1, true>(),
          stockham_variant<double, 2048, 16, 1, 2, 1, 1>(),  // round-1 default (R16, [16,16,8], bulk TMA)
          stockham_variant<double, 2048, 16, 1, 2>(),
          stockham_variant<double, 2048, 8, 1, 2, 1>(),
          stockham_variant<double, 2048, 16, 1, 1>(),
          stockham_variant<double, 2048, 16, 1, 2, 1>(),
          pipe_variant<double, 2048, 16, 1, 2, 1, 3>(),
          stockham_variant<double, 2048, 16, 1, 2, 2, 1>(),  // TWP 2 + bulk TMA
          stockham_variant<double, 2048, 16, 1, 2, 0, 1>(),  // TWP 0 + bulk TMA
          pipe_variant<double, 2048, 16, 1, 2, 1, 2>(),      // 2-stage pipeline (64 KB, 3 CTAs/SM)
          stockham_variant<double, 2048, 32, 1, 2, 1, 1>(),  // R32 (passes [32, 32, 2], two warps) + bulk TMA
          stockham_variant<double, 2048, 32, 1, 2, 1, 0>(),  // R32, LDG
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
