// Kernel variants of fp64 N = 1024 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f64_1024(int log2n) {
  switch (log2n) {
    case 10:
      return {
          // default (round 2): one warp per sequence, R = 32, passes [32, 32]
          // (one exchange, __syncwarp only), one bulk TMA copy per sequence.
          // Sustained power-capped load: 6350 vs 5976 GB/s for the round-1
          // R16 default (0.99 vs 0.94 of the copy's own sustained rate); real
          // input 6.80 vs 6.15 TB/s; burst -1.8 % (profiles/r02_wide_radix_study.txt).
          stockham_variant<double, 1024, 32, 1, 2, 1, 1, true>(),
          stockham_variant<double, 1024, 16, 1, 2, 1>(),     // round-1 default (R16 [16,16,4], LDG)
          stockham_variant<double, 1024, 16, 2, 2, 1>(),
          stockham_variant<double, 1024, 16, 1, 2>(),
          stockham_variant<double, 1024, 8, 1, 2>(),
          stockham_variant<double, 1024, 16, 2, 2, 1, 1>(),
          stockham_variant<double, 1024, 16, 1, 2, 2>(),     // TWP 2
          stockham_variant<double, 1024, 16, 1, 2, 0, 1>(),  // TWP 0 + bulk TMA
          stockham_variant<double, 1024, 32, 1, 2, 1, 0>(),  // R32, LDG
          stockham_variant<double, 1024, 32, 2, 2, 1, 1>(),  // R32, bulk TMA, 2 sequences per CTA
          stockham_variant<double, 1024, 32, 1, 2, 3, 1, true>(),  // TWP 3: burst and sustained within 0.1 % of entry 0
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
