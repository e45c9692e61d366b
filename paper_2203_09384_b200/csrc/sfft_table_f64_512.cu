// Kernel variants of fp64 N = 512 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f64_512(int log2n) {
  switch (log2n) {
    case 9:
      return {
          // default (round 2): R = 32, passes [32, 16] instead of [16, 16, 2];
          // 16 threads per sequence, 2 sequences per warp, one bulk TMA copy
          // per CTA.  Sustained 1.065 vs 1.029 of the copy (uncapped box),
          // burst -1 % (profiles/r02_wide_radix_study.txt).
          stockham_variant<double, 512, 32, 2, 2, 1, 1, true>(),
          stockham_variant<double, 512, 16, 4, 2, 1>(),     // round-1 default (R16 [16,16,2], LDG)
          stockham_variant<double, 512, 16, 2, 2>(),
          stockham_variant<double, 512, 8, 2, 1>(),
          stockham_variant<double, 512, 16, 4, 2>(),
          stockham_variant<double, 512, 16, 4, 2, 2>(),     // TWP 2
          stockham_variant<double, 512, 32, 2, 2, 1, 0>(),  // R32, LDG
          stockham_variant<double, 512, 32, 4, 2, 1, 1>(),  // R32, bulk TMA, 4 sequences per CTA
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
