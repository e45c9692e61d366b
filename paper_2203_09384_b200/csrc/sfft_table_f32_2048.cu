// Kernel variants of fp32 N = 2048 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f32_2048(int log2n) {
  switch (log2n) {
    case 11:
      return {
          // default: two-level twiddles (TWP 2) -- ramp-2048 |error| 0.072 against
          // 0.129 for TWP 1, inside the reference's own 0.1 bound
          // (tests/test_stats.py:211-222); burst equal, sustained -0.7 %
          // (profiles/r02_twiddle_policy.txt)
          stockham_variant<float, 2048, 16, 1, 1, 2, 0, true>(),
          stockham_variant<float, 2048, 16, 1, 1>(),
          stockham_variant<float, 2048, 16, 1, 2>(),
          stockham_variant<float, 2048, 32, 1, 1>(),
          stockham_variant<float, 2048, 16, 1, 1, 1, 1>(),
          stockham_variant<float, 2048, 32, 1, 1, 1>(),
          stockham_variant<float, 2048, 32, 2, 1, 1>(),
          stockham_variant<float, 2048, 16, 1, 1, 1>(),  // round-1 default (TWP 1)
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
