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
          stockham_variant<double, 2048, 16, 1, 2, 2, 1, true>(),
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
