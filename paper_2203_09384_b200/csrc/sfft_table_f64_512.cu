// Kernel variants of fp64 N = 512 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f64_512(int log2n) {
  switch (log2n) {
    case 9:
      return {
          stockham_variant<double, 512, 16, 4, 2, 1, 0, true>(),
          stockham_variant<double, 512, 16, 2, 2>(),
          stockham_variant<double, 512, 8, 2, 1>(),
          stockham_variant<double, 512, 16, 4, 2>(),
          stockham_variant<double, 512, 16, 4, 2, 2, 0, true>(),
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
