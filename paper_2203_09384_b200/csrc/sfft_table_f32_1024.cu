// Kernel variants of fp32 N = 1024 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f32_1024(int log2n) {
  switch (log2n) {
    case 10:
      return {
          stockham_variant<float, 1024, 32, 2, 1, 1, 0, true>(),
          stockham_variant<float, 1024, 16, 1, 1, 1, 1>(),
          stockham_variant<float, 1024, 16, 1, 1, 1>(),
          stockham_variant<float, 1024, 16, 1, 1>(),
          stockham_variant<float, 1024, 32, 4, 1>(),
          stockham_variant<float, 1024, 16, 2, 1>(),
          stockham_variant<float, 1024, 16, 2, 1, 1, 1>(),
          stockham_variant<float, 1024, 32, 4, 1, 1>(),
          pipe_variant<float, 1024, 16, 2, 1, 1, 3>(),
          stockham_variant<float, 1024, 32, 2, 1, 2, 0, true>(),
          stockham_variant<float, 1024, 32, 4, 1, 1, 1>(),  // r02 study: R32 + bulk TMA, 4 sequences
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
