// Kernel variants of fp64 N = 2, 4, 8, 16, 32, 64, 128, 256 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f64_small(int log2n) {
  switch (log2n) {
    case 1:
      return {
          tile_variant<double, 2, 4, 4, true>(),
          tile_variant<double, 2, 2, 8>(),
      };
    case 2:
      return {
          tile_variant<double, 4, 2, 4, true>(),
          tile_variant<double, 4, 1, 8>(),
      };
    case 3:
      return {
          tile_variant<double, 8, 1, 4, true>(),
          tile_variant<double, 8, 2, 4>(),
      };
    case 4:
      return {
          tile_variant<double, 16, 1, 4, true>(),
          stockham_variant<double, 16, 8, 64, 2>(),
      };
    case 5:
      return {
          stockham_variant<double, 32, 8, 32, 1, 1, 0, true>(),
          stockham_variant<double, 32, 8, 32, 2>(),
          stockham_variant<double, 32, 8, 32, 1>(),
          stockham_variant<double, 32, 8, 32, 1, 2, 0, true>(),
      };
    case 6:
      return {
          stockham_variant<double, 64, 8, 16, 1, 1, 0, true>(),
          stockham_variant<double, 64, 8, 16, 2>(),
          stockham_variant<double, 64, 8, 16, 1>(),
          stockham_variant<double, 64, 8, 16, 1, 2, 0, true>(),
      };
    case 7:
      return {
          stockham_variant<double, 128, 16, 16, 2, 1, 0, true>(),
          stockham_variant<double, 128, 8, 8, 1>(),
          stockham_variant<double, 128, 16, 16, 2>(),
          stockham_variant<double, 128, 16, 16, 2, 2, 0, true>(),
      };
    case 8:
      return {
          stockham_variant<double, 256, 16, 8, 2, 1, 0, true>(),
          stockham_variant<double, 256, 8, 4, 1>(),
          stockham_variant<double, 256, 16, 8, 2>(),
          stockham_variant<double, 256, 16, 8, 2, 2, 0, true>(),
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
