// Kernel variants of fp32 N = 2, 4, 8, 16, 32, 64, 128, 256 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f32_small(int log2n) {
  switch (log2n) {
    case 1:
      return {
          tile_variant<float, 2, 8, 4, true>(),
          tile_variant<float, 2, 4, 8>(),
      };
    case 2:
      return {
          tile_variant<float, 4, 4, 4, true>(),
          tile_variant<float, 4, 2, 8>(),
      };
    case 3:
      return {
          tile_variant<float, 8, 4, 4, true>(),
          tile_variant<float, 8, 2, 4>(),
      };
    case 4:
      return {
          tile_variant<float, 16, 2, 4, true>(),
          tile_variant<float, 16, 1, 8>(),
      };
    case 5:
      return {
          tile_variant<float, 32, 1, 4, true>(),
          stockham_variant<float, 32, 8, 32, 1>(),
      };
    case 6:
      return {
          stockham_variant<float, 64, 8, 16, 1, 1, 0, true>(),
          stockham_variant<float, 64, 16, 32, 1>(),
          stockham_variant<float, 64, 8, 16, 1>(),
          stockham_variant<float, 64, 8, 16, 1, 2, 0, true>(),
      };
    case 7:
      return {
          stockham_variant<float, 128, 16, 16, 1, 1, 0, true>(),
          stockham_variant<float, 128, 16, 16, 1>(),
          stockham_variant<float, 128, 8, 8, 1>(),
          stockham_variant<float, 128, 16, 16, 2, 1>(),
          stockham_variant<float, 128, 16, 16, 2>(),
          stockham_variant<float, 128, 16, 16, 1, 2, 0, true>(),
      };
    case 8:
      return {
          stockham_variant<float, 256, 16, 8, 1, 0, 0, true>(),
          stockham_variant<float, 256, 16, 8, 2>(),
          stockham_variant<float, 256, 16, 8, 1, 1>(),
          stockham_variant<float, 256, 16, 8, 1, 0, 1>(),
          stockham_variant<float, 256, 16, 8, 1, 2, 0, true>(),
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
