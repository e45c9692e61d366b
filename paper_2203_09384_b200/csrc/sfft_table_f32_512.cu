// Kernel variants of fp32 N = 512 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f32_512(int log2n) {
  switch (log2n) {
    case 9:
      return {
          // real input with __launch_bounds__ min-blocks 6: ptxas schedules it
          // differently (128 registers, no spill) and it reads real rows at
          // 6.87 vs 6.80 TB/s (+1.0 %); a cap at 80 registers spills and
          // loses (6.71) -- profiles/r02_real_input_regcap.txt
          stockham_variant<float, 512, 32, 4, 1, 1, 0, true, 6>(),
          stockham_variant<float, 512, 16, 2, 1>(),
          stockham_variant<float, 512, 16, 4, 1>(),
          stockham_variant<float, 512, 16, 4, 1, 1>(),
          stockham_variant<float, 512, 32, 8, 1, 1>(),
          stockham_variant<float, 512, 32, 4, 1, 2, 0, true>(),
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
