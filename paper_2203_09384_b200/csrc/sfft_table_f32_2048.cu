// Kernel variants of fp32 N = 2048 (one translation unit per group,
// so the instantiations compile in parallel; see build.py).  Entry 0 is the
// planner's default; the rest stay compiled for tuning and are parity-tested.
#include "sfft_variants.cuh"

namespace sfft_impl {

std::vector<Variant> table_f32_2048(int log2n) {
  switch (log2n) {
    case 11:
      return {
          // default (round 2): one warp per sequence, R = 64, passes [64, 32]
          // (one exchange, __syncwarp only), one bulk TMA copy per sequence,
          // TWP 1.  Under sustained power-capped load it holds 6.49-6.85 TB/s
          // where the round-1 R16 design held 6.09-6.57 (+4-7 %, >= 1.0x the
          // copy's own sustained rate); real input 6.50 vs 6.08 TB/s; burst
          // -1.2 % (profiles/r02_wide_radix_study.txt).  Ramp-2048 |error|
          // 0.066 < 0.1, the reference's bound (tests/test_stats.py:211-222).
          // Real input with a register cap of 168 (min 12 CTAs/SM): the real
          // loader's kernel otherwise takes 216 registers, 8 CTAs/SM instead of
          // the complex kernel's 12; capped 6.52 vs 6.34 TB/s of its traffic
          // (+2.9 %, bit-identical; profiles/r02_real_input_regcap.txt)
          stockham_variant<float, 2048, 64, 1, 1, 1, 1, true, 12>(),
          stockham_variant<float, 2048, 16, 1, 1, 2>(),     // R16 TWP 2 LDG (round-2 interim default)
          stockham_variant<float, 2048, 16, 1, 1>(),
          stockham_variant<float, 2048, 16, 1, 2>(),
          stockham_variant<float, 2048, 32, 1, 1>(),
          stockham_variant<float, 2048, 16, 1, 1, 1, 1>(),
          stockham_variant<float, 2048, 32, 1, 1, 1>(),
          stockham_variant<float, 2048, 32, 2, 1, 1>(),
          stockham_variant<float, 2048, 16, 1, 1, 1>(),     // round-1 default (R16 TWP 1 LDG)
          stockham_variant<float, 2048, 16, 1, 1, 2, 1>(),  // R16 TWP 2 + bulk TMA
          stockham_variant<float, 2048, 64, 1, 1, 1, 0>(),  // R64, LDG
          stockham_variant<float, 2048, 64, 4, 1, 1, 0>(),  // R64, LDG, 4 sequences per CTA
          stockham_variant<float, 2048, 64, 2, 1, 1, 1>(),  // R64, bulk TMA, 2 sequences per CTA
          stockham_variant<float, 2048, 64, 1, 1, 2, 1>(),  // R64, TWP 2, bulk TMA (ramp |error| 0.128 > 0.1)
      };
    default:
      return {};
  }
}

}  // namespace sfft_impl
