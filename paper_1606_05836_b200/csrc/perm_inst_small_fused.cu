// Instantiation unit: fused small-n full permanent (one cooperative launch: sweep + grid
// barrier + canonical combine), Glynn n <= 22 and Ryser n <= 21, compensated, plain and separate-addition.
#include "perm_registry.h"
namespace permb200 {
void register_small_fused(FusedLauncher (*t)[kNMax + 1]) {
  fill_sweep_small_fused<kGlynn, kComp, 1>(t[0], std::make_integer_sequence<int, 22>{});
  fill_sweep_small_fused<kRyser, kComp, 1>(t[1], std::make_integer_sequence<int, 21>{});
  fill_sweep_small_fused<kGlynn, kPlain, 1>(t[4], std::make_integer_sequence<int, 22>{});
  fill_sweep_small_fused<kRyser, kPlain, 1>(t[5], std::make_integer_sequence<int, 21>{});
  fill_sweep_small_fused<kGlynn, kSep, 1>(t[6], std::make_integer_sequence<int, 22>{});
  fill_sweep_small_fused<kRyser, kSep, 1>(t[7], std::make_integer_sequence<int, 21>{});
}
}  // namespace permb200
