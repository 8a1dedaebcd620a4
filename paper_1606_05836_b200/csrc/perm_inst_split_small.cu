// Instantiation unit: row-split sweep (4 lanes per chunk) for small n (2^m terms, m <= 21):
// Glynn n = 8 .. 22, Ryser n = 8 .. 21, compensated / plain / separate-addition modes; the plain
// sweep and the fused one-launch full permanent.  t[alg][n] (PERM_ALG_* codes 0, 1, 4, 5, 6, 7).
#include "perm_registry.h"
#include "perm_kernels_split.cuh"
namespace permb200 {
void register_split_small(SweepLauncher (*t)[kNMax + 1], FusedLauncher (*f)[kNMax + 1]) {
  fill_split<kGlynn, kComp, 4, 8>(t[0], std::make_integer_sequence<int, 15>{});
  fill_split<kRyser, kComp, 4, 8>(t[1], std::make_integer_sequence<int, 14>{});
  fill_split<kGlynn, kPlain, 4, 8>(t[4], std::make_integer_sequence<int, 15>{});
  fill_split<kRyser, kPlain, 4, 8>(t[5], std::make_integer_sequence<int, 14>{});
  fill_split<kGlynn, kSep, 4, 8>(t[6], std::make_integer_sequence<int, 15>{});
  fill_split<kRyser, kSep, 4, 8>(t[7], std::make_integer_sequence<int, 14>{});
  fill_split_fused<kGlynn, kComp, 4, 8>(f[0], std::make_integer_sequence<int, 15>{});
  fill_split_fused<kRyser, kComp, 4, 8>(f[1], std::make_integer_sequence<int, 14>{});
  fill_split_fused<kGlynn, kPlain, 4, 8>(f[4], std::make_integer_sequence<int, 15>{});
  fill_split_fused<kRyser, kPlain, 4, 8>(f[5], std::make_integer_sequence<int, 14>{});
  fill_split_fused<kGlynn, kSep, 4, 8>(f[6], std::make_integer_sequence<int, 15>{});
  fill_split_fused<kRyser, kSep, 4, 8>(f[7], std::make_integer_sequence<int, 14>{});
}
}  // namespace permb200
