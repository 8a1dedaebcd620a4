// Instantiation unit: small-n sweep (shared-memory column table, m <= kSmallLog2 = 21) for
// Glynn n <= 22 and Ryser n <= 21, compensated, plain and separate-addition accumulation.
// t[alg]: PERM_ALG_GLYNN (0), PERM_ALG_RYSER (1), PERM_ALG_GLYNN_PLAIN (4), PERM_ALG_RYSER_PLAIN (5), PERM_ALG_GLYNN_SEP (6), PERM_ALG_RYSER_SEP (7).
#include "perm_registry.h"
namespace permb200 {
void register_small(SweepLauncher (*t)[kNMax + 1]) {
  fill_sweep_small<kGlynn, kComp, 1>(t[0], std::make_integer_sequence<int, 22>{});
  fill_sweep_small<kRyser, kComp, 1>(t[1], std::make_integer_sequence<int, 21>{});
  fill_sweep_small<kGlynn, kPlain, 1>(t[4], std::make_integer_sequence<int, 22>{});
  fill_sweep_small<kRyser, kPlain, 1>(t[5], std::make_integer_sequence<int, 21>{});
  fill_sweep_small<kGlynn, kSep, 1>(t[6], std::make_integer_sequence<int, 22>{});
  fill_sweep_small<kRyser, kSep, 1>(t[7], std::make_integer_sequence<int, 21>{});
}
}  // namespace permb200
