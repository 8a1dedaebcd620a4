// Instantiation unit: row-split sweep (2 lanes per chunk) for large n, compensated mode:
// Glynn n = 52 .. 64, Ryser n = 52 .. 63 (4n registers of row sums no longer fit one thread).
#include "perm_registry.h"
#include "perm_kernels_split.cuh"
namespace permb200 {
void register_split_large(SweepLauncher (*t)[kNMax + 1]) {
  fill_split<kGlynn, kComp, 2, 52>(t[0], std::make_integer_sequence<int, 13>{});
  fill_split<kRyser, kComp, 2, 52>(t[1], std::make_integer_sequence<int, 12>{});
}
}  // namespace permb200
