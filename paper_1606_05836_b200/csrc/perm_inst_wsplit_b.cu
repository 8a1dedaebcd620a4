// Instantiation unit: warp-pair row-split sweep (perm_kernels_wsplit.cuh), compensated mode,
// Glynn n = 56 .. 64, Ryser n = 56 .. 63 (this TU holds its own constant column slot).
#include "perm_registry.h"
#include "perm_kernels_wsplit.cuh"
namespace permb200 {
void register_wsplit_b(SweepLauncher (*t)[kNMax + 1]) {
  fill_wsplit<kGlynn, kComp, 56>(t[0], std::make_integer_sequence<int, 9>{});
  fill_wsplit<kRyser, kComp, 56>(t[1], std::make_integer_sequence<int, 8>{});
}
}  // namespace permb200
