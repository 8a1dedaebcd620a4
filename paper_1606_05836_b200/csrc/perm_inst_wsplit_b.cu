// Instantiation unit: warp-pair row-split sweep (perm_kernels_wsplit.cuh), compensated mode,
// Glynn and Ryser n = 56 .. 60 (this TU holds its own constant column slot).  n = 61 .. 64 stay on
// the 2-lane split of one warp (perm_kernels_split.cuh): measured 2026-10-21 (wsplit_bench, 2368
// units of 2^21 terms) FP64 issue 0.596 (warp pair) vs 0.680 (2-lane) at n = 64 and, in the library,
// 0.562 vs 0.714 at n = 62, against 0.743 vs 0.728 at n = 60 (profiles/r02_wsplit_bench.log).
#include "perm_registry.h"
#include "perm_kernels_wsplit.cuh"
namespace permb200 {
void register_wsplit_b(SweepLauncher (*t)[kNMax + 1]) {
  fill_wsplit<kGlynn, kComp, 56>(t[0], std::make_integer_sequence<int, 5>{});
  fill_wsplit<kRyser, kComp, 56>(t[1], std::make_integer_sequence<int, 5>{});
}
}  // namespace permb200
