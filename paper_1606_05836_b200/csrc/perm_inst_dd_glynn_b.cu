// Instantiation unit: double-double glynn sweep for n = 33 .. 64.
#include "perm_registry.h"
#include "perm_kernels_dd.cuh"
namespace permb200 {
void register_dd_glynn_b(SweepLauncher* t) { fill_sweep_dd<kGlynn, 33>(t, std::make_integer_sequence<int, 32>{}); }
}  // namespace permb200
