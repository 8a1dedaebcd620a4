// Instantiation unit: double-double glynn sweep for n = 1 .. 32.
#include "perm_registry.h"
#include "perm_kernels_dd.cuh"
namespace permb200 {
void register_dd_glynn_a(SweepLauncher* t) { fill_sweep_dd<kGlynn, 1>(t, std::make_integer_sequence<int, 32>{}); }
}  // namespace permb200
