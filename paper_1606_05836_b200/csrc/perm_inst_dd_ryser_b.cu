// Instantiation unit: double-double ryser sweep for n = 33 .. 63.
#include "perm_registry.h"
#include "perm_kernels_dd.cuh"
namespace permb200 {
void register_dd_ryser_b(SweepLauncher* t) { fill_sweep_dd<kRyser, 33>(t, std::make_integer_sequence<int, 31>{}); }
}  // namespace permb200
