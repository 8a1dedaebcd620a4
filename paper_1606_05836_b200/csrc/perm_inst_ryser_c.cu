// Instantiation unit: kRyser for n = 39 .. 51 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_ryser_c(SweepLauncher* t) { fill_sweep<kRyser, 39>(t, std::make_integer_sequence<int, 13>{}); }
}  // namespace permb200
