// Instantiation unit: kGlynn for n = 39 .. 51 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_glynn_c(SweepLauncher* t) { fill_sweep<kGlynn, 39>(t, std::make_integer_sequence<int, 13>{}); }
}  // namespace permb200
