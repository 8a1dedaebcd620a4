// Instantiation unit (plain-accumulation mode): kGlynn for n = 39 .. 51 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_plain_glynn_c(SweepLauncher* t) { fill_sweep_plain<kGlynn, 39>(t, std::make_integer_sequence<int, 13>{}); }
}  // namespace permb200
