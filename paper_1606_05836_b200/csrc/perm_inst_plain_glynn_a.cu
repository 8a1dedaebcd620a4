// Instantiation unit (plain-accumulation mode): kGlynn for n = 1 .. 24 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_plain_glynn_a(SweepLauncher* t) { fill_sweep_plain<kGlynn, 1>(t, std::make_integer_sequence<int, 24>{}); }
}  // namespace permb200
