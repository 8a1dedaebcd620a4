// Instantiation unit (plain-accumulation mode): kRyser for n = 25 .. 38 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_plain_ryser_b(SweepLauncher* t) { fill_sweep_plain<kRyser, 25>(t, std::make_integer_sequence<int, 14>{}); }
}  // namespace permb200
