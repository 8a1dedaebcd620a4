// Instantiation unit (plain-accumulation mode): kRyser for n = 1 .. 24 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_plain_ryser_a(SweepLauncher* t) { fill_sweep_plain<kRyser, 1>(t, std::make_integer_sequence<int, 24>{}); }
}  // namespace permb200
