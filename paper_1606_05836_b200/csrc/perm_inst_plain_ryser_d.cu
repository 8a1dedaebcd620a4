// Instantiation unit (plain-accumulation mode): kRyser for n = 52 .. 64 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_plain_ryser_d(SweepLauncher* t) { fill_sweep_plain<kRyser, 52>(t, std::make_integer_sequence<int, 13>{}); }
}  // namespace permb200
