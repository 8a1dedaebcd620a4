// Instantiation unit (plain-accumulation mode): kRyser for n = 39 .. 51 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_plain_ryser_c(SweepLauncher* t) { fill_sweep_plain<kRyser, 39>(t, std::make_integer_sequence<int, 13>{}); }
}  // namespace permb200
