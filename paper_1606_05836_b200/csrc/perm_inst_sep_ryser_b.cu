// Instantiation unit (separate-addition precision mode, Table AV): kRyser for n = 25 .. 40.
#include "perm_registry.h"
namespace permb200 {
void register_sep_ryser_b(SweepLauncher* t) { fill_sweep_sep<kRyser, 25>(t, std::make_integer_sequence<int, 16>{}); }
}  // namespace permb200
