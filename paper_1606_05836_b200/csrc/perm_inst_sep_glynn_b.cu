// Instantiation unit (separate-addition precision mode, Table AV): kGlynn for n = 25 .. 40.
#include "perm_registry.h"
namespace permb200 {
void register_sep_glynn_b(SweepLauncher* t) { fill_sweep_sep<kGlynn, 25>(t, std::make_integer_sequence<int, 16>{}); }
}  // namespace permb200
