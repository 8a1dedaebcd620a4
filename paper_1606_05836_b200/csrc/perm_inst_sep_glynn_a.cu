// Instantiation unit (separate-addition precision mode, Table AV): kGlynn for n = 1 .. 24.
#include "perm_registry.h"
namespace permb200 {
void register_sep_glynn_a(SweepLauncher* t) { fill_sweep_sep<kGlynn, 1>(t, std::make_integer_sequence<int, 24>{}); }
}  // namespace permb200
