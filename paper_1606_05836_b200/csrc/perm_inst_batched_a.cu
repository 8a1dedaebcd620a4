// Instantiation unit: batched for n = 1 .. 32 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_batched_a(BatchedLauncher* t) { fill_batched<1>(t, std::make_integer_sequence<int, 32>{}); }
}  // namespace permb200
