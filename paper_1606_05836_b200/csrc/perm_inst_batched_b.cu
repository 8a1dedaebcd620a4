// Instantiation unit: batched for n = 33 .. 64 (each TU holds its own constant column slots).
#include "perm_registry.h"
namespace permb200 {
void register_batched_b(BatchedLauncher* t) { fill_batched<33>(t, std::make_integer_sequence<int, 32>{}); }
}  // namespace permb200
