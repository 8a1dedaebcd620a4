// perm_registry.h — per-translation-unit launcher registration (one template instance per n).
#pragma once
#include "perm_kernels.cuh"

namespace permb200 {
void register_glynn_a(SweepLauncher* t);
void register_glynn_b(SweepLauncher* t);
void register_glynn_c(SweepLauncher* t);
void register_glynn_d(SweepLauncher* t);
void register_ryser_a(SweepLauncher* t);
void register_ryser_b(SweepLauncher* t);
void register_ryser_c(SweepLauncher* t);
void register_ryser_d(SweepLauncher* t);
void register_plain_glynn_a(SweepLauncher* t);
void register_plain_glynn_b(SweepLauncher* t);
void register_plain_glynn_c(SweepLauncher* t);
void register_plain_glynn_d(SweepLauncher* t);
void register_plain_ryser_a(SweepLauncher* t);
void register_plain_ryser_b(SweepLauncher* t);
void register_plain_ryser_c(SweepLauncher* t);
void register_plain_ryser_d(SweepLauncher* t);
void register_dd_glynn_a(SweepLauncher* t);
void register_dd_glynn_b(SweepLauncher* t);
void register_dd_ryser_a(SweepLauncher* t);
void register_dd_ryser_b(SweepLauncher* t);
void register_sep_glynn_a(SweepLauncher* t);
void register_sep_glynn_b(SweepLauncher* t);
void register_sep_ryser_a(SweepLauncher* t);
void register_sep_ryser_b(SweepLauncher* t);
void register_small(SweepLauncher (*t)[kNMax + 1]);
void register_small_fused(FusedLauncher (*t)[kNMax + 1]);
void register_split_large(SweepLauncher (*t)[kNMax + 1]);
void register_wsplit_a(SweepLauncher (*t)[kNMax + 1]);
void register_wsplit_b(SweepLauncher (*t)[kNMax + 1]);
void register_batched_a(BatchedLauncher* t);
void register_batched_b(BatchedLauncher* t);
}  // namespace permb200
