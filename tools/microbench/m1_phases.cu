// M1 (n = 20 single permanent) anatomy: the fused small-n kernel (perm_kernels.cuh
// sweep_small_fused_kernel) on the canonical plan, timed back to back with CUDA events, and --
// when built with -DPERMB200_PHASE_TIMES -- its phases (staging, column table, walk, block tree,
// grid barrier, final reduce) from %globaltimer / clock64 stamps.  A/B of compile-time shapes:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_1606_05836_b200/csrc [-DPERMB200_PHASE_TIMES] [-DPERMB200_SMALL_BUILD=0] \
//        tools/microbench/m1_phases.cu -o tools/microbench/m1_phases_X
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "perm_kernels.cuh"
using namespace permb200;

template <int N, int ALG>
void run(int c, int wb, int ub, const char* name) {
  const int m = ALG == kGlynn ? N - 1 : N;
  const long long units = 1LL << ub;
  std::vector<double2> h(N * N);
  unsigned long long x = 88172645463325252ULL;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v.x = ((double)(x >> 11) / 9007199254740992.0 - 0.5) / N;
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v.y = ((double)(x >> 11) / 9007199254740992.0 - 0.5) / N;
  }
  double2 *dA, *out;
  Dd2* parts;
  cudaMalloc(&dA, sizeof(double2) * N * N);
  cudaMalloc(&out, sizeof(double2));
  cudaMalloc(&parts, sizeof(Dd2) * units);
  cudaMemcpy(dA, h.data(), sizeof(double2) * N * N, cudaMemcpyHostToDevice);
  SweepArgs a;
  a.A = dA; a.unit_out = parts; a.lo = 0; a.hi = 1ull << m; a.unit_lo = 0;
  a.c = c; a.lam = m - c - wb - ub; a.block_bits = wb; a.slot = 0; a.col_base = 0; a.zero = 0;
  const FinishArgs f{out, nullptr, ALG == kGlynn ? 1 : 0, -(N - 1), 1, 0};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 20; ++i) launch_sweep_small_fused<N, ALG, kComp>(a, f, units, 0);
  cudaDeviceSynchronize();
  const int calls = 200;
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    for (int i = 0; i < calls; ++i) launch_sweep_small_fused<N, ALG, kComp>(a, f, units, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double2 r;
  cudaMemcpy(&r, out, sizeof(double2), cudaMemcpyDeviceToHost);
  printf("%s n=%d c=%d wb=%d units=%lld: %.2f us/call back to back  out %.17g %.17g  %s\n", name, N, c, wb, units,
         best * 1e3 / calls, r.x, r.y, cudaGetErrorString(cudaGetLastError()));
#ifdef PERMB200_PHASE_TIMES
  const char* ph[] = {"entry", "staged A", "column table", "walk", "block tree", "grid barrier", "final reduce"};
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z[16] = {0};
    z[0] = ~0ull;
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    launch_sweep_small_fused<N, ALG, kComp>(a, f, units, 0);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(z, g_phase, sizeof(z));
    printf("  phases (us after first block entry, latest block / mean block cycles):");
    for (int k = 1; k <= 6; ++k) {
      const double n_blocks = (k == 6) ? 1.0 : (double)units;
      printf("  %s %.2f/%.0f", ph[k], z[k] ? (z[k] - z[0]) * 1e-3 : -1.0, z[8 + k] / n_blocks);
    }
    printf("\n");
  }
#endif
  cudaFree(dA); cudaFree(out); cudaFree(parts);
}

int main() {
  // canonical R = 1 plans (perm_api.cu make_plan): Glynn n = 20 c = 5, Ryser n = 20 c = 6
  run<20, kGlynn>(5, 7, 7, "glynn");
  run<20, kRyser>(6, 7, 7, "ryser");
  // alternatives: more, shorter chunks; fewer threads per block
  run<20, kGlynn>(4, 7, 8, "glynn");
  run<20, kGlynn>(5, 6, 8, "glynn");
  run<20, kGlynn>(6, 7, 6, "glynn");
  return 0;
}
