// Standalone timing of the production sweep kernel (perm_kernels.cuh launch_sweep) for a few n
// on short custom-plan units, for A/B comparison of compile-time code shapes without touching
// the library (build twice with different -D switches, run both in one GPU session).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_1606_05836_b200/csrc tools/microbench/sweep_bench.cu -o /tmp/sweep_bench
//   /tmp/sweep_bench            -> one line per n: terms/s and FP64 issue fraction
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "perm_kernels.cuh"
using namespace permb200;

template <int N, int ALG>
void run(int waves) {
  const int c = 11, lam = 4, wb = 7;
  const int m = ALG == kGlynn ? N - 1 : N;
  const long long units = 296LL * waves;
  std::vector<double2> h(N * N);
  unsigned long long x = 88172645463325252ULL;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v.x = ((double)(x >> 11) / 9007199254740992.0 - 0.5) / N;
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v.y = ((double)(x >> 11) / 9007199254740992.0 - 0.5) / N;
  }
  double2 *dA, *staging;
  Dd2* out;
  cudaMalloc(&dA, sizeof(double2) * N * N);
  cudaMalloc(&staging, sizeof(double2) * kTabRows * kNMax);
  cudaMalloc(&out, sizeof(Dd2) * units);
  cudaMemcpy(dA, h.data(), sizeof(double2) * N * N, cudaMemcpyHostToDevice);
  SweepArgs a;
  a.A = dA; a.unit_out = out; a.lo = 0; a.hi = 1ull << m; a.unit_lo = 0;
  a.c = c; a.lam = lam; a.block_bits = wb; a.slot = 0; a.col_base = 0; a.zero = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch_sweep<N, ALG, kComp>(a, units, staging, 0);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    launch_sweep<N, ALG, kComp>(a, units, staging, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double terms = (double)units * (1ull << (c + lam + wb));
  Dd2 r;
  cudaMemcpy(&r, out, sizeof(Dd2), cudaMemcpyDeviceToHost);
  printf("n=%d alg=%d units=%lld %.3f ms %.4e terms/s fp64_issue %.4f  unit0 %.17g %s\n", N, ALG, units, best,
         terms / (best * 1e-3), terms * (6 * N - 2) / (best * 1e-3) / (148.0 * 64 * 1.965e9), r.re_hi,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(dA); cudaFree(staging); cudaFree(out);
}

int main(int argc, char** argv) {
  const int waves = argc > 1 ? atoi(argv[1]) : 8;
  run<32, kGlynn>(waves);
  run<40, kGlynn>(waves);
  run<44, kGlynn>(waves);
  run<46, kGlynn>(waves);
  run<48, kGlynn>(waves);
  run<49, kGlynn>(waves);
  run<50, kGlynn>(waves);
  run<51, kGlynn>(waves);
  run<50, kRyser>(waves);
  return 0;
}
