// A/B timing of the three large-n sweep mappings on the same custom plan (c = 11, lam = 4,
// 64 leaves per unit, 148 * 8 * waves units): one lane per chunk (launch_sweep, perm_kernels.cuh),
// the 2-lane row split (launch_split, perm_kernels_split.cuh) and the warp-pair row split
// (launch_wsplit, perm_kernels_wsplit.cuh).  Prints terms/s, the FP64 issue fraction at 6n-2
// instructions per term and the relative difference of each variant's total from the
// one-lane total (different product / accumulation orders: rounding-level differences).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_1606_05836_b200/csrc tools/microbench/wsplit_bench.cu -o /tmp/wsplit_bench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "perm_kernels.cuh"
#include "perm_kernels_split.cuh"
#include "perm_kernels_wsplit.cuh"
using namespace permb200;

template <int N, int ALG>
void run(int waves) {
  const int c = 11, lam = 4, wb = 6;
  const int m = ALG == kGlynn ? N - 1 : N;
  const long long units = 148LL * 8 * waves;
  std::vector<double2> h(N * N);
  unsigned long long x = 88172645463325252ULL;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v.x = ((double)(x >> 11) / 9007199254740992.0 - 0.5) / N * 2.5;
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v.y = ((double)(x >> 11) / 9007199254740992.0 - 0.5) / N * 2.5;
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
  std::vector<Dd2> ho(units);
  double ref_re = 0, ref_im = 0;
  for (int variant = 0; variant < 3; ++variant) {
    auto launch = [&]() {
      if (variant == 0) return launch_sweep<N, ALG, kComp>(a, units, staging, 0);
      if (variant == 1) return launch_split<N, ALG, kComp, 2>(a, units, staging, 0);
      return launch_wsplit<N, ALG, kComp>(a, units, staging, 0);
    };
    cudaError_t le = launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaMemcpy(ho.data(), out, sizeof(Dd2) * units, cudaMemcpyDeviceToHost);
    double sr = 0, si = 0;
    for (auto& d : ho) { sr += d.re_hi + d.re_lo; si += d.im_hi + d.im_lo; }
    if (variant == 0) { ref_re = sr; ref_im = si; }
    const double rel = std::hypot(sr - ref_re, si - ref_im) / std::hypot(ref_re, ref_im);
    const double terms = (double)units * (1ull << (c + lam + wb));
    printf("n=%d alg=%d %-7s units=%lld %9.3f ms %.4e terms/s fp64_issue %.4f rel_vs_onelane %.2e %s/%s\n", N, ALG,
           variant == 0 ? "onelane" : variant == 1 ? "split2" : "wsplit", units, best, terms / (best * 1e-3),
           terms * (6 * N - 2) / (best * 1e-3) / (148.0 * 64 * 1.965e9), rel, cudaGetErrorString(le),
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
  cudaFree(dA); cudaFree(staging); cudaFree(out);
}

int main(int argc, char** argv) {
  const int waves = argc > 1 ? atoi(argv[1]) : 2;
  run<48, kGlynn>(waves);
  run<50, kGlynn>(waves);
  run<50, kRyser>(waves);
  run<51, kGlynn>(waves);
  run<52, kGlynn>(waves);
  run<54, kGlynn>(waves);
  run<56, kGlynn>(waves);
  run<60, kGlynn>(waves);
  run<64, kGlynn>(waves);
  return 0;
}
