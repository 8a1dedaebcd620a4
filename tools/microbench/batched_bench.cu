// Standalone timing of the production batched kernel (perm_kernels.cuh launch_batched) on a
// synthetic 4096 x 16x16 batch, for A/B comparison of compile-time code shapes (build with
// different -D switches, run all in one GPU session).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "perm_kernels.cuh"
using namespace permb200;

template <int N>
void run(long long B) {
  std::vector<double2> h((size_t)B * N * N);
  unsigned long long x = 88172645463325252ULL;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v.x = ((double)(x >> 11) / 9007199254740992.0 - 0.5) / 4;
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v.y = ((double)(x >> 11) / 9007199254740992.0 - 0.5) / 4;
  }
  double2 *dA, *out;
  cudaMalloc(&dA, sizeof(double2) * h.size());
  cudaMalloc(&out, sizeof(double2) * B);
  cudaMemcpy(dA, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice);
  BatchedArgs a;
  a.A = dA; a.out = out; a.out_abs2 = nullptr; a.batch = B;
  const int m = N - 1, wb = 7, rem = m - wb;
  a.block_bits = wb; a.c = rem < kCMax ? rem : kCMax; a.lam = rem - a.c;
  a.scale_exp = -(N - 1); a.zero = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch_batched<N>(a, (int)B, 0);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    launch_batched<N>(a, (int)B, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double terms = (double)B * (1ull << (N - 1));
  double2 r;
  cudaMemcpy(&r, out, sizeof(double2), cudaMemcpyDeviceToHost);
  printf("batched n=%d B=%lld %.4f ms %.4e terms/s fp64_issue %.4f  out0 %.17g %s\n", N, B, best,
         terms / (best * 1e-3), terms * (6 * N - 2) / (best * 1e-3) / (148.0 * 64 * 1.965e9), r.x,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(dA); cudaFree(out);
}

int main(int argc, char** argv) {
  const long long B = argc > 1 ? atoll(argv[1]) : 4096;
  run<16>(B);
  run<16>(B * 8);
  return 0;
}
