#include <cuda_runtime.h>
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  double2 r; r.x = __fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)); r.y = __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)); return r; }
template <int N, int NC>
__device__ __forceinline__ double2 prodc(const double2 (&s)[N]) {
  double2 c[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) c[k] = s[k];
#pragma unroll
  for (int i = NC; i < N; ++i) c[i % NC] = cmul(c[i % NC], s[i]);
#pragma unroll
  for (int w = 1; w < NC; w *= 2)
#pragma unroll
    for (int k = 0; k + w < NC; k += 2 * w) c[k] = cmul(c[k], c[k + w]);
  return c[0];
}
template <int N> struct ColParam { double2 col[16][N]; };
template <int N, int U, int NC>
__global__ void __launch_bounds__(128) sweep_uc(const __grid_constant__ ColParam<N> p, double2* out, int steps, int zero) {
  double2 s[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { s[i].x = 1.0 + 1e-3 * (threadIdx.x + i); s[i].y = 1e-3 * i; }
  double2 acc = {0, 0};
  for (int t = 0; t < steps; t += U) {
    const int tz = t * zero;   // opaque 0: defeats hoisting of the column loads out of the loop
#pragma unroll
    for (int r = 0; r < U; ++r) {
      const int b = (r == 0) ? ((__ffs(t + U) - 1) & 15) : (__ffs(r) - 1) + tz;
#pragma unroll
      for (int i = 0; i < N; ++i) { double2 v = p.col[b][i]; s[i].x = __dadd_rn(s[i].x, v.x); s[i].y = __dadd_rn(s[i].y, v.y); }
      double2 P = prodc<N, NC>(s);
      if (r & 1) { acc.x = __dsub_rn(acc.x, P.x); acc.y = __dsub_rn(acc.y, P.y); }
      else { acc.x = __dadd_rn(acc.x, P.x); acc.y = __dadd_rn(acc.y, P.y); }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
#define INST(N,U,NC) template __global__ void sweep_uc<N,U,NC>(const __grid_constant__ ColParam<N>, double2*, int, int);
INST(50,4,4) INST(50,8,4) INST(40,4,4) INST(56,4,4) INST(32,4,4) INST(16,4,4) INST(64,4,4) INST(60,4,4)
#include <cstdio>
template <int N, int U, int NC>
void run(int nsm, double2* dout) {
  ColParam<N> p;
  for (int c = 0; c < 16; ++c) for (int i = 0; i < N; ++i) { p.col[c][i].x = 1e-9 * (c + i); p.col[c][i].y = -1e-9 * i; }
  const int steps = 1 << 13;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {2, 4, 8}) {
    int grid = nsm * bps;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      sweep_uc<N, U, NC><<<grid, 128>>>(p, dout, steps, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double terms = (double)grid * 128 * steps, ops = terms * (6.0 * N - 2);
      if (rep == 2) printf("N=%d U=%d NC=%d grid=%d: %.3f ms %.3e terms/s  FP64 instr-lanes %.2f T/s (%.1f%% of 17.0)\n", N, U, NC, grid, ms,
                           terms / (ms * 1e-3), ops / (ms * 1e-3) / 1e12, 100 * ops / (ms * 1e-3) / 17.0e12);
    }
  }
}
int main() {
  double2* dout; cudaMalloc(&dout, sizeof(double2) * 148 * 8 * 128);
  run<16,4,4>(148, dout); run<32,4,4>(148, dout); run<40,4,4>(148, dout); run<50,4,4>(148, dout); run<50,8,4>(148, dout);
  run<56,4,4>(148, dout); run<60,4,4>(148, dout); run<64,4,4>(148, dout);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
