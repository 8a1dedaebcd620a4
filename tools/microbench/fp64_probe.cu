// FP64 pipe probes for the Gray-code sweep design (SURVEY §8d "FP64 DFMA peak
// microbenchmark"; §7 step 8 "column operand delivery via LDS broadcast vs
// constant operands").  Not part of the product library.
//
//   dfma_peak        : 8 independent DFMA chains per thread, full chip
//   sweep_lds<N>     : N complex row sums in registers; every step adds a column
//                      read from shared memory (uniform address = broadcast),
//                      then an N-way complex product (the a4 step shape)
//   sweep_param<N>   : same, but the column operands come from a
//                      __grid_constant__ kernel parameter (constant bank)
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void dfma_peak(double* out, int iters, double x, double y) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, x, y); a1 = fma(a1, x, y); a2 = fma(a2, x, y); a3 = fma(a3, x, y);
      a4 = fma(a4, x, y); a5 = fma(a5, x, y); a6 = fma(a6, x, y); a7 = fma(a7, x, y);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  double2 r;
  r.x = __fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y));
  r.y = __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x));
  return r;
}

template <int N>
__device__ __forceinline__ double2 prod4(const double2 (&s)[N]) {
  double2 c0 = s[0], c1 = s[1], c2 = s[2], c3 = s[3];
#pragma unroll
  for (int i = 4; i < N; i += 4) {
    c0 = cmul(c0, s[i]);
    if (i + 1 < N) c1 = cmul(c1, s[i + 1]);
    if (i + 2 < N) c2 = cmul(c2, s[i + 2]);
    if (i + 3 < N) c3 = cmul(c3, s[i + 3]);
  }
  return cmul(cmul(c0, c1), cmul(c2, c3));
}

template <int N>
struct ColParam { double2 col[8][N]; };

template <int N>
__global__ void __launch_bounds__(128) sweep_lds(const double2* __restrict__ M, double2* out, int steps) {
  __shared__ double2 sm[32 * N];
  for (int i = threadIdx.x; i < 32 * N; i += blockDim.x) sm[i] = M[i % (8 * N)];
  __syncthreads();
  double2 s[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { s[i].x = 1.0 + 1e-3 * (threadIdx.x + i); s[i].y = 1e-3 * i; }
  double2 acc = {0, 0};
  for (int t = 0; t < steps; t += 8) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int col = (r == 0) ? (8 + (__ffs(t + 8) & 15)) : (__ffs(r) - 1);
      const double2* cp = sm + col * N;
#pragma unroll
      for (int i = 0; i < N; ++i) { double2 v = cp[i]; s[i].x = __dadd_rn(s[i].x, v.x); s[i].y = __dadd_rn(s[i].y, v.y); }
      double2 P = prod4<N>(s);
      if (r & 1) { acc.x = __dsub_rn(acc.x, P.x); acc.y = __dsub_rn(acc.y, P.y); }
      else { acc.x = __dadd_rn(acc.x, P.x); acc.y = __dadd_rn(acc.y, P.y); }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int N>
__global__ void __launch_bounds__(128) sweep_param(const __grid_constant__ ColParam<N> p, const double2* __restrict__ M, double2* out, int steps) {
  __shared__ double2 sm[32 * N];
  for (int i = threadIdx.x; i < 32 * N; i += blockDim.x) sm[i] = M[i % (8 * N)];
  __syncthreads();
  double2 s[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { s[i].x = 1.0 + 1e-3 * (threadIdx.x + i); s[i].y = 1e-3 * i; }
  double2 acc = {0, 0};
  for (int t = 0; t < steps; t += 8) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r == 0) {
        const double2* cp = sm + (8 + (__ffs(t + 8) & 15)) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) { double2 v = cp[i]; s[i].x = __dadd_rn(s[i].x, v.x); s[i].y = __dadd_rn(s[i].y, v.y); }
      } else {
        const int col = __ffs(r) - 1;
#pragma unroll
        for (int i = 0; i < N; ++i) { s[i].x = __dadd_rn(s[i].x, p.col[col][i].x); s[i].y = __dadd_rn(s[i].y, p.col[col][i].y); }
      }
      double2 P = prod4<N>(s);
      if (r & 1) { acc.x = __dsub_rn(acc.x, P.x); acc.y = __dsub_rn(acc.y, P.y); }
      else { acc.x = __dadd_rn(acc.x, P.x); acc.y = __dadd_rn(acc.y, P.y); }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int N>
void run_sweeps(int nsm, double2* dM, double2* dout) {
  ColParam<N> p;
  for (int c = 0; c < 8; ++c) for (int i = 0; i < N; ++i) { p.col[c][i].x = 1e-9 * (c + i); p.col[c][i].y = -1e-9 * i; }
  const int steps = 1 << 14;
  for (int bps : {1, 2}) {
    int grid = nsm * bps * 4;
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (int variant = 0; variant < 2; ++variant) {
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        if (variant == 0) sweep_lds<N><<<grid, 128>>>(dM, dout, steps);
        else sweep_param<N><<<grid, 128>>>(p, dM, dout, steps);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        double terms = (double)grid * 128 * steps;
        double ops = terms * (6.0 * N - 2);
        if (rep == 2)
          printf("N=%d %s grid=%d: %.3f ms  %.3e terms/s  %.2f TFLOP-instr/s (x2 = %.2f TF-equiv)\n", N,
                 variant ? "param" : "lds  ", grid, ms, terms / (ms * 1e-3), ops / (ms * 1e-3) / 1e12,
                 2 * ops / (ms * 1e-3) / 1e12);
      }
    }
  }
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("%s SMs=%d clockRate=%d kHz regsPerSM=%d smemPerSM=%zu\n", prop.name, prop.multiProcessorCount, clk,
         prop.regsPerMultiprocessor, prop.sharedMemPerMultiprocessor);
  const int nsm = prop.multiProcessorCount;
  double* dout; CK(cudaMalloc(&dout, sizeof(double2) * nsm * 16 * 1024));
  const int iters = 20000;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int wps : {4, 8, 16, 32}) {
    int grid = nsm * (wps / 4);  // 128-thread blocks
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(e0));
      dfma_peak<<<grid, 128>>>(dout, iters, 0.999999, 1e-7);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      double fl = 2.0 * 8 * 16 * (double)iters * grid * 128;
      if (rep == 2) printf("dfma_peak warps/SM=%d: %.3f ms %.2f TFLOP/s\n", wps, ms, fl / (ms * 1e-3) / 1e12);
    }
  }
  // sustained: ~5 s of DFMA
  {
    int grid = nsm * 4;
    CK(cudaEventRecord(e0));
    for (int k = 0; k < 20; ++k) dfma_peak<<<grid, 128>>>(dout, iters * 4, 0.999999, 1e-7);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double fl = 20 * 2.0 * 8 * 16 * (double)iters * 4 * grid * 128;
    printf("dfma_peak sustained (%.1f s): %.2f TFLOP/s\n", ms / 1e3, fl / (ms * 1e-3) / 1e12);
  }
  double2* dM; CK(cudaMalloc(&dM, sizeof(double2) * 64 * 64));
  {
    double2 h[64 * 64];
    for (int i = 0; i < 64 * 64; ++i) { h[i].x = 1e-9 * (i % 17); h[i].y = -1e-9 * (i % 13); }
    CK(cudaMemcpy(dM, h, sizeof(h), cudaMemcpyHostToDevice));
  }
  run_sweeps<16>(nsm, dM, (double2*)dout);
  run_sweeps<32>(nsm, dM, (double2*)dout);
  run_sweeps<40>(nsm, dM, (double2*)dout);
  run_sweeps<50>(nsm, dM, (double2*)dout);
  return 0;
}
