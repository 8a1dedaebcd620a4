// FP64 issue rate vs warps per scheduler and independent chains per thread (the M1 question:
// can ONE warp per SM sub-partition keep the FP64 pipe busy?).  K independent DFMA chains per
// thread, 148 blocks of W threads (W / 128 warps per scheduler), fraction of the nominal
// 148 SM x 64 lanes x 1.965 GHz rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/fp64_warps.cu -o tools/microbench/fp64_warps
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, int iters, double x, double y) {
  double a[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32 / K + 1; ++u) {
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = fma(a[k], x, y);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
void run(double* d) {
  for (int W : {32, 64, 128, 256, 512}) {
    const int iters = 4000;
    chains<K><<<148, W>>>(d, 10, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chains<K><<<148, W>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double instr = 148.0 * W * iters * (double)K * (32 / K + 1);
    printf("K=%2d warps/scheduler=%4.2f  fp64 frac %.3f  (%.3f ms)\n", K, W / 128.0,
           instr / (ms * 1e-3) / (148.0 * 64 * 1.965e9), ms);
  }
}

int main() {
  double* d;
  cudaMalloc(&d, sizeof(double) * 148 * 512);
  run<1>(d); run<2>(d); run<4>(d); run<8>(d); run<16>(d);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
