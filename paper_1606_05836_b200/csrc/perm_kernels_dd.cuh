// perm_kernels_dd.cuh — double-double precision mode of the Gray-code sweep.
//
// Same method, same canonical plan shape and reduction tree as the FP64 sweep
// (perm_kernels.cuh), but every row sum, every partial product and every term is carried
// as an unevaluated sum hi + lo of two doubles (~2^-104 relative), so
//   * integer matrices whose every partial product and partial sum stays below ~2^104 are
//     evaluated EXACTLY (J_20: 20!, J_20 - I: D_20 -- neither fits one double; reading R9),
//   * Ryser's cancellation (the paper's precision finding) is pushed ~2^51 further
//     down: relative error ~ n * 2^-104 * kappa instead of n * 2^-53 * kappa.
//
// PAPER.md: Eq. (2), Eq. (1), Alg. A1/A2 loop bodies P:220-229 / P:251-260.
//
// Layout: the n complex dd row sums of a thread live in SHARED memory (32 B per row per
// thread; ss[(2 i + part) * T + tid], part 0 = (re_hi, re_lo), part 1 = (im_hi, im_lo);
// consecutive threads -> consecutive 16 B, conflict-free 128-bit accesses), because 8n
// registers per thread would not fit for n > 24.  Columns are read from the matrix in global
// memory with warp-uniform addresses (one broadcast sector per load, L1-resident).
#pragma once

#include "perm_kernels.cuh"

namespace permb200 {
namespace ddm {

struct dd { double hi, lo; };
struct cdd { dd re, im; };

// (hi, lo) + b, b a double: TwoSum, fold the low part, renormalise.  Exact when the true sum
// is representable as a double-double (e.g. integers below 2^106).
__device__ __forceinline__ dd add_d(dd a, double b) {
  double s, e;
  two_sum(a.hi, b, s, e);
  e = __dadd_rn(e, a.lo);
  dd r;
  fast_two_sum(s, e, r.hi, r.lo);
  return r;
}

__device__ __forceinline__ dd add_dd(dd a, dd b) {
  dd r;
  dd_add(a.hi, a.lo, b.hi, b.lo, r.hi, r.lo);
  return r;
}

// x*y + SG*z*w in double-double: leading products split exactly (TwoProd), their sum by
// TwoSum, the first-order cross terms folded with FMAs, renormalised by TwoSum (the leading
// sum may cancel, so the fast variant's |s| >= |t| precondition does not hold).
template <int SG>
__device__ __forceinline__ dd dot2(dd x, dd y, dd z, dd w) {
  const double p1 = __dmul_rn(x.hi, y.hi);
  const double e1 = __fma_rn(x.hi, y.hi, -p1);
  const double zs = SG > 0 ? z.hi : -z.hi;
  const double zl = SG > 0 ? z.lo : -z.lo;
  const double p2 = __dmul_rn(zs, w.hi);
  const double e2 = __fma_rn(zs, w.hi, -p2);
  double s, e3;
  two_sum(p1, p2, s, e3);
  double t = __dadd_rn(__dadd_rn(e1, e2), e3);
  t = __fma_rn(x.hi, y.lo, t);
  t = __fma_rn(x.lo, y.hi, t);
  t = __fma_rn(zs, w.lo, t);
  t = __fma_rn(zl, w.hi, t);
  dd r;
  two_sum(s, t, r.hi, r.lo);
  return r;
}

__device__ __forceinline__ cdd cmul(const cdd& a, const cdd& b) {
  cdd r;
  r.re = dot2<-1>(a.re, b.re, a.im, b.im);
  r.im = dot2<+1>(a.re, b.im, a.im, b.re);
  return r;
}

// Independent product chains (i mod kDdChains): the dd multiply is a ~22-deep dependent
// chain per component, and shared-memory residency limits a block to 2 warps, so the
// chains are what hides the FP64 latency (ncu r01_dd_n32: "wait" stalls dominate).
constexpr int kDdChains = 4;
// Stride (in double2) between a thread's consecutive row-sum slots = the largest dd block.
// A compile-time stride lets the compiler prove that the store of row i and the load of row
// i+1 do not alias, so the rows' independent update chains interleave.
constexpr int kDdStride = 64;
// n <= kDdHiRegMax: the hi halves of the row sums live in registers (4n) and only the lo halves
// in shared memory (16 B per row per thread): half the shared memory per thread, 4 blocks of
// 64 threads per SM instead of 3 (n = 32); one product chain keeps that within 255 registers.
constexpr int kDdHiRegMax = 32;
__host__ __device__ constexpr int dd_smem_parts(int N) { return N <= kDdHiRegMax ? 1 : 2; }

template <int N, int ALG>
struct DdWalker {
  static constexpr bool kHiRegs = N <= kDdHiRegMax;
  double2* ss;
  double2 h[kHiRegs ? N : 1];
  dd ar, ai;
  __device__ __forceinline__ cdd load(int i) const {
    if (kHiRegs) {
      const double2 l = ss[i * kDdStride];
      return cdd{dd{h[i].x, l.x}, dd{h[i].y, l.y}};
    }
    const double2 r = ss[(2 * i) * kDdStride], m = ss[(2 * i + 1) * kDdStride];
    return cdd{dd{r.x, r.y}, dd{m.x, m.y}};
  }
  __device__ __forceinline__ void store(int i, const cdd& v) {
    if (kHiRegs) {
      h[i] = make_double2(v.re.hi, v.im.hi);
      ss[i * kDdStride] = make_double2(v.re.lo, v.im.lo);
      return;
    }
    ss[(2 * i) * kDdStride] = make_double2(v.re.hi, v.re.lo);
    ss[(2 * i + 1) * kDdStride] = make_double2(v.im.hi, v.im.lo);
  }

  // Row sums for code G from the row-major matrix A: Glynn s_i = a_i1 +
  // sum_{j>=2} delta_j a_ij (bit j-2 of G set <=> delta_j = -1), Ryser s_i = sum_{j in S} a_ij.
  __device__ __forceinline__ void build(const double2* __restrict__ A, uint64_t G) {
    // kHiRegs: rows unrolled so h[i] is a register; else a runtime row loop (code size)
#pragma unroll
    for (int i0 = 0; i0 < (kHiRegs ? N : 1); ++i0)
#pragma unroll 1
    for (int i1 = 0; i1 < (kHiRegs ? 1 : N); ++i1) {
      const int i = kHiRegs ? i0 : i1;
      const double2* row = A + i * N;
      cdd s{dd{0.0, 0.0}, dd{0.0, 0.0}};
      if (ALG == kGlynn) { const double2 v = __ldg(row); s.re.hi = v.x; s.im.hi = v.y; }
#pragma unroll 4
      for (int j = (ALG == kGlynn) ? 1 : 0; j < N; ++j) {
        const int bit = (ALG == kGlynn) ? (int)((G >> (j - 1)) & 1) : (int)((G >> j) & 1);
        const double w = (ALG == kGlynn) ? (bit ? -1.0 : 1.0) : (bit ? 1.0 : 0.0);
        const double2 v = __ldg(row + j);
        s.re = add_d(s.re, w * v.x);      // w in {-1, 0, 1}: exact
        s.im = add_d(s.im, w * v.y);
      }
      store(i, s);
    }
  }

  // Walk Gray indices [ga, gb) (inside one aligned chunk) into (ar, ai).  Step g flips code
  // bit b = ctz(g) with direction bit (b+1) of g: the row sums move by
  // sg * column(col0 + b), sg = +-2 (Glynn, exact) or +-1 (Ryser).  The flip and the product
  // of the new row sums share one pass over the rows; the first term flips by 0 (exact).
  __device__ __forceinline__ void walk(const double2* __restrict__ A, uint64_t ga, uint64_t gb) {
    constexpr int col0 = (ALG == kGlynn) ? 1 : 0;
    constexpr bool kNegBase = (ALG == kRyser) && (N & 1);
    build(A, ga ^ (ga >> 1));
    ar = dd{0.0, 0.0};
    ai = dd{0.0, 0.0};
    double sg = 0.0;
    int col = 0;
    constexpr int NC = (N <= kDdHiRegMax) ? 1 : (N < kDdChains ? N : kDdChains);
    for (uint64_t g = ga;;) {
      cdd c[NC];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        cdd s = load(i);
        const double2 v = __ldg(A + i * N + col);
        s.re = add_d(s.re, __dmul_rn(sg, v.x));
        s.im = add_d(s.im, __dmul_rn(sg, v.y));
        store(i, s);
        c[i % NC] = (i < NC) ? s : cmul(c[i % NC], s);
      }
      // pairwise tree over the chains (order fixed by N)
#pragma unroll
      for (int w = 1; w < NC; w *= 2) {
#pragma unroll
        for (int k = 0; k + w < NC; k += 2 * w) c[k] = cmul(c[k], c[k + w]);
      }
      cdd p = c[0];
      if (((g & 1) != 0) != kNegBase) {
        p.re.hi = -p.re.hi; p.re.lo = -p.re.lo; p.im.hi = -p.im.hi; p.im.lo = -p.im.lo;
      }
      ar = add_dd(ar, p.re);
      ai = add_dd(ai, p.im);
      if (++g >= gb) break;
      const int b = __ffsll((long long)g) - 1;
      const int d = (int)((g >> (b + 1)) & 1);
      // Glynn: d = 1 -> delta back to +1 -> +2a; d = 0 -> -2a.  Ryser: d = 1 -> leaves S -> -a.
      sg = (ALG == kGlynn) ? (d ? 2.0 : -2.0) : (d ? -1.0 : 1.0);
      col = col0 + b;
    }
  }
};

// One block = one unit of the dd plan (perm_api.cu make_plan, block_bits <= 6); thread =
// leaf of 2^lam chunks.  Dynamic shared memory: 2 N kDdStride double2 (row sums) + blockDim
// Dd2 (tree).
template <int N, int ALG>
__global__ void __launch_bounds__(kDdStride, N <= kDdHiRegMax ? 4 : 1) sweep_dd_kernel(const SweepArgs args) {
  extern __shared__ double2 smem[];
  Dd2* red = reinterpret_cast<Dd2*>(smem + dd_smem_parts(N) * N * kDdStride);
  DdWalker<N, ALG> w;
  w.ss = smem + threadIdx.x;
  PERM_CHECK(in_dyn_smem(w.ss + (dd_smem_parts(N) * N - 1) * kDdStride, sizeof(double2)));
  const uint64_t unit = (uint64_t)(args.unit_lo + blockIdx.x);
  const uint64_t leaf_id = (unit << args.block_bits) + threadIdx.x;
  Dd2 acc{0.0, 0.0, 0.0, 0.0};
  uint64_t k0, k1;
  leaf_chunk_window(leaf_id, args.c, args.lam, args.lo, args.hi, k0, k1);
  for (uint64_t k = k0; k < k1; ++k) {
    const uint64_t q = (leaf_id << args.lam) + k;
    const uint64_t g0 = q << args.c, g1 = g0 + (1ull << args.c);
    const uint64_t ga = g0 > args.lo ? g0 : args.lo;
    const uint64_t gb = g1 < args.hi ? g1 : args.hi;
    if (ga < gb) {
      w.walk(args.A, ga, gb);
      Dd2 part;
      fast_two_sum(w.ar.hi, w.ar.lo, part.re_hi, part.re_lo);
      fast_two_sum(w.ai.hi, w.ai.lo, part.im_hi, part.im_lo);
      acc = dd2_add(acc, part);
    }
  }
  block_tree(red, acc);
  if (threadIdx.x == 0) args.unit_out[blockIdx.x] = red[0];
}

template <int N, int ALG>
cudaError_t launch_sweep_dd(const SweepArgs& a, int64_t units, double2*, cudaStream_t st) {
  const int threads = 1 << a.block_bits;
  const size_t smem = sizeof(double2) * dd_smem_parts(N) * N * kDdStride + sizeof(Dd2) * threads;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sweep_dd_kernel<N, ALG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  sweep_dd_kernel<N, ALG><<<(unsigned)units, threads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace ddm

template <int ALG, int LO, int... Is>
void fill_sweep_dd(SweepLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &ddm::launch_sweep_dd<LO + Is, ALG>), ...);
}

}  // namespace permb200
