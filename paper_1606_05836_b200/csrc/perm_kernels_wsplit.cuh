// perm_kernels_wsplit.cuh — the Gray-code sweep with each chunk's n row sums split over a PAIR OF
// WARPS (lane l of warp 2p and lane l of warp 2p + 1 walk the same chunk), for large n.
// Included by perm_inst_wsplit.cu after perm_kernels.cuh.
//
// Same method as perm_kernels.cuh (Eq. (2) P:66-68 / Eq. (1) P:62-64 walked in Gray-code order:
// one +-column update of the row sums and one n-way complex product per term), different mapping:
//   * the lower warp (K = 0) of a pair holds rows [0, N0), the upper warp (K = 1) rows [N0, n)
//     (N0 = ceil(n / 2)); each flips only its rows and multiplies them into a half product;
//   * because K is a property of the WARP, every flip's step vector is still a warp-uniform
//     constant-bank operand (LDCU -> uniform register -> DADD), as in the one-lane sweep -- the
//     2-lane split (perm_kernels_split.cuh) had to read its columns from shared memory into
//     vector registers and measured 0.62-0.71 of the FP64 issue rate at n = 52..62;
//   * the two half products of a term meet through shared memory, 4 terms per exchange: per
//     loop iteration (terms r = 0..3) the lower warp finishes terms 0, 1 and the upper warp
//     terms 2, 3; each writes the half products the other needs into a double-buffered slot,
//     one named barrier (bar.sync, 64 threads) per iteration, then term = cmul(lower, upper) --
//     always in that operand order, so both warps form identical terms (n >= 60: 2 terms per
//     exchange, the lower warp finishing the even terms and the upper warp the odd ones);
//   * each warp accumulates the terms it finished (8 of every 16: plain sums, then the Sum2
//     cascade); the leaf partial is lower + upper (double-double), and the upper warps feed
//     exact zeros to the block tree (tree over threads = canonical tree over leaves).
// Why: from n = 52, 4n registers of row sums no longer fit one thread next to the product
// chains; two warps hold ~2n each, which also halves the per-thread register footprint at
// n = 48..51 (more resident warps).
// Chunk-start builds read the row-major matrix from global memory (L1/L2; once per 2^c terms),
// so the kernel needs no shared-memory matrix copy (n = 64: 64 KB per block).  Ragged end units
// and chunks shorter than 2^kMinFastC run the one-lane sweep_kernel's generic walk instead.
#pragma once

#include "perm_kernels.cuh"

namespace permb200 {

// Terms per exchange of the warp pair: 4, or 2 for N >= PERMB200_WSPLIT_U2_FROM.  The two warps of a
// pair run DIFFERENT loop bodies (K = 0 / K = 1), ~3n/2 x 16 B of SASS per term each: with 4 terms
// per iteration 38 KB together at n = 60 and 41 KB at n = 64, against a 32 KB L1.5 instruction
// cache.  Measured 2026-10-21 (wsplit_bench, 2368 units of 2^21 terms; 4 terms / 2 terms): FP64
// issue 0.864 / 0.853 (n = 52), 0.834 / 0.795 (56), 0.743 / 0.774 (60), 0.596 / 0.779 (64); library,
// 888 units: 0.777 / 0.75 (58), 0.718 / 0.747 (60) -- so 2 terms from n = 60.
#ifndef PERMB200_WSPLIT_U2_FROM        // A/B switch (tools/microbench/wsplit_bench.cu)
#define PERMB200_WSPLIT_U2_FROM 60
#endif
__host__ __device__ constexpr bool wsplit_u2(int N) { return N >= PERMB200_WSPLIT_U2_FROM; }

__device__ __forceinline__ void pair_barrier(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

// Product chains of a half product (NR rows): independent chains (i mod NC), then a pairwise
// tree; fixed order per (N, K).
__host__ __device__ constexpr int wsplit_chains(int NR) { return NR >= 16 ? 4 : NR >= 4 ? 2 : 1; }

template <int N, int ALG, int MODE, int K>
struct HalfWalker {
  static constexpr int N0 = (N + 1) / 2;
  static constexpr int OFF = K ? N0 : 0;          // first row of this warp
  static constexpr int NR = K ? N - N0 : N0;      // rows of this warp
  static constexpr int NC = wsplit_chains(NR);
  static constexpr bool PLAIN = (MODE == kPlain);
  static constexpr double kSgnDir1 = (ALG == kGlynn) ? 1.0 : -1.0;
  static constexpr double kSgnDir0 = (ALG == kGlynn) ? -1.0 : 1.0;
  static constexpr bool kNegBase = (ALG == kRyser) && (N & 1);

  double2 s[NR];
  double arh, arl, aih, ail;

  __device__ __forceinline__ void zero_acc() { arh = arl = aih = ail = 0.0; }

  __device__ __forceinline__ void acc_add(double re, double im) {
    if (PLAIN) { arh = __dadd_rn(arh, re); aih = __dadd_rn(aih, im); return; }
    double s_, e_;
    two_sum(arh, re, s_, e_);
    arh = s_; arl = __dadd_rn(arl, e_);
    two_sum(aih, im, s_, e_);
    aih = s_; ail = __dadd_rn(ail, e_);
  }

  // Chunk-start row sums of this warp's rows for code G, from the row-major,
  // unscaled matrix in global memory: s_i = a_i1 + sum_{j>=2} delta_j a_ij (Glynn; delta_1 = +1),
  // s_i = sum_{j in S} a_ij (Ryser).  fma(+-1, a, s) = RN(s +- a): the same bits as the
  // one-lane build's fma(+-0.5, 2a, s).  8 rows per pass bound the registers the loads take.
  __device__ __forceinline__ void build(const double2* __restrict__ A, uint64_t G) {
    constexpr int RB = 8;
#pragma unroll
    for (int r0 = 0; r0 < NR; r0 += RB) {
#pragma unroll
      for (int j = r0; j < r0 + RB; ++j)
        if (j < NR) s[j] = (ALG == kGlynn) ? __ldg(A + (size_t)(OFF + j) * N) : make_double2(0.0, 0.0);
#pragma unroll 1
      for (int col = (ALG == kGlynn) ? 1 : 0; col < N; ++col) {
        const int bit = (ALG == kGlynn) ? (int)((G >> (col - 1)) & 1) : (int)((G >> col) & 1);
        const double w = (ALG == kGlynn) ? (bit ? -1.0 : 1.0) : (bit ? 1.0 : 0.0);
#pragma unroll
        for (int j = r0; j < r0 + RB; ++j)
          if (j < NR) {
            const double2 v = __ldg(A + (size_t)(OFF + j) * N + col);
            s[j].x = __fma_rn(w, v.x, s[j].x);
            s[j].y = __fma_rn(w, v.y, s[j].y);
          }
      }
    }
  }

  static __device__ __forceinline__ int plus_row(int b) { return 2 * b + (ALG == kGlynn ? 1 : 0); }

  __device__ __forceinline__ void flip_row(const ConstColumns& cols, int row) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const double2 v = cols.get(row, OFF + j);
      s[j].x = __dadd_rn(s[j].x, v.x);
      s[j].y = __dadd_rn(s[j].y, v.y);
    }
  }

  __device__ __forceinline__ void flip_signed(const ConstColumns& cols, int row, double sg) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const double2 v = cols.get(row, OFF + j);
      s[j].x = __fma_rn(sg, v.x, s[j].x);
      s[j].y = __fma_rn(sg, v.y, s[j].y);
    }
  }

  __device__ __forceinline__ double2 half_product() const {
    double2 c[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) c[q] = s[q];
#pragma unroll
    for (int j = NC; j < NR; ++j) c[j % NC] = cmul(c[j % NC], s[j]);
#pragma unroll
    for (int w = 1; w < NC; w *= 2) {
#pragma unroll
      for (int q = 0; q + w < NC; q += 2 * w) c[q] = cmul(c[q], c[q + w]);
    }
    return c[0];
  }

  // Uniform half-walk (Walker::half_walk's visiting order, rows and flips).  xb: this pair's
  // exchange buffer, xb[((slot * 2 + side) * 2 + e) * 32 + lane], side = the writing warp's K.
  // H / 4 iterations (an even count for c >= kMinFastC), so the slot alternation runs on
  // across half-walks and chunks.
  __device__ __forceinline__ void half_walk(const ConstColumns& cols, int T0, int H, int zero, double2* xb, int bar,
                                            int lane) {
    double mr = 0.0, mi = 0.0;
    int slot = 0;
    if constexpr (wsplit_u2(N)) {
    // 2 terms per exchange (half the loop body, see wsplit_u2): the lower warp finishes the even
    // terms, the upper warp the odd ones; one barrier per 2 terms.
    for (int t = -2; t < H - 2; t += 2) {
      const int tz = t * zero;
      double2 keep = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int b = (r == 0) ? ((__ffs(t + 2) - 1) & 15) : 0;
        const int d = (r == 0) ? (((T0 + t + 2) >> (b + 1)) & 1) : (((t + 2) >> 1) & 1);
        const int row = (r == 0) ? (2 * b + d) : (d + tz);
        flip_row(cols, row);
        const double2 p = half_product();
        if (r == K) keep = p;
        else xb[((slot * 2 + K) * 2) * 32 + lane] = p;
      }
      pair_barrier(bar);
      {
        const double2 o = xb[((slot * 2 + (1 - K)) * 2) * 32 + lane];
        const double2 term = (K == 0) ? cmul(keep, o) : cmul(o, keep);    // cmul(lower, upper)
        if ((K != 0) != kNegBase) { mr = __dsub_rn(mr, term.x); mi = __dsub_rn(mi, term.y); }
        else { mr = __dadd_rn(mr, term.x); mi = __dadd_rn(mi, term.y); }
      }
      slot ^= 1;
      if (((t + 2) & 14) == 14) {
        acc_add(mr, mi);
        mr = 0.0; mi = 0.0;
      }
    }
    acc_add(mr, mi);
    } else {
    for (int t = -4; t < H - 4; t += 4) {
      const int tz = t * zero;
      double2 keep0 = make_double2(0.0, 0.0), keep1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int b = (r == 0) ? ((__ffs(t + 4) - 1) & 15) : (__ffs(r) - 1);
        const int d = (r == 0) ? (((T0 + t + 4) >> (b + 1)) & 1) : (r == 1) ? 0 : (r == 2) ? (((t + 4) >> 2) & 1) : 1;
        const int row = (r == 0) ? (2 * b + d) : (2 * b + d + tz);
        flip_row(cols, row);
        const double2 p = half_product();
        const bool mine = (K == 0) ? (r < 2) : (r >= 2);
        if (mine) {
          if ((r & 1) == 0) keep0 = p;
          else keep1 = p;
        } else {
          xb[((slot * 2 + K) * 2 + (r & 1)) * 32 + lane] = p;
        }
      }
      pair_barrier(bar);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double2 o = xb[((slot * 2 + (1 - K)) * 2 + e) * 32 + lane];
        const double2 h = e ? keep1 : keep0;
        const double2 term = (K == 0) ? cmul(h, o) : cmul(o, h);    // cmul(lower, upper)
        // term r = 2K + e: the sign alternates with the parity of r (= parity of g)
        if ((e != 0) != kNegBase) { mr = __dsub_rn(mr, term.x); mi = __dsub_rn(mi, term.y); }
        else { mr = __dadd_rn(mr, term.x); mi = __dadd_rn(mi, term.y); }
      }
      slot ^= 1;
      if (((t + 4) & 12) == 12) {
        acc_add(mr, mi);
        mr = 0.0; mi = 0.0;
      }
    }
    acc_add(mr, mi);
    }
  }

  __device__ __forceinline__ void fast_chunk(const ConstColumns& cols, const double2* __restrict__ A, uint64_t q, int c,
                                             int zero, double2* xb, int bar, int lane) {
    const uint64_t g0 = q << c;
    build(A, g0 ^ (g0 >> 1));
    const int H = 1 << (c - 1);
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      if (h == 1) flip_signed(cols, plus_row(c - 1), (q & 1) ? kSgnDir1 : kSgnDir0);
      half_walk(cols, h * H, H, zero, xb, bar, lane);
    }
  }

  __device__ __forceinline__ Dd2 result() const {
    if (PLAIN) return Dd2{arh, 0.0, aih, 0.0};
    Dd2 r;
    fast_two_sum(arh, arl, r.re_hi, r.re_lo);
    fast_two_sum(aih, ail, r.im_hi, r.im_lo);
    return r;
  }
};

// One full aligned chunk as its own ptxas allocation unit (keeps the half-walk's loop counter in
// a uniform register and the column operands on LDCU, as chunk_fast does).
template <int N, int ALG, int MODE, int K>
__device__ __noinline__ Dd2 wsplit_chunk_fast(const ConstColumns cols, const double2* __restrict__ A, uint64_t q, int c,
                                              int zero, double2* xb, int bar, int lane) {
  HalfWalker<N, ALG, MODE, K> w;
  w.zero_acc();
  w.fast_chunk(cols, A, q, c, zero, xb, bar, lane);
  return w.result();
}

// Exchange buffer per warp pair: 2 slots x 2 sides x 2 terms x 32 lanes.
constexpr int kXbPerPair = 2 * 2 * 2 * 32;

// One block = one unit of the canonical plan lying inside [lo, hi) (c >= kMinFastC):
// 2^block_bits leaves (5 <= block_bits <= 6), each leaf a lane of a warp pair.  Only the fast
// path lives here (no shared-memory matrix, no one-lane Walker: a noinline callee's registers
// count against the kernel, and the one-lane generic walk needs all of them).  Dynamic shared
// memory: [blockDim Dd2: tree][blockDim/2 Dd2: upper partials][pairs * kXbPerPair double2].
// Resident blocks per SM the register allocation targets: 3 (<= 168 registers, 12 warps/SM)
// where ptxas keeps the half-walk loop free of spills at that cap (n <= 55 except 54,
// -Xptxas -v + tools/sass_loop_stats.py), else 2 (<= 255 registers, 8 warps/SM).
#ifdef PERMB200_WSPLIT_MINB            // A/B switch (tools/microbench/wsplit_bench.cu)
__host__ __device__ constexpr int wsplit_min_blocks(int) { return PERMB200_WSPLIT_MINB; }
#else
__host__ __device__ constexpr int wsplit_min_blocks(int N) { return (N <= 55 && N != 54) ? 3 : 2; }
#endif
template <int N, int ALG, int MODE>
__global__ void __launch_bounds__(kMaxBlock, wsplit_min_blocks(N)) wsplit_kernel(const SweepArgs args) {
  extern __shared__ double2 smem[];
  const int nt = blockDim.x;
  Dd2* red = reinterpret_cast<Dd2*>(smem);
  Dd2* upper = red + nt;
  double2* xball = reinterpret_cast<double2*>(upper + nt / 2);
  // warp index through a shuffle from lane 0: ptxas then knows K is warp-uniform, so the
  // K-branches below are not divergent and the half-walks keep their uniform-register column
  // path (with K = (threadIdx.x >> 5) & 1 every column load fell back to per-thread LDC)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int K = warp & 1, pair = warp >> 1;
  const uint64_t unit = (uint64_t)(args.unit_lo + blockIdx.x);
  const uint64_t leaf_id = (unit << args.block_bits) + (uint64_t)(pair * 32 + lane);
  const ConstColumns cols{args.col_base};
  double2* xb = xball + pair * kXbPerPair;
  Dd2 acc{0.0, 0.0, 0.0, 0.0};
  const uint64_t nch = 1ull << args.lam;
  for (uint64_t kk = 0; kk < nch; ++kk) {
    const uint64_t q = (leaf_id << args.lam) + kk;
    if (K == 0) acc = part_add<MODE>(acc, wsplit_chunk_fast<N, ALG, MODE, 0>(cols, args.A, q, args.c, args.zero, xb, 1 + pair, lane));
    else acc = part_add<MODE>(acc, wsplit_chunk_fast<N, ALG, MODE, 1>(cols, args.A, q, args.c, args.zero, xb, 1 + pair, lane));
  }
  if (K == 1) upper[pair * 32 + lane] = acc;
  __syncthreads();
  // leaf partial = lower + upper; the upper warps feed exact zeros to the tree over threads
  const Dd2 mine = (K == 0) ? part_add<MODE>(acc, upper[pair * 32 + lane]) : Dd2{0.0, 0.0, 0.0, 0.0};
  block_tree<MODE>(red, mine);
  if (threadIdx.x == 0) args.unit_out[blockIdx.x] = red[0];
}

// Ragged end units (and every unit when c < kMinFastC): the one-lane generic walk (Walker,
// all n rows per thread; rare, so its register spills do not matter) over the same canonical
// leaves, tree over leaves.  Shared memory: [N*N transposed matrix][blockDim Dd2: tree]
// [blockDim Dd2: Walker chunk accumulators] (sweep_kernel's layout).
template <int N, int ALG, int MODE>
__global__ void __launch_bounds__(kMaxBlock) wsplit_ragged_kernel(const SweepArgs args) {
  extern __shared__ double2 smem[];
  double2* at = smem;
  Dd2* red = reinterpret_cast<Dd2*>(smem + N * N);
  stage_transposed<N>(args.A, at, (ALG == kGlynn) ? 2.0 : 1.0);
  __syncthreads();
  const ConstColumns cols{args.col_base};
  const uint64_t leaf_id = ((uint64_t)(args.unit_lo + blockIdx.x) << args.block_bits) + threadIdx.x;
  const Dd2 mine = walk_leaf<N, ALG, false, MODE>(cols, at, leaf_id, args.c, args.lam, args.lo, args.hi, args.zero);
  block_tree<MODE>(red, mine);
  if (threadIdx.x == 0) args.unit_out[blockIdx.x] = red[0];
}

// Launch over units [unit_lo, unit_lo + units): the units inside [lo, hi) run wsplit_kernel;
// the (at most two) ragged end units -- or all units when c < kMinFastC -- run
// wsplit_ragged_kernel.
template <int N, int ALG, int MODE>
cudaError_t launch_wsplit(const SweepArgs& a, int64_t units, double2* staging, cudaStream_t st) {
  if (a.block_bits < 5 || a.block_bits > 6) return cudaErrorInvalidValue;   // pairs of whole warps
  auto ragged = [&](int64_t u, int64_t cnt) -> cudaError_t {
    SweepArgs r = a;
    r.unit_lo = u;
    r.unit_out = a.unit_out + (u - a.unit_lo);
    const int threads = 1 << a.block_bits;
    const size_t smem = sizeof(double2) * N * N + 2 * sizeof(Dd2) * threads;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(wsplit_ragged_kernel<N, ALG, MODE>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    wsplit_ragged_kernel<N, ALG, MODE><<<(unsigned)cnt, threads, smem, st>>>(r);
    return cudaGetLastError();
  };
  if (a.c < kMinFastC) return ragged(a.unit_lo, units);
  const int ubits = a.block_bits + a.lam + a.c;
  int64_t u0 = a.unit_lo, u1 = a.unit_lo + units;        // interior units [u0, u1)
  cudaError_t e = cudaSuccess;
  if (((uint64_t)u0 << ubits) < a.lo) e = ragged(u0++, 1);
  if (e == cudaSuccess && u1 > u0 && ((uint64_t)u1 << ubits) > a.hi) e = ragged(--u1, 1);
  if (e != cudaSuccess || u1 <= u0) return e;
  const int c_tab = a.c < kCMax ? a.c : kCMax;
  const int col0 = (ALG == kGlynn) ? 1 : 0;
  stage_columns_kernel<<<1, 256, 0, st>>>(a.A, N, col0, c_tab, (ALG == kGlynn) ? 2.0 : 1.0, staging);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbolAsync(c_cols, staging, sizeof(double2) * kTabRows * kNMax,
                              sizeof(double2) * (size_t)a.slot * kTabRows * kNMax, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  const int threads = 2 << a.block_bits;
  const size_t smem = sizeof(Dd2) * (threads + threads / 2) + sizeof(double2) * (threads / 64) * kXbPerPair;
  SweepArgs f = a;
  f.unit_lo = u0;
  f.unit_out = a.unit_out + (u0 - a.unit_lo);
  wsplit_kernel<N, ALG, MODE><<<(unsigned)(u1 - u0), threads, smem, st>>>(f);
  return cudaGetLastError();
}

// Kernel launches made by one launch_wsplit call (the library's launch counter).
inline int wsplit_launches(const SweepArgs& a, int64_t units) {
  if (a.c < kMinFastC) return 1;
  const int ubits = a.block_bits + a.lam + a.c;
  int64_t u0 = a.unit_lo, u1 = a.unit_lo + units;
  int n = 0;
  if (((uint64_t)u0 << ubits) < a.lo) { ++u0; ++n; }
  if (u1 > u0 && ((uint64_t)u1 << ubits) > a.hi) { --u1; ++n; }
  return n + (u1 > u0 ? 2 : 0);
}

}  // namespace permb200

#include <utility>
namespace permb200 {
template <int ALG, int MODE, int LO, int... Is>
void fill_wsplit(SweepLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &launch_wsplit<LO + Is, ALG, MODE>), ...);
}
}  // namespace permb200
