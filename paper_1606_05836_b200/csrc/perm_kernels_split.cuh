// perm_kernels_split.cuh — the Gray-code sweep with each chunk's n row sums SPLIT over a group
// of R = 2 consecutive lanes, for n >= 52.  Included by perm_inst_split_large.cu after
// perm_kernels.cuh.
//
// Same method as perm_kernels.cuh (Eq. (2) P:66-68 / Eq. (1), walked in Gray-code
// order, one +-column update and one n-way product per term), different mapping:
//   * lane k of a group holds rows [k NR, (k+1) NR) (NR = ceil(n / R); rows >= n are padding
//     fixed at 1 + 0i, an exact multiplicative identity of cmul), flips only those rows and
//     multiplies them into a lane partial product;
//   * the group combines the lane partials with shuffles, always as cmul(lower lanes, upper
//     lanes), so every lane ends with the same, uniquely ordered term; every lane accumulates it
//     (the accumulators of a group are identical) and only lane 0 feeds the block tree (the
//     others contribute exact zeros, so the tree over threads equals the canonical tree over
//     leaves = groups);
//   * the step vectors come from a per-block shared-memory table with the padded row stride
//     NP = R NR: a warp reads R distinct addresses per flip (one wavefront).
// Why: from n = 52, 4n registers of row sums exceed what one thread can hold next to the
// product chains (round 1: local-memory spills in the hot loop); two lanes hold 2n each.  (A
// 4-lane variant for small n was measured slower than one lane per chunk on M1 and removed:
// profiles/r02_m1_latency_split4.log.)
#pragma once

#include "perm_kernels.cuh"

namespace permb200 {

__host__ __device__ constexpr int split_rows(int N, int R) { return (N + R - 1) / R; }
__host__ __device__ constexpr int split_chains(int NR) { return NR >= 12 ? 4 : NR >= 4 ? 2 : 1; }

template <int N, int ALG, int MODE, int R>
struct SplitWalker {
  static constexpr int NR = split_rows(N, R);
  static constexpr int NP = NR * R;
  static constexpr int NC = split_chains(NR);
  static constexpr double kScale = (ALG == kGlynn) ? 2.0 : 1.0;
  static constexpr double kSgnDir1 = (ALG == kGlynn) ? 1.0 : -1.0;
  static constexpr double kSgnDir0 = (ALG == kGlynn) ? -1.0 : 1.0;
  static constexpr bool kNegBase = (ALG == kRyser) && (N & 1);
  static constexpr bool PLAIN = (MODE == kPlain);

  double2 s[NR];                  // this lane's row sums
  double arh, arl, aih, ail;      // accumulator (kSep: even / odd sums in hi / lo)
  int k;                          // lane within the group
  unsigned gmask;                 // the group's lanes (shuffles stay inside the group: groups of
                                  // one warp may walk different ragged chunk windows)

  __device__ __forceinline__ void zero_acc() { arh = arl = aih = ail = 0.0; }

  __device__ __forceinline__ void acc_add(double re, double im) {
    if (PLAIN) { arh = __dadd_rn(arh, re); aih = __dadd_rn(aih, im); return; }
    double s_, e_;
    two_sum(arh, re, s_, e_);
    arh = s_; arl = __dadd_rn(arl, e_);
    two_sum(aih, im, s_, e_);
    aih = s_; ail = __dadd_rn(ail, e_);
  }
  __device__ __forceinline__ void acc_add_sep(double er, double ei, double orr, double oi) {
    arh = __dadd_rn(arh, er); arl = __dadd_rn(arl, orr);
    aih = __dadd_rn(aih, ei); ail = __dadd_rn(ail, oi);
  }

  // Chunk-start row sums of this lane's rows for code G, from the transposed,
  // pre-scaled matrix at[j N + i] = kScale a_ij.
  __device__ __forceinline__ void build(const double2* __restrict__ at, uint64_t G) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int i = k * NR + j;
      if (i < N) {
        if (ALG == kGlynn) s[j] = make_double2(0.5 * at[i].x, 0.5 * at[i].y);   // delta_1 = +1; exact
        else s[j] = make_double2(0.0, 0.0);
      } else {
        s[j] = make_double2(1.0, 0.0);                                           // padding row
      }
    }
#pragma unroll 1
    for (int col = (ALG == kGlynn) ? 1 : 0; col < N; ++col) {
      const int bit = (ALG == kGlynn) ? (int)((G >> (col - 1)) & 1) : (int)((G >> col) & 1);
      const double w = (ALG == kGlynn) ? (bit ? -0.5 : 0.5) : (bit ? 1.0 : 0.0);
      const double2* cp = at + col * N;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const int i = k * NR + j;
        if (i < N) {
          const double2 v = cp[i];
          s[j].x = __fma_rn(w, v.x, s[j].x);
          s[j].y = __fma_rn(w, v.y, s[j].y);
        }
      }
    }
  }

  static __device__ __forceinline__ int plus_row(int b) { return 2 * b + (ALG == kGlynn ? 1 : 0); }

  __device__ __forceinline__ void flip_row(const double2* tab, int row) {
    const double2* t = tab + row * NP + k * NR;
    PERM_CHECK(row >= 0 && row < kTabRows && in_dyn_smem(t, NR * sizeof(double2)));
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const double2 v = t[j];
      s[j].x = __dadd_rn(s[j].x, v.x);
      s[j].y = __dadd_rn(s[j].y, v.y);
    }
  }

  __device__ __forceinline__ void flip_signed(const double2* tab, int row, double sg) {
    const double2* t = tab + row * NP + k * NR;
    PERM_CHECK(row >= 0 && row < kTabRows && in_dyn_smem(t, NR * sizeof(double2)));
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const double2 v = t[j];
      s[j].x = __fma_rn(sg, v.x, s[j].x);
      s[j].y = __fma_rn(sg, v.y, s[j].y);
    }
  }

  // Term product: lane partial over NC chains, then the group's shuffle tree.
  __device__ __forceinline__ double2 product() const {
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
    double2 p = c[0];
#pragma unroll
    for (int lvl = 1; lvl < R; lvl *= 2) {
      double2 o;
      o.x = __shfl_xor_sync(gmask, p.x, lvl);
      o.y = __shfl_xor_sync(gmask, p.y, lvl);
      const bool upper = (k & lvl) != 0;           // lower lanes' product is the left operand
      p = cmul(upper ? o : p, upper ? p : o);
    }
    return p;
  }

  // Uniform half-walk: Walker::half_walk's visiting order, flips and accumulation.
  __device__ __forceinline__ void half_walk(const double2* tab, int T0, int H) {
    double mr = 0.0, mi = 0.0;
    double orr = 0.0, oi = 0.0;
    for (int t = -4; t < H - 4; t += 4) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int b = (r == 0) ? ((__ffs(t + 4) - 1) & 15) : (__ffs(r) - 1);
        const int d = (r == 0) ? (((T0 + t + 4) >> (b + 1)) & 1) : (r == 1) ? 0 : (r == 2) ? (((t + 4) >> 2) & 1) : 1;
        flip_row(tab, 2 * b + d);
        const double2 p = product();
        if (MODE == kSep) {
          if (r & 1) { orr = __dadd_rn(orr, p.x); oi = __dadd_rn(oi, p.y); }
          else { mr = __dadd_rn(mr, p.x); mi = __dadd_rn(mi, p.y); }
        } else if (((r & 1) != 0) != kNegBase) { mr = __dsub_rn(mr, p.x); mi = __dsub_rn(mi, p.y); }
        else { mr = __dadd_rn(mr, p.x); mi = __dadd_rn(mi, p.y); }
      }
      if (((t + 4) & 12) == 12) {
        if (MODE == kSep) { acc_add_sep(mr, mi, orr, oi); orr = 0.0; oi = 0.0; }
        else acc_add(mr, mi);
        mr = 0.0; mi = 0.0;
      }
    }
    if (MODE == kSep) acc_add_sep(mr, mi, orr, oi);
    else acc_add(mr, mi);
  }

  __device__ __forceinline__ void fast_chunk(const double2* tab, const double2* __restrict__ at, uint64_t q, int c) {
    const uint64_t g0 = q << c;
    build(at, g0 ^ (g0 >> 1));
    const int H = 1 << (c - 1);
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      if (h == 1) flip_signed(tab, plus_row(c - 1), (q & 1) ? kSgnDir1 : kSgnDir0);
      half_walk(tab, h * H, H);
    }
  }

  // Ragged piece [ga, gb) of one chunk: per-term flips straight from the transposed matrix.
  __device__ __forceinline__ void generic_walk(const double2* __restrict__ at, uint64_t ga, uint64_t gb) {
    constexpr int col0 = (ALG == kGlynn) ? 1 : 0;
    build(at, ga ^ (ga >> 1));
    for (uint64_t g = ga;; ) {
      double2 p = product();
      if (MODE == kSep) {
        if (g & 1) acc_add_sep(0.0, 0.0, p.x, p.y);
        else acc_add_sep(p.x, p.y, 0.0, 0.0);
      } else {
        const bool neg = ((g & 1) != 0) != kNegBase;
        if (neg) { p.x = -p.x; p.y = -p.y; }
        acc_add(p.x, p.y);
      }
      if (++g >= gb) break;
      const int b = __ffsll((long long)g) - 1;
      const double sg = ((g >> (b + 1)) & 1) ? kSgnDir1 : kSgnDir0;
      const double2* cp = at + (col0 + b) * N;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const int i = k * NR + j;
        if (i < N) {
          const double2 v = cp[i];
          s[j].x = __fma_rn(sg, v.x, s[j].x);
          s[j].y = __fma_rn(sg, v.y, s[j].y);
        }
      }
    }
  }

  __device__ __forceinline__ Dd2 result() const {
    if (MODE == kSep) return Dd2{arh, arl, aih, ail};
    if (PLAIN) return Dd2{arh, 0.0, aih, 0.0};
    Dd2 r;
    fast_two_sum(arh, arl, r.re_hi, r.re_lo);
    fast_two_sum(aih, ail, r.im_hi, r.im_lo);
    return r;
  }
};

template <int N, int ALG, int MODE, int R>
__device__ __noinline__ Dd2 split_chunk_fast(const double2* tab, const double2* __restrict__ at, uint64_t q, int c, int k) {
  SplitWalker<N, ALG, MODE, R> w;
  w.k = k;
  w.gmask = ((1u << R) - 1) << ((threadIdx.x & 31) & ~(R - 1));
  w.zero_acc();
  w.fast_chunk(tab, at, q, c);
  return w.result();
}

template <int N, int ALG, int MODE, int R>
__device__ __noinline__ Dd2 split_chunk_generic(const double2* __restrict__ at, uint64_t ga, uint64_t gb, int k) {
  SplitWalker<N, ALG, MODE, R> w;
  w.k = k;
  w.gmask = ((1u << R) - 1) << ((threadIdx.x & 31) & ~(R - 1));
  w.zero_acc();
  w.generic_walk(at, ga, gb);
  return w.result();
}

// Signed step-vector table with the padded row stride NP: tab[(2b+d) NP + i], zero for padding
// rows and for bits >= c (Glynn: d = 1 -> +2a, d = 0 -> -2a; Ryser: d = 1 -> -a, d = 0 -> +a).
template <int N, int ALG, int NP>
__device__ __forceinline__ void build_tab_split(const double2* at, double2* tab, int c) {
  constexpr int col0 = (ALG == kGlynn) ? 1 : 0;
  for (int idx = threadIdx.x; idx < kTabRows * NP; idx += blockDim.x) {
    const int row = idx / NP, i = idx - row * NP;
    const int bb = row >> 1, d = row & 1;
    double2 v = make_double2(0.0, 0.0);
    if (bb < c && col0 + bb < N && i < N) {
      v = at[(col0 + bb) * N + i];
      const bool neg = (ALG == kGlynn) ? !d : d;
      if (neg) { v.x = -v.x; v.y = -v.y; }
    }
    PERM_CHECK(in_dyn_smem(tab + idx, sizeof(double2)));
    tab[idx] = v;
  }
}

// One block = one unit of the canonical plan: 2^block_bits leaves (groups) x R lanes.
template <int N, int ALG, int MODE, int R>
__global__ void __launch_bounds__(kMaxBlock) sweep_split_kernel(const SweepArgs args) {
  constexpr int NR = split_rows(N, R), NP = NR * R;
  extern __shared__ double2 smem[];
  // [N*N: at][kTabRows*NP: tab][blockDim Dd2: tree]
  double2* at = smem;
  double2* tab = smem + N * N;
  Dd2* red = reinterpret_cast<Dd2*>(smem + N * N + kTabRows * NP);
  stage_transposed<N>(args.A, at, (ALG == kGlynn) ? 2.0 : 1.0);
  __syncthreads();
  build_tab_split<N, ALG, NP>(at, tab, args.c < kCMax ? args.c : kCMax);
  __syncthreads();
  const int k = threadIdx.x % R;
  const uint64_t unit = (uint64_t)(args.unit_lo + blockIdx.x);
  const uint64_t leaf_id = (unit << args.block_bits) + threadIdx.x / R;
  const int ubits = args.block_bits + args.lam + args.c;
  const bool inside = (unit << ubits) >= args.lo && ((unit + 1) << ubits) <= args.hi;
  Dd2 acc{0.0, 0.0, 0.0, 0.0};
  uint64_t k0 = 0, k1 = 1ull << args.lam;
  const bool fast = inside && args.c >= kMinFastC;
  if (!fast) leaf_chunk_window(leaf_id, args.c, args.lam, args.lo, args.hi, k0, k1);
  for (uint64_t kk = k0; kk < k1; ++kk) {
    const uint64_t q = (leaf_id << args.lam) + kk;
    if (fast) {
      acc = part_add<MODE>(acc, split_chunk_fast<N, ALG, MODE, R>(tab, at, q, args.c, k));
    } else {
      const uint64_t g0 = q << args.c, g1 = g0 + (1ull << args.c);
      const uint64_t ga = g0 > args.lo ? g0 : args.lo;
      const uint64_t gb = g1 < args.hi ? g1 : args.hi;
      if (ga < gb) acc = part_add<MODE>(acc, split_chunk_generic<N, ALG, MODE, R>(at, ga, gb, k));
    }
  }
  const Dd2 mine = (k == 0) ? acc : Dd2{0.0, 0.0, 0.0, 0.0};
  block_tree<MODE>(red, mine);
  if (threadIdx.x == 0) args.unit_out[blockIdx.x] = red[0];
}

template <int N, int R>
constexpr size_t split_smem(int threads) {
  return sizeof(double2) * (N * N + kTabRows * split_rows(N, R) * R) + sizeof(Dd2) * threads;
}

template <int N, int ALG, int MODE, int R>
cudaError_t launch_split(const SweepArgs& a, int64_t units, double2*, cudaStream_t st) {
  const int threads = (1 << a.block_bits) * R;
  const size_t smem = split_smem<N, R>(threads);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sweep_split_kernel<N, ALG, MODE, R>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  sweep_split_kernel<N, ALG, MODE, R><<<(unsigned)units, threads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace permb200

#include <utility>
namespace permb200 {
template <int ALG, int MODE, int R, int LO, int... Is>
void fill_split(SweepLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &launch_split<LO + Is, ALG, MODE, R>), ...);
}
}  // namespace permb200
