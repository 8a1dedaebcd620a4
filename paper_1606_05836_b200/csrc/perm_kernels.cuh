// perm_kernels.cuh — sm_100a FP64 Gray-code sweep kernels for Glynn (BB/FG, Eq. 2) and
// Ryser (Eq. 1) permanents.  Included only by the perm_inst_*.cu translation units, each
// of which instantiates a range of n (one template instantiation per n keeps the n
// complex row sums register-resident: DESIGN.md §Kernels).
//
// PAPER.md citations ("P:<line>"):
//   Eq. (2) P:66-68  perm = 2^-(N-1) sum_delta (prod delta_k) prod_i sum_j delta_j a_ij
//   Eq. (1) P:62-64  perm = (-1)^N sum_S (-1)^|S| prod_i sum_{j in S} a_ij
//   Alg. A2 loop body P:251-260 (delta decode, row sums, product, signed accumulate)
//   Alg. A1 loop body P:220-229
//   per-process partial + one ALLREDUCE
//
// What differs from the paper's loop ("O(2^N N^2)"): consecutive terms are visited in
// Gray-code order so each term costs ONE +-2*column (Glynn) / +-column (Ryser) update of
// the n row sums plus one n-way complex product: O(n) per term (north_star).
//
// Structure of one thread's work:
//   leaf  = 2^lam chunks, walked in order, one compensated accumulator;
//   chunk = 2^c Gray indices: O(n^2) row-sum build from the code (drift reset), then two
//           half-walks of 2^(c-1) steps separated by the one flip whose direction is
//           per-thread (Gray bit c-1 flips with direction = bit c of g = bit 0 of q);
//   in a half-walk every thread flips the SAME column b = ctz(t) with the SAME direction
//   at the same step, so the column is a warp-uniform operand: it is read from the
//   constant bank with a uniform index (LDCU -> uniform register -> DFMA operand), which
//   costs no vector register and no shared-memory bandwidth.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace permb200 {

enum { kGlynn = 0, kRyser = 1 };

// Accumulation modes of the FP64 sweep (template parameter MODE):
//   kComp  compensated: 16-term plain sums -> Sum2 cascade -> double-double partials (default)
//   kPlain plain FP64 everywhere, the paper's "Perm = Perm +- delta" (reading R12)
//   kSep   the paper's "separate addition" (Table AV): the terms of even and
//          of odd Gray index (|S| / number of -1 in delta even or odd) are summed separately in
//          plain FP64 -- partials carry (even, odd) in the (hi, lo) slots -- and subtracted once,
//          at the very end (finish_root).
enum { kComp = 0, kPlain = 1, kSep = 2 };

constexpr int kNMax = 64;      // largest n
constexpr int kCMax = 12;      // largest chunk_bits
// Smallest chunk_bits of the uniform-column fast path: half_walk takes the direction of the bit-1
// flip from bit 2 of its local step, which equals bit 2 of the chunk index only when the second
// half starts at a multiple of 8, i.e. c >= 4 (c = 3 measured wrong results, r02 M1 plan sweep).
constexpr int kMinFastC = 4;
constexpr int kTabBits = 16;   // Gray bits covered by a column table (rows for bits >= c are zero)
constexpr int kTabRows = 2 * kTabBits;   // row 2b+d = signed step vector of bit b, direction d
constexpr int kSlots = 1;      // constant-memory column slots per translation unit (32 KB each)
constexpr int kMaxBlock = 128; // threads per block (block_bits <= 7)


// Bounds-checked build (python -m paper_1606_05836_b200.build --checked -> libpermb200_checked.so;
// compute-sanitizer is closed on this pool): every shared-memory table / tree / accumulator
// access and every index that comes from device data is checked; a failed check prints the
// condition and traps (the launch fails with cudaErrorLaunchFailure).
#ifdef PERMB200_CHECKED
#define PERM_CHECK(cond)                                                                     \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("permb200 check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                               \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define PERM_CHECK(cond) do { } while (0)
#endif

// Phase timers (tools/microbench/m1_phases.cu only; compiled out of the library): block-level
// timestamps of the fused small-n kernel -- slot k holds the max over blocks of the %globaltimer
// value at the end of phase k (slot 0: the min at kernel entry), slots 8+k the sum over blocks
// of the block's clock64 cycles spent in phase k.
#ifdef PERMB200_PHASE_TIMES
__device__ unsigned long long g_phase[16];
__device__ __forceinline__ unsigned long long perm_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PERM_PHASE_START(var)                                                      \
  long long var = clock64();                                                       \
  if (threadIdx.x == 0) atomicMin(&g_phase[0], perm_gtimer())
#define PERM_PHASE(k, var)                                                         \
  do {                                                                             \
    if (threadIdx.x == 0) {                                                        \
      const long long now_ = clock64();                                            \
      atomicMax(&g_phase[k], perm_gtimer());                                       \
      atomicAdd(&g_phase[8 + (k)], (unsigned long long)(now_ - var));              \
      var = now_;                                                                  \
    }                                                                              \
  } while (0)
#else
#define PERM_PHASE_START(var) do { } while (0)
#define PERM_PHASE(k, var) do { } while (0)
#endif

// Bytes of dynamic shared memory of the running launch (for PERM_CHECK of smem offsets).
__device__ __forceinline__ unsigned dyn_smem_bytes() {
  unsigned r;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}
// true if [p, p + bytes) lies inside this block's dynamic shared memory
__device__ __forceinline__ bool in_dyn_smem(const void* p, size_t bytes) {
  extern __shared__ double2 smem_base_[];
  const char* b = reinterpret_cast<const char*>(smem_base_);
  const char* q = reinterpret_cast<const char*>(p);
  return q >= b && q + bytes <= b + dyn_smem_bytes();
}

struct Dd2 { double re_hi, re_lo, im_hi, im_lo; };

// Arguments of one sweep launch (plain struct, passed by value).
struct SweepArgs {
  const double2* A;      // device, row-major n*n
  Dd2* unit_out;         // device, one partial per launched unit (blockIdx.x)
  uint64_t lo, hi;       // clip range of Gray indices
  int64_t unit_lo;       // global index of the unit run by blockIdx.x == 0
  int c, lam, block_bits;
  int slot;              // constant-memory column slot
  int col_base;          // slot * kTabRows * kNMax, precomputed on the host: an index formed by
                         // multiplying in the kernel defeats ptxas' uniform-register path
  int zero;              // always 0; opaque to the compiler (keeps column loads in the loop)
};

struct BatchedArgs {
  const double2* A;      // device, batch * n*n
  double2* out;          // device, batch (nullptr: |perm|^2 only)
  double* out_abs2;      // device, batch: |perm|^2 (boson-sampling probability numerator) or nullptr
  int64_t batch;
  int c, lam, block_bits;
  int scale_exp;         // -(n-1)
  int zero;
};

// ------------------------------------------------------------------ FP64 building blocks
// All rounding steps are explicit (__dadd_rn / __dmul_rn / __fma_rn) so --fmad cannot
// change them (reading R6).
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  double2 r;
  r.x = __fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y));
  r.y = __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x));
  return r;
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

__device__ __forceinline__ void fast_two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(s, a));
}

// double-double + double-double (accurate variant); result normalised.
__device__ __forceinline__ void dd_add(double ah, double al, double bh, double bl, double& rh, double& rl) {
  double s, e, t, f;
  two_sum(ah, bh, s, e);
  two_sum(al, bl, t, f);
  e = __dadd_rn(e, t);
  fast_two_sum(s, e, s, e);
  e = __dadd_rn(e, f);
  fast_two_sum(s, e, rh, rl);
}

__device__ __forceinline__ Dd2 dd2_add(const Dd2& a, const Dd2& b) {
  Dd2 r;
  dd_add(a.re_hi, a.re_lo, b.re_hi, b.re_lo, r.re_hi, r.re_lo);
  dd_add(a.im_hi, a.im_lo, b.im_hi, b.im_lo, r.im_hi, r.im_lo);
  return r;
}

// Register budget near the 255-register cap (4n registers of row sums).  ptxas's allocation of
// the half-walk loop is erratic there, so two shape parameters are chosen per n from the SASS
// of the loop (tools/sass_loop_stats.py over all variants, 2026-10-20; register moves /
// local-memory spill instructions per 4 terms):
//   acc_in_smem: the chunk's Sum2 accumulator lives in a per-thread shared-memory slot
//     (touched once per 16 terms) instead of 8 registers;
//   product_chains: independent chains of the n-way complex product.
//   n <= 50: smem accumulator + 4 chains: 10 / 0 (register accumulator: n = 50 206 / 28 with
//     4 chains, 32 / 2 with 3);  n = 51: smem + 3: 10 / 0;  n = 52: registers + 3: 68 / 28;
//   n = 53: smem + 3: 192 / 20;  n >= 54: registers + 2: 70 / 16 (n = 54) .. 184 / 40 (56).
__host__ __device__ constexpr bool acc_in_smem(int N) { return N <= 51 || N == 53; }
// Chunk-start build shape (Walker::build): rows per pass and columns per loop iteration.
#ifndef PERMB200_SMALL_BUILD          // A/B switch (tools/microbench/m1_phases.cu)
#define PERMB200_SMALL_BUILD 1
#endif
// WIDE: the column source's kernel has registers to spare (not the batched kernel, which is
// capped at 128 registers for 4 blocks/SM and spilled with the wide build).
__host__ __device__ constexpr int build_rows(int N, bool WIDE) { return (PERMB200_SMALL_BUILD && WIDE && N <= 24) ? N : 8; }
__host__ __device__ constexpr int build_col_unroll(int N, bool WIDE) {
  return (PERMB200_SMALL_BUILD && WIDE && N <= 24) ? 2 : 1;
}

#ifndef PERMB200_N50_CHAINS            // A/B switch for the M5 size (tools/microbench/sweep_bench.cu)
#define PERMB200_N50_CHAINS 4
#endif
__host__ __device__ constexpr int product_chains(int N) {
  return N == 50 ? PERMB200_N50_CHAINS : N < 4 ? N : N <= 50 ? 4 : N <= 53 ? 3 : 2;
}

// Product of the n row sums: NC independent chains (i mod NC) then a pairwise tree.
// The order depends only on N, so every kernel/launch shape computes identical terms.
template <int N>
__device__ __forceinline__ double2 row_product(const double2 (&s)[N]) {
  constexpr int NC = product_chains(N);
  double2 c[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) c[k] = s[k];
#pragma unroll
  for (int i = NC; i < N; ++i) c[i % NC] = cmul(c[i % NC], s[i]);
#pragma unroll
  for (int w = 1; w < NC; w *= 2) {
#pragma unroll
    for (int k = 0; k + w < NC; k += 2 * w) c[k] = cmul(c[k], c[k + w]);
  }
  return c[0];
}

// ------------------------------------------------------------------ column sources
// Flip of Gray bit b touches matrix column col0 + b (Glynn col0 = 1: bit b <-> delta_{b+2};
// Ryser col0 = 0: bit b <-> column b).
//
// ConstColumns: table[slot][2b+d][i] = signed step vector of Gray bit b flipped with direction d
// (b < c; zero rows for c <= b < 16), so every flip is one DADD with a uniform operand.
// Declared per translation unit (static): each TU stages its own copy.
static __constant__ double2 c_cols[kSlots * kTabRows * kNMax];

// Batched / small kernels: keep the bit-0 step vector (used by two of every four flips) in
// registers for the whole chunk instead of re-reading it from shared memory (A/B switch for
// tools/microbench/batched_bench.cu).
#ifndef PERMB200_ROW_AHEAD             // A/B switch (tools/microbench/sweep_bench.cu)
#define PERMB200_ROW_AHEAD 1
#endif
#ifndef PERMB200_N50_AHEAD
#define PERMB200_N50_AHEAD 0
#endif
__host__ __device__ constexpr bool row_ahead(int N) {
  return PERMB200_ROW_AHEAD && (N <= 46 || N == 49 || (N == 50 && PERMB200_N50_AHEAD));
}
#ifndef PERMB200_BIT0_CACHE
#define PERMB200_BIT0_CACHE 0
#endif
// Terms per half-walk loop iteration: 4 (bit-0 flips with compile-time directions), or 2 for
// N >= PERMB200_UNROLL2_FROM (half the loop body: the n = 50 body of 4 terms is ~30 KB of SASS
// against a 32 KB L1.5 instruction cache; the bit-0 direction becomes a loop-carried uniform
// value).  Same flips, same terms, same accumulation order: bit-identical results.
#ifndef PERMB200_UNROLL2_FROM          // A/B switch (tools/microbench/sweep_bench.cu)
#define PERMB200_UNROLL2_FROM 999
#endif
__host__ __device__ constexpr bool walk_unroll2(int N) { return N >= PERMB200_UNROLL2_FROM; }

struct ConstColumns {
  static constexpr bool kSmemAccOk = true;    // see Walker::kSmemAcc
  static constexpr bool kWideBuild = true;    // Walker::build: all rows per pass for n <= 24
  static constexpr bool kBit0Cached = false;  // uniform LDCU operands cost no vector registers
  int base;
  __device__ __forceinline__ double2 get(int row, int i) const {
    PERM_CHECK(row >= 0 && row < kTabRows && i >= 0 && i < kNMax && base >= 0 &&
               base + row * kNMax + i < kSlots * kTabRows * kNMax);
    return c_cols[base + row * kNMax + i];
  }
};

// SmemColumns: a per-block shared-memory table with the same layout as the constant one:
// tab[(2b+d)*N + i] = signed step vector of Gray bit b, direction d (zero rows for b >= c).
template <int N, bool WIDE = true>
struct SmemColumns {
  // The batched kernel reads its columns from shared memory; with shared-memory accumulators
  // too (and their layout) M2 measured 28 % slower (1.11 vs 0.865 ms): registers there.
  static constexpr bool kSmemAccOk = false;
  static constexpr bool kWideBuild = WIDE;
  static constexpr bool kBit0Cached = PERMB200_BIT0_CACHE;
  const double2* tab;
  __device__ __forceinline__ double2 get(int row, int i) const {
    PERM_CHECK(row >= 0 && row < kTabRows && i >= 0 && i < N && in_dyn_smem(tab + row * N + i, sizeof(double2)));
    return tab[row * N + i];
  }
};

// Plain (uncompensated) FP64 addition of two partials: the paper's accumulation
// ("Perm = Perm +- delta"; reading R12) used by the PLAIN mode; only the hi
// halves are used, lo stays 0.
__device__ __forceinline__ Dd2 plain2_add(const Dd2& a, const Dd2& b) {
  return Dd2{__dadd_rn(a.re_hi, b.re_hi), 0.0, __dadd_rn(a.im_hi, b.im_hi), 0.0};
}

// Separate-addition partials (kSep): (even, odd) sums in the (hi, lo) slots, each added in
// plain FP64 on its own.
__device__ __forceinline__ Dd2 sep2_add(const Dd2& a, const Dd2& b) {
  return Dd2{__dadd_rn(a.re_hi, b.re_hi), __dadd_rn(a.re_lo, b.re_lo), __dadd_rn(a.im_hi, b.im_hi),
             __dadd_rn(a.im_lo, b.im_lo)};
}

template <int MODE>
__device__ __forceinline__ Dd2 part_add(const Dd2& a, const Dd2& b) {
  return MODE == kComp ? dd2_add(a, b) : MODE == kPlain ? plain2_add(a, b) : sep2_add(a, b);
}

// ------------------------------------------------------------------ the walker
// MODE = kComp: compensated accumulation (Sum2 cascade + dd partials, the default);
// kPlain: every accumulation in plain FP64 (the precision lab's "plain" mode, §8(f)2: same
// terms, same order, only the compensation removed); kSep: even / odd terms summed apart.
template <int N, int ALG, int MODE = kComp, bool SMEM_ACC = acc_in_smem(N)>
struct Walker {
  static constexpr bool PLAIN = (MODE == kPlain);
  double2 s[N];                  // row sums (registers)
  // Cascaded (Sum2) double-double accumulator of the chunk (PLAIN: hi halves only): in
  // registers, or (acc_in_smem(N)) in this thread's shared-memory slot, which the kernels place
  // right after their N*N matrix copy and blockDim reduction entries.
  static constexpr bool kSmemAcc = SMEM_ACC;
  double arh, arl, aih, ail;     // kSep: arh/aih even sums, arl/ail odd sums
  Dd2* accs;

  // Column sources hold STEP VECTORS u = kScale * column (Glynn 2a: exact doubling; Ryser a).
  // Direction bit d of a flip: Glynn d=1 -> delta back to +1 -> +u, d=0 -> delta to -1 -> -u;
  // Ryser d=1 -> column leaves S -> -u, d=0 -> joins S -> +u.
  static constexpr double kScale = (ALG == kGlynn) ? 2.0 : 1.0;
  static constexpr double kSgnDir1 = (ALG == kGlynn) ? 1.0 : -1.0;
  static constexpr double kSgnDir0 = (ALG == kGlynn) ? -1.0 : 1.0;
  // term sign base: Glynn (-1)^g ; Ryser (-1)^(N+g)
  static constexpr bool kNegBase = (ALG == kRyser) && (N & 1);

  __device__ __forceinline__ void zero_acc() {
    if (kSmemAcc) {
      extern __shared__ double2 smem_acc[];
      accs = reinterpret_cast<Dd2*>(smem_acc + N * N) + blockDim.x + threadIdx.x;
      PERM_CHECK(in_dyn_smem(accs, sizeof(Dd2)));
      *accs = Dd2{0.0, 0.0, 0.0, 0.0};
    } else {
      arh = arl = aih = ail = 0.0;
    }
  }

  // kSep: the even-g and odd-g block sums enter their own plain accumulators.
  __device__ __forceinline__ void acc_add_sep(double er, double ei, double orr, double oi) {
    if (kSmemAcc) {
      Dd2 a = *accs;
      a.re_hi = __dadd_rn(a.re_hi, er); a.re_lo = __dadd_rn(a.re_lo, orr);
      a.im_hi = __dadd_rn(a.im_hi, ei); a.im_lo = __dadd_rn(a.im_lo, oi);
      *accs = a;
      return;
    }
    arh = __dadd_rn(arh, er); arl = __dadd_rn(arl, orr);
    aih = __dadd_rn(aih, ei); ail = __dadd_rn(ail, oi);
  }

  __device__ __forceinline__ void acc_add(double re, double im) {
    if (kSmemAcc) {
      Dd2 a = *accs;
      if (PLAIN) {
        a.re_hi = __dadd_rn(a.re_hi, re);
        a.im_hi = __dadd_rn(a.im_hi, im);
      } else {
        double s_, e_;
        two_sum(a.re_hi, re, s_, e_);
        a.re_hi = s_; a.re_lo = __dadd_rn(a.re_lo, e_);
        two_sum(a.im_hi, im, s_, e_);
        a.im_hi = s_; a.im_lo = __dadd_rn(a.im_lo, e_);
      }
      *accs = a;
      return;
    }
    if (PLAIN) {
      arh = __dadd_rn(arh, re);
      aih = __dadd_rn(aih, im);
      return;
    }
    double s_, e_;
    two_sum(arh, re, s_, e_);
    arh = s_; arl = __dadd_rn(arl, e_);
    two_sum(aih, im, s_, e_);
    aih = s_; ail = __dadd_rn(ail, e_);
  }

  // Chunk-start row sums for code G ("Convert iter to the set delta ...
  // Calculate s"), O(n^2), from the transposed, pre-scaled matrix in shared memory.  Rows are done
  // RB at a time with a runtime column loop, which bounds the registers the loads take: 8 rows
  // for large n; all rows, two columns per iteration, for n <= 24, where the build is a large
  // share of a chunk (M1: 32-term chunks) and was bound by the shared-memory load latency of
  // each 8-row column slice (m1_phases: ~6000 of the walk's 15500 cycles per block).  Every row
  // sum is accumulated over the same columns in the same order: the same bits either way.
  template <bool WIDE = false>
  __device__ __forceinline__ void build(const double2* __restrict__ at, uint64_t G) {
    constexpr int RB = build_rows(N, WIDE);
#pragma unroll
    for (int r0 = 0; r0 < N; r0 += RB) {
#pragma unroll
      for (int i = r0; i < r0 + RB; ++i)
        if (i < N) {
          if (ALG == kGlynn) s[i] = make_double2(0.5 * at[i].x, 0.5 * at[i].y);  // delta_1 = +1; exact
          else s[i] = make_double2(0.0, 0.0);          // Ryser: S starts empty
        }
#pragma unroll (build_col_unroll(N, WIDE))
      for (int j = (ALG == kGlynn) ? 1 : 0; j < N; ++j) {
        const int bit = (ALG == kGlynn) ? (int)((G >> (j - 1)) & 1) : (int)((G >> j) & 1);
        // at holds kScale * a: weight delta_j / 2 (Glynn) reproduces RN(s + delta_j a_ij) exactly
        const double w = (ALG == kGlynn) ? (bit ? -0.5 : 0.5) : (bit ? 1.0 : 0.0);
        const double2* col = at + j * N;
#pragma unroll
        for (int i = r0; i < r0 + RB; ++i)
          if (i < N) {
            const double2 v = col[i];
            s[i].x = __fma_rn(w, v.x, s[i].x);
            s[i].y = __fma_rn(w, v.y, s[i].y);
          }
      }
    }
  }

  // Row of the signed table holding +u_b (Glynn: d = 1 -> +u; Ryser: d = 0 -> +u).
  static __device__ __forceinline__ int plus_row(int b) { return 2 * b + (ALG == kGlynn ? 1 : 0); }

  // s_i <- s_i + table[row]_i : one DADD per real component, the signed step vector being
  // the uniform (UR) operand.
  template <class Cols>
  __device__ __forceinline__ void flip_row(const Cols& cols, int row) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double2 v = cols.get(row, i);
      s[i].x = __dadd_rn(s[i].x, v.x);
      s[i].y = __dadd_rn(s[i].y, v.y);
    }
  }

  // s_i <- s_i + sg * table[row]_i with a per-thread sign sg = +-1 (the one mid-chunk flip).
  template <class Cols>
  __device__ __forceinline__ void flip_signed(const Cols& cols, int row, double sg) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double2 v = cols.get(row, i);
      s[i].x = __fma_rn(sg, v.x, s[i].x);
      s[i].y = __fma_rn(sg, v.y, s[i].y);
    }
  }
  // Uniform half-walk.  State on entry = row sums at local index T0; visits local indices
  // T0 .. T0+H-1 (H = 2^(c-1) >= 16).  Iteration t (t = -4, 0, 4, ..., H-8) visits
  // T0+t+4 .. T0+t+7:  r=0 flips Gray bit b = ctz(t+4) (t = -4: bit 15, all-zero table
  // rows: no flip), r=1 bit 0, r=2 bit 1, r=3 bit 0.  Direction of the flip into index g is
  // bit (b+1) of g, so r=1 -> 0, r=3 -> 1, r=2 -> bit 2 of t+4 and r=0
  // -> bit b+1 of T0+t+4: all warp-uniform.  Terms alternate in sign (parity of G(g) =
  // parity of g); plain sums over 16 terms, then the compensated (Sum2) accumulator.
  //
  // The loop is written in exactly this shape on purpose: one flip call site per unrolled
  // step with (b, sg) selected by r, and the opaque tz = t*zero in the compile-time
  // column indices.  ptxas then keeps t in a uniform register and reads the columns with
  // LDCU (uniform operand, no vector register); other spellings of the same loop made it
  // fall back to per-thread LDC + spills (tests/test_build_sass.py guards this).
  // Row of the step-r = 0 flip into local index T0 + t + 4: Gray bit b = ctz(t + 4) (t = -4: bit
  // 15, an all-zero table row), direction bit b + 1 of the index.
  static __device__ __forceinline__ int head_row(int T0, int t) {
    const int b = (__ffs(t + 4) - 1) & 15;
    return 2 * b + (((T0 + t + 4) >> (b + 1)) & 1);
  }

  template <class Cols>
  __device__ __forceinline__ void half_walk(const Cols& cols, int T0, int H, int zero, const double2 (&u0)[N]) {
    double mr = 0.0, mi = 0.0;      // kSep: even-g block sums
    double orr = 0.0, oi = 0.0;     // kSep only: odd-g block sums
    // PERMB200_ROW_AHEAD: the step-0 row of the NEXT iteration is computed during this one (a
    // loop-carried uniform value), so the loop head's column loads do not wait behind the
    // ctz / shift chain (ncu source view, n = 50: the runtime-row flips at steps 0 and 2 carried
    // ~all of the short-scoreboard stalls; the constant-row bit-0 flips none).
    // Per n (spill-free SASS only, tools/sass_loop_stats.py: on for n <= 46 and n = 49; at n = 48,
    // 50, 51 the extra live value tipped ptxas into spills).
    constexpr bool kAhead = row_ahead(N);
    if constexpr (walk_unroll2(N) && MODE != kSep && !Cols::kBit0Cached) {
      // 2 terms per iteration: local indices T0+t+2 (Gray bit ctz(t+2); t = -2: the all-zero
      // row of bit 15) and T0+t+3 (bit 0, direction = bit 1 of the index).
      for (int t = -2; t < H - 2; t += 2) {
        const int tz = t * zero;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int b = (r == 0) ? ((__ffs(t + 2) - 1) & 15) : 0;
          const int d = (r == 0) ? (((T0 + t + 2) >> (b + 1)) & 1) : (((t + 2) >> 1) & 1);
          const int row = (r == 0) ? (2 * b + d) : (d + tz);
          flip_row(cols, row);
          const double2 p = row_product<N>(s);
          if (((r & 1) != 0) != kNegBase) { mr = __dsub_rn(mr, p.x); mi = __dsub_rn(mi, p.y); }
          else { mr = __dadd_rn(mr, p.x); mi = __dadd_rn(mi, p.y); }
        }
        if (((t + 2) & 14) == 14) {
          acc_add(mr, mi);
          mr = 0.0; mi = 0.0;
        }
      }
      acc_add(mr, mi);
      return;
    }
    int row0_next = head_row(T0, -4);
    for (int t = -4; t < H - 4; t += 4) {
      const int tz = t * zero;
      const int row0 = row0_next;
      if (kAhead) row0_next = head_row(T0, t + 4);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int b = (r == 0) ? ((__ffs(t + 4) - 1) & 15) : (__ffs(r) - 1);
        const int d = (r == 0) ? (((T0 + t + 4) >> (b + 1)) & 1) : (r == 1) ? 0 : (r == 2) ? (((t + 4) >> 2) & 1) : 1;
        const int row = (r == 0) ? (kAhead ? row0 : 2 * b + d) : (2 * b + d + tz);
        if (Cols::kBit0Cached && (r & 1)) {
          // bit 0 from registers: r = 1 adds table row 0, r = 3 row 1 = -(row 0)
#pragma unroll
          for (int i = 0; i < N; ++i) {
            if (r == 1) { s[i].x = __dadd_rn(s[i].x, u0[i].x); s[i].y = __dadd_rn(s[i].y, u0[i].y); }
            else { s[i].x = __dsub_rn(s[i].x, u0[i].x); s[i].y = __dsub_rn(s[i].y, u0[i].y); }
          }
        } else {
          flip_row(cols, row);
        }
        const double2 p = row_product<N>(s);
        if (MODE == kSep) {          // parity of g = parity of r (T0 and t + 4 are multiples of 4)
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

  // Full aligned chunk q (Gray indices [q 2^c, (q+1) 2^c)), c >= kMinFastC.
  template <class Cols>
  __device__ __forceinline__ void fast_chunk(const Cols& cols, const double2* __restrict__ at, uint64_t q, int c, int zero) {
    const uint64_t g0 = q << c;
    build<Cols::kWideBuild>(at, g0 ^ (g0 >> 1));
    const int H = 1 << (c - 1);
    double2 u0[N];                  // Cols::kBit0Cached: table row 0 (bit 0, direction 0)
    if (Cols::kBit0Cached) {
#pragma unroll
      for (int i = 0; i < N; ++i) u0[i] = cols.get(0, i);
    }
    // One copy of the half-walk loop serves both halves (two inlined copies of the n = 50
    // loop body overflow the instruction cache).
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      // direction = bit c of g = bit 0 of q: per-thread sign on the +u row (uniform index)
      if (h == 1) flip_signed(cols, plus_row(c - 1), (q & 1) ? kSgnDir1 : kSgnDir0);
      half_walk(cols, h * H, H, zero, u0);
    }
  }

  // Generic walk over [ga, gb) inside one aligned chunk (ragged range ends, tiny n):
  // per-thread columns from shared memory, per-term compensated accumulation.
  __device__ __forceinline__ void generic_walk(const double2* __restrict__ at, uint64_t ga, uint64_t gb) {
    constexpr int col0 = (ALG == kGlynn) ? 1 : 0;
    build(at, ga ^ (ga >> 1));
    for (uint64_t g = ga;; ) {
      double2 p = row_product<N>(s);
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
      const double2* col = at + (col0 + b) * N;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double2 v = col[i];
        s[i].x = __fma_rn(sg, v.x, s[i].x);
        s[i].y = __fma_rn(sg, v.y, s[i].y);
      }
    }
  }

  __device__ __forceinline__ Dd2 result() const {
    if (MODE == kSep) return kSmemAcc ? *accs : Dd2{arh, arl, aih, ail};
    if (kSmemAcc) {
      const Dd2 a = *accs;
      if (PLAIN) return Dd2{a.re_hi, 0.0, a.im_hi, 0.0};
      Dd2 r;
      fast_two_sum(a.re_hi, a.re_lo, r.re_hi, r.re_lo);
      fast_two_sum(a.im_hi, a.im_lo, r.im_hi, r.im_lo);
      return r;
    }
    if (PLAIN) return Dd2{arh, 0.0, aih, 0.0};
    Dd2 r;
    fast_two_sum(arh, arl, r.re_hi, r.re_lo);
    fast_two_sum(aih, ail, r.im_hi, r.im_lo);
    return r;
  }
};

// One full aligned chunk q, c >= kMinFastC, as its own (non-inlined) function.  Keeping the walk
// in a separate ptxas allocation unit is what lets ptxas hold the half-walk loop counter in
// a uniform register and feed the column operands from LDCU; inlined into the leaf loop
// (a loop nest with the build's loop) it fell back to per-thread LDC and spilled.
template <int N, int ALG, int MODE, bool SA, class Cols>
__device__ __noinline__ Dd2 chunk_fast(const Cols cols, const double2* __restrict__ at, uint64_t q, int c, int zero) {
  Walker<N, ALG, MODE, SA> w;
  w.zero_acc();
  w.fast_chunk(cols, at, q, c, zero);
  return w.result();
}

// Ragged piece [ga, gb) of one chunk (range ends, tiny n).
template <int N, int ALG, int MODE, bool SA>
__device__ __noinline__ Dd2 chunk_generic(const double2* __restrict__ at, uint64_t ga, uint64_t gb) {
  Walker<N, ALG, MODE, SA> w;
  w.zero_acc();
  w.generic_walk(at, ga, gb);
  return w.result();
}

// Chunks k in [k0, k1) of leaf `leaf_id` (chunks q = leaf_id 2^lam + k of 2^c Gray indices)
// that intersect [lo, hi): a ragged range touching a few chunks of a long leaf (large n:
// 2^27 chunks per leaf) must not iterate over the rest.
__device__ __forceinline__ void leaf_chunk_window(uint64_t leaf_id, int c, int lam, uint64_t lo, uint64_t hi,
                                                  uint64_t& k0, uint64_t& k1) {
  const uint64_t first = leaf_id << lam, nchunks = 1ull << lam;
  const uint64_t qlo = lo >> c, qhi = (hi + (1ull << c) - 1) >> c;     // chunks [qlo, qhi) meet [lo, hi)
  k0 = qlo > first ? qlo - first : 0;
  k1 = qhi > first ? qhi - first : 0;
  if (k0 > nchunks) k0 = nchunks;
  if (k1 > nchunks) k1 = nchunks;
}

// One leaf = 2^lam consecutive chunks walked in order by one thread; chunk partials are
// combined in order with double-double additions.  kFast: every chunk lies inside the
// range and c >= kMinFastC (decided by the caller from block-uniform values).
template <int N, int ALG, bool kFast, int MODE, class Cols>
__device__ __forceinline__ Dd2 walk_leaf(const Cols& cols, const double2* __restrict__ at, uint64_t leaf_id,
                                         int c, int lam, uint64_t lo, uint64_t hi, int zero) {
  // shared-memory chunk accumulator only in the sweep kernel (ConstColumns; its smem layout
  // puts the slots after the matrix copy and the reduction entries)
  constexpr bool SA = Cols::kSmemAccOk && acc_in_smem(N);
  Dd2 acc{0.0, 0.0, 0.0, 0.0};
  // Fast path: all 2^lam chunks (this exact loop shape keeps ptxas's uniform-register column
  // path, tests/test_build_sass.py).  Ragged path: only chunks [k0, k1) meeting [lo, hi).
  uint64_t k0 = 0, k1 = 1ull << lam;
  if (!kFast) leaf_chunk_window(leaf_id, c, lam, lo, hi, k0, k1);
  for (uint64_t k = k0; k < k1; ++k) {
    const uint64_t q = (leaf_id << lam) + k;
    if (kFast) {
      acc = part_add<MODE>(acc, chunk_fast<N, ALG, MODE, SA>(cols, at, q, c, zero));
    } else {
      const uint64_t g0 = q << c, g1 = g0 + (1ull << c);
      const uint64_t ga = g0 > lo ? g0 : lo;
      const uint64_t gb = g1 < hi ? g1 : hi;
      if (ga < gb) acc = part_add<MODE>(acc, chunk_generic<N, ALG, MODE, SA>(at, ga, gb));
    }
  }
  return acc;
}

// Transposed, pre-scaled copy of one n*n row-major matrix into shared memory:
// at[j*N + i] = scale * a_ij (scale 2 for Glynn, exact; 1 for Ryser).
template <int N>
__device__ __forceinline__ void stage_transposed(const double2* __restrict__ A, double2* at, double scale) {
  for (int k = threadIdx.x; k < N * N; k += blockDim.x) {
    const int i = k / N, j = k - i * N;
    double2 v = A[k];
    v.x *= scale;
    v.y *= scale;
    PERM_CHECK(in_dyn_smem(at + j * N + i, sizeof(double2)));
    at[j * N + i] = v;
  }
}

// Canonical block reduction: contiguous pairwise tree over the block's threads (leaves),
// node = left + right in double-double: at level o (1, 2, 4, ...) thread t (a multiple of 2o)
// adds the node of t + o.  Result valid in red[0] for thread 0 (blockDim a power of two).
// Levels below 32 run inside each warp with shuffles (lane t takes lane t + o's node: the same
// pairs, left + right, so the same bits as the shared-memory tree); the warp roots then go
// through shared memory once and warp 0 finishes the levels above with shuffles -- one block
// barrier instead of log2(blockDim) (m1_phases: the 7-level tree took ~2250 cycles per block).
__device__ __forceinline__ Dd2 shfl_down_dd2(const Dd2& v, int o, unsigned mask) {
  return Dd2{__shfl_down_sync(mask, v.re_hi, o), __shfl_down_sync(mask, v.re_lo, o),
             __shfl_down_sync(mask, v.im_hi, o), __shfl_down_sync(mask, v.im_lo, o)};
}

// Levels o < width (a power of two <= 32) among the lanes in `mask` (every lane that executes).
template <int MODE>
__device__ __forceinline__ Dd2 warp_tree(Dd2 v, int lane, int width, unsigned mask) {
  for (int o = 1; o < width; o <<= 1) {
    const Dd2 u = shfl_down_dd2(v, o, mask);
    if ((lane & (2 * o - 1)) == 0) v = part_add<MODE>(v, u);
  }
  return v;
}

template <int MODE = kComp>
__device__ __forceinline__ void block_tree(Dd2* red, const Dd2& mine) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nw = (nt + 31) >> 5;
  // a block smaller than a warp has only its nt lanes
  Dd2 v = warp_tree<MODE>(mine, lane, nt < 32 ? nt : 32, nt < 32 ? ((1u << nt) - 1u) : 0xffffffffu);
  if (nw == 1) {
    if (tid == 0) red[0] = v;
    return;
  }
  PERM_CHECK(in_dyn_smem(red + warp, sizeof(Dd2)));
  __syncthreads();                       // red may still be read by an earlier use
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? red[lane] : Dd2{0.0, 0.0, 0.0, 0.0};
    v = warp_tree<MODE>(v, lane, nw, 0xffffffffu);
    if (lane == 0) red[0] = v;
  }
}

// ------------------------------------------------------------------ kernels
// One block = one unit of the canonical plan.  Dynamic shared memory: N*N double2
// (transposed matrix) + blockDim Dd2 (reduction).
template <int N, int ALG, int MODE>
__global__ void __launch_bounds__(kMaxBlock) sweep_kernel(const SweepArgs args) {
  extern __shared__ double2 smem[];
  // [N*N: at][blockDim Dd2: tree][blockDim Dd2: chunk accumulators (Walker)]
  double2* at = smem;
  Dd2* red = reinterpret_cast<Dd2*>(smem + N * N);
  stage_transposed<N>(args.A, at, Walker<N, ALG>::kScale);
  __syncthreads();

  const ConstColumns cols{args.col_base};
  const uint64_t unit = (uint64_t)(args.unit_lo + blockIdx.x);
  const uint64_t leaf_id = (unit << args.block_bits) + threadIdx.x;
  const int ubits = args.block_bits + args.lam + args.c;          // log2(unit terms)
  const bool inside = (unit << ubits) >= args.lo && ((unit + 1) << ubits) <= args.hi;
  Dd2 mine;
  if (inside && args.c >= kMinFastC) mine = walk_leaf<N, ALG, true, MODE>(cols, at, leaf_id, args.c, args.lam, args.lo, args.hi, args.zero);
  else mine = walk_leaf<N, ALG, false, MODE>(cols, at, leaf_id, args.c, args.lam, args.lo, args.hi, args.zero);

  block_tree<MODE>(red, mine);
  if (threadIdx.x == 0) args.unit_out[blockIdx.x] = red[0];
}

// Signed step-vector table of one matrix in shared memory, the layout of the constant one:
// tab[(2b+d)*N + i] = step of Gray bit b (< c) flipped with direction d; zero rows beyond c.
// at = the pre-scaled transposed matrix (Glynn 2a, Ryser a).
template <int N, int ALG>
__device__ __forceinline__ void build_tab(const double2* at, double2* tab, int c) {
  constexpr int col0 = (ALG == kGlynn) ? 1 : 0;
  for (int k = threadIdx.x; k < kTabRows * N; k += blockDim.x) {
    const int row = k / N, i = k - row * N;
    const int bb = row >> 1, d = row & 1;
    double2 v = make_double2(0.0, 0.0);
    if (bb < c && col0 + bb < N) {
      v = at[(col0 + bb) * N + i];
      // Glynn: d=1 -> +2a, d=0 -> -2a;  Ryser: d=1 -> -a, d=0 -> +a
      const bool neg = (ALG == kGlynn) ? !d : d;
      if (neg) { v.x = -v.x; v.y = -v.y; }
    }
    PERM_CHECK(in_dyn_smem(tab + k, sizeof(double2)));
    tab[k] = v;
  }
}

// Small-n single permanents (2^m terms, m <= kSmallLog2): the same walk with the step vectors
// read from a per-block shared-memory table (SmemColumns) instead of the constant bank, so a
// call needs no column-staging kernel, no constant-memory copy and no slot fencing -- two
// launches (this + combine) instead of four.  The terms and their order are the sweep
// kernel's (same table values, same flips, same accumulation), i.e. bit-identical results.
constexpr int kSmallLog2 = 21;

template <int N, int ALG, int MODE>
__global__ void __launch_bounds__(kMaxBlock) sweep_small_kernel(const SweepArgs args) {
  extern __shared__ double2 smem[];
  // [N*N: at][kTabRows*N: tab][blockDim Dd2: tree]  (register chunk accumulators)
  double2* at = smem;
  double2* tab = smem + N * N;
  Dd2* red = reinterpret_cast<Dd2*>(smem + N * N + kTabRows * N);
  stage_transposed<N>(args.A, at, Walker<N, ALG>::kScale);
  __syncthreads();
  build_tab<N, ALG>(at, tab, args.c < kCMax ? args.c : kCMax);
  __syncthreads();
  const SmemColumns<N> cols{tab};
  const uint64_t unit = (uint64_t)(args.unit_lo + blockIdx.x);
  const uint64_t leaf_id = (unit << args.block_bits) + threadIdx.x;
  const int ubits = args.block_bits + args.lam + args.c;
  const bool inside = (unit << ubits) >= args.lo && ((unit + 1) << ubits) <= args.hi;
  Dd2 mine;
  if (inside && args.c >= kMinFastC) mine = walk_leaf<N, ALG, true, MODE>(cols, at, leaf_id, args.c, args.lam, args.lo, args.hi, args.zero);
  else mine = walk_leaf<N, ALG, false, MODE>(cols, at, leaf_id, args.c, args.lam, args.lo, args.hi, args.zero);
  block_tree<MODE>(red, mine);
  if (threadIdx.x == 0) args.unit_out[blockIdx.x] = red[0];
}

// Final step of a permanent: the unscaled root partial -> out (complex128, x 2^-(n-1) for
// Glynn, reading R3) and/or out_dd (optionally scaled, both halves exactly); zero components
// canonicalised to +0 (reading R11).  Shared by combine_kernel and the fused small-n kernel
// so both produce the same bits.
struct FinishArgs {
  double2* out;
  Dd2* out_dd;
  int do_scale, scale_exp, scale_dd;
  int sep;      // 0; or kSep partials: +1 / -1 = sign of (even - odd) (Ryser, odd n: -1)
};

__device__ __forceinline__ void finish_root(const Dd2& r, const FinishArgs& f) {
  const int e = f.do_scale ? f.scale_exp : 0;
  if (f.sep) {
    // separate addition: the ONE subtraction of the odd-index sum from the even-index sum
    // ("(0+2+4+6)-(1+3+5+7)"), then the exact sign and power-of-two factors
    if (f.out_dd) {
      Dd2 o = r;
      if (f.scale_dd) {
        o.re_hi = ldexp(o.re_hi, e); o.re_lo = ldexp(o.re_lo, e);
        o.im_hi = ldexp(o.im_hi, e); o.im_lo = ldexp(o.im_lo, e);
      }
      *f.out_dd = o;
    }
    if (f.out) {
      double re = ldexp(__dsub_rn(r.re_hi, r.re_lo), e) * (double)f.sep;
      double im = ldexp(__dsub_rn(r.im_hi, r.im_lo), e) * (double)f.sep;
      if (re == 0.0) re = 0.0;
      if (im == 0.0) im = 0.0;
      *f.out = make_double2(re, im);
    }
    return;
  }
  if (f.out_dd) {
    Dd2 o = r;
    if (f.scale_dd) {            // exact power-of-two scaling of both halves
      o.re_hi = ldexp(o.re_hi, e); o.re_lo = ldexp(o.re_lo, e);
      o.im_hi = ldexp(o.im_hi, e); o.im_lo = ldexp(o.im_lo, e);
      if (o.re_hi == 0.0) { o.re_hi = 0.0; o.re_lo = 0.0; }
      if (o.im_hi == 0.0) { o.im_hi = 0.0; o.im_lo = 0.0; }
    }
    *f.out_dd = o;
  }
  if (f.out) {
    double re = __dadd_rn(ldexp(r.re_hi, e), ldexp(r.re_lo, e));
    double im = __dadd_rn(ldexp(r.im_hi, e), ldexp(r.im_lo, e));
    if (re == 0.0) re = 0.0;
    if (im == 0.0) im = 0.0;
    *f.out = make_double2(re, im);
  }
}

// Small-n full permanent in ONE cooperative launch: every block sweeps its unit (as
// sweep_small_kernel), a grid barrier, then block 0 reduces the unit partials with the
// canonical tree (units <= blockDim, a power of two: block_tree over blockDim entries with
// zero padding pairs them exactly as combine_kernel does) and finishes.  Same bits as sweep +
// combine, one launch fewer (M1: the combine launch measured ~5 us of a ~20 us call).
template <int N, int ALG, int MODE>
__global__ void __launch_bounds__(kMaxBlock) sweep_small_fused_kernel(const SweepArgs args, const FinishArgs fin) {
  extern __shared__ double2 smem[];
  PERM_PHASE_START(ph_t);
  double2* at = smem;
  double2* tab = smem + N * N;
  Dd2* red = reinterpret_cast<Dd2*>(smem + N * N + kTabRows * N);
  stage_transposed<N>(args.A, at, Walker<N, ALG>::kScale);
  __syncthreads();
  PERM_PHASE(1, ph_t);
  build_tab<N, ALG>(at, tab, args.c < kCMax ? args.c : kCMax);
  __syncthreads();
  PERM_PHASE(2, ph_t);
  const SmemColumns<N> cols{tab};
  const uint64_t unit = (uint64_t)(args.unit_lo + blockIdx.x);
  const uint64_t leaf_id = (unit << args.block_bits) + threadIdx.x;
  Dd2 mine;
  if (args.c >= kMinFastC) mine = walk_leaf<N, ALG, true, MODE>(cols, at, leaf_id, args.c, args.lam, args.lo, args.hi, args.zero);
  else mine = walk_leaf<N, ALG, false, MODE>(cols, at, leaf_id, args.c, args.lam, args.lo, args.hi, args.zero);
  PERM_PHASE(3, ph_t);
  block_tree<MODE>(red, mine);
  if (threadIdx.x == 0) args.unit_out[blockIdx.x] = red[0];
  PERM_PHASE(4, ph_t);
  cooperative_groups::this_grid().sync();
  PERM_PHASE(5, ph_t);
  if (blockIdx.x == 0) {
    // units (a power of two) <= 8 * blockDim: thread t first reduces the aligned segment
    // [t S, (t+1) S) (the bottom levels of the canonical tree), then the block tree
    const int S = gridDim.x > blockDim.x ? (int)(gridDim.x / blockDim.x) : 1;
    Dd2 stack[4];
    int top = 0;
    for (int k = 0; k < S; ++k) {
      const unsigned idx = threadIdx.x * S + k;
      Dd2 v = idx < gridDim.x ? args.unit_out[idx] : Dd2{0.0, 0.0, 0.0, 0.0};
      int lvl = 0;
      for (int kk = k; kk & 1; kk >>= 1) { v = part_add<MODE>(stack[lvl], v); ++lvl; }
      stack[lvl] = v;
      if (lvl > top) top = lvl;
    }
    const Dd2 v = stack[top];
    block_tree<MODE>(red, v);
    if (threadIdx.x == 0) finish_root(red[0], fin);
    PERM_PHASE(6, ph_t);
  }
}

// Batched Glynn: block b computes Perm(A_b) completely (boson sampling needs
// many permanents of n x n submatrices).  Columns come from the block's shared-memory copy
// (warp-uniform addresses: broadcast LDS).
// Resident blocks per SM the batched kernel is compiled for: the shared-memory column operands
// are loaded into vector registers, so ptxas's default allocation (n = 16: 168 registers, 3
// blocks/SM, 9.2 waves for M2's 4096 permanents; ncu profiles/r01_batched_m2_*) leaves warps
// idle.  At 4 blocks (<= 128 registers) chunk_fast<16> still has no spills (only the kernel
// body spills a few values across the chunk call).
#ifdef PERMB200_BATCHED_MINB          // A/B experiments (tools/microbench/batched_bench.cu)
__host__ __device__ constexpr int batched_min_blocks(int N) { return N <= 16 ? PERMB200_BATCHED_MINB : N <= 20 ? 3 : 1; }
#else
__host__ __device__ constexpr int batched_min_blocks(int N) { return N <= 16 ? 4 : N <= 20 ? 3 : 1; }
#endif

template <int N>
__global__ void __launch_bounds__(kMaxBlock, batched_min_blocks(N)) batched_kernel(const BatchedArgs args) {
  extern __shared__ double2 smem[];
  // [N*N: at][kTabRows*N: tab][blockDim Dd2: tree]  (register chunk accumulators)
  double2* at = smem;
  double2* tab = smem + N * N;
  Dd2* red = reinterpret_cast<Dd2*>(smem + N * N + kTabRows * N);
  for (int64_t b = blockIdx.x; b < args.batch; b += gridDim.x) {
    __syncthreads();
    stage_transposed<N>(args.A + b * (int64_t)(N * N), at, 2.0);
    __syncthreads();
    for (int k = threadIdx.x; k < kTabRows * N; k += blockDim.x) {
      const int row = k / N, i = k - row * N;
      const int bb = row >> 1, d = row & 1;
      double2 v = make_double2(0.0, 0.0);
      if (bb < args.c && 1 + bb < N) {
        v = at[(1 + bb) * N + i];      // 2a (pre-scaled); Glynn: d=1 -> +2a, d=0 -> -2a
        if (!d) { v.x = -v.x; v.y = -v.y; }
      }
      PERM_CHECK(in_dyn_smem(tab + k, sizeof(double2)));
      tab[k] = v;
    }
    __syncthreads();
    const SmemColumns<N, false> cols{tab};
    const uint64_t terms = 1ull << (N - 1);
    Dd2 mine;
    if (args.c >= kMinFastC) mine = walk_leaf<N, kGlynn, true, false>(cols, at, threadIdx.x, args.c, args.lam, 0, terms, args.zero);
    else mine = walk_leaf<N, kGlynn, false, false>(cols, at, threadIdx.x, args.c, args.lam, 0, terms, args.zero);
    block_tree(red, mine);
    if (threadIdx.x == 0) {
      const Dd2 r = red[0];
      double re = __dadd_rn(ldexp(r.re_hi, args.scale_exp), ldexp(r.re_lo, args.scale_exp));
      double im = __dadd_rn(ldexp(r.im_hi, args.scale_exp), ldexp(r.im_lo, args.scale_exp));
      if (re == 0.0) re = 0.0;   // canonical +0
      if (im == 0.0) im = 0.0;
      if (args.out) args.out[b] = make_double2(re, im);
      // P(S|T) ~ |Perm(U_ST)|^2: one fused multiply-add of the rounded components
      if (args.out_abs2) args.out_abs2[b] = __fma_rn(re, re, __dmul_rn(im, im));
    }
  }
}

// Column staging: table[b][i] = a_{i, col0+b}, b < c  (written to a device buffer, then
// copied into this TU's constant slot with cudaMemcpyToSymbolAsync).
static __global__ void stage_columns_kernel(const double2* __restrict__ A, int n, int col0, int c, double scale,
                                     double2* table) {
  for (int k = threadIdx.x; k < kTabRows * kNMax; k += blockDim.x) {
    const int row = k / kNMax, i = k - row * kNMax;
    const int b = row >> 1, d = row & 1;
    double2 v = make_double2(0.0, 0.0);
    if (b < c && i < n && col0 + b < n) {
      v = A[(size_t)i * n + col0 + b];
      // Glynn (col0 = 1): d=1 -> +2a, d=0 -> -2a;  Ryser (col0 = 0): d=1 -> -a, d=0 -> +a
      const double sg = (col0 == 1) ? (d ? scale : -scale) : (d ? -scale : scale);
      v.x *= sg;      // x(+-2) and x(+-1) are exact
      v.y *= sg;
    }
    table[k] = v;
  }
}

// ------------------------------------------------------------------ launchers
using SweepLauncher = cudaError_t (*)(const SweepArgs&, int64_t units, double2* staging, cudaStream_t);
using BatchedLauncher = cudaError_t (*)(const BatchedArgs&, int grid, cudaStream_t);

template <int N, int ALG, int MODE = kComp>
cudaError_t launch_sweep(const SweepArgs& a, int64_t units, double2* staging, cudaStream_t st) {
  const int c_tab = a.c < kCMax ? a.c : kCMax;
  const int col0 = (ALG == kGlynn) ? 1 : 0;
  if (a.c >= kMinFastC) {
    stage_columns_kernel<<<1, 256, 0, st>>>(a.A, N, col0, c_tab, (ALG == kGlynn) ? 2.0 : 1.0, staging);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cudaMemcpyToSymbolAsync(c_cols, staging, sizeof(double2) * kTabRows * kNMax,
                                sizeof(double2) * (size_t)a.slot * kTabRows * kNMax, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  const int threads = 1 << a.block_bits;
  const size_t smem = sizeof(double2) * N * N + 2 * sizeof(Dd2) * threads;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<N, ALG, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  sweep_kernel<N, ALG, MODE><<<(unsigned)units, threads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N, int ALG, int MODE>
cudaError_t launch_sweep_small(const SweepArgs& a, int64_t units, double2*, cudaStream_t st) {
  const int threads = 1 << a.block_bits;
  const size_t smem = sizeof(double2) * (N * N + kTabRows * N) + sizeof(Dd2) * threads;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sweep_small_kernel<N, ALG, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  sweep_small_kernel<N, ALG, MODE><<<(unsigned)units, threads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N, int ALG, int MODE>
cudaError_t launch_sweep_small_fused(const SweepArgs& a, const FinishArgs& f, int64_t units, cudaStream_t st) {
  const int threads = 1 << a.block_bits;
  const size_t smem = sizeof(double2) * (N * N + kTabRows * N) + sizeof(Dd2) * threads;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sweep_small_fused_kernel<N, ALG, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // every block of a cooperative launch must be co-resident: resident blocks per SM x SMs,
  // computed once per instantiation (and block size) -- one device model per process
  static int cap_threads = 0, cap_blocks = 0;
  if (cap_threads != threads) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_small_fused_kernel<N, ALG, MODE>,
                                                                  threads, smem);
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    cap_blocks = per_sm * sms;
    cap_threads = threads;
  }
  if (cap_blocks < units) return cudaErrorCooperativeLaunchTooLarge;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)units);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sweep_small_fused_kernel<N, ALG, MODE>, a, f);
}

template <int N>
cudaError_t launch_batched(const BatchedArgs& a, int grid, cudaStream_t st) {
  const int threads = 1 << a.block_bits;
  const size_t smem = sizeof(double2) * (N * N + kTabRows * N) + sizeof(Dd2) * threads;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(batched_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  batched_kernel<N><<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace permb200

// Instantiate launchers for n in [LO, HI] of algorithm ALG and register them in a table.
#include <utility>
namespace permb200 {
template <int ALG, int LO, int... Is>
void fill_sweep(SweepLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &launch_sweep<LO + Is, ALG, kComp>), ...);
}
template <int ALG, int LO, int... Is>
void fill_sweep_plain(SweepLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &launch_sweep<LO + Is, ALG, kPlain>), ...);
}
template <int ALG, int LO, int... Is>
void fill_sweep_sep(SweepLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &launch_sweep<LO + Is, ALG, kSep>), ...);
}
template <int ALG, int MODE, int LO, int... Is>
void fill_sweep_small(SweepLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &launch_sweep_small<LO + Is, ALG, MODE>), ...);
}
using FusedLauncher = cudaError_t (*)(const SweepArgs&, const FinishArgs&, int64_t units, cudaStream_t);
template <int ALG, int MODE, int LO, int... Is>
void fill_sweep_small_fused(FusedLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &launch_sweep_small_fused<LO + Is, ALG, MODE>), ...);
}
template <int LO, int... Is>
void fill_batched(BatchedLauncher* table, std::integer_sequence<int, Is...>) {
  ((table[LO + Is] = &launch_batched<LO + Is>), ...);
}
}  // namespace permb200
