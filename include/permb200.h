/*
 * permb200.h — C ABI of the B200 permanent engine (libpermb200.so).
 *
 * The problem: given an N x N complex matrix A, return
 *   Perm(A) = sum over permutations sigma of prod_i a_{i,sigma(i)}.
 * Two evaluation formulas, both walked in Gray-code order on the GPU:
 *   BB/FG (Glynn), Eq. (2), PAPER.md:66-68:
 *     Perm(A) = 2^{-(N-1)} * sum_delta (prod_k delta_k) prod_i sum_j delta_j a_ij,
 *     delta_1 = +1, delta_k in {-1,+1}; 2^{N-1} terms.
 *   Ryser, Eq. (1), PAPER.md:62-64:
 *     Perm(A) = (-1)^N sum_{S subset [N]} (-1)^{|S|} prod_i sum_{j in S} a_ij; 2^N terms.
 *
 * Index conventions (readings R2, R4, R5):
 *   - a "Gray index" g ranges over [0, 2^{N-1}) (Glynn) or [0, 2^N) (Ryser); its code is
 *     G(g) = g ^ (g >> 1).  Glynn: bit b of G set <=> delta_{b+2} = -1 (1-based), i.e.
 *     column b+1 (0-based) carries a minus sign.  Ryser: bit b of G set <=> column b
 *     (0-based) is in S.
 *   - term(g) = sign(g) * prod_i rowsum_i(G(g)), sign = prod_k delta_k = (-1)^{popcount G}
 *     (Glynn) or (-1)^{N - popcount G} (Ryser; the (-1)^N of Eq. (1) is folded per term).
 *   - a "partial" is the UNSCALED sum of term(g) over a range of g, as complex
 *     double-double.  The final factor 2^{-(N-1)} (Glynn) is applied exactly once, by
 *     perm_combine / perm_glynn (PAPER.md:262-263 divides after ALLREDUCE; reading R3:
 *     always, not only for odd N).
 *
 * Data layout: matrices are row-major n*n perm_c128 (interleaved re, im; identical to
 * torch.complex128 / numpy complex128 / cuDoubleComplex).  Batches are `batch` such
 * matrices back to back.
 *
 * Ownership and asynchrony: the CALLER owns every buffer.  Functions taking device
 * pointers enqueue work on `stream` (a cudaStream_t passed as void*; NULL = legacy
 * default stream) on the CURRENT device and return immediately; outputs are valid after
 * the stream is synchronised.  Temporary workspace is taken stream-ordered (cudaMallocFromPoolAsync,
 * a library-owned per-device pool that keeps up to 256 MiB cached) on
 * `stream` and released on it.  Concurrent calls on different streams / devices are
 * safe (the per-device constant-memory column slots are fenced with events).
 * Functions suffixed _host take HOST pointers and are synchronous.
 *
 * Deliberate deviations from SURVEY §8(b)'s conventions (measured trade-offs):
 *   - "no persistent library allocations": the library keeps a per-device stream-ordered
 *     memory pool (release threshold 256 MiB) for its workspaces -- the default pool remapped
 *     pages on every synchronous call (4.2 ms instead of tens of us for n = 20);
 *   - "no __constant__ matrix symbol": FP64 sweeps of more than 2^21 terms stage the signed
 *     column table in a per-translation-unit __constant__ slot so every column operand is a
 *     uniform-register LDCU read (this is what holds the FP64 pipe at ~90 %).  Consequences:
 *     such sweeps on one device serialise across streams (event-fenced slot reuse), and they
 *     refuse CUDA-graph capture (PERM_ECUDA); small n, the dd mode and the batched kernel use
 *     shared memory and are concurrent and capturable.
 *
 * Errors: every function returns PERM_OK (0) or an error code; nothing is written on
 * PERM_EINVAL.  Asynchronous device faults surface at the caller's next synchronisation.
 * Input VALUES are not checked: NaN / Inf propagate.  Results never contain -0.0.
 */
#ifndef PERMB200_H
#define PERMB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } perm_c128;                          /* 16 B */
typedef struct { double re_hi, re_lo, im_hi, im_lo; } perm_dd_c128;  /* 32 B */

enum {
  PERM_OK = 0,
  PERM_EINVAL = 1,   /* null pointer, n < 1, n > perm_max_n() (Ryser: n > 63), batch < 0, lo > hi,
                        hi > #terms, count < 1, bad alg */
  PERM_ECUDA = 2,    /* CUDA runtime / launch error (message via perm_strerror(PERM_ECUDA)) */
  PERM_ENOTIMPL = 3
};

/* Algorithm codes.  *_DD: the double-double precision mode: the same Gray
 * walk with every row sum, partial product and term carried as hi + lo (~2^-104 relative);
 * about 10x the FP64 instruction count per term.  Integer matrices whose partial products
 * and partial sums stay below 2^104 are evaluated exactly (e.g. J_20 -> 20!, J_20 - I -> D_20,
 * both beyond one double; reading R9). */
/* *_PLAIN: the FP64 sweep with every accumulation in plain (uncompensated) FP64 -- the
 * paper's "Perm = Perm +- delta" -- for the precision lab's
 * compensated-vs-plain accumulation discrepancy.  Same terms, same order,
 * same speed; partials carry lo = 0 and perm_combine adds them in plain FP64. */
/* *_SEP: the paper's "separate addition" summation order (Table AV):
 * the terms of even and of odd Gray index (even / odd |S|, resp. number of delta = -1) are
 * summed separately in plain FP64 and subtracted once at the end.  Partials carry the even
 * sum in the hi slots and the odd sum in the lo slots (re_hi = sum_even Re, re_lo = sum_odd
 * Re, ...); perm_combine adds them componentwise and finishes with (even - odd) times
 * (-1)^n (Ryser) / 2^{-(n-1)} (Glynn).  Precision-lab mode, n <= 40. */
enum { PERM_ALG_GLYNN = 0, PERM_ALG_RYSER = 1, PERM_ALG_GLYNN_DD = 2, PERM_ALG_RYSER_DD = 3,
       PERM_ALG_GLYNN_PLAIN = 4, PERM_ALG_RYSER_PLAIN = 5, PERM_ALG_GLYNN_SEP = 6, PERM_ALG_RYSER_SEP = 7 };

/* The canonical evaluation plan for (n, alg).  It depends only on (n, alg), never on
 * the GPU count, so any partition of the unit range reproduces the single-GPU result
 * bit for bit.
 *   terms      = 2^log2_terms (2^{n-1} Glynn, 2^n Ryser)
 *   chunk      = 2^chunk_bits consecutive Gray indices walked by one leaf from a fresh
 *                O(n^2) row-sum build (the drift reset)
 *   leaf       = 2^leaf_bits chunks, walked in order by one group of `lanes` threads into one
 *                dd partial; lanes = 1, or 2 (n >= 52, compensated mode) with the n row sums
 *                split over the two: lane l of a PAIR OF WARPS (rows [0, ceil(n/2)) in the
 *                even warp, the rest in the odd one; the plan's block_bits is 6) -- or two
 *                adjacent lanes of one warp for custom plans with block_bits < 5
 *   unit       = 2^block_bits leaves (one thread block of 2^block_bits * lanes threads) -> one
 *                dd partial
 *   units      = 2^unit_bits; unit_terms = terms / units */
typedef struct {
  int n, alg;
  int log2_terms, chunk_bits, leaf_bits, block_bits, unit_bits;
  int lanes;
  uint64_t unit_terms;
  int64_t units;
} perm_plan_t;

/* Largest supported n (64 for Glynn; Ryser stops at 63 because its 2^n Gray indices
 * must fit in uint64).  The FP64 sweep keeps every row sum in registers for all n: one thread
 * per chunk (4n registers) up to n = 51, two threads per chunk (2n registers each, one per
 * warp of a warp pair) from 52 on (the plain and separate-addition modes keep one thread per
 * chunk there and spill). */
int perm_max_n(void);

/* Human-readable text for a status code (for PERM_ECUDA: the last CUDA error seen by
 * this thread). */
const char* perm_strerror(int code);

/* Fill *plan for (n, alg).  PERM_EINVAL for bad n/alg or null plan. */
int perm_plan(int n, int alg, perm_plan_t* plan);

/* ---- single permanent (device pointers) -------------------------------------------- */
/* PAPER.md:60 (problem), Eq. (2) PAPER.md:66-68 / Alg. A2 PAPER.md:238-263 (BB/FG), Eq. (1)
 * PAPER.md:62-64 / Alg. A1 PAPER.md:206-235 (Ryser); the final factor and the single reduction
 * after the per-process partial sums: PAPER.md:230-232, :261-263 (reading R3: always 2^{-(N-1)}). */
/* out[0] = Perm(A) by Eq. (2) (perm_glynn) or Eq. (1) (perm_ryser).  A: device, n*n.
 * out: device, 1 element.  = perm_sweep_units over all units + perm_combine. */
int perm_glynn(const perm_c128* A, int n, perm_c128* out, void* stream);
int perm_ryser(const perm_c128* A, int n, perm_c128* out, void* stream);

/* ---- double-double precision mode (device pointers) -------------------------------- */
/* Same formulas; motivated by the paper's precision finding (FIG. 4). */
/* out[0] = Perm(A) as a complex double-double (re_hi, re_lo, im_hi, im_lo), already scaled by
 * 2^{-(N-1)} (Glynn; exact).  Same plan/tree structure as the FP64 entry points with
 * alg = PERM_ALG_GLYNN_DD / PERM_ALG_RYSER_DD.  A: device, n*n; out: device, 1 element.
 * Zero components are +0 in both halves.  PERM_EINVAL as perm_glynn / perm_ryser. */
int perm_glynn_dd(const perm_c128* A, int n, perm_dd_c128* out, void* stream);
int perm_ryser_dd(const perm_c128* A, int n, perm_dd_c128* out, void* stream);

/* ---- building blocks for multi-GPU partitions --------------------------------------- */
/* The paper's per-process contiguous ranges and one ALLREDUCE (PAPER.md:204, :217-219, :230,
 * :248-251, :261); here canonical units + a fixed reduction tree (bit-identical partitions). */
/* Sweep kernel only: unit partials for units [unit_lo, unit_hi) of plan(n, alg), written
 * to unit_partials[0 .. unit_hi-unit_lo) (device).  One kernel launch (plus a tiny
 * column-staging kernel).  Partials are unscaled. */
int perm_sweep_units(const perm_c128* A, int n, int alg, int64_t unit_lo, int64_t unit_hi,
                     perm_dd_c128* unit_partials, void* stream);

/* Experiments / profiling: the same sweep kernel on a NON-canonical plan of (n, alg) with the
 * given chunk_bits (5..12), leaf_bits (>= 0) and block_bits (0..7; dd: 0..6); units =
 * 2^(log2_terms - chunk_bits - leaf_bits - block_bits) (<= 2^40).  Lets a profiler run the
 * n = 50 kernel on short units (the canonical n = 50 unit is 2^32 terms, ~10 s per block).
 * Partials follow that plan's unit numbering; combining all of them gives Perm(A) up to
 * rounding (not bit-identical to the canonical plan). */
int perm_sweep_units_custom(const perm_c128* A, int n, int alg, int chunk_bits, int leaf_bits, int block_bits,
                            int64_t unit_lo, int64_t unit_hi, perm_dd_c128* unit_partials, void* stream);

/* Unscaled partial over Gray indices [lo, hi) (any lo <= hi <= #terms; ragged ends are
 * walked by the library).  partial: device, 1 element.  If [lo, hi) is an aligned
 * power-of-two block of units, the value equals that node of the canonical tree. */
int perm_glynn_range(const perm_c128* A, int n, uint64_t lo, uint64_t hi, perm_dd_c128* partial, void* stream);
int perm_ryser_range(const perm_c128* A, int n, uint64_t lo, uint64_t hi, perm_dd_c128* partial, void* stream);
/* The same for any algorithm code (FP64 or double-double). */
int perm_range(const perm_c128* A, int n, int alg, uint64_t lo, uint64_t hi, perm_dd_c128* partial, void* stream);

/* Canonical pairwise tree over `count` partials (device; zero-padded to a power of two:
 * node = left + right in double-double, left = lower indices).  Writes the unscaled root
 * to out_dd (device, may be NULL) and, if out (device) is not NULL, the final value:
 * root * 2^{-(n-1)} (alg = GLYNN) or root (RYSER), rounded to complex128. */
int perm_combine(const perm_dd_c128* partials, int64_t count, int n, int alg,
                 perm_c128* out, perm_dd_c128* out_dd, void* stream);

/* ---- batched (device pointers): one permanent per thread block ---------------------- */
/* Boson sampling needs many permanents of n x n submatrices of one unitary. */
/* out[b] = Perm(A_b) by Eq. (2), b < batch.  A: device, batch*n*n; out: device, batch.
 * batch == 0 is a no-op returning PERM_OK. */
int perm_glynn_batched(const perm_c128* A, int n, int64_t batch, perm_c128* out, void* stream);

/* out[b] = |Perm(A_b)|^2, the boson-sampling probability numerator P(S|T) ~ |Perm(U_ST)|^2
 * (FIG. 1), computed in the kernel from the rounded permanent as
 * fma(re, re, im * im).  out: device, batch doubles.  Otherwise as perm_glynn_batched. */
int perm_glynn_batched_abs2(const perm_c128* A, int n, int64_t batch, double* out, void* stream);

/* ---- summation-order experiments (precision lab, Table AV) --- */
/* out[0] = (partials[order[0]] + partials[order[1]] + ... + partials[order[count-1]]) added
 * SEQUENTIALLY in plain FP64 in the given order (each partial first rounded to hi + lo), times
 * 2^{-(n-1)} for Glynn algs.  With the chunk partials of a plain-mode sweep (e.g.
 * perm_sweep_units_custom with chunk_bits 5, leaf_bits 0, block_bits 0: 32-term chunks) and a
 * random permutation as `order`, this is the paper's "random order" summation at 32-term
 * granularity; the identity order is its "original order".  partials, order: device; order
 * must be a permutation of [0, count) (not checked: device data).  One thread adds (the
 * order IS the experiment); count < 1 or null pointers -> PERM_EINVAL. */
int perm_sum_ordered(const perm_dd_c128* partials, int64_t count, const int64_t* order, int n, int alg,
                     perm_c128* out, void* stream);

/* ---- host-buffer entry points (synchronous; copies inside) -------------------------- */
int perm_glynn_host(const perm_c128* A, int n, perm_c128* out);
int perm_ryser_host(const perm_c128* A, int n, perm_c128* out);
int perm_glynn_batched_host(const perm_c128* A, int n, int64_t batch, perm_c128* out);
int perm_glynn_batched_abs2_host(const perm_c128* A, int n, int64_t batch, double* out);

/* ---- instrumentation ------------------------------------------------------------------ */
/* Number of CUDA kernels this library has launched since it was loaded (all devices and
 * threads; the column-staging kernel counts).  bench.py reads it around its timed region. */
long long perm_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* PERMB200_H */
