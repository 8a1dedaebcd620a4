/*
 * perm_oracle.c — CPU ORACLE for the permanent hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code, header, table or helper with the
 * CUDA path under paper_1606_05836_b200/ (task rule ③); it is built separately with
 * `gcc -O2 -ffp-contract=off` (no FMA contraction, no fast-math) so every rounding
 * step below is the one written.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:<line>"):
 *   - the definition  perm(A) = sum_sigma prod_i a_{i,sigma(i)}        (P:60 notation)
 *     -> oracle_naive (n <= 10), double-double
 *   - BB/FG (Glynn), Eq. (2), P:66-68:
 *       perm(A) = 2^{-(N-1)} sum_delta (prod_k delta_k) prod_i sum_j delta_j a_ij,
 *       delta_1 = +1.  Reading R2: Gray/iter bit b <-> delta_{b+2}
 *       (1-based), a set bit means delta = -1.
 *     -> oracle_glynn_faithful: Alg. A2 loop body literally, row sums
 *        recomputed from scratch for every iter, ascending iter order, double-double.
 *     -> oracle_glynn_gray: the same sum walked in Gray-code order g -> G(g)=g^(g>>1),
 *        one +-2*column row-sum update per step (BASELINE.json north_star), all in
 *        double-double, contiguous ranges per host thread combined in range order.
 *   - Ryser, Eq. (1):  perm(A) = (-1)^N sum_S (-1)^{|S|} prod_i sum_{j in S} a_ij,
 *       bit b <-> column b+1 in S (1-based).  Per-term sign (-1)^{N-|S|} (reading R5).
 *     -> oracle_ryser_faithful (Alg. A1 body) and oracle_ryser_gray.
 *   - exact Gaussian-integer Glynn/Ryser in __int128 (overflow-checked) for integer
 *     matrices, with the exactness bounds used by the bit-exact parity class.
 *
 * All partial-sum entry points return the UNSCALED signed sum over iter/Gray index
 * range [lo, hi) as double-double (re_hi, re_lo, im_hi, im_lo); the caller applies
 * 2^{-(n-1)} (Glynn) exactly once (reading R3).
 *
 * Matrices are n*n complex128, row-major, interleaved (re, im): A[2*(i*n+j)] = Re a_ij.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ double-double */
typedef struct { double hi, lo; } dd;
typedef struct { dd re, im; } ddc;

static dd two_sum(double a, double b) {          /* Knuth: a + b = s + e exactly */
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  dd r = {s, e};
  return r;
}
static dd quick_two_sum(double a, double b) {    /* requires |a| >= |b| */
  double s = a + b;
  double e = b - (s - a);
  dd r = {s, e};
  return r;
}
static dd two_prod(double a, double b) {         /* a * b = p + e exactly (fma) */
  double p = a * b;
  double e = fma(a, b, -p);
  dd r = {p, e};
  return r;
}
static dd dd_add(dd a, dd b) {                   /* IEEE-style accurate dd addition */
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
static dd dd_neg(dd a) { dd r = {-a.hi, -a.lo}; return r; }
static dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
static dd dd_from(double a) { dd r = {a, 0.0}; return r; }
static dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
static ddc ddc_add(ddc a, ddc b) { ddc r = {dd_add(a.re, b.re), dd_add(a.im, b.im)}; return r; }
static ddc ddc_sub(ddc a, ddc b) { ddc r = {dd_sub(a.re, b.re), dd_sub(a.im, b.im)}; return r; }
static ddc ddc_mul(ddc a, ddc b) {               /* (ar + i ai)(br + i bi) */
  ddc r;
  r.re = dd_sub(dd_mul(a.re, b.re), dd_mul(a.im, b.im));
  r.im = dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re));
  return r;
}
static ddc ddc_zero(void) { ddc r = {{0, 0}, {0, 0}}; return r; }
static ddc ddc_from(double re, double im) { ddc r = {dd_from(re), dd_from(im)}; return r; }
static double ddc_abs_approx(ddc a) { return hypot(a.re.hi + a.re.lo, a.im.hi + a.im.lo); }
static void ddc_store(ddc a, double* out4) {
  out4[0] = a.re.hi; out4[1] = a.re.lo; out4[2] = a.im.hi; out4[3] = a.im.lo;
}

static int popcount64(uint64_t x) { int c = 0; while (x) { x &= x - 1; ++c; } return c; }
static int ctz64(uint64_t x) { int c = 0; while (!(x & 1)) { x >>= 1; ++c; } return c; }
static uint64_t gray(uint64_t g) { return g ^ (g >> 1); }

#define RE(A, n, i, j) ((A)[2 * ((size_t)(i) * (n) + (j))])
#define IM(A, n, i, j) ((A)[2 * ((size_t)(i) * (n) + (j)) + 1])

/* ------------------------------------------------------------------ naive (definition) */
/* sum over all permutations sigma of prod_i a_{i, sigma(i)}; recursive over rows,
 * lexicographic in sigma.  n <= 10 (10! * 10 complex dd products). */
static void naive_rec(const double* A, int n, int row, int* used, ddc prefix, ddc* acc) {
  if (row == n) { *acc = ddc_add(*acc, prefix); return; }
  for (int j = 0; j < n; ++j) {
    if (used[j]) continue;
    used[j] = 1;
    naive_rec(A, n, row + 1, used, ddc_mul(prefix, ddc_from(RE(A, n, row, j), IM(A, n, row, j))), acc);
    used[j] = 0;
  }
}

int oracle_naive(const double* A, int n, double* out4) {
  if (n < 1 || n > 10 || !A || !out4) return 1;
  int used[10] = {0};
  ddc acc = ddc_zero();
  naive_rec(A, n, 0, used, ddc_from(1.0, 0.0), &acc);
  ddc_store(acc, out4);
  return 0;
}

/* ------------------------------------------------------------------ faithful loops */
/* Alg. A2 body, iter in [lo, hi) ascending: delta from the bits of iter,
 * s_i = sum_j delta_j a_ij from scratch (Eq. 2 row sums), product over rows i = 1..N,
 * +/- by the parity of the number of -1 entries. */
int oracle_glynn_faithful(const double* A, int n, uint64_t lo, uint64_t hi, double* out4) {
  if (n < 1 || n > 62 || lo > hi || hi > (1ull << (n - 1)) || !A || !out4) return 1;
  ddc acc = ddc_zero();
  ddc* s = (ddc*)malloc(sizeof(ddc) * n);
  for (uint64_t it = lo; it < hi; ++it) {
    for (int i = 0; i < n; ++i) {
      s[i] = ddc_from(RE(A, n, i, 0), IM(A, n, i, 0));               /* delta_1 = +1 */
      for (int j = 1; j < n; ++j) {
        ddc a = ddc_from(RE(A, n, i, j), IM(A, n, i, j));
        s[i] = ((it >> (j - 1)) & 1) ? ddc_sub(s[i], a) : ddc_add(s[i], a);
      }
    }
    ddc p = s[0];
    for (int i = 1; i < n; ++i) p = ddc_mul(p, s[i]);
    acc = (popcount64(it) & 1) ? ddc_sub(acc, p) : ddc_add(acc, p);
  }
  free(s);
  ddc_store(acc, out4);
  return 0;
}

/* Alg. A1 body: S from the bits of iter, s_i = sum_{j in S} a_ij,
 * term sign (-1)^{N-|S|} (Eq. 1 with the (-1)^N folded in per term, reading R5). */
int oracle_ryser_faithful(const double* A, int n, uint64_t lo, uint64_t hi, double* out4) {
  if (n < 1 || n > 62 || lo > hi || hi > (1ull << n) || !A || !out4) return 1;
  ddc acc = ddc_zero();
  ddc* s = (ddc*)malloc(sizeof(ddc) * n);
  for (uint64_t it = lo; it < hi; ++it) {
    for (int i = 0; i < n; ++i) {
      s[i] = ddc_zero();
      for (int j = 0; j < n; ++j)
        if ((it >> j) & 1) s[i] = ddc_add(s[i], ddc_from(RE(A, n, i, j), IM(A, n, i, j)));
    }
    ddc p = s[0];
    for (int i = 1; i < n; ++i) p = ddc_mul(p, s[i]);
    acc = ((n - popcount64(it)) & 1) ? ddc_sub(acc, p) : ddc_add(acc, p);
  }
  free(s);
  ddc_store(acc, out4);
  return 0;
}

/* ------------------------------------------------------------------ Gray-code walks */
/* One host thread walks Gray indices g in [lo, hi): at g = lo the row sums are built
 * from the code G(lo); each later step flips the single code bit b = ctz(g)
 * (G(g) ^ G(g-1) = 2^b) and adds +-2*column (Glynn) or +-column (Ryser) to every
 * row sum.  Terms are signed by the parity of the code, accumulated in double-double.
 * l1 accumulates |term| (double, approximate) for the error bounds. */
typedef struct {
  const double* A; int n; int ryser; uint64_t lo, hi;
  ddc acc; double l1; double l1c;
} walk_job;

static void* walk_range(void* arg) {
  walk_job* w = (walk_job*)arg;
  const double* A = w->A;
  const int n = w->n;
  ddc acc = ddc_zero();
  double l1 = 0.0, l1c = 0.0;
  if (w->lo < w->hi) {
    ddc* s = (ddc*)malloc(sizeof(ddc) * n);
    /* rowabs_i = sum_j |a_ij|: the scale of the rounding error of any row sum of row i */
    double* rowabs = (double*)malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
      rowabs[i] = 0.0;
      for (int j = 0; j < n; ++j) rowabs[i] += hypot(RE(A, n, i, j), IM(A, n, i, j));
    }
    uint64_t G = gray(w->lo);
    for (int i = 0; i < n; ++i) {
      if (!w->ryser) {
        s[i] = ddc_from(RE(A, n, i, 0), IM(A, n, i, 0));
        for (int j = 1; j < n; ++j) {
          ddc a = ddc_from(RE(A, n, i, j), IM(A, n, i, j));
          s[i] = ((G >> (j - 1)) & 1) ? ddc_sub(s[i], a) : ddc_add(s[i], a);
        }
      } else {
        s[i] = ddc_zero();
        for (int j = 0; j < n; ++j)
          if ((G >> j) & 1) s[i] = ddc_add(s[i], ddc_from(RE(A, n, i, j), IM(A, n, i, j)));
      }
    }
    for (uint64_t g = w->lo;; ) {
      ddc p = s[0];
      for (int i = 1; i < n; ++i) p = ddc_mul(p, s[i]);
      int neg = w->ryser ? ((n - popcount64(G)) & 1) : (popcount64(G) & 1);
      acc = neg ? ddc_sub(acc, p) : ddc_add(acc, p);
      const double ap = ddc_abs_approx(p);
      l1 += ap;
      /* componentwise error scale: |term| * sum_i rowabs_i / |s_i| (first-order relative
       * error of the product when each row sum carries an error ~ u * rowabs_i) */
      if (ap > 0.0) {
        double kappa = 0.0;
        for (int i = 0; i < n; ++i) kappa += rowabs[i] / ddc_abs_approx(s[i]);
        l1c += ap * kappa;
      }
      if (++g >= w->hi) break;
      const int b = ctz64(g);
      const uint64_t Gn = gray(g);
      const int now_set = (int)((Gn >> b) & 1);
      const int j = w->ryser ? b : b + 1;
      for (int i = 0; i < n; ++i) {
        ddc a = ddc_from(RE(A, n, i, j), IM(A, n, i, j));
        if (!w->ryser) a = ddc_add(a, a);                 /* 2 a_ij (exact) */
        /* Glynn: set bit = delta becomes -1 -> subtract; Ryser: set bit = column joins S -> add */
        const int subtract = w->ryser ? !now_set : now_set;
        s[i] = subtract ? ddc_sub(s[i], a) : ddc_add(s[i], a);
      }
      G = Gn;
    }
    free(s);
    free(rowabs);
  }
  w->acc = acc;
  w->l1 = l1;
  w->l1c = l1c;
  return 0;
}

static int walk_threaded(const double* A, int n, int ryser, uint64_t lo, uint64_t hi, int threads,
                         double* out4, double* l1_out, double* l1c_out) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  uint64_t len = hi - lo;
  if ((uint64_t)threads > len) threads = len ? (int)len : 1;
  walk_job* jobs = (walk_job*)calloc(threads, sizeof(walk_job));
  pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t].A = A; jobs[t].n = n; jobs[t].ryser = ryser;
    jobs[t].lo = lo + (uint64_t)((unsigned __int128)len * t / threads);
    jobs[t].hi = lo + (uint64_t)((unsigned __int128)len * (t + 1) / threads);
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], 0, walk_range, &jobs[t]);
  walk_range(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], 0);
  ddc acc = ddc_zero();
  double l1 = 0.0, l1c = 0.0;
  for (int t = 0; t < threads; ++t) { acc = ddc_add(acc, jobs[t].acc); l1 += jobs[t].l1; l1c += jobs[t].l1c; }
  ddc_store(acc, out4);
  if (l1_out) *l1_out = l1;
  if (l1c_out) *l1c_out = l1c;
  free(jobs); free(tid);
  return 0;
}

int oracle_glynn_gray(const double* A, int n, uint64_t lo, uint64_t hi, int threads, double* out4, double* l1) {
  if (n < 1 || n > 64 || lo > hi || hi > (1ull << (n - 1)) || !A || !out4) return 1;
  return walk_threaded(A, n, 0, lo, hi, threads, out4, l1, 0);
}

int oracle_ryser_gray(const double* A, int n, uint64_t lo, uint64_t hi, int threads, double* out4, double* l1) {
  if (n < 1 || n > 63 || lo > hi || hi > (1ull << n) || !A || !out4) return 1;
  return walk_threaded(A, n, 1, lo, hi, threads, out4, l1, 0);
}

/* Same walks, also returning l1c = sum_terms |term| * sum_i (sum_j |a_ij|) / |s_i|, the
 * componentwise error scale used by the parity bound of DESIGN.md reading R10b. */
int oracle_gray_ex(const double* A, int n, int ryser, uint64_t lo, uint64_t hi, int threads, double* out4,
                   double* l1, double* l1c) {
  if (n < 1 || !A || !out4 || lo > hi) return 1;
  if (!ryser && (n > 64 || hi > (1ull << (n - 1)))) return 1;
  if (ryser && (n > 63 || hi > (1ull << n))) return 1;
  return walk_threaded(A, n, ryser, lo, hi, threads, out4, l1, l1c);
}

/* ------------------------------------------------------------------ exact Gaussian integers */
/* Integer matrix entries (re, im as int64).  Glynn numerator / Ryser sum evaluated
 * exactly in __int128 with overflow checks.  Also returns, for the bit-exact parity
 * class, l1 = sum over terms of (|Re t| + |Im t|) and maxprod = max over terms of
 * prod_i max(1, |Re s_i| + |Im s_i|), a bound on every partial product of row sums in
 * any order (saturating at 2^126).  Return 2 on overflow. */
typedef __int128 i128;
typedef struct { i128 re, im; } ci128;

static int add_ovf(i128 a, i128 b, i128* r) { return __builtin_add_overflow(a, b, r); }
static int mul_ovf(i128 a, i128 b, i128* r) { return __builtin_mul_overflow(a, b, r); }
static int cmul_exact(ci128 a, ci128 b, ci128* r) {
  i128 t1, t2, t3, t4;
  if (mul_ovf(a.re, b.re, &t1) || mul_ovf(a.im, b.im, &t2) || mul_ovf(a.re, b.im, &t3) || mul_ovf(a.im, b.re, &t4))
    return 1;
  if (__builtin_sub_overflow(t1, t2, &r->re) || add_ovf(t3, t4, &r->im)) return 1;
  return 0;
}
static i128 iabs128(i128 x) { return x < 0 ? -x : x; }

static void store_i128(i128 v, int64_t* out2) {  /* two's complement split: hi (signed), lo (unsigned bits) */
  out2[0] = (int64_t)(v >> 64);
  out2[1] = (int64_t)(uint64_t)v;
}

int oracle_exact_int(const int64_t* Are, const int64_t* Aim, int n, int ryser,
                     int64_t* out_re2, int64_t* out_im2, int64_t* l1_2, double* maxprod) {
  if (n < 1 || n > 40 || !Are || !Aim) return 1;
  const uint64_t T = ryser ? (1ull << n) : (1ull << (n - 1));
  ci128* s = (ci128*)calloc(n, sizeof(ci128));
  ci128 acc = {0, 0};
  i128 l1 = 0;
  const i128 cap = ((i128)1) << 126;
  i128 maxp = 0;
  int rc = 0;
  for (uint64_t g = 0; g < T && !rc; ++g) {
    uint64_t G = gray(g);
    if (g == 0) {
      for (int i = 0; i < n; ++i) {          /* G(0) = 0: Glynn all delta = +1, Ryser S empty */
        s[i].re = 0;
        s[i].im = 0;
        if (!ryser)
          for (int j = 0; j < n; ++j) { s[i].re += Are[i * n + j]; s[i].im += Aim[i * n + j]; }
      }
    } else {
      const int b = ctz64(g);
      const int now_set = (int)((G >> b) & 1);
      const int j = ryser ? b : b + 1;
      const int sgn = ryser ? (now_set ? 1 : -1) : (now_set ? -1 : 1);
      const int mult = ryser ? 1 : 2;
      for (int i = 0; i < n; ++i) {
        s[i].re += (i128)sgn * mult * Are[i * n + j];
        s[i].im += (i128)sgn * mult * Aim[i * n + j];
      }
    }
    ci128 p = s[0];
    i128 bound = iabs128(s[0].re) + iabs128(s[0].im);
    if (bound < 1) bound = 1;
    for (int i = 1; i < n && !rc; ++i) {
      if (cmul_exact(p, s[i], &p)) rc = 2;
      i128 f = iabs128(s[i].re) + iabs128(s[i].im);
      if (f < 1) f = 1;
      if (bound > cap / f) bound = cap; else bound *= f;
    }
    if (rc) break;
    if (bound > maxp) maxp = bound;
    int neg = ryser ? ((n - popcount64(G)) & 1) : (popcount64(G) & 1);
    if (neg) { p.re = -p.re; p.im = -p.im; }
    if (add_ovf(acc.re, p.re, &acc.re) || add_ovf(acc.im, p.im, &acc.im)) rc = 2;
    if (add_ovf(l1, iabs128(p.re) + iabs128(p.im), &l1)) rc = 2;
  }
  free(s);
  if (rc) return rc;
  if (out_re2) store_i128(acc.re, out_re2);
  if (out_im2) store_i128(acc.im, out_im2);
  if (l1_2) store_i128(l1, l1_2);
  if (maxprod) *maxprod = (double)maxp;
  return 0;
}

/* ------------------------------------------------------------------ dd helpers for callers */
/* Exact dd sum of two dd values (used by tests to combine range partials the oracle's way). */
void oracle_dd_add(const double* a4, const double* b4, double* out4) {
  ddc a = {{a4[0], a4[1]}, {a4[2], a4[3]}};
  ddc b = {{b4[0], b4[1]}, {b4[2], b4[3]}};
  ddc_store(ddc_add(a, b), out4);
}
