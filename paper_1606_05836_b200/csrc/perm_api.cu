// perm_api.cu — C ABI of libpermb200.so (declared in include/permb200.h): argument
// checks, the canonical plan, constant-slot fencing, workspace, the combine kernel.
//
// PAPER.md: the per-process partial sums and the single ALLREDUCE followed by the final
// division (Alg. A2) become: unit partials (sweep kernel) -> canonical
// pairwise tree (combine kernel) -> x 2^-(n-1) exactly once (reading R3).
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <string>

#include "../../include/permb200.h"
#include "perm_registry.h"
#include "perm_kernels_wsplit.cuh"   // wsplit_launches

using namespace permb200;

namespace {

thread_local std::string g_last_error;

// Kernels this library has launched (all devices, all threads): perm_launch_count().
std::atomic<long long> g_launches{0};
inline void note_launch(int k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return PERM_ECUDA;
}

#define CUDA_TRY(expr, where)                       \
  do {                                              \
    cudaError_t e_ = (expr);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

struct DeviceSlots {
  std::mutex mu;
  bool init = false;
  int next = 0;
  cudaEvent_t ev[kSlots];
  bool used[kSlots] = {};
};
DeviceSlots g_slots[64];

// Per-device stream-ordered memory pool for the library's temporary workspaces (staging table,
// unit partials, host-entry copies).  The default pool's release threshold is 0: it returns
// its memory at every synchronisation, so the next cudaMallocAsync maps fresh pages -- measured
// 4.2 ms for a synchronous n = 20 call (tools/latency_probe.py).  This pool keeps up to
// 256 MiB cached instead; concurrent streams allocate from it safely.
struct DevicePool {
  std::once_flag once;
  cudaMemPool_t pool = nullptr;
  cudaError_t err = cudaSuccess;
};
DevicePool g_pools[64];

cudaError_t ws_alloc(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  DevicePool& dp = g_pools[dev];
  std::call_once(dp.once, [&] {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    dp.err = cudaMemPoolCreate(&dp.pool, &props);
    if (dp.err == cudaSuccess) {
      uint64_t thr = 256ull << 20;
      dp.err = cudaMemPoolSetAttribute(dp.pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  if (dp.err != cudaSuccess) return dp.err;
  // under stream capture: a plain stream-ordered allocation becomes a graph memory node
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess) return e;
  if (cs != cudaStreamCaptureStatusNone) return cudaMallocAsync(p, bytes, st);
  return cudaMallocFromPoolAsync(p, bytes, dp.pool, st);
}

std::once_flag g_tables_once;
constexpr int kAlgs = 8;
SweepLauncher g_sweep[kAlgs][kNMax + 1];   // [alg][n]: GLYNN, RYSER, GLYNN_DD, RYSER_DD, GLYNN_PLAIN, RYSER_PLAIN, GLYNN_SEP, RYSER_SEP
SweepLauncher g_small[kAlgs][kNMax + 1];   // small-n shared-memory-column sweep (m <= kSmallLog2)
FusedLauncher g_small_fused[kAlgs][kNMax + 1];   // the same + grid barrier + combine, one launch
SweepLauncher g_split[kAlgs][kNMax + 1];   // 2-lane row split (perm_kernels_split.cuh): fallback
SweepLauncher g_wsplit[kAlgs][kNMax + 1];  // warp-pair row split (perm_kernels_wsplit.cuh): n >= 52
BatchedLauncher g_batched[kNMax + 1];

void init_tables() {
  std::call_once(g_tables_once, [] {
    register_glynn_a(g_sweep[kGlynn]);
    register_glynn_b(g_sweep[kGlynn]);
    register_glynn_c(g_sweep[kGlynn]);
    register_glynn_d(g_sweep[kGlynn]);
    register_ryser_a(g_sweep[kRyser]);
    register_ryser_b(g_sweep[kRyser]);
    register_ryser_c(g_sweep[kRyser]);
    register_ryser_d(g_sweep[kRyser]);
    register_plain_glynn_a(g_sweep[PERM_ALG_GLYNN_PLAIN]);
    register_plain_glynn_b(g_sweep[PERM_ALG_GLYNN_PLAIN]);
    register_plain_glynn_c(g_sweep[PERM_ALG_GLYNN_PLAIN]);
    register_plain_glynn_d(g_sweep[PERM_ALG_GLYNN_PLAIN]);
    register_plain_ryser_a(g_sweep[PERM_ALG_RYSER_PLAIN]);
    register_plain_ryser_b(g_sweep[PERM_ALG_RYSER_PLAIN]);
    register_plain_ryser_c(g_sweep[PERM_ALG_RYSER_PLAIN]);
    register_plain_ryser_d(g_sweep[PERM_ALG_RYSER_PLAIN]);
    register_dd_glynn_a(g_sweep[PERM_ALG_GLYNN_DD]);
    register_dd_glynn_b(g_sweep[PERM_ALG_GLYNN_DD]);
    register_dd_ryser_a(g_sweep[PERM_ALG_RYSER_DD]);
    register_dd_ryser_b(g_sweep[PERM_ALG_RYSER_DD]);
    register_sep_glynn_a(g_sweep[PERM_ALG_GLYNN_SEP]);
    register_sep_glynn_b(g_sweep[PERM_ALG_GLYNN_SEP]);
    register_sep_ryser_a(g_sweep[PERM_ALG_RYSER_SEP]);
    register_sep_ryser_b(g_sweep[PERM_ALG_RYSER_SEP]);
    register_small(g_small);
    register_small_fused(g_small_fused);
    register_split_large(g_split);
    register_wsplit_a(g_wsplit);
    register_wsplit_b(g_wsplit);
    register_batched_a(g_batched);
    register_batched_b(g_batched);
  });
}

int ceil_log2(long long v) {
  int k = 0;
  while ((1LL << k) < v) ++k;
  return k;
}

bool valid_alg(int alg) { return alg >= PERM_ALG_GLYNN && alg <= PERM_ALG_RYSER_SEP; }
// alg = formula (bit 0: 0 Glynn, 1 Ryser) + 2 * arithmetic mode (0 FP64, 1 dd, 2 plain FP64,
// 3 separate addition)
bool is_glynn(int alg) { return (alg & 1) == 0; }
bool is_plain(int alg) { return alg == PERM_ALG_GLYNN_PLAIN || alg == PERM_ALG_RYSER_PLAIN; }
bool is_dd(int alg) { return alg == PERM_ALG_GLYNN_DD || alg == PERM_ALG_RYSER_DD; }
bool is_sep(int alg) { return alg == PERM_ALG_GLYNN_SEP || alg == PERM_ALG_RYSER_SEP; }
// accumulation mode of the FP64 sweep / combine (perm_kernels.cuh kComp / kPlain / kSep)
int mode_of(int alg) { return is_plain(alg) ? kPlain : is_sep(alg) ? kSep : kComp; }
// the one subtraction of separate addition: even - odd, times (-1)^n for Ryser (Eq. (1))
int sep_sign(int n, int alg) { return !is_sep(alg) ? 0 : (!is_glynn(alg) && (n & 1)) ? -1 : 1; }

// Lanes per chunk (leaf) of the FP64 sweep: 2 for n >= kSplitLargeN in the compensated mode (4n
// row-sum registers do not fit one thread), else 1.  Two lanes = the same lane of a warp pair
// (perm_kernels_wsplit.cuh: constant-bank columns, half products exchanged through shared
// memory), or -- custom plans with block_bits < 5 -- two adjacent lanes of one warp
// (perm_kernels_split.cuh).  Small n (m <= kSmallLog2) walks one thread per chunk: the
// 4-lane split measured slower on M1 (n = 20: 26.7 / 47.2 us per Glynn / Ryser call against
// 18.5 / 22.6 us for one lane, profiles/r02_m1_latency_split4.log) -- at ~1 warp per scheduler the
// FP64 pipe, not the per-thread chain, bounds it, and the split adds shuffles and a combine cmul.
constexpr int kSplitLargeN = 52;
int split_lanes(int n, int alg) {
  if (is_dd(alg)) return 1;
  const int m = is_glynn(alg) ? n - 1 : n;
  if (m <= kSmallLog2) return 1;
  if (n >= kSplitLargeN && mode_of(alg) == kComp) return 2;
  return 1;
}
int lanes_log2(int R) { return R == 2 ? 1 : 0; }

void make_plan(int n, int alg, perm_plan_t* p) {
  const int m = is_glynn(alg) ? n - 1 : n;
  const int R = split_lanes(n, alg);
  // FP64 sweep: up to 128 threads per unit (row sums in registers; leaves of R lanes); dd
  // sweep: up to 64 (row sums in shared memory, 32 B per row per thread).
  const int wmax = is_dd(alg) ? 6 : 7 - lanes_log2(R);
  int wbits, c, ubits, lam;
  if (m < 5) {
    wbits = 0; c = m; ubits = 0; lam = 0;      // tiny: one thread, generic walk
  } else {
    wbits = m - 5 < wmax ? m - 5 : wmax;
    const int rem = m - wbits;
    int ct = ceil_log2(33LL * n);              // chunk build <= ~1% of the sweep's FP64 ops
    if (ct < 5) ct = 5;
    if (ct > kCMax) ct = kCMax;
    const int ub_min = rem - 5 < 7 ? rem - 5 : 7;
    c = rem - ub_min < ct ? rem - ub_min : ct;
    if (c < 5) c = 5;
    // Units: 2^17 up to 2^39 terms; beyond, 2^(m-29) (capped at 2^22) so a unit stays ~2^29
    // terms (~3 s per wave at n = 50).  Long units make every wave one lock-step phase: the
    // two co-resident blocks of an SM build their chunks at the same moments, and a single
    // 2^32-term wave measured 0.83 of the FP64 issue rate against 0.87 for 8 short waves
    // (tools/profile_sweep.py --custom, 2026-10-20).  Short units also make checkpoint
    // segments and multi-GPU shares finer.
    int ucap = m - 29;
    if (ucap < 17) ucap = 17;
    if (ucap > 22) ucap = 22;
    ubits = rem - c < ucap ? rem - c : ucap;
    lam = rem - c - ubits;
  }
  p->n = n; p->alg = alg;
  p->log2_terms = m; p->chunk_bits = c; p->leaf_bits = lam; p->block_bits = wbits; p->unit_bits = ubits;
  p->lanes = R;
  p->units = 1LL << ubits;
  p->unit_terms = 1ULL << (m - ubits);
}

bool valid_n(int n) { return n >= 1 && n <= kNMax; }
// Ryser has 2^n terms: n = 64 would overflow the 64-bit Gray index.  The separate-addition
// precision mode is compiled for n <= kSepNMax (the paper's Table AV stops at N = 32).
constexpr int kSepNMax = 40;
bool valid_n_alg(int n, int alg) {
  return valid_alg(alg) && valid_n(n) && (is_glynn(alg) ? true : n <= 63) && (!is_sep(alg) || n <= kSepNMax);
}

// Canonical tree over `count` partials (zero-padded to P = 2^k): one block of up to 1024
// threads; thread t reduces the aligned segment [t*S, (t+1)*S) with the binary-counter
// method (node = left + right), then a pairwise tree over the segment roots in smem.
__global__ void combine_kernel(const Dd2* __restrict__ parts, int64_t count, int64_t P, int do_scale,
                               int scale_exp, double2* out, Dd2* out_dd, int scale_dd, int mode, int sep) {
  __shared__ Dd2 red[1024];
  const int64_t T = P < 1024 ? P : 1024;
  const int64_t S = P / T;
  const int tid = threadIdx.x;
  if (tid < T) {
    Dd2 stack[40];
    int top_level = 0;
    for (int64_t k = 0; k < S; ++k) {
      const int64_t idx = tid * S + k;
      Dd2 v = idx < count ? parts[idx] : Dd2{0.0, 0.0, 0.0, 0.0};
      int lvl = 0;
      for (int64_t kk = k; kk & 1; kk >>= 1) {
        v = mode == kPlain ? plain2_add(stack[lvl], v) : mode == kSep ? sep2_add(stack[lvl], v) : dd2_add(stack[lvl], v);
        ++lvl;
      }
      stack[lvl] = v;
      if (lvl > top_level) top_level = lvl;
    }
    red[tid] = stack[top_level];
  }
  __syncthreads();
  for (int64_t o = 1; o < T; o <<= 1) {
    if ((tid & (2 * o - 1)) == 0 && tid + o < T)
      red[tid] = mode == kPlain ? plain2_add(red[tid], red[tid + o])
                 : mode == kSep ? sep2_add(red[tid], red[tid + o]) : dd2_add(red[tid], red[tid + o]);
    __syncthreads();
  }
  if (tid == 0) finish_root(red[0], FinishArgs{out, out_dd, do_scale, scale_exp, scale_dd, sep});
}

// Sequential plain-FP64 sum of `count` partials in a caller-given order (the paper's "original"
// and "random" summation orders, Table AV): the order is the point, so the additions
// form ONE dependent chain.  Warp 1 gathers batches of 1024 partials (rounded hi + lo) into a
// double-buffered shared-memory tile while thread 0 adds the previous batch in order.
__global__ void __launch_bounds__(64) ordered_sum_kernel(const Dd2* __restrict__ parts,
                                                         const int64_t* __restrict__ order, int64_t count,
                                                         FinishArgs f) {
  constexpr int B = 1024;
  __shared__ double2 buf[2][B];
  const int tid = threadIdx.x;
  const int64_t nb = (count + B - 1) / B;
  auto load = [&](int64_t b, int slot) {
    for (int k = tid - 32; k < B; k += 32) {
      const int64_t idx = b * B + k;
      double2 v = make_double2(0.0, 0.0);
      if (idx < count) {
        PERM_CHECK(order[idx] >= 0 && order[idx] < count);
        const Dd2 p = parts[order[idx]];
        v = make_double2(__dadd_rn(p.re_hi, p.re_lo), __dadd_rn(p.im_hi, p.im_lo));
      }
      buf[slot][k] = v;
    }
  };
  if (tid >= 32 && nb > 0) load(0, 0);
  __syncthreads();
  double sr = 0.0, si = 0.0;
  for (int64_t b = 0; b < nb; ++b) {
    if (tid >= 32) {
      if (b + 1 < nb) load(b + 1, (int)((b + 1) & 1));
    } else if (tid == 0) {
      const int m = (int)(count - b * B < B ? count - b * B : B);
      const double2* t = buf[b & 1];
      for (int k = 0; k < m; ++k) { sr = __dadd_rn(sr, t[k].x); si = __dadd_rn(si, t[k].y); }
    }
    __syncthreads();
  }
  if (tid == 0) finish_root(Dd2{sr, 0.0, si, 0.0}, f);
}

int run_combine(const Dd2* parts, int64_t count, int n, int alg, double2* out, Dd2* out_dd, cudaStream_t st,
                int scale_dd = 0) {
  int64_t P = 1;
  while (P < count) P <<= 1;
  combine_kernel<<<1, 1024, 0, st>>>(parts, count, P, is_glynn(alg), -(n - 1), out, out_dd, scale_dd, mode_of(alg),
                                     sep_sign(n, alg));
  CUDA_TRY(cudaGetLastError(), "combine_kernel launch");
  note_launch();
  return PERM_OK;
}

// Sweep over units [u_lo, u_hi) clipped to Gray indices [lo, hi); partials -> out[0..).
int run_sweep(const perm_c128* A, const perm_plan_t& P, int64_t u_lo, int64_t u_hi, uint64_t lo, uint64_t hi,
              Dd2* out, double2* staging, cudaStream_t st) {
  init_tables();
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev < 0 || dev >= 64) { g_last_error = "device ordinal >= 64"; return PERM_ECUDA; }
  SweepArgs a;
  a.A = reinterpret_cast<const double2*>(A);
  a.unit_out = out;
  a.lo = lo; a.hi = hi;
  a.unit_lo = u_lo;
  a.c = P.chunk_bits; a.lam = P.leaf_bits; a.block_bits = P.block_bits;
  a.zero = 0;
  const bool wsplit = P.lanes > 1 && g_wsplit[P.alg][P.n] && P.block_bits >= 5 && P.block_bits <= 6;
  if (P.lanes > 1 && !wsplit && g_split[P.alg][P.n]) {
    // 2-lane row split (plans with fewer than 32 leaves per unit): columns from shared memory,
    // capturable, no constant slot
    a.slot = 0; a.col_base = 0;
    CUDA_TRY(g_split[P.alg][P.n](a, u_hi - u_lo, staging, st), "split sweep launch");
    note_launch();
    return PERM_OK;
  }
  if (!is_dd(P.alg) && P.log2_terms <= kSmallLog2 && g_small[P.alg][P.n]) {
    // small n: columns from shared memory, no staging / constant slot / fencing
    a.slot = 0; a.col_base = 0;
    CUDA_TRY(g_small[P.alg][P.n](a, u_hi - u_lo, staging, st), "small sweep launch");
    note_launch();
    return PERM_OK;
  }
  {
    // The constant-slot path fences the slot with events recorded outside any graph; it is
    // not capturable.  Fail loudly (small n, the dd mode and the batched kernel are).
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
    if (cs != cudaStreamCaptureStatusNone && !is_dd(P.alg)) {
      g_last_error = "stream capture: the constant-memory column path (more than 2^21 terms) cannot be "
                     "captured in a CUDA graph; capture small n, the dd mode or perm_glynn_batched";
      return PERM_ECUDA;
    }
  }
  if (is_dd(P.alg)) {            // the dd sweep reads its columns from A: no constant slot
    a.slot = 0; a.col_base = 0;
    CUDA_TRY(g_sweep[P.alg][P.n](a, u_hi - u_lo, staging, st), "dd sweep launch");
    note_launch();
    return PERM_OK;
  }
  DeviceSlots& ds = g_slots[dev];
  std::lock_guard<std::mutex> lk(ds.mu);
  if (!ds.init) {
    for (int k = 0; k < kSlots; ++k) CUDA_TRY(cudaEventCreateWithFlags(&ds.ev[k], cudaEventDisableTiming), "cudaEventCreate");
    ds.init = true;
  }
  const int slot = ds.next;
  ds.next = (ds.next + 1) % kSlots;
  // the constant slot may still be read by an earlier sweep on another stream: fence it
  if (ds.used[slot]) CUDA_TRY(cudaStreamWaitEvent(st, ds.ev[slot], 0), "cudaStreamWaitEvent");
  a.slot = slot;
  a.col_base = slot * kTabRows * kNMax;
  if (wsplit) {
    // warp-pair row split: constant-bank columns like the one-lane sweep (+ ragged end units)
    CUDA_TRY(g_wsplit[P.alg][P.n](a, u_hi - u_lo, staging, st), "warp-split sweep launch");
    note_launch(wsplit_launches(a, u_hi - u_lo));
  } else {
    CUDA_TRY(g_sweep[P.alg][P.n](a, u_hi - u_lo, staging, st), "sweep launch");
    note_launch(a.c >= kMinFastC ? 2 : 1);   // column staging (fast path) + sweep
  }
  CUDA_TRY(cudaEventRecord(ds.ev[slot], st), "cudaEventRecord");
  ds.used[slot] = true;
  return PERM_OK;
}

constexpr size_t kStagingBytes = sizeof(double2) * kTabRows * kNMax;

// out (complex128) and/or out_dd (scaled double-double) of the full permanent.
int full_perm(const perm_c128* A, int n, int alg, perm_c128* out, cudaStream_t st, perm_dd_c128* out_dd = nullptr) {
  if (!A || (!out && !out_dd) || !valid_n_alg(n, alg)) return PERM_EINVAL;
  perm_plan_t P;
  make_plan(n, alg, &P);
  void* ws = nullptr;
  const size_t bytes = kStagingBytes + sizeof(Dd2) * (size_t)P.units;
  CUDA_TRY(ws_alloc(&ws, bytes, st), "workspace alloc");
  double2* staging = static_cast<double2*>(ws);
  Dd2* parts = reinterpret_cast<Dd2*>(static_cast<char*>(ws) + kStagingBytes);
  const uint64_t T = 1ULL << P.log2_terms;
  int rc = -1;
  init_tables();
  if (P.lanes == 1 && !is_dd(alg) && P.log2_terms <= kSmallLog2 && g_small_fused[alg][n] &&
      P.units <= (8LL << P.block_bits)) {
    // small n: sweep + combine in one cooperative launch (same bits as the two-kernel path)
    SweepArgs a;
    a.A = reinterpret_cast<const double2*>(A);
    a.unit_out = parts;
    a.lo = 0; a.hi = T;
    a.unit_lo = 0;
    a.c = P.chunk_bits; a.lam = P.leaf_bits; a.block_bits = P.block_bits;
    a.slot = 0; a.col_base = 0; a.zero = 0;
    const FinishArgs f{reinterpret_cast<double2*>(out), reinterpret_cast<Dd2*>(out_dd), is_glynn(alg) ? 1 : 0,
                       -(n - 1), 1, sep_sign(n, alg)};
    cudaError_t le = g_small_fused[alg][n](a, f, P.units, st);
    if (le == cudaSuccess) {
      rc = PERM_OK;
      note_launch();
    } else if (le != cudaErrorCooperativeLaunchTooLarge) {
      rc = cuda_fail(le, "fused small launch");
    }
    // cudaErrorCooperativeLaunchTooLarge: the grid cannot be co-resident (another kernel owns
    // the SMs' registers / shared memory): the same sweep + combine as two launches below
  }
  if (rc == -1) {
    rc = run_sweep(A, P, 0, P.units, 0, T, parts, staging, st);
    if (rc == PERM_OK)
      rc = run_combine(parts, P.units, n, alg, reinterpret_cast<double2*>(out), reinterpret_cast<Dd2*>(out_dd), st, 1);
  }
  cudaError_t e = cudaFreeAsync(ws, st);
  if (rc == PERM_OK && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return rc;
}

int range_perm(const perm_c128* A, int n, int alg, uint64_t lo, uint64_t hi, perm_dd_c128* partial, cudaStream_t st) {
  if (!A || !partial || !valid_n_alg(n, alg)) return PERM_EINVAL;
  perm_plan_t P;
  make_plan(n, alg, &P);
  const uint64_t T = 1ULL << P.log2_terms;
  if (lo > hi || hi > T) return PERM_EINVAL;
  if (lo == hi) {
    CUDA_TRY(cudaMemsetAsync(partial, 0, sizeof(perm_dd_c128), st), "cudaMemsetAsync");
    return PERM_OK;
  }
  const int64_t u_lo = (int64_t)(lo / P.unit_terms);
  const int64_t u_hi = (int64_t)((hi + P.unit_terms - 1) / P.unit_terms);
  void* ws = nullptr;
  const size_t bytes = kStagingBytes + sizeof(Dd2) * (size_t)(u_hi - u_lo);
  CUDA_TRY(ws_alloc(&ws, bytes, st), "workspace alloc");
  double2* staging = static_cast<double2*>(ws);
  Dd2* parts = reinterpret_cast<Dd2*>(static_cast<char*>(ws) + kStagingBytes);
  int rc = run_sweep(A, P, u_lo, u_hi, lo, hi, parts, staging, st);
  if (rc == PERM_OK) rc = run_combine(parts, u_hi - u_lo, n, alg, nullptr, reinterpret_cast<Dd2*>(partial), st);
  cudaError_t e = cudaFreeAsync(ws, st);
  if (rc == PERM_OK && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return rc;
}

void make_batched_plan(int n, int* block_bits, int* c, int* lam) {
  const int m = n - 1;
  if (m < 5) { *block_bits = 0; *c = m; *lam = 0; return; }
  int wb = m - 5 < 7 ? m - 5 : 7;
  const int rem = m - wb;
  int cc = rem < kCMax ? rem : kCMax;
  *block_bits = wb; *c = cc; *lam = rem - cc;
}

}  // namespace

extern "C" {

int perm_max_n(void) { return kNMax; }

const char* perm_strerror(int code) {
  switch (code) {
    case PERM_OK: return "ok";
    case PERM_EINVAL: return "invalid argument";
    case PERM_ECUDA: return g_last_error.empty() ? "CUDA error" : g_last_error.c_str();
    case PERM_ENOTIMPL: return "not implemented";
    default: return "unknown status";
  }
}

int perm_plan(int n, int alg, perm_plan_t* plan) {
  if (!plan || !valid_n_alg(n, alg)) return PERM_EINVAL;
  make_plan(n, alg, plan);
  return PERM_OK;
}

int perm_glynn(const perm_c128* A, int n, perm_c128* out, void* stream) {
  return full_perm(A, n, PERM_ALG_GLYNN, out, static_cast<cudaStream_t>(stream));
}

int perm_ryser(const perm_c128* A, int n, perm_c128* out, void* stream) {
  return full_perm(A, n, PERM_ALG_RYSER, out, static_cast<cudaStream_t>(stream));
}

int perm_glynn_dd(const perm_c128* A, int n, perm_dd_c128* out, void* stream) {
  if (!out) return PERM_EINVAL;
  return full_perm(A, n, PERM_ALG_GLYNN_DD, nullptr, static_cast<cudaStream_t>(stream), out);
}

int perm_ryser_dd(const perm_c128* A, int n, perm_dd_c128* out, void* stream) {
  if (!out) return PERM_EINVAL;
  return full_perm(A, n, PERM_ALG_RYSER_DD, nullptr, static_cast<cudaStream_t>(stream), out);
}

int perm_range(const perm_c128* A, int n, int alg, uint64_t lo, uint64_t hi, perm_dd_c128* partial, void* stream) {
  return range_perm(A, n, alg, lo, hi, partial, static_cast<cudaStream_t>(stream));
}

int perm_sweep_units(const perm_c128* A, int n, int alg, int64_t unit_lo, int64_t unit_hi,
                     perm_dd_c128* unit_partials, void* stream) {
  if (!A || !unit_partials || !valid_n_alg(n, alg)) return PERM_EINVAL;
  perm_plan_t P;
  make_plan(n, alg, &P);
  if (unit_lo < 0 || unit_lo > unit_hi || unit_hi > P.units) return PERM_EINVAL;
  if (unit_lo == unit_hi) return PERM_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* ws = nullptr;
  CUDA_TRY(ws_alloc(&ws, kStagingBytes, st), "workspace alloc");
  const uint64_t lo = (uint64_t)unit_lo * P.unit_terms, hi = (uint64_t)unit_hi * P.unit_terms;
  int rc = run_sweep(A, P, unit_lo, unit_hi, lo, hi, reinterpret_cast<Dd2*>(unit_partials), static_cast<double2*>(ws), st);
  cudaError_t e = cudaFreeAsync(ws, st);
  if (rc == PERM_OK && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return rc;
}

int perm_sweep_units_custom(const perm_c128* A, int n, int alg, int chunk_bits, int leaf_bits, int block_bits,
                            int64_t unit_lo, int64_t unit_hi, perm_dd_c128* unit_partials, void* stream) {
  if (!A || !unit_partials || !valid_n_alg(n, alg)) return PERM_EINVAL;
  perm_plan_t P;
  make_plan(n, alg, &P);
  const int wmax = is_dd(alg) ? 6 : 7 - lanes_log2(P.lanes);
  if (chunk_bits < kMinFastC || chunk_bits > kCMax || leaf_bits < 0 || block_bits < 0 || block_bits > wmax ||
      chunk_bits + leaf_bits + block_bits > P.log2_terms || P.log2_terms - chunk_bits - leaf_bits - block_bits > 40)
    return PERM_EINVAL;
  P.chunk_bits = chunk_bits; P.leaf_bits = leaf_bits; P.block_bits = block_bits;
  P.unit_bits = P.log2_terms - chunk_bits - leaf_bits - block_bits;
  P.units = 1LL << P.unit_bits;
  P.unit_terms = 1ULL << (P.log2_terms - P.unit_bits);
  if (unit_lo < 0 || unit_lo > unit_hi || unit_hi > P.units || unit_hi - unit_lo > (1LL << 31) - 1) return PERM_EINVAL;
  if (unit_lo == unit_hi) return PERM_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* ws = nullptr;
  CUDA_TRY(ws_alloc(&ws, kStagingBytes, st), "workspace alloc");
  const uint64_t lo = (uint64_t)unit_lo * P.unit_terms, hi = (uint64_t)unit_hi * P.unit_terms;
  int rc = run_sweep(A, P, unit_lo, unit_hi, lo, hi, reinterpret_cast<Dd2*>(unit_partials), static_cast<double2*>(ws), st);
  cudaError_t e = cudaFreeAsync(ws, st);
  if (rc == PERM_OK && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return rc;
}

int perm_glynn_range(const perm_c128* A, int n, uint64_t lo, uint64_t hi, perm_dd_c128* partial, void* stream) {
  return range_perm(A, n, PERM_ALG_GLYNN, lo, hi, partial, static_cast<cudaStream_t>(stream));
}

int perm_ryser_range(const perm_c128* A, int n, uint64_t lo, uint64_t hi, perm_dd_c128* partial, void* stream) {
  return range_perm(A, n, PERM_ALG_RYSER, lo, hi, partial, static_cast<cudaStream_t>(stream));
}

int perm_combine(const perm_dd_c128* partials, int64_t count, int n, int alg, perm_c128* out,
                 perm_dd_c128* out_dd, void* stream) {
  if (!partials || count < 1 || !valid_n_alg(n, alg)) return PERM_EINVAL;
  if (!out && !out_dd) return PERM_EINVAL;
  return run_combine(reinterpret_cast<const Dd2*>(partials), count, n, alg, reinterpret_cast<double2*>(out),
                     reinterpret_cast<Dd2*>(out_dd), static_cast<cudaStream_t>(stream));
}

static int batched(const perm_c128* A, int n, int64_t batch, perm_c128* out, double* out_abs2, void* stream) {
  if (!valid_n(n) || batch < 0) return PERM_EINVAL;
  if (batch == 0) return PERM_OK;
  if (!A || (!out && !out_abs2)) return PERM_EINVAL;
  init_tables();
  BatchedArgs a;
  a.A = reinterpret_cast<const double2*>(A);
  a.out = reinterpret_cast<double2*>(out);
  a.out_abs2 = out_abs2;
  a.batch = batch;
  make_batched_plan(n, &a.block_bits, &a.c, &a.lam);
  a.scale_exp = -(n - 1);
  a.zero = 0;
  const int grid = batch < (1LL << 30) ? (int)batch : (1 << 30);
  CUDA_TRY(g_batched[n](a, grid, static_cast<cudaStream_t>(stream)), "batched launch");
  note_launch();
  return PERM_OK;
}

int perm_glynn_batched(const perm_c128* A, int n, int64_t batch, perm_c128* out, void* stream) {
  if (!out && batch > 0) return PERM_EINVAL;
  return batched(A, n, batch, out, nullptr, stream);
}

int perm_glynn_batched_abs2(const perm_c128* A, int n, int64_t batch, double* out, void* stream) {
  if (!out && batch > 0) return PERM_EINVAL;
  return batched(A, n, batch, nullptr, out, stream);
}

int perm_sum_ordered(const perm_dd_c128* partials, int64_t count, const int64_t* order, int n, int alg,
                     perm_c128* out, void* stream) {
  if (!partials || !order || !out || count < 1 || !valid_n_alg(n, alg)) return PERM_EINVAL;
  const FinishArgs f{reinterpret_cast<double2*>(out), nullptr, is_glynn(alg) ? 1 : 0, -(n - 1), 0, 0};
  ordered_sum_kernel<<<1, 64, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<const Dd2*>(partials),
                                                                        order, count, f);
  CUDA_TRY(cudaGetLastError(), "ordered_sum_kernel launch");
  note_launch();
  return PERM_OK;
}

long long perm_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

static int host_call(const perm_c128* A, int n, int64_t batch, void* out, int which) {
  if (!A || !out || !valid_n(n) || batch < 0) return PERM_EINVAL;
  if (batch == 0) return PERM_OK;
  cudaStream_t st = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
  void* dA = nullptr;
  void* dO = nullptr;
  const size_t abytes = sizeof(perm_c128) * (size_t)n * n * batch;
  const size_t obytes = (which == 3 ? sizeof(double) : sizeof(perm_c128)) * batch;
  int rc = PERM_OK;
  cudaError_t e = ws_alloc(&dA, abytes, st);
  if (e == cudaSuccess) e = ws_alloc(&dO, obytes, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dA, A, abytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) rc = cuda_fail(e, "host entry: alloc/copy in");
  if (rc == PERM_OK) {
    const perm_c128* a = static_cast<const perm_c128*>(dA);
    perm_c128* o = static_cast<perm_c128*>(dO);
    if (which == 0) rc = perm_glynn(a, n, o, st);
    else if (which == 1) rc = perm_ryser(a, n, o, st);
    else if (which == 2) rc = perm_glynn_batched(a, n, batch, o, st);
    else rc = perm_glynn_batched_abs2(a, n, batch, static_cast<double*>(dO), st);
  }
  if (rc == PERM_OK) {
    e = cudaMemcpyAsync(out, dO, obytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "host entry: copy out");
  }
  if (dA) cudaFreeAsync(dA, st);
  if (dO) cudaFreeAsync(dO, st);
  e = cudaStreamSynchronize(st);
  if (rc == PERM_OK && e != cudaSuccess) rc = cuda_fail(e, "host entry: synchronize");
  cudaStreamDestroy(st);
  return rc;
}

int perm_glynn_host(const perm_c128* A, int n, perm_c128* out) { return host_call(A, n, 1, out, 0); }
int perm_ryser_host(const perm_c128* A, int n, perm_c128* out) { return host_call(A, n, 1, out, 1); }
int perm_glynn_batched_host(const perm_c128* A, int n, int64_t batch, perm_c128* out) {
  return host_call(A, n, batch, out, 2);
}
int perm_glynn_batched_abs2_host(const perm_c128* A, int n, int64_t batch, double* out) {
  return host_call(A, n, batch, out, 3);
}

}  // extern "C"
