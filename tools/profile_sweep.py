"""Profiling driver (ncu target): run one kernel of the hot path on a slice of its canonical
units, so `ncu --set full` replays stay short.

    python tools/profile_sweep.py [--workload M4] [--fraction 64 | --units U] [--alg glynn] [--reps 2]
    python tools/profile_sweep.py --workload M2 --batched [--reps 2]
    python tools/profile_sweep.py --workload M5 --custom 11,4,7 --units 296   # short n = 50 units

--alg: glynn | ryser | glynn_dd | ryser_dd.  --batched times perm_glynn_batched on M2.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="M4")
ap.add_argument("--fraction", type=int, default=64)
ap.add_argument("--units", type=int, default=0, help="sweep exactly this many units (overrides --fraction)")
ap.add_argument("--alg", default="glynn")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--batched", action="store_true")
ap.add_argument("--custom", default="", help="c,leaf_bits,block_bits: non-canonical plan (perm_sweep_units_custom)")
ap.add_argument("--n", type=int, default=0, help="an n x n Gaussian matrix instead of --workload")
a = ap.parse_args()
A = torch.from_numpy(synth.gaussian(a.n, 9000 + a.n) if a.n else synth.workload(a.workload)).cuda()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if a.batched:
    B, n = A.shape[0], A.shape[1]
    for r in range(a.reps):
        e0.record()
        pb.glynn_batched(A)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        terms = B * (1 << (n - 1))
        print(f"batched B={B} n={n} {ms:.3f} ms {terms / ms * 1e3:.4e} terms/s "
              f"instr {terms * (6 * n - 2) / (ms * 1e-3) / (148 * 64 * 1.965e9):.3f}")
    sys.exit(0)
n = A.shape[0]
alg = pb._alg(a.alg)
P = pb.plan(n, alg)
if a.custom:
    c, lam, wb = (int(x) for x in a.custom.split(","))
    ub = P.log2_terms - c - lam - wb
    P = pb.Plan(n, alg, P.log2_terms, c, lam, wb, ub, 1 << (P.log2_terms - ub), 1 << ub, P.lanes)
units = a.units or max(1, P.units // a.fraction)
for r in range(a.reps):
    e0.record()
    if a.custom:
        parts = pb.sweep_units_custom(A, alg, P.chunk_bits, P.leaf_bits, P.block_bits, 0, units)
    else:
        parts = pb.sweep_units(A, alg, 0, units)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    terms = units * P.unit_terms
    print(f"n={n} alg={a.alg} units={units}/{P.units} {ms:.2f} ms {terms / ms * 1e3:.4e} terms/s "
          f"alg {terms * (8 * n - 4) / ms / 1e9:.2f} TFLOP/s instr {terms * (6 * n - 2) / (ms * 1e-3) / (148 * 64 * 1.965e9):.3f}")
