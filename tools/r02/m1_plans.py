"""M1 (n = 20, 2^19 Glynn terms) plan experiment: device time of the small-n sweep kernel
for several chunk / block shapes, each measured as 64 back-to-back calls captured in ONE CUDA
graph (so host submission does not hide the kernel time), plus the canonical full call.

    python tools/r02/m1_plans.py [--n 20] [--alg glynn]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=20)
ap.add_argument("--alg", default="glynn")
ap.add_argument("--reps", type=int, default=64)
a = ap.parse_args()
A = torch.from_numpy(synth.gaussian(a.n, 20)).cuda()
alg = pb._alg(a.alg)
P = pb.plan(a.n, alg)
m = P.log2_terms


def graph_time(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best


out = {"n": a.n, "alg": a.alg, "canonical_plan": P.__dict__, "rows": []}
fn_full = pb.glynn if alg == pb.ALG_GLYNN else pb.ryser
out["canonical_full_call_us"] = graph_time(lambda: fn_full(A), a.reps)
ref = complex(fn_full(A).item())
wmax = 7 - (P.lanes.bit_length() - 1)
for c in (4, 5, 6, 7):
    for wb in range(wmax - 2, wmax + 1):
        lam = 0
        ub = m - c - wb - lam
        if ub < 0:
            continue
        units = 1 << ub
        t = graph_time(lambda: pb.sweep_units_custom(A, alg, c, lam, wb, 0, units), a.reps)
        parts = pb.sweep_units_custom(A, alg, c, lam, wb, 0, units)
        v = complex(pb.combine(parts, a.n, alg)[0].item())
        row = {"c": c, "block_bits": wb, "units": units, "threads": (units << wb) * P.lanes, "sweep_us": t,
               "rel_vs_canonical": abs(v - ref) / abs(ref)}
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
parts = pb.sweep_units(A, alg, 0, P.units)
out["combine_only_us"] = graph_time(lambda: pb.combine(parts, a.n, alg), a.reps)
print(json.dumps(out))
