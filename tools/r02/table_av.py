"""The paper's Table AV: errors of Ryser's algorithm on J_N under
four summation orders -- original (sequential in index order), random (sequential in a seeded
random order), merge (pairwise tree) and separate (sum of the added minus sum of the subtracted
terms) -- re-run on the B200 kernels, N = 8..32, next to the compensated FP64 and double-double
modes.  The GPU analogue of each order (include/permb200.h):
  original  perm_sum_ordered, identity order, over the 32-term chunk partials of a plain sweep
  random    perm_sum_ordered, synth.permutation order, same partials
  merge     perm_combine (canonical pairwise tree, plain adds) over the same partials
  separate  PERM_ALG_RYSER_SEP (even / odd index terms summed apart, one subtraction)
Exact value N! (integer).  Error rate = |value - N!| / N! (the paper's metric).

    python tools/r02/table_av.py [--nmax 32] [--out gpurun_out/r02_precision]
"""
import argparse
import csv
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nmin", type=int, default=8)
ap.add_argument("--nmax", type=int, default=32)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "r02_precision"))
a = ap.parse_args()
os.makedirs(a.out, exist_ok=True)
dev = torch.device("cuda:0")
rows = []
for N in range(a.nmin, a.nmax + 1):
    t0 = time.time()
    A = torch.from_numpy(synth.ones(N)).to(dev)
    exact = math.factorial(N)
    P = pb.plan(N, pb.ALG_RYSER_PLAIN)
    count = P.terms >> 5
    parts = pb.sweep_units_custom(A, pb.ALG_RYSER_PLAIN, 5, 0, 0, 0, count)
    ident = torch.arange(count, dtype=torch.int64, device=dev)
    order = torch.from_numpy(synth.permutation(count, 977 + N)).to(dev)
    vals = {
        "original": pb.sum_ordered(parts, ident, N, "ryser_plain"),
        "random": pb.sum_ordered(parts, order, N, "ryser_plain"),
        "merge": pb.combine(parts, N, "ryser_plain")[0],
        "separate": pb.perm_alg(A, "ryser_sep"),
        "fp64_compensated": pb.ryser(A),
        "plain_sweep": pb.perm_alg(A, "ryser_plain"),
    }
    del parts, ident, order
    row = {"N": N, "theor": float(exact)}
    for k, v in vals.items():
        x = complex(v.item()).real
        row[k] = x
        row[k + "_err"] = abs(x - exact) / exact
    dd = pb.dd_to_complex(pb.ryser_dd(A)).real
    row["dd"] = dd
    row["dd_err"] = abs(dd - exact) / exact
    row["seconds"] = time.time() - t0
    rows.append(row)
    torch.cuda.empty_cache()
    print(json.dumps(row), flush=True)
keys = list(rows[0].keys())
with open(os.path.join(a.out, "table_AV_ryser_orders.csv"), "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=keys)
    w.writeheader()
    w.writerows(rows)
with open(os.path.join(a.out, "table_AV_ryser_orders.json"), "w") as f:
    json.dump({"cite": "PAPER.md:977-1040 (Table AV), P:365", "rows": rows}, f, indent=1)
