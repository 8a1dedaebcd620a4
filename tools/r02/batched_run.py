"""Batched boson-sampling probabilities at scale (FIG. 1:
P(S|T) ~ |Perm(U_ST)|^2): B >= 10^5 independent 16 x 16 submatrices of one Haar(256) unitary
(first 16 columns, seeded random 16-row subsets -- the M2 recipe with a larger batch),
|perm|^2 computed in the batched kernel (perm_glynn_batched_abs2), timed on the device
(inputs resident) and end to end through the host-buffer entry point; a sample of items is
checked against the CPU oracle.

    python tools/r02/batched_run.py [--batch 131072] [--out gpurun_out/batched.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402
from bench import ClockSampler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=131072)
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "batched.json"))
a = ap.parse_args()
t0 = time.time()
As = synth.haar_batch(a.batch, 256, a.n, 16, 17)
gen_s = time.time() - t0
dA = torch.from_numpy(As).cuda()
n, B = a.n, a.batch
terms = B * (1 << (n - 1))
for _ in range(3):
    pb.glynn_batched_abs2(dA)
torch.cuda.synchronize()
clk = ClockSampler(0)
clk.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
times = []
for _ in range(a.reps):
    e0.record()
    p2 = pb.glynn_batched_abs2(dA)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
clocks = clk.stop()
ms = float(np.median(times))
t1 = time.perf_counter()
p2h = pb.glynn_batched_abs2_host(As)
e2e_ms = (time.perf_counter() - t1) * 1e3
p2d = p2.cpu().numpy()
assert np.array_equal(p2h, p2d)
worst = 0.0
for b in range(0, B, max(1, B // 64)):
    ref = abs(oracle.glynn(As[b]).value) ** 2
    worst = max(worst, abs(p2d[b] - ref) / ref)
res = {"what": "batched |perm|^2, 16x16 submatrices of Haar(256)", "batch": B, "n": n,
       "device_ms": ms, "permanents_per_s": B / (ms * 1e-3), "terms_per_s": terms / (ms * 1e-3),
       "fp64_issue_frac": terms * (6 * n - 2) / (ms * 1e-3) / (148 * 64 * 1.965e9),
       "e2e_ms": e2e_ms, "e2e_permanents_per_s": B / (e2e_ms * 1e-3),
       "h2d_bytes": int(As.nbytes), "d2h_bytes": 8 * B, "input_gen_s": gen_s,
       "oracle_sample_items": len(range(0, B, max(1, B // 64))), "oracle_worst_rel": worst,
       "sum_p2": float(p2d.sum()), "clocks": clocks, "launches_per_call": 1}
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
