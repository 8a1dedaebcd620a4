"""Race detector proxy (compute-sanitizer's racecheck is closed on this GPU pool): every kernel
family is run many times -- back to back and concurrently on 4 streams -- on the same input, and
every result must be bit-identical to the first.  A shared-memory race (a missing barrier in a
tree, a slot read before it is written) shows up as run-to-run differences in the low bits of
double-double partials long before it corrupts a value visibly.

    python tools/r02/determinism.py [--reps 100]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=100)
a = ap.parse_args()
dev = torch.device("cuda:0")


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(dev)


A20, A24, A52 = T(synth.gaussian(20, 1)), T(synth.gaussian(24, 2)), T(synth.gaussian(52, 3))
A60 = T(synth.gaussian(60, 4))
As = T(synth.haar_batch(512, 256, 16, 16, 17))
cases = {
    "fused split n=20 glynn": lambda s: pb.glynn(A20),
    "fused split n=20 ryser": lambda s: pb.ryser(A20),
    "const-slot n=24 glynn": lambda s: pb.glynn(A24),
    "split units n=20 (dd partials)": lambda s: pb.sweep_units(A20, "glynn", 0, pb.plan(20).units),
    "dd n=20": lambda s: pb.glynn_dd(A20),
    "sep n=20": lambda s: pb.perm_alg(A20, "glynn_sep"),
    "batched n=16": lambda s: pb.glynn_batched(As),
    "2-lane split n=52 range": lambda s: pb.glynn_range(A52, 777, 777 + (1 << 15)),
    # warp-pair split (perm_kernels_wsplit.cuh): shared-memory exchange + named barriers;
    # n = 52: 4 terms per exchange, n = 60: 2 terms per exchange
    "warp-pair n=52 units": lambda s: pb.sweep_units_custom(A52, "glynn", 5, 0, 6, 1000, 1296),
    "warp-pair n=60 units": lambda s: pb.sweep_units_custom(A60, "ryser", 6, 8, 6, 1000, 1296),
}
streams = [torch.cuda.Stream(dev) for _ in range(4)]
bad = 0
for name, fn in cases.items():
    ref = fn(None).clone()
    torch.cuda.synchronize()
    outs = []
    for r in range(a.reps):
        st = streams[r % 4]
        with torch.cuda.stream(st):
            outs.append(fn(st))
    torch.cuda.synchronize()
    diff = sum(0 if torch.equal(o, ref) else 1 for o in outs)
    bad += diff
    print(f"{name}: {a.reps} runs (4 streams), {diff} differ from the first", flush=True)
print("determinism ok" if bad == 0 else f"determinism FAILED: {bad} differing runs")
sys.exit(1 if bad else 0)
