"""Small invocations of every kernel family for compute-sanitizer (VERDICT r01
item 9): the n = 20 fused cooperative small-n path, the n = 24 constant-slot sweep + combine,
the batched kernel (n = 16, plus |perm|^2), the double-double sweep (n = 20), the separate-
addition mode and the ordered sum.  Each result is checked against the CPU oracle, so the
same command is a plain correctness run when not under the sanitizer.

    python tools/r02/sanitize_cases.py
    compute-sanitizer --tool memcheck  python tools/r02/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/r02/sanitize_cases.py --small
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--small", action="store_true", help="smaller sizes (racecheck is slow)")
a = ap.parse_args()
dev = torch.device("cuda:0")


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(dev)


def rel(x, y):
    return abs(x - y) / abs(y)


n1 = 16 if a.small else 20
A = synth.gaussian(n1, 20)
ref = oracle.glynn(A).value
g = complex(pb.glynn(T(A)).item())                       # fused cooperative small-n path
assert rel(g, ref) < 1e-9, ("fused", g, ref)
r = complex(pb.ryser(T(A)).item())
assert rel(r, ref) < 1e-7, ("fused ryser", r, ref)
n2 = 23 if a.small else 24                               # > 2^21 terms: constant-slot sweep + combine
B = synth.gaussian(n2, 24)
refB = oracle.glynn(B).value
gB = complex(pb.glynn(T(B)).item())
assert rel(gB, refB) < 1e-9, ("const", gB, refB)
As = synth.haar_batch(64 if a.small else 256, 256, 16, 16, 17)   # batched
out = pb.glynn_batched(T(As)).cpu().numpy()
p2 = pb.glynn_batched_abs2(T(As)).cpu().numpy()
for b in range(0, As.shape[0], 17):
    want = oracle.glynn(As[b]).value
    assert rel(complex(out[b]), want) < 1e-9 and abs(p2[b] - abs(want) ** 2) <= 3e-9 * abs(want) ** 2
d = pb.dd_to_complex(pb.glynn_dd(T(A)))                  # double-double sweep
assert rel(d, ref) < 1e-12, ("dd", d, ref)
s = complex(pb.perm_alg(T(A), "glynn_sep").item())       # separate addition
assert rel(s, ref) < 1e-7, ("sep", s, ref)
P = pb.plan(n1, pb.ALG_GLYNN_PLAIN)                      # chunk partials + ordered sum
cnt = P.terms >> 5
parts = pb.sweep_units_custom(T(A), "glynn_plain", 5, 0, 0, 0, cnt)
o = complex(pb.sum_ordered(parts, torch.from_numpy(synth.permutation(cnt, 5)).to(dev), n1, "glynn_plain").item())
assert rel(o, ref) < 1e-7, ("ordered", o, ref)
C = synth.gaussian(52, 52)                               # 2-lane row-split sweep (n >= 52), ragged range
lo, hi = 12345, 12345 + (1 << 13)
rp = oracle.partial_ex(C, lo, hi)
gp = pb.dd_to_complex(pb.glynn_range(T(C), lo, hi))
assert abs(gp - rp.dd.to_complex()) <= 1e-9 * rp.l1, ("split large", gp, rp.dd.to_complex())
torch.cuda.synchronize()
print("sanitize_cases ok", n1, n2, pb.launch_count(), "launches")
