"""Write oracle-computed expected values to tests/golden/ (calls ONLY oracle/ and synth/).

    python tools/make_golden.py m2 m3 [--threads T]

m2: config 1 -- 4096 x (16x16) Haar(256) submatrices, Glynn, double-double oracle
m3: config 2 -- n=32 Gaussian (seed 32), Glynn and Ryser, double-double oracle (~1 core-hour each)
Each file records the input recipe, the SHA-256 of the input bytes, the oracle's dd value
(hex floats) and sum|term| (L1), so a test can refuse a mismatched input.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def _dd_hex(d: oracle.DD):
    return [float(x).hex() for x in d.as4()]


def make_m2(threads):
    As = synth.workload("M2")
    t0 = time.time()
    vals = []
    for b in range(As.shape[0]):
        r = oracle.glynn(As[b], threads=threads)
        vals.append({"dd": _dd_hex(r.dd), "l1": r.l1})
    doc = {"config": synth.WORKLOADS["M2"]["desc"], "sha256": synth.sha256(As), "shape": list(As.shape),
           "oracle": "oracle.glynn (double-double Gray walk), value scaled by 2^-(n-1)",
           "seconds": time.time() - t0, "values": vals}
    with open(os.path.join(GOLDEN, "m2_batched_n16.json"), "w") as f:
        json.dump(doc, f)
    print("m2 done", time.time() - t0)


def make_m3(threads):
    A = synth.workload("M3")
    out = {"config": synth.WORKLOADS["M3"]["desc"], "sha256": synth.sha256(A), "n": 32}
    for alg, fn in (("glynn", oracle.glynn), ("ryser", oracle.ryser)):
        t0 = time.time()
        r = fn(A, threads=threads)
        out[alg] = {"dd": _dd_hex(r.dd), "value": [r.value.real, r.value.imag], "l1": r.l1,
                    "seconds": time.time() - t0, "threads": threads}
        print(alg, r.value, time.time() - t0, flush=True)
        with open(os.path.join(GOLDEN, "m3_n32.json"), "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="+", choices=["m2", "m3"])
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    a = ap.parse_args()
    for w in a.which:
        {"m2": make_m2, "m3": make_m3}[w](a.threads)
