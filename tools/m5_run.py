"""The full M5 permanent (BASELINE.json configs[4]: n = 50 iid complex Gaussian, 2^49 Gray-code
terms) on ONE B200, run as checkpointed segments across several time-limited GPU sessions
(paper_1606_05836_b200/runner.py).  Each session resumes from the ledger it
is given, sweeps segments until its time budget, and leaves the updated ledger behind; the
last one combines all unit partials into the permanent (bit-identical to a one-shot run).

    python tools/m5_run.py --ledger-in runs/m5 --out gpurun_out/m5 --budget-s 1700

Per-segment device times (CUDA events) go to <out>/segments.csv; the finished run writes
<out>/m5_result.json (value, total device seconds, terms/s, extrapolated 8-GPU seconds).
"""
import argparse
import csv
import glob
import json
import os
import shutil
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402
from paper_1606_05836_b200.runner import run_checkpointed  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alg", default="glynn")
    ap.add_argument("--ledger-in", default=os.path.join(ROOT, "runs", "m5"))
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "m5"))
    ap.add_argument("--budget-s", type=float, default=1700.0)
    ap.add_argument("--segment-units", type=int, default=2368)
    a = ap.parse_args()
    t_start = time.monotonic()
    os.makedirs(a.out, exist_ok=True)
    for f in glob.glob(os.path.join(a.ledger_in, "*")):          # resume from the previous session
        if os.path.abspath(os.path.dirname(f)) != os.path.abspath(a.out):
            shutil.copy(f, a.out)
    dev = torch.device("cuda:0")
    A = torch.from_numpy(synth.workload("M5")).to(dev)
    alg = pb._alg(a.alg)
    P = pb.plan(50, alg)
    seg_csv = os.path.join(a.out, "segments.csv")
    new = not os.path.exists(seg_csv)
    fh = open(seg_csv, "a", newline="")
    w = csv.writer(fh)
    if new:
        w.writerow(["segment", "unit_lo", "unit_hi", "terms", "device_ms", "terms_per_s", "wall_time"])
    ev = {}

    def sweep(A_, a_, lo, hi):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = pb.sweep_units(A_, a_, lo, hi)
        e1.record()
        e1.synchronize()
        ev["ms"] = e0.elapsed_time(e1)
        return out

    def on_segment(k, lo, hi):
        terms = (hi - lo) * P.unit_terms
        w.writerow([k, lo, hi, terms, f"{ev['ms']:.3f}", f"{terms / (ev['ms'] * 1e-3):.6e}", f"{time.time():.1f}"])
        fh.flush()

    deadline = t_start + a.budget_s
    val, done = run_checkpointed(A, alg, os.path.join(a.out, f"m5_{a.alg}"), segment_units=a.segment_units,
                                 deadline=deadline, sweep=sweep, on_segment=on_segment)
    fh.close()
    rows = list(csv.DictReader(open(seg_csv)))
    dev_s = sum(float(r["device_ms"]) for r in rows) * 1e-3
    terms = sum(int(r["terms"]) for r in rows)
    status = {"complete": bool(done), "segments_done": len(rows), "segments_total": -(-P.units // a.segment_units),
              "device_seconds_so_far": dev_s, "terms_so_far": terms,
              "terms_per_s": terms / dev_s if dev_s else None, "plan": P.__dict__}
    if done:
        v = complex(val.item())
        status.update({"value": [v.real, v.imag], "device_seconds_total": dev_s,
                       "extrapolated_8gpu_seconds": dev_s / 8,
                       "note": "device time = sum of per-segment CUDA-event sweep times on one B200; 8 GPUs "
                               "split the same units 8 ways (one all_reduce of the partial table)"})
    with open(os.path.join(a.out, "m5_status.json"), "w") as f:
        json.dump(status, f, indent=1)
    print(json.dumps(status))


if __name__ == "__main__":
    main()
