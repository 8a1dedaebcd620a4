"""Per-config performance sweep (BASELINE.json configs M1-M5 on one GPU), written as one JSON
object.  Not the driver's bench line (bench.py is); this records the numbers DESIGN.md §6
quotes for the other configs.

    python tools/perf_configs.py [--out gpurun_out/perf_configs.json] [--m5-units 296] [--skip M1,M2,...]

  M1  n=20: Glynn / Ryser latency per call (CUDA events over back-to-back calls)
  M2  4096 x 16x16 batched Glynn: permanents/s, terms/s, FP64 fraction
  M3  n=32: Glynn / Ryser seconds, terms/s
  M4  n=40: Glynn + Ryser full permanents; Glynn-Ryser discrepancy (class X)
  M5  n=50: sweep of the first 2368 canonical units (8 waves of 2 resident blocks x 148
      SMs; Glynn and Ryser), per-GPU terms/s and the extrapolated 1- and 8-GPU seconds
  DD  the double-double mode on M1 (n=20) and M3 (n=32): ms and terms/s
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402
from bench import ClockSampler  # noqa: E402

PEAK_INSTR = 148 * 64 * 1.965e9          # FP64 pipe instructions/s


def ev_time(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def rates(n, terms, ms, per_term_instr=None):
    s = ms * 1e-3
    k = per_term_instr if per_term_instr is not None else 6 * n - 2
    return {"ms": ms, "terms_per_s": terms / s, "alg_tflops": terms * (8 * n - 4) / s / 1e12,
            "fp64_instr_frac": terms * k / s / PEAK_INSTR}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "perf_configs.json"))
    ap.add_argument("--m5-units", type=int, default=2368, help="units per M5 sample (8 waves of 2 resident blocks x 148 SMs)")
    ap.add_argument("--skip", default="")
    a = ap.parse_args()
    skip = set(a.skip.split(",")) if a.skip else set()
    dev = torch.device("cuda:0")
    res = {"gpu": torch.cuda.get_device_name(0)}

    if "M1" not in skip:
        A = torch.from_numpy(synth.workload("M1")).to(dev)
        for fn in (pb.glynn, pb.ryser):
            fn(A)
        r = {}
        for name, fn, T in (("glynn", pb.glynn, 1 << 19), ("ryser", pb.ryser, 1 << 20)):
            ms, v = ev_time(lambda: fn(A), 200)
            r[name] = {"us_per_call": ms * 1e3, "terms_per_s": T / (ms * 1e-3), "value": [v.item().real, v.item().imag]}
        res["M1"] = r

    if "M2" not in skip:
        As = torch.from_numpy(synth.workload("M2")).to(dev)
        pb.glynn_batched(As)
        ms, _ = ev_time(lambda: pb.glynn_batched(As), 20)
        B, n = As.shape[0], As.shape[1]
        terms = B * (1 << (n - 1))
        res["M2"] = {"batch": B, "n": n, "permanents_per_s": B / (ms * 1e-3), **rates(n, terms, ms)}

    if "M3" not in skip:
        A = torch.from_numpy(synth.workload("M3")).to(dev)
        r = {}
        for name, fn, T in (("glynn", pb.glynn, 1 << 31), ("ryser", pb.ryser, 1 << 32)):
            fn(A)
            ms, v = ev_time(lambda: fn(A), 3)
            r[name] = {**rates(32, T, ms), "value": [v.item().real, v.item().imag]}
        # M3 asks for the oracle timed on the box's host cores: a bounded sample of the same
        # matrix (bench.py's cpu_oracle_rate), extrapolated to the full 2^31 terms
        from bench import _cores, cpu_oracle_rate
        cores = _cores()
        rate, S, dt = cpu_oracle_rate(synth.workload("M3"), 8.0, cores)
        r["oracle_cpu"] = {"terms_per_s": rate, "cores": cores, "sample_terms": S, "sample_seconds": dt,
                           "glynn_full_seconds_extrapolated": (1 << 31) / rate,
                           "gpu_over_cpu": r["glynn"]["terms_per_s"] / rate}
        res["M3"] = r

    if "M4" not in skip:
        A = torch.from_numpy(synth.workload("M4")).to(dev)
        r = {}
        for name, fn, T in (("glynn", pb.glynn, 1 << 39), ("ryser", pb.ryser, 1 << 40)):
            ms, v = ev_time(lambda: fn(A), 1)
            r[name] = {**rates(40, T, ms), "value": [v.item().real, v.item().imag]}
        g = complex(*r["glynn"]["value"])
        rr = complex(*r["ryser"]["value"])
        r["glynn_ryser_rel_discrepancy"] = abs(g - rr) / abs(g)
        res["M4"] = r

    if "M5" not in skip:
        A = torch.from_numpy(synth.workload("M5")).to(dev)
        r = {}
        for name, alg in (("glynn", pb.ALG_GLYNN), ("ryser", pb.ALG_RYSER)):
            P = pb.plan(50, alg)
            units = a.m5_units
            pb.range_partial(A, alg, 0, 4096)          # loads the n = 50 kernel
            clk = ClockSampler(0)
            clk.start()
            ms, _ = ev_time(lambda: pb.sweep_units(A, alg, 0, units), 1)
            clocks = clk.stop()
            terms = units * P.unit_terms
            x = rates(50, terms, ms)
            x["full_seconds_1gpu_extrapolated"] = P.terms / x["terms_per_s"]
            x["full_seconds_8gpu_extrapolated"] = P.terms / x["terms_per_s"] / 8
            x["units_swept"] = units
            x["clocks"] = clocks
            if clocks.get("sm_mhz"):
                x["fp64_instr_frac_at_measured_clock"] = x["fp64_instr_frac"] * 1965.0 / clocks["sm_mhz"]
            r[name] = x
        res["M5"] = r

    if "DD" not in skip:
        r = {}
        for wl, n in (("M1", 20), ("M3", 32)):
            A = torch.from_numpy(synth.workload(wl)).to(dev)
            for name, fn, T in (("glynn_dd", pb.glynn_dd, 1 << (n - 1)), ("ryser_dd", pb.ryser_dd, 1 << n)):
                fn(A)
                ms, v = ev_time(lambda: fn(A), 3)
                r[f"{wl}_{name}"] = {"ms": ms, "terms_per_s": T / (ms * 1e-3), "dd": v.cpu().tolist()}
        res["DD"] = r

    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
