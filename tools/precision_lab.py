"""GPU precision lab: the paper's precision experiments (PAPER.md "Precision
Performance" P:134-163, FIG. 4 P:138-146, Tables AI-AIV) re-run on the B200 kernels,
in the paper's table format, for every arithmetic mode of the library:

  fp64   the production sweep (Gray order, compensated accumulation)      PERM_ALG_GLYNN / RYSER
  plain  the same sweep with plain FP64 accumulation (the paper's loop)   PERM_ALG_*_PLAIN
  dd     the double-double sweep                                          PERM_ALG_*_DD

Inputs are synthetic and carry no paper data:
  all-r  N x N matrices with every entry r (Tables AI-AIV: r = 1, 0.1, 10, 0.2 real and
         1+i, 10+10i complex; N = 17..36).  Theoretical value r^N N!, evaluated
         EXACTLY for the double nearest r (Fraction(float(r))), i.e. the exact permanent of
         the matrix the GPU actually received.
  haar   n x n submatrices of Haar(n^2) unitaries (the paper's MATLAB random unitaries,
         P:1045, are not available): Glynn-Ryser relative discrepancy
         |P_BB/FG - P_Ryser| / |P_BB/FG| (P:1045's metric) and each FP64 mode's error against
         the dd value.
  M4     (--m4) the bench matrix (n = 40): all six modes, errors against the dd Glynn value.

    python tools/precision_lab.py [--out-dir gpurun_out/precision] [--nmax 36] [--m4]

Writes one CSV per paper table (Size, Value, Comput. (Re, Im), Theor. (Re, Im), Abs. Error,
Relative Error Rate) plus precision_lab.json with everything.
"""
import argparse
import csv
import json
import math
import os
import sys
import time
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402

MODES = {"fp64": ("glynn", "ryser"), "plain": ("glynn_plain", "ryser_plain"), "dd": ("glynn_dd", "ryser_dd")}


def run(A: torch.Tensor, formula: int, mode: str):
    """-> (complex value, exact (re, im) Fractions of what the GPU returned, seconds)."""
    alg = MODES[mode][formula]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "dd":
        d = (pb.glynn_dd if formula == 0 else pb.ryser_dd)(A).cpu().numpy()
        fr = (Fraction(float(d[0])) + Fraction(float(d[1])), Fraction(float(d[2])) + Fraction(float(d[3])))
        v = complex(float(d[0]) + float(d[1]), float(d[2]) + float(d[3]))
    else:
        v = complex(pb.perm_alg(A, alg).item())
        fr = (Fraction(v.real), Fraction(v.imag))
    return v, fr, time.perf_counter() - t0


def cabs(re: Fraction, im: Fraction) -> float:
    return math.hypot(float(re), float(im))


def all_r_tables(dev, nmin, nmax, out_dir, res):
    values = [("1", 1.0), ("0.1", 0.1), ("10", 10.0), ("0.2", 0.2), ("1+i", 1 + 1j), ("10+10i", 10 + 10j)]
    rows = []
    for name, r in values:
        rr = complex(r)
        fr_re, fr_im = Fraction(float(rr.real)), Fraction(float(rr.imag))
        for n in range(nmin, nmax + 1):
            A = torch.full((n, n), rr, dtype=torch.complex128, device=dev)
            # exact r^n n! for the double-rounded r (complex power by repeated multiplication)
            pr, pi = Fraction(1), Fraction(0)
            for _ in range(n):
                pr, pi = pr * fr_re - pi * fr_im, pr * fr_im + pi * fr_re
            f = math.factorial(n)
            th = (pr * f, pi * f)
            th_abs = cabs(*th)
            for formula, fname in ((0, "BB/FG"), (1, "Ryser")):
                for mode in MODES:
                    v, fr, dt = run(A, formula, mode)
                    err = cabs(fr[0] - th[0], fr[1] - th[1])
                    rows.append({"table": f"{fname} {'complex' if rr.imag else 'real'}", "formula": fname,
                                 "mode": mode, "N": n, "r": name, "comp_re": v.real, "comp_im": v.imag,
                                 "theor_re": float(th[0]), "theor_im": float(th[1]), "abs_error": err,
                                 "rel_error": err / th_abs, "seconds": dt})
            print(f"all-r r={name} n={n} done", flush=True)
    res["all_r"] = rows
    for fname in ("BB/FG", "Ryser"):
        for kind in ("real", "complex"):
            path = os.path.join(out_dir, f"table_{fname.replace('/', '')}_{kind}.csv")
            with open(path, "w", newline="") as fh:
                w = csv.writer(fh)
                w.writerow(["Size of Matrix", "Value of Elements", "Mode", "Comput. Re", "Comput. Im", "Theor. Re",
                            "Theor. Im", "Abs. Error", "Relative Error Rate"])
                for x in rows:
                    if x["table"] == f"{fname} {kind}":
                        w.writerow([x["N"], x["r"], x["mode"], f"{x['comp_re']:.6E}", f"{x['comp_im']:.6E}",
                                    f"{x['theor_re']:.6E}", f"{x['theor_im']:.6E}", f"{x['abs_error']:.3E}",
                                    f"{x['rel_error']:.3E}"])


def haar_table(dev, sizes, out_dir, res):
    rows = []
    for n in sizes:
        A = torch.from_numpy(synth.haar_submatrix(n * n, n, 700 + n, 800 + n)).to(dev)
        vals = {}
        for formula, fname in ((0, "BB/FG"), (1, "Ryser")):
            for mode in MODES:
                vals[(fname, mode)] = run(A, formula, mode)[0]
        ref = vals[("BB/FG", "dd")]
        row = {"N": n, "ref_dd_glynn": [ref.real, ref.imag],
               "glynn_ryser_rel_discrepancy_fp64": abs(vals[("BB/FG", "fp64")] - vals[("Ryser", "fp64")]) / abs(vals[("BB/FG", "fp64")]),
               "glynn_ryser_rel_discrepancy_dd": abs(vals[("BB/FG", "dd")] - vals[("Ryser", "dd")]) / abs(ref)}
        for (fname, mode), v in vals.items():
            row[f"rel_err_{fname.replace('/', '')}_{mode}"] = abs(v - ref) / abs(ref)
        rows.append(row)
        print(f"haar n={n} done", flush=True)
    res["haar"] = rows
    with open(os.path.join(out_dir, "table_random_unitary.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        keys = [k for k in rows[0] if k not in ("ref_dd_glynn",)]
        w.writerow(keys)
        for r in rows:
            w.writerow([r[k] if isinstance(r[k], int) else f"{r[k]:.3E}" for k in keys])


def m4_report(dev, res):
    A = torch.from_numpy(synth.workload("M4")).to(dev)
    vals, secs = {}, {}
    for formula, fname in ((0, "BB/FG"), (1, "Ryser")):
        for mode in MODES:
            v, _, dt = run(A, formula, mode)
            vals[f"{fname}_{mode}"] = v
            secs[f"{fname}_{mode}"] = dt
            print(f"M4 {fname} {mode} {dt:.1f} s", flush=True)
    ref = vals["BB/FG_dd"]
    res["M4"] = {"values": {k: [v.real, v.imag] for k, v in vals.items()}, "seconds": secs,
                 "rel_err_vs_dd_glynn": {k: abs(v - ref) / abs(ref) for k, v in vals.items()},
                 "glynn_ryser_rel_discrepancy_fp64": abs(vals["BB/FG_fp64"] - vals["Ryser_fp64"]) / abs(vals["BB/FG_fp64"]),
                 "plain_vs_compensated_rel_discrepancy_glynn": abs(vals["BB/FG_plain"] - vals["BB/FG_fp64"]) / abs(ref),
                 "plain_vs_compensated_rel_discrepancy_ryser": abs(vals["Ryser_plain"] - vals["Ryser_fp64"]) / abs(ref)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "gpurun_out", "precision"))
    ap.add_argument("--nmin", type=int, default=17)
    ap.add_argument("--nmax", type=int, default=36)
    ap.add_argument("--haar", default="16,20,24,28,32,36")
    ap.add_argument("--m4", action="store_true")
    a = ap.parse_args()
    os.makedirs(a.out_dir, exist_ok=True)
    dev = torch.device("cuda:0")
    res = {"gpu": torch.cuda.get_device_name(0), "modes": MODES}
    all_r_tables(dev, a.nmin, a.nmax, a.out_dir, res)
    haar_table(dev, [int(x) for x in a.haar.split(",") if x], a.out_dir, res)
    if a.m4:
        m4_report(dev, res)
    with open(os.path.join(a.out_dir, "precision_lab.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print("ok")


if __name__ == "__main__":
    main()
