"""Summarise the measured Glynn-Ryser discrepancy ladder of round 2 (full FP64 Glynn and Ryser
permanents of synth.gaussian(n, 50) at n = 46 and 48, run as checkpointed segments by
tools/r02/ladder_session.sh) together with round 1's n = 40 / 42 / 44 rungs
(profiles/r01_discrepancy_ladder.json), in the paper's metric |P_BB/FG - P_Ryser| / |P_BB/FG|
(FIG. 5 P:148-157, Table).  The n = 50 value is then an extrapolation
over two rungs instead of six.

    python tools/r02/ladder_summary.py [--runs runs/ladder] [--out profiles/r02_discrepancy_ladder.json]
"""
import argparse
import csv
import glob
import json
import os
import statistics

ap = argparse.ArgumentParser()
ap.add_argument("--runs", default="runs/ladder")
ap.add_argument("--r01", default="profiles/r01_discrepancy_ladder.json")
ap.add_argument("--out", default="profiles/r02_discrepancy_ladder.json")
a = ap.parse_args()


def job(n, alg):
    d = os.path.join(a.runs, f"g{n}_{alg}")
    rows = []
    for f in sorted(glob.glob(os.path.join(d, "segments.rank*.csv"))):
        rows += list(csv.DictReader(open(f)))
    st = json.load(open(os.path.join(d, "m5_status.json"))) if os.path.exists(os.path.join(d, "m5_status.json")) else {}
    dev_s = sum(float(r["device_ms"]) for r in rows) * 1e-3
    terms = sum(int(r["terms"]) for r in rows)
    sm = [float(r["sm_mhz"]) for r in rows if r.get("sm_mhz") not in (None, "", "None")]
    return {
        "complete": bool(st.get("complete")), "value": st.get("value"),
        "segments": len({int(r["segment"]) for r in rows}), "segments_total": st.get("segments_total"),
        "sessions": len({r.get("session") for r in rows}),
        "device_seconds": dev_s, "terms": terms, "terms_per_s": terms / dev_s if dev_s else None,
        "fp64_issue_frac_nominal": terms / dev_s * (6 * n - 2) / (148 * 64 * 1.965e9) if dev_s and not alg.endswith("_dd") else None,
        "sm_mhz_min": min(sm) if sm else None, "sm_mhz_median": statistics.median(sm) if sm else None,
        "throttle_reasons": sorted({x for r in rows for x in (r.get("reasons") or "").split("|") if x}),
    }


rungs = []
r01 = json.load(open(a.r01))
for r in r01["rows"]:
    rungs.append({"n": r["n"], "glynn_ryser_rel_discrepancy": r["glynn_ryser_rel_discrepancy"],
                  "source": a.r01, "glynn": r["glynn"], "ryser": r["ryser"],
                  **{k: r[k] for k in ("rel_err_glynn_vs_dd", "rel_err_ryser_vs_dd") if k in r}})
new = {}
import re
sizes = sorted({int(m.group(1)) for d in glob.glob(os.path.join(a.runs, "g*_*"))
                for m in [re.match(r"g(\d+)_", os.path.basename(d))] if m})
for n in sizes:
    g, r = job(n, "glynn"), job(n, "ryser")
    new[n] = {"glynn": g, "ryser": r}
    rung = None
    if g["complete"] and r["complete"]:
        G = complex(*g["value"])
        R = complex(*r["value"])
        rung = {"n": n, "glynn_ryser_rel_discrepancy": abs(G - R) / abs(G), "source": f"{a.runs}/g{n}_*",
                "glynn": g["value"], "ryser": r["value"]}
        rungs.append(rung)
    if os.path.isdir(os.path.join(a.runs, f"g{n}_glynn_dd")):
        d = job(n, "glynn_dd")
        new[n]["glynn_dd"] = d
        if rung and d["complete"]:
            D = complex(*d["value"])
            rung["glynn_dd"] = d["value"]
            rung["rel_err_glynn_vs_dd"] = abs(complex(*g["value"]) - D) / abs(D)
            rung["rel_err_ryser_vs_dd"] = abs(complex(*r["value"]) - D) / abs(D)
rungs.sort(key=lambda x: x["n"])
# The discrepancy is Ryser's rounding error over |perm|, and |perm| of one Gaussian realisation
# fluctuates by an order of magnitude around its e^(-n/2)-like trend, so the rungs are not
# monotone: fit log10(d) = a + b n over ALL measured rungs (least squares), report the residual
# scatter, and give the n = 50 figure as a band (fit +- 1 sigma of the residuals), not a point.
import math
ext = None
for x in rungs:
    G, R = complex(*x["glynn"]), complex(*x["ryser"])
    x["abs_discrepancy"] = abs(G - R)
    x["abs_glynn"] = abs(G)
if len(rungs) >= 3:
    xs = [x["n"] for x in rungs]
    ys = [math.log10(x["glynn_ryser_rel_discrepancy"]) for x in rungs]
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    b = sum((u - mx) * (v - my) for u, v in zip(xs, ys)) / sum((u - mx) ** 2 for u in xs)
    a0 = my - b * mx
    resid = [v - (a0 + b * u) for u, v in zip(xs, ys)]
    sd = math.sqrt(sum(r * r for r in resid) / max(1, len(xs) - 2))
    p50 = a0 + b * 50
    ext = {"fit": "log10(d) = a + b n, least squares over all rungs", "rungs_used": xs, "a": a0, "b_per_n": b,
           "factor_per_n": 10 ** b, "residual_sigma_log10": sd, "n50_estimate": 10 ** p50,
           "n50_band_1sigma": [10 ** (p50 - sd), 10 ** (p50 + sd)],
           "note": "an extrapolation: the full n = 50 Ryser run (2^50 terms, ~5.7 GPU-hours on one B200) was not "
                   "affordable in this round's GPU budget; the rungs are measured"}
res = {"family": "synth.gaussian(n, 50) (the M5 family, iid complex Gaussian, variance 1/n)",
       "metric": "|P_BBFG - P_Ryser| / |P_BBFG| (PAPER.md:1045), both FP64 compensated accumulation on one B200",
       "rungs": rungs, "runs_r02": {str(k): v for k, v in new.items()}, "extrapolation_n50": ext}
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps({"rungs": [(x["n"], x["glynn_ryser_rel_discrepancy"]) for x in rungs], "extrapolation": ext}))
