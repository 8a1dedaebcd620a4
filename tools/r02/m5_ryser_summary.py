"""Summarise the round-2 full n = 50 Ryser run (tools/m5_run.py --alg ryser, per-session ledgers
and segment logs with SM clocks) into profiles/r02_m5_ryser_full.json, with the measured
Glynn-Ryser discrepancy |P_G - P_R| / |P_G| against the round-1 full Glynn run (the paper's
central precision comparison: PAPER.md:146, :148-157 FIG. 5, :1042-1075).

    python tools/r02/m5_ryser_summary.py <dir with segments.rank*.csv> [m5_status.json] \
        --glynn profiles/r01_m5_full.json --out profiles/r02_m5_ryser_full.json
"""
import argparse
import csv
import glob
import json
import os
import statistics

ap = argparse.ArgumentParser()
ap.add_argument("segdir")
ap.add_argument("status", nargs="?", default=None)
ap.add_argument("--glynn", default="profiles/r01_m5_full.json")
ap.add_argument("--out", default="profiles/r02_m5_ryser_full.json")
a = ap.parse_args()
rows = []
for f in sorted(glob.glob(os.path.join(a.segdir, "segments.rank*.csv"))):
    rows += list(csv.DictReader(open(f)))
segs = {int(r["segment"]) for r in rows}
dev_s = sum(float(r["device_ms"]) for r in rows) * 1e-3
terms = sum(int(r["terms"]) for r in rows)
sm = [float(r["sm_mhz"]) for r in rows if r.get("sm_mhz") not in (None, "", "None")]
reasons = sorted({x for r in rows for x in (r.get("reasons") or "").split("|") if x})
sessions = sorted({r.get("session", "") for r in rows})
status = json.load(open(a.status)) if a.status and os.path.exists(a.status) else {}
res = {
    "config": "M5 (BASELINE.json configs[4]): n = 50 iid complex Gaussian, variance 1/n (synth.workload('M5')), "
              "Ryser (Eq. (1), P:62-64), FP64 compensated accumulation, 2^50 Gray-code terms, canonical plan, "
              "ONE B200",
    "complete": bool(status.get("complete")),
    "value": status.get("value"),
    "segments_logged": len(rows), "distinct_segments": len(segs), "sessions": len(sessions),
    "terms_logged": terms, "device_seconds": dev_s, "terms_per_s": terms / dev_s if dev_s else None,
    "fp64_issue_frac_nominal": terms / dev_s * (6 * 50 - 2) / (148 * 64 * 1.965e9) if dev_s else None,
    "clocks": {"segments_with_clock": len(sm), "sm_mhz_min": min(sm) if sm else None,
               "sm_mhz_median": statistics.median(sm) if sm else None, "reasons": reasons},
    "how": "tools/m5_run.py --alg ryser: checkpointed segments of 2368 units (runner.py) over time-limited gpurun "
           "sessions, each writing its own ledger; per-segment CUDA-event device times and nvidia-smi SM clocks "
           "sampled during the segment; combined value bit-identical to a one-shot run (tests/test_gpu_runner.py)",
}
if len(rows) != len(segs):
    res["note_duplicates"] = ("some segments were computed in more than one session (a session whose ledger "
                              "was not shipped to the next); the ledgers' union is used, device time above "
                              "counts every logged segment")
if res["complete"] and os.path.exists(a.glynn):
    g = json.load(open(a.glynn))
    G, R = complex(*g["value"]), complex(*res["value"])
    res["glynn_value"] = g["value"]
    res["glynn_ryser_discrepancy"] = {
        "rel": abs(G - R) / abs(G), "abs": abs(G - R),
        "what": "|P_G - P_R| / |P_G|, P_G = full n = 50 BB/FG run (profiles/r01_m5_full.json), P_R = this run",
        "cite": "PAPER.md:146 (FIG. 4 text), :148-157 (FIG. 5), :1042-1075 (Table ResultsComparing)"}
with open(a.out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
