"""Summarise a finished tools/m5_run.py run (ledger dir with segments.csv and m5_status.json)
into the JSON kept under profiles/.

    python tools/m5_summary.py runs/m5 profiles/r01_m5_full.json
    python tools/m5_summary.py runs/m5p profiles/r01_m5_plain_full.json profiles/r01_m5_full.json
"""
import csv
import json
import sys


def main():
    src, out = sys.argv[1], sys.argv[2]
    rows = list(csv.DictReader(open(f"{src}/segments.csv")))
    status = json.load(open(f"{src}/m5_status.json"))
    rates = [float(r["terms_per_s"]) for r in rows]
    dev_s = sum(float(r["device_ms"]) for r in rows) * 1e-3
    terms = sum(int(r["terms"]) for r in rows)
    # sessions = runs of segments without a wall-clock gap above 5 minutes
    walls = [float(r["wall_time"]) for r in rows]
    sessions = 1 + sum(1 for a, b in zip(walls[:-1], walls[1:]) if b - a > 300)
    alg = (status.get("plan") or {}).get("alg", 0)
    mode = {0: "FP64 compensated accumulation", 4: "FP64 PLAIN accumulation (PERM_ALG_GLYNN_PLAIN)",
            2: "double-double"}.get(alg, f"alg {alg}")
    res = {
        "config": "M5 (BASELINE.json configs[4]): n = 50 iid complex Gaussian, variance 1/n (synth.workload('M5')), "
                  f"BB/FG (Glynn), {mode}, 2^49 Gray-code terms, canonical plan, ONE B200",
        "complete": status.get("complete"),
        "value": status.get("value"),
        "segments": len(rows), "sessions": sessions,
        "terms": terms, "device_seconds": dev_s, "terms_per_s": terms / dev_s,
        "segment_terms_per_s_min": min(rates), "segment_terms_per_s_max": max(rates),
        "fp64_issue_frac_nominal": terms / dev_s * (6 * 50 - 2) / (148 * 64 * 1.965e9),
        "extrapolated_8gpu_seconds": dev_s / 8,
        "paper_context_minutes": "Tianhe-2 full system predicted 77.41-112.44 min (P:129)",
        "how": "tools/m5_run.py: checkpointed segments of 2368 units (paper_1606_05836_b200/runner.py), "
               "resumed across time-limited gpurun sessions; device time = sum of per-segment CUDA-event "
               "times; the combined value is bit-identical to a one-shot run (tests/test_gpu_runner.py)",
        "parity": "sampled windows vs the oracle (tests/test_gpu_configs.py::test_m5_windows_vs_oracle); "
                  "no oracle can walk 2^49 terms",
        "plan": status.get("plan"),
    }
    if len(sys.argv) > 3 and res["complete"]:         # compare with another finished run (e.g. compensated)
        other = json.load(open(sys.argv[3]))
        v, w = complex(*res["value"]), complex(*other["value"])
        res["rel_discrepancy_vs"] = {"file": sys.argv[3], "rel": abs(v - w) / abs(w)}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
