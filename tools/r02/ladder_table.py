"""Print the DESIGN.md section 6.1 ladder table rows from profiles/r02_discrepancy_ladder.json."""
import json
import sys

r = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_discrepancy_ladder.json"))
runs = r.get("runs_r02", {})
for x in r["rungs"]:
    n = x["n"]
    j = runs.get(str(n), {})
    g, ry = j.get("glynn", {}), j.get("ryser", {})
    t = f"{g['device_seconds']:.0f} / {ry['device_seconds']:.0f} s" if g else ""
    f = f"{g['fp64_issue_frac_nominal']:.3f} / {ry['fp64_issue_frac_nominal']:.3f}" if g else ""
    gd = f"{x['rel_err_glynn_vs_dd']:.1e}" if "rel_err_glynn_vs_dd" in x else "—"
    rd = f"{x['rel_err_ryser_vs_dd']:.1e}" if "rel_err_ryser_vs_dd" in x else "—"
    print(f"| {n} | {x['glynn_ryser_rel_discrepancy']:.2e} | {x['abs_discrepancy']:.1e} | {x['abs_glynn']:.1e} | {gd} | {rd} | {t} | {f} |")
print(json.dumps(r.get("extrapolation_n50"), indent=1))
