"""Glynn-Ryser and compensated-vs-plain discrepancies as n grows toward M5 (BASELINE.json
configs[4] asks for them at n = 50, where a Ryser run is 2^50 terms ~ 5.7 GPU-hours): the same
iid complex Gaussian family as M5 (variance 1/n, synth.gaussian(n, 50)) at n = 40, 42, 44, with
FP64 Glynn, FP64 Ryser, plain-accumulation Glynn, and the double-double Glynn value as the
reference where affordable (n <= 42).  The paper's metric |P_BB/FG - P_Ryser| / |P_BB/FG|
 is reported, plus each mode's error against dd.

    python tools/discrepancy_ladder.py [--sizes 40,42,44] [--dd-max 42] [--out gpurun_out/ladder.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v = fn()
    torch.cuda.synchronize()
    return v, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="40,42,44")
    ap.add_argument("--dd-max", type=int, default=42)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ladder.json"))
    a = ap.parse_args()
    rows = []
    for n in (int(x) for x in a.sizes.split(",")):
        A = torch.from_numpy(synth.gaussian(n, 50)).cuda()
        r = {"n": n, "seconds": {}}
        for name, fn in (("glynn", lambda: pb.glynn(A)), ("ryser", lambda: pb.ryser(A)),
                         ("glynn_plain", lambda: pb.perm_alg(A, "glynn_plain"))):
            v, dt = timed(fn)
            r[name] = complex(v.item())
            r["seconds"][name] = dt
        if n <= a.dd_max:
            v, dt = timed(lambda: pb.glynn_dd(A))
            r["glynn_dd"] = pb.dd_to_complex(v.cpu().numpy())
            r["seconds"]["glynn_dd"] = dt
        g = r["glynn"]
        r["glynn_ryser_rel_discrepancy"] = abs(g - r["ryser"]) / abs(g)
        r["plain_vs_compensated_rel_discrepancy"] = abs(r["glynn_plain"] - g) / abs(g)
        if "glynn_dd" in r:
            ref = r["glynn_dd"]
            for k in ("glynn", "ryser", "glynn_plain"):
                r[f"rel_err_{k}_vs_dd"] = abs(r[k] - ref) / abs(ref)
        for k in ("glynn", "ryser", "glynn_plain", "glynn_dd"):
            if k in r:
                r[k] = [r[k].real, r[k].imag]
        rows.append(r)
        print(json.dumps(r), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"gpu": torch.cuda.get_device_name(0), "family": "synth.gaussian(n, 50)", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
