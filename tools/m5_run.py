"""A full single permanent of a BASELINE.json config (default M5: n = 50 iid complex Gaussian;
Glynn 2^49 / Ryser 2^50 Gray-code terms) run as checkpointed segments across several
time-limited GPU sessions (paper_1606_05836_b200/runner.py).  Each session
resumes from the ledgers it is given, sweeps segments until its time budget, and writes its
own per-session ledger; the last one combines all unit partials into the permanent
(bit-identical to a one-shot run).

    python tools/m5_run.py --alg ryser --ledger-in runs/m5r --out gpurun_out/m5r --budget-s 2400
    torchrun --nproc-per-node 8 tools/m5_run.py ...        # N GPUs: ranks claim segments

Rank-aware: under torchrun every rank uses cuda:LOCAL_RANK, one NCCL process group, and a
TCPStore on MASTER_PORT+1 for dynamic segment claims (a slow GPU takes fewer segments).
Per-segment device times (CUDA events) and the SM clock / throttle reasons sampled by
nvidia-smi during the segment go to <out>/segments.rank<r>.csv; the finished run writes
<out>/m5_status.json with the value, total device seconds and terms/s.
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
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_1606_05836_b200.runner import run_checkpointed  # noqa: E402

FIELDS = ["segment", "unit_lo", "unit_hi", "terms", "device_ms", "terms_per_s", "wall_time", "rank",
          "sm_mhz", "sm_max_mhz", "reasons", "session"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alg", default="glynn")
    ap.add_argument("--workload", default="M5", help="a synth.WORKLOADS name, or gauss50:<n> = synth.gaussian(n, 50)")
    ap.add_argument("--ledger-in", default=os.path.join(ROOT, "runs", "m5"))
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "m5"))
    ap.add_argument("--budget-s", type=float, default=1700.0)
    ap.add_argument("--segment-units", type=int, default=2368)
    ap.add_argument("--max-segments", type=int, default=None, help="stop after this many segments (tests)")
    ap.add_argument("--session", default=None, help="tag of this session's ledger (default: a timestamp)")
    a = ap.parse_args()
    t_start = time.monotonic()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > torch.cuda.device_count():
        raise SystemExit(f"{world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    store = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        store = dist.TCPStore(os.environ["MASTER_ADDR"], int(os.environ["MASTER_PORT"]) + 1, world, rank == 0)
    session = a.session or time.strftime("s%Y%m%d%H%M%S", time.gmtime())
    if world > 1:
        obj = [session]
        dist.broadcast_object_list(obj, src=0)
        session = obj[0]
    # Work directory: the previous sessions' ledgers and segment logs are copied in; only THIS
    # session's files are copied to --out at the end (gpurun merges back <= 64 MiB per call,
    # while the ledgers of a 2^21-unit run total 64 MiB).
    work = os.path.join("/tmp", f"m5work_{a.workload.replace(':', '_')}_{a.alg}_{session}")
    os.makedirs(a.out, exist_ok=True)
    if rank == 0:
        os.makedirs(work, exist_ok=True)
        for f in glob.glob(os.path.join(a.ledger_in, "*")):          # resume from the previous sessions
            if os.path.isfile(f):
                shutil.copy(f, work)
    if world > 1:
        dist.barrier()
    if a.workload.startswith("gauss50:"):
        # the M5 family at another size (Glynn-Ryser discrepancy ladder): synth.gaussian(n, 50)
        A = torch.from_numpy(synth.gaussian(int(a.workload.split(":")[1]), 50)).to(dev)
    else:
        A = torch.from_numpy(synth.workload(a.workload)).to(dev)
    n = A.shape[0]
    alg = pb._alg(a.alg)
    P = pb.plan(n, alg)
    seg_csv = os.path.join(work, f"segments.rank{rank}.{session}.csv")
    new = not os.path.exists(seg_csv)
    fh = open(seg_csv, "a", newline="")
    w = csv.DictWriter(fh, fieldnames=FIELDS)
    if new:
        w.writeheader()
    ev = {}

    def sweep(A_, a_, lo, hi):
        clk = ClockSampler(local_rank)
        clk.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = pb.sweep_units(A_, a_, lo, hi)
        e1.record()
        e1.synchronize()
        ev["clk"] = clk.stop()
        ev["ms"] = e0.elapsed_time(e1)
        return out

    def on_segment(k, lo, hi):
        terms = (hi - lo) * P.unit_terms
        c = ev["clk"]
        w.writerow({"segment": k, "unit_lo": lo, "unit_hi": hi, "terms": terms, "device_ms": f"{ev['ms']:.3f}",
                    "terms_per_s": f"{terms / (ev['ms'] * 1e-3):.6e}", "wall_time": f"{time.time():.1f}",
                    "rank": rank, "sm_mhz": c.get("sm_mhz"), "sm_max_mhz": c.get("sm_max_mhz"),
                    "reasons": "|".join(c.get("reasons", [])), "session": session})
        fh.flush()
        # Mirror this session's ledger + log into --out after EVERY segment (hidden temporary
        # name + rename): a session killed by the GPU-call time limit keeps all finished segments.
        for src in (os.path.join(work, f"m5_{a.alg}.rank{rank}.{session}.npz"), seg_csv):
            if os.path.exists(src):
                tmp = os.path.join(a.out, ".tmp-" + os.path.basename(src))
                shutil.copy(src, tmp)
                os.replace(tmp, os.path.join(a.out, os.path.basename(src)))

    deadline = t_start + a.budget_s
    val, done = run_checkpointed(A, alg, os.path.join(work, f"m5_{a.alg}"), segment_units=a.segment_units,
                                 deadline=deadline, max_segments=a.max_segments, sweep=sweep, on_segment=on_segment, store=store, tag=session)
    fh.close()
    for f in glob.glob(os.path.join(work, f"*.rank{rank}.{session}.*")):   # this session's ledger + log
        shutil.copy(f, a.out)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    rows = []
    for f in sorted(glob.glob(os.path.join(work, "segments*.csv"))):
        rows += list(csv.DictReader(open(f)))
    dev_s = sum(float(r["device_ms"]) for r in rows) * 1e-3
    terms = sum(int(r["terms"]) for r in rows)
    status = {"workload": a.workload, "alg": a.alg, "n": n, "complete": bool(done), "segments_done": len(rows),
              "segments_total": -(-P.units // a.segment_units), "device_seconds_so_far": dev_s,
              "terms_so_far": terms, "terms_per_s": terms / dev_s if dev_s else None, "plan": P.__dict__,
              "world": world, "session": session}
    if done:
        v = complex(val.item())
        status.update({"value": [v.real, v.imag], "device_seconds_total": dev_s,
                       "note": "device time = sum of per-segment CUDA-event sweep times (each rank's own); "
                               "the units are split over the ranks by dynamic claims, one all_reduce of the "
                               "partial table"})
    with open(os.path.join(a.out, "m5_status.json"), "w") as f:
        json.dump(status, f, indent=1)
    print(json.dumps(status))


if __name__ == "__main__":
    main()
