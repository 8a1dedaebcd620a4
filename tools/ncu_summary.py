"""Summarise an ncu report (.ncu-rep, read with `ncu -i ... --page raw --csv`) into the JSON
kept under profiles/: launch shape, occupancy limits, FP64-pipe utilisation, issue activity,
DRAM traffic, local-memory traffic and the PC-sampled stall reasons.

    python tools/ncu_summary.py <report.ncu-rep> <out.json> --kernel "<what>" --command "<cmd>" [--note ...]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps", "launch__waves_per_multiprocessor",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--command", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    out = {"kernel": a.kernel, "command": a.command, "note": a.note,
           "metrics": {k: list(d[k]) for k in KEYS if k in d},
           "stalls_pc_sampled": {}}
    for h in hdr:
        if "pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
            v = d[h][1]
            if v not in ("", "0"):
                out["stalls_pc_sampled"][h.split("stalled_")[1]] = int(float(v))
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
