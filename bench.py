#!/usr/bin/env python
"""Benchmark: BB/FG (Glynn) Gray-code terms/s for one permanent (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload M4]

Workload (BASELINE.json configs[3], "M4"): one 40 x 40 complex128 submatrix of a seeded
1600 x 1600 Haar unitary (synthetic: the paper's MATLAB matrices are not available), BB/FG
over 2^39 Gray-code terms, partitioned over the N GPUs of one node (strong scaling: the
total work is fixed) with one NCCL all_reduce.  One step = one full permanent.

Under torchrun (N > 1) every rank runs its share; the per-step device time is the max over
ranks.  Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle (the only
reference this paper-tier task has) on the host cores; under torchrun only rank 0 works.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

SM_COUNT = 148                 # B200 (B200_PROFILING.md)
SM_MAX_MHZ = 1965.0            # clocks.max.sm (B200_PROFILING.md / MEASURED_PEAKS.json)
FP64_FMA_PER_SM_CLK = 64       # FP64 lanes per SM (measured 34 TFLOP/s DFMA)
FP64_PEAK_TFLOPS = SM_COUNT * FP64_FMA_PER_SM_CLK * 2 * SM_MAX_MHZ * 1e6 / 1e12   # 37.2
# Sustained DFMA rate measured on this pool's B200 (tools/microbench/fp64_probe.cu, 8 independent
# DFMA chains per thread, 32 warps/SM, 0.9 s, 1965 MHz throughout): profiles/r01_fp64_probe.log
FP64_MEASURED_TFLOPS = 33.84


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None, "samples": len(sm), "reasons": sorted(reasons)}


def cpu_oracle_rate(A: np.ndarray, seconds: float, threads: int):
    """Time the CPU oracle (double-double Gray walk, oracle/perm_oracle.c) on a bounded
    sample of the workload's Gray-index range: the first S terms, S a power of two sized
    for about `seconds` of work."""
    import oracle
    n = A.shape[0]
    probe = 1 << 14
    t0 = time.perf_counter()
    oracle.glynn_partial(A, 0, probe * threads, threads=threads)
    dt = time.perf_counter() - t0
    rate = probe * threads / max(dt, 1e-9)
    S = 1 << max(10, int(np.floor(np.log2(max(rate * seconds, 1024)))))
    S = min(S, 1 << (n - 1))
    t0 = time.perf_counter()
    oracle.glynn_partial(A, 0, S, threads=threads)
    dt = time.perf_counter() - t0
    return S / dt, S, dt


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    A = synth.workload(args.workload)
    n = A.shape[0]
    cores = _cores()
    step_seconds = max(2.0, args.cpu_seconds / max(1, args.steps))
    for _ in range(args.warmup):
        cpu_oracle_rate(A, 0.5, cores)
    rates, samples, times = [], [], []
    for _ in range(args.steps):
        r, S, dt = cpu_oracle_rate(A, step_seconds, cores)
        rates.append(r)
        samples.append(S)
        times.append(dt)
    value = float(np.mean(rates))
    sample = f"first {samples[-1]} Gray indices of n={n} (of 2^{n - 1}) per step, double-double oracle, {cores} threads"
    line = {"impl": "reference", "metric": "BB/FG Gray-code terms/s", "value": value, "unit": "terms/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(times)) * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 (double-double)", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {synth.WORKLOADS[args.workload]['desc']}", "n": n,
                       "terms": 1 << (n - 1), "sample_terms_per_step": samples[-1]},
            "cpu_baseline": {"value": value, "unit": "terms/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "terms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1606_05836_b200 as pb
    from paper_1606_05836_b200 import dist as pdist

    dev_index = local_rank % torch.cuda.device_count()   # ranks share a GPU only in gloo tests
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    A_np = synth.workload(args.workload)
    n = A_np.shape[0]
    alg = pb.ALG_GLYNN
    P = pb.plan(n, alg)
    terms = P.terms
    A = torch.from_numpy(A_np).to(dev)
    A_pinned = torch.from_numpy(A_np).pin_memory()
    ulo, uhi = pdist.unit_range(P.units, world, rank)
    my_terms = (uhi - ulo) * P.unit_terms
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    stream = torch.cuda.current_stream(dev)
    sweep_ms = []

    def step(time_sweep: bool):
        # one full permanent: sweep my units -> subtree root -> one all_reduce -> combine
        if time_sweep:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        parts = pb.sweep_units(A, alg, ulo, uhi)
        if time_sweep:
            e1.record(stream)
        root = pb.combine(parts, n, alg, scale=False)[1]
        roots = pdist.gather_roots(root, world, rank)
        val, _ = pb.combine(roots, n, alg, scale=True)
        if time_sweep:
            sweep_ms.append((e0, e1))
        return val

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        v = step(False)
        flush.zero_()
    barrier()
    clocks = ClockSampler(dev_index)
    clocks.start()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    t_start.record(stream)
    for k in range(args.steps):
        v = step(True)
        if k + 1 < args.steps:
            flush.zero_()        # L2 flushed between timed steps
    t_end.record(stream)
    barrier()
    clk = clocks.stop()
    ms_total = t_start.elapsed_time(t_end)
    sweep_avg = float(np.mean([a.elapsed_time(b) for a, b in sweep_ms]))
    value_c = complex(v.item())
    mx = torch.tensor([ms_total, sweep_avg], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    ms_total, sweep_max = float(mx[0]), float(mx[1])

    # end to end through the public API with host buffers (C-ABI perm_glynn_host at N=1)
    e2e_ms = []
    for k in range(max(1, args.e2e_steps)):
        barrier()
        t0 = time.perf_counter()
        if world == 1:
            r = pb.glynn_host(A_np)
        else:
            Ad = A_pinned.to(dev, non_blocking=True)
            r = complex(pdist.perm_dist(Ad, "glynn").item())
        barrier()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_t = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_ms_step = float(e2e_t[0])
    assert r == value_c, (r, value_c)      # the host path computes the same bits

    if rank != 0:
        return 0
    ms_step = ms_total / args.steps
    value = terms / (ms_step * 1e-3)
    flop_per_term = 8 * n - 4          # n complex adds + (n-1) complex mults + accumulate
    achieved = my_terms * flop_per_term / (sweep_max * 1e-3) / 1e12
    fp64_instr_per_term = 6 * n - 2
    instr_frac = my_terms * fp64_instr_per_term / (sweep_max * 1e-3) / (SM_COUNT * FP64_FMA_PER_SM_CLK * SM_MAX_MHZ * 1e6)
    traffic = None       # dram read+write bytes of the profiled sweep launch (profiles/traffic.json)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"glynn_n{n}")
        except (ValueError, OSError):
            traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = _cores()
        rate, S, dt = cpu_oracle_rate(A_np, args.cpu_seconds, cores)
        cpu = {"value": rate, "unit": "terms/s", "cores": cores, "kind": "oracle",
               "sample": f"first {S} of 2^{n - 1} Gray indices of the same matrix, double-double oracle, {dt:.1f} s"}
    line = {
        "metric": "BB/FG Gray-code terms/s", "value": value, "unit": "terms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {synth.WORKLOADS[args.workload]['desc']}", "n": n,
                   "terms": terms, "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": f"Gray-index range partition over {world} GPU(s), one NCCL all_reduce",
                   "plan": {"chunk_bits": P.chunk_bits, "leaf_bits": P.leaf_bits, "block_bits": P.block_bits,
                            "units": P.units}},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "traffic_note": "dram read+write bytes of the bench's full sweep launch under ncu "
                                     "(profiles/r01_sweep_m4_dram.csv, profiles/traffic.json)",
                     "kernel": "sweep_kernel (perm_sweep_units)", "flop_per_term": flop_per_term,
                     "fp64_instr_frac": instr_frac,
                     "peak_note": "derived FP64 FMA peak 148 SM x 64 lanes x 2 x 1.965 GHz (DESIGN.md §Roofline)",
                     "measured_peak": FP64_MEASURED_TFLOPS,
                     "frac_of_measured": achieved / FP64_MEASURED_TFLOPS,
                     "fp64_issue_frac_of_measured": instr_frac * FP64_PEAK_TFLOPS / FP64_MEASURED_TFLOPS,
                     "measured_peak_note": "sustained DFMA microbenchmark, profiles/r01_fp64_probe.log; "
                                           "algorithmic ceiling (8n-4)/(2(6n-2)) = 0.664 of any DFMA peak"},
        "e2e": {"value": terms / (e2e_ms_step * 1e-3), "unit": "terms/s", "h2d_bytes_per_step": 16 * n * n,
                "d2h_bytes_per_step": 16, "ms_per_step": e2e_ms_step},
        "gpu_launches": 4 * args.steps,
        "clocks": clk,
        "result": [value_c.real, value_c.imag],
        "paper_context": {"tianhe2_bbfg_hybrid_256_nodes_n40_s": 132.35, "derived_terms_per_s": 4.15e9,
                          "cite": "PAPER.md:562 (Table preTestBBFG)"},
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    # The metric's third part ("n=50 permanent seconds at 8 GPUs") is not a bench step (2^49
    # terms, 2.9 h on one GPU): it was measured once, in checkpointed sessions, by
    # tools/m5_run.py; quoted here from its record.
    m5 = os.path.join(ROOT, "profiles", "r01_m5_full.json")
    if os.path.exists(m5):
        try:
            r = json.load(open(m5))
            line["n50_full_run"] = {"device_seconds_1gpu": r["device_seconds"], "terms_per_s": r["terms_per_s"],
                                    "extrapolated_8gpu_seconds": r["extrapolated_8gpu_seconds"],
                                    "value": r["value"], "source": "profiles/r01_m5_full.json (tools/m5_run.py)"}
        except (ValueError, KeyError, OSError):
            pass
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="M4", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.workload == "M2":
        raise SystemExit("M2 is a batched parity config; bench the single-permanent workloads")
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("PERMB200_DIST_BACKEND", "nccl")    # gloo: CPU-side test of the N>1 logic
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
