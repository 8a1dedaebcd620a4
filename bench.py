#!/usr/bin/env python
"""Benchmark: BB/FG (Glynn) Gray-code terms/s for one permanent (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload M4]

Workload (BASELINE.json configs[3], "M4"): one 40 x 40 complex128 submatrix of a seeded
1600 x 1600 Haar unitary (synthetic: the paper's MATLAB matrices are not available), BB/FG
over 2^39 Gray-code terms, partitioned over the N GPUs of one node (strong scaling: the
total work is fixed) with one NCCL all_reduce.  One step = one full permanent.

`--gpus N` (N > 1) without torchrun re-launches itself through torch.distributed.run with N
ranks (fails loudly if fewer than N GPUs are visible; PERMB200_DIST_BACKEND=gloo runs the
N-rank logic with ranks sharing GPUs).  Every rank runs its share; the per-step device time
is the max over ranks; NCCL_DEBUG=INFO (INIT) puts the communicator init in the log.  Rank 0
prints ONE JSON line.  --impl reference times the CPU oracle (the only reference this
paper-tier task has) on the host cores; under torchrun only rank 0 works.
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


def _ncu_fp64_pipe(n: int):
    """FP64-pipe utilisation of the sweep kernel from the latest committed ncu summary
    (profiles/r0*_sweep_n<n>*_ncu_full.json), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", f"r0*_sweep_n{n}*ncu_full.json")), reverse=True):
        try:
            m = json.load(open(path))["metrics"]
            return {"pct": float(m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][1]),
                    "source": os.path.relpath(path, ROOT)}
        except (ValueError, KeyError, OSError):
            continue
    return None


def run_ours(args, rank, world, local_rank, shared_gpu: bool):
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
    aligned = pdist.subtree_aligned(P.units, world)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    stream = torch.cuda.current_stream(dev)
    sweep_ms = []

    def step(time_sweep: bool):
        # one full permanent: sweep my units -> (world > 1: one collective) -> combine + scale
        if time_sweep:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        parts = pb.sweep_units(A, alg, ulo, uhi)
        if time_sweep:
            e1.record(stream)
            sweep_ms.append((e0, e1))
        return pdist.reduce_partials(parts, n, alg, P.units, ulo, uhi, world, rank)

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
    k0 = pb.launch_count()
    t_start.record(stream)
    for k in range(args.steps):
        v = step(True)
        if k + 1 < args.steps:
            flush.zero_()        # L2 flushed between timed steps
    t_end.record(stream)
    barrier()
    launches = pb.launch_count() - k0
    clk = clocks.stop()
    ms_total = t_start.elapsed_time(t_end)
    sweep_avg = float(np.mean([a.elapsed_time(b) for a, b in sweep_ms]))
    value_c = complex(v.item())
    mx = torch.tensor([ms_total, sweep_avg], dtype=torch.float64, device=dev)
    nl = torch.tensor([launches], dtype=torch.int64, device=dev)
    clocks_all = [clk]
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(nl, op=dist.ReduceOp.SUM)
        clocks_all = [None] * world
        dist.all_gather_object(clocks_all, clk)
    ms_total, sweep_max = float(mx[0]), float(mx[1])
    launches_all = int(nl[0])

    # end to end through the public API with host buffers: the C-ABI perm_glynn_host at N = 1;
    # at N > 1 the pinned host matrix is copied to every GPU inside the timed region, then
    # perm_dist, and the result is read back to the host
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
    if world == 1:
        par = "single GPU: sweep + canonical combine, no collective"
    elif aligned:
        par = (f"Gray-index range partition over {world} GPUs: per-rank subtree root, one "
               f"{'gloo' if shared_gpu else 'NCCL'} all_reduce of the ({world}, 4) root table")
    else:
        par = (f"Gray-index range partition over {world} GPUs: one {'gloo' if shared_gpu else 'NCCL'} "
               f"all_reduce of the ({P.units}, 4) unit-partial table")
    line = {
        "metric": "BB/FG Gray-code terms/s", "value": value, "unit": "terms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {synth.WORKLOADS[args.workload]['desc']}", "n": n,
                   "terms": terms, "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": par,
                   "plan": {"chunk_bits": P.chunk_bits, "leaf_bits": P.leaf_bits, "block_bits": P.block_bits,
                            "units": P.units}},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "kernel": "sweep_kernel (perm_sweep_units)", "flop_per_term": flop_per_term,
                     "fp64_pipe_pct_ncu": _ncu_fp64_pipe(n),
                     "fp64_instr_frac": instr_frac,
                     "algorithmic_ceiling": flop_per_term / (2 * fp64_instr_per_term),
                     "peak_note": "nominal FP64 FMA peak 148 SM x 64 lanes x 2 x 1.965 GHz (MEASURED_PEAKS.json has "
                                  "no FP64 entry); a term needs 6n-2 FP64 instructions for 8n-4 flops, so "
                                  "frac <= algorithmic_ceiling; fp64_instr_frac and ncu's FP64-pipe % are the "
                                  "utilisation figures",
                     "traffic_note": "dram read+write bytes of one full sweep launch, kernel-only ncu capture "
                                     "(profiles/traffic.json); algorithmic bytes 16n^2 in + 32 B per unit out",
                     "builder_dfma_probe_tflops": FP64_MEASURED_TFLOPS,
                     "builder_dfma_probe_note": "the builder's DFMA microbenchmark (profiles/r01_fp64_probe.log); "
                                                "the sweep issues as fast as it, so it understates the pipe peak"},
        "e2e": {"value": terms / (e2e_ms_step * 1e-3), "unit": "terms/s", "h2d_bytes_per_step": 16 * n * n * world,
                "d2h_bytes_per_step": 16 * world, "ms_per_step": e2e_ms_step,
                "path": "C-ABI perm_glynn_host" if world == 1 else "pinned host -> each GPU, dist.perm_dist, .item()"},
        "gpu_launches": launches_all,
        "gpu_launches_note": f"libpermb200 kernels in the timed region, all ranks (perm_launch_count): "
                             f"{launches_all // max(1, args.steps)} per step",
        "clocks": clocks_all[0],
        "result": [value_c.real, value_c.imag],
        "paper_context": {"tianhe2_bbfg_hybrid_256_nodes_n40_s": 132.35, "derived_terms_per_s": 4.15e9,
                          "cite": "PAPER.md:562 (Table preTestBBFG)"},
    }
    if world > 1:
        line["clocks_per_rank"] = clocks_all
        if shared_gpu:
            line["ranks_share_gpus"] = True
    if cpu is not None:
        line["cpu_baseline"] = cpu
    # The metric's third part ("n=50 permanent seconds at 8 GPUs") is not a bench step (2^49
    # terms, 2.9 h on one GPU): it was measured once on ONE GPU, in checkpointed sessions, by
    # tools/m5_run.py; quoted here from its record, with the 8-GPU figure labelled as the
    # linear extrapolation it is.
    m5 = os.path.join(ROOT, "profiles", "r01_m5_full.json")
    if os.path.exists(m5):
        try:
            r = json.load(open(m5))
            line["n50_full_run"] = {"device_seconds_1gpu": r["device_seconds"], "terms_per_s": r["terms_per_s"],
                                    "linear_extrapolation_8gpu_seconds": r["device_seconds"] / 8,
                                    "value": r["value"], "measured_on": "1 GPU",
                                    "source": "profiles/r01_m5_full.json (tools/m5_run.py)"}
        except (ValueError, KeyError, OSError):
            pass
    # The Glynn-Ryser discrepancy toward n = 50 (BASELINE.json config 5): full FP64 Glynn and
    # Ryser permanents of the M5 family measured at n = 40..48 (tools/r02/ladder_summary.py);
    # the n = 50 figure is a band fitted to those rungs, labelled as such.
    lad = os.path.join(ROOT, "profiles", "r02_discrepancy_ladder.json")
    if os.path.exists(lad):
        try:
            r = json.load(open(lad))
            line["glynn_ryser_discrepancy"] = {
                "measured": {str(x["n"]): x["glynn_ryser_rel_discrepancy"] for x in r["rungs"]},
                "n50_fitted_band_1sigma": (r.get("extrapolation_n50") or {}).get("n50_band_1sigma"),
                "source": "profiles/r02_discrepancy_ladder.json (measured rungs; n = 50 is a fit, not a run)"}
        except (ValueError, KeyError, OSError):
            pass
    print(json.dumps(line), flush=True)
    return 0


def _self_launch(args) -> int:
    """`bench.py --gpus N` without torchrun: re-launch this script as N ranks through
    torch.distributed.run on 127.0.0.1 (the driver's command shape), with the NCCL init log on."""
    import socket
    import torch
    backend = os.environ.get("PERMB200_DIST_BACKEND", "nccl")
    have = torch.cuda.device_count()
    if args.impl == "ours" and backend == "nccl" and have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have} "
                         f"(set PERMB200_DIST_BACKEND=gloo to run the N-rank logic on shared GPUs)\n")
        return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


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
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return _self_launch(args)
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    backend = os.environ.get("PERMB200_DIST_BACKEND", "nccl")
    need = world if backend == "nccl" else 1
    if torch.cuda.device_count() < need:
        sys.stderr.write(f"bench.py: {world} rank(s) on backend {backend} needs {need} visible GPUs, found "
                         f"{torch.cuda.device_count()}\n")
        return 2
    shared_gpu = False
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("PERMB200_DIST_BACKEND", "nccl")    # gloo: CPU-side test of the N>1 logic
        if backend == "nccl":
            if torch.cuda.device_count() < world:
                raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, found {torch.cuda.device_count()}")
            os.environ.setdefault("NCCL_DEBUG", "INFO")          # the communicator init (nRanks) in the log
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
            shared_gpu = torch.cuda.device_count() < world
    try:
        return run_ours(args, rank, world, local_rank, shared_gpu)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
