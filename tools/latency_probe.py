"""M1 latency anatomy: per-call wall time of back-to-back pb.glynn calls vs the GPU-side time
(CUDA events around the whole batch of calls) vs the kernels' own durations.

    python tools/latency_probe.py [--n 20] [--calls 500]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1606_05836_b200 as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=20)
ap.add_argument("--calls", type=int, default=500)
a = ap.parse_args()
A = torch.from_numpy(synth.gaussian(a.n, 20)).cuda()
for fn in (pb.glynn, pb.ryser):
    for _ in range(20):
        fn(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(a.calls):
        fn(A)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{fn.__name__} n={a.n}: host submit {(t1 - t0) / a.calls * 1e6:.1f} us/call, "
          f"device span {e0.elapsed_time(e1) / a.calls * 1e3:.1f} us/call, wall {(t2 - t0) / a.calls * 1e6:.1f} us/call")
    # one call, synchronous latency
    lat = []
    for _ in range(50):
        torch.cuda.synchronize()
        s = time.perf_counter()
        fn(A)
        torch.cuda.synchronize()
        lat.append(time.perf_counter() - s)
    lat.sort()
    print(f"{fn.__name__} n={a.n}: single-call synchronous latency median {lat[len(lat) // 2] * 1e6:.1f} us")

# CUDA-graph replay of the same call (PermGraph): input copy + replay per permanent
for alg in ("glynn", "ryser"):
    g = pb.PermGraph(a.n, alg)
    for _ in range(20):
        g(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(a.calls):
        g(A)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"graph {alg} n={a.n}: host submit {(t1 - t0) / a.calls * 1e6:.1f} us/call, "
          f"device span {e0.elapsed_time(e1) / a.calls * 1e3:.1f} us/call, wall {(t2 - t0) / a.calls * 1e6:.1f} us/call")
