"""Checkpointed, straggler-tolerant sweeps: one permanent run as a sequence of
unit SEGMENTS that can be interrupted, resumed, and claimed dynamically by the ranks of a
process group -- with a result bit-identical to the one-shot perm_glynn / perm_ryser.

Why it is exact: the canonical plan (include/permb200.h perm_plan_t) fixes every unit's
partial sum independently of which launch, GPU or rank computes it, and perm_combine reduces
the unit partials with a fixed tree.  So a run only has to collect every unit partial once;
the order in which segments are computed, the ranks that computed them and the interruptions
in between cannot change a bit.

Motivation: node failures ended multi-hour runs on Tianhe-2
("the node cn1561 failed during the execution, leading to the job termination"); n >= 52
permanents take hours even on 8 B200s.

  ledger   per-rank file <prefix>.rank<r>.npz: input SHA-256, plan, segment size, the unit
           partials of the segments this rank finished, and their indices; written atomically
           (tmp + rename) after every segment.
  resume   every rank loads ALL ledgers under the prefix (shared filesystem: one node), takes
           the union of finished segments, and only the remaining ones are claimed.
  claims   world > 1: segment k of the remaining list goes to the rank whose store.add() on a
           per-run counter returned k -- fast GPUs take more segments, a slow one fewer.
  gather   one all_reduce(SUM) of the (units, 4) partial table in which every unit has exactly
           one non-zero contributor (exact), then perm_combine on every rank.
"""
from __future__ import annotations

import glob
import hashlib
import os
import time
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


@dataclass
class Ledger:
    n: int
    alg: int
    units: int
    segment_units: int
    sha256: str
    seg_done: np.ndarray        # (k,) int64 segment indices finished by the writer
    parts: np.ndarray           # (k * segment_units, 4) float64, partials of those segments in order

    def save(self, path: str) -> None:
        tmp = path + ".tmp.npz"
        np.savez(tmp, n=self.n, alg=self.alg, units=self.units, segment_units=self.segment_units,
                 sha256=self.sha256, seg_done=self.seg_done, parts=self.parts)
        os.replace(tmp, path)

    @classmethod
    def load(cls, path: str) -> "Ledger":
        z = np.load(path, allow_pickle=False)
        return cls(int(z["n"]), int(z["alg"]), int(z["units"]), int(z["segment_units"]), str(z["sha256"]),
                   z["seg_done"].astype(np.int64), z["parts"].astype(np.float64))


def matrix_sha256(A: torch.Tensor) -> str:
    return hashlib.sha256(A.detach().to("cpu").contiguous().numpy().tobytes()).hexdigest()


def _segments(units: int, segment_units: int) -> list[tuple[int, int]]:
    return [(s, min(s + segment_units, units)) for s in range(0, units, segment_units)]


def _load_all(prefix: str, n: int, alg: int, units: int, seg_units: int, sha: str):
    """Union of the finished segments in every ledger under `prefix` -> {segment: (len, 4) parts}."""
    done = {}
    for path in sorted(glob.glob(prefix + ".rank*.npz")):
        L = Ledger.load(path)
        if (L.n, L.alg, L.units, L.segment_units, L.sha256) != (n, alg, units, seg_units, sha):
            raise ValueError(f"{path}: ledger of a different job (n/alg/plan/segment size/input differ)")
        off = 0
        for k in L.seg_done.tolist():
            lo, hi = k * seg_units, min((k + 1) * seg_units, units)
            done[k] = L.parts[off:off + (hi - lo)]
            off += hi - lo
    return done


def run_checkpointed(A: torch.Tensor, alg="glynn", prefix: Optional[str] = None, segment_units: int = 0,
                     group=None, store=None, max_segments: Optional[int] = None, deadline: Optional[float] = None,
                     sweep: Optional[Callable] = None, combine: Optional[Callable] = None,
                     on_segment: Optional[Callable] = None):
    """Perm(A) by `alg` as claimed, checkpointed segments of the canonical plan's units.

    Returns (value, complete): value is the 0-d complex128 permanent (None if this call stopped
    early because `max_segments` segments were computed by this rank -- a simulated failure
    for tests -- or because time.monotonic() passed `deadline`; the ledgers keep the work),
    identical on every rank and bit-identical to the one-shot computation.
    `on_segment(k, lo, hi)` is called after each segment this rank computes (progress logs).
    `prefix`: ledger path prefix (None: no checkpointing).  `segment_units`: units per segment
    (0: units / 64).  `store`: torch.distributed Store for the claim counter (default: the
    default group's store).  `sweep` / `combine` default to the CUDA kernels."""
    import paper_1606_05836_b200 as pb
    sweep = sweep or pb.sweep_units
    combine = combine or pb.combine
    a = pb._alg(alg)
    n = A.shape[0]
    P = pb.plan(n, a)
    seg_units = segment_units or max(1, P.units // 64)
    segs = _segments(P.units, seg_units)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sha = matrix_sha256(A)

    if world > 1:
        dist.barrier(group)                              # every ledger of a previous run is on disk
    done = _load_all(prefix, n, a, P.units, seg_units, sha) if prefix else {}
    loaded = set(done)
    remaining = [k for k in range(len(segs)) if k not in done]

    # claim counter for this run: a fresh key per call (rank 0 draws the run id)
    key = None
    if world > 1:
        # the default group's rendezvous store (torchrun's TCPStore); pass `store` explicitly to
        # avoid this private accessor
        store = store or dist.distributed_c10d._get_default_store()
        ids = [int(store.add(f"permb200/run/{sha[:16]}/{a}", 1)) if rank == 0 else 0]
        dist.broadcast_object_list(ids, src=0, group=group)
        key = f"permb200/claim/{sha[:16]}/{a}/{ids[0]}"

    mine_k, mine_parts = [], []
    if prefix:                                       # keep what this rank already finished
        own = prefix + f".rank{rank}.npz"
        if os.path.exists(own):
            L = Ledger.load(own)
            mine_k, mine_parts = L.seg_done.tolist(), [L.parts]
    computed = 0
    computed_k = []
    stopped = False
    next_local = 0
    while True:
        if (max_segments is not None and computed >= max_segments) or \
                (deadline is not None and time.monotonic() > deadline):
            stopped = True
            break
        if world > 1:
            idx = int(store.add(key, 1)) - 1
        else:
            idx = next_local
            next_local += 1
        if idx >= len(remaining):
            break
        k = remaining[idx]
        lo, hi = segs[k]
        p = sweep(A, a, lo, hi).to("cpu").numpy().astype(np.float64).reshape(hi - lo, 4)
        done[k] = p
        mine_k.append(k)
        mine_parts.append(p)
        computed_k.append(k)
        computed += 1
        if prefix:
            Ledger(n, a, P.units, seg_units, sha, np.asarray(mine_k, np.int64),
                   np.concatenate(mine_parts, axis=0)).save(prefix + f".rank{rank}.npz")
        if on_segment is not None:
            on_segment(k, lo, hi)

    stop_any = torch.tensor([1 if stopped else 0], dtype=torch.int64)
    table = np.zeros((P.units, 4), np.float64)
    # every unit gets exactly one contributor: the rank that computed it in this call, or
    # rank 0 for the units loaded from ledgers
    for k in computed_k + (sorted(loaded) if rank == 0 else []):
        lo, hi = segs[k]
        table[lo:hi] = done[k]
    if world > 1:
        dev = A.device if A.is_cuda and dist.get_backend(group) == "nccl" else torch.device("cpu")
        t = torch.from_numpy(table).to(dev)
        s = stop_any.to(dev)
        dist.all_reduce(s, op=dist.ReduceOp.MAX, group=group)
        if int(s.item()):
            return None, False
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)   # exact: one contributor per unit
        table_t = t.to(A.device)
    else:
        if stopped:
            return None, False
        table_t = torch.from_numpy(table).to(A.device)
    val, _ = combine(table_t, n, a, scale=True)
    return val, True
