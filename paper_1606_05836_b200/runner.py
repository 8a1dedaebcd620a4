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

  ledger   per-rank file <prefix>.rank<r>[.<tag>].npz: input SHA-256, plan, segment size, the
           unit partials of the segments this rank finished, and their indices; written
           atomically (hidden temporary file + rename) after every segment.
  resume   rank 0 loads ALL ledgers under the prefix (shared filesystem: one node), takes the
           union of finished segments and broadcasts it; only the remaining ones are claimed.
  claims   world > 1 with a shared Store: segment k of the remaining list goes to the rank whose
           store.add() on a per-run counter returned k -- fast GPUs take more segments, a slow
           one fewer; without a Store: static round robin.
  gather   one all_reduce(SUM) of the (units, 4) partial table in which every unit has exactly
           one non-zero contributor (exact), then perm_combine on every rank.
"""
from __future__ import annotations

import glob
import hashlib
import os
import re
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
        """Atomic write: a temporary file the ledger glob cannot match (`<prefix>.tmp-...`),
        written through a file handle, then renamed over `path`."""
        d, b = os.path.split(path)
        tmp = os.path.join(d, ".tmp-" + b)
        with open(tmp, "wb") as f:
            np.savez(f, n=self.n, alg=self.alg, units=self.units, segment_units=self.segment_units,
                     sha256=self.sha256, seg_done=self.seg_done, parts=self.parts)
            f.flush()
            os.fsync(f.fileno())
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


def ledger_path(prefix: str, rank: int, tag: str = "") -> str:
    """<prefix>.rank<r>.npz, or <prefix>.rank<r>.<tag>.npz for a per-session ledger."""
    return prefix + f".rank{rank}" + (f".{tag}" if tag else "") + ".npz"


_LEDGER_RE = re.compile(r"\.rank\d+(?:\.[A-Za-z0-9_-]+)?\.npz$")


def ledger_files(prefix: str) -> list[str]:
    """Every finished ledger under `prefix` (temporary files never match)."""
    base = os.path.basename(prefix)
    out = []
    for path in sorted(glob.glob(prefix + ".rank*.npz")):
        name = os.path.basename(path)
        if name.startswith(base) and _LEDGER_RE.fullmatch(name[len(base):]):
            out.append(path)
    return out


def _load_all(prefix: str, n: int, alg: int, units: int, seg_units: int, sha: str):
    """Union of the finished segments in every ledger under `prefix` -> {segment: (len, 4) parts}."""
    done = {}
    for path in ledger_files(prefix):
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
                     on_segment: Optional[Callable] = None, tag: str = ""):
    """Perm(A) by `alg` as claimed, checkpointed segments of the canonical plan's units.

    Returns (value, complete): value is the 0-d complex128 permanent (None if this call stopped
    early because `max_segments` segments were computed by this rank -- a simulated failure
    for tests -- or because time.monotonic() passed `deadline`; the ledgers keep the work),
    identical on every rank and bit-identical to the one-shot computation.
    `on_segment(k, lo, hi)` is called after each segment this rank computes (progress logs).
    `prefix`: ledger path prefix (None: no checkpointing).  `tag`: this call writes its own
    ledger file <prefix>.rank<r>.<tag>.npz (per-session ledgers; default: one cumulative file
    per rank).  `segment_units`: units per segment (0: units / 64).
    `store`: a torch.distributed Store shared by the ranks (e.g. a TCPStore) for dynamic
    segment claims; without one, world > 1 falls back to a static round-robin assignment of
    the remaining segments.  `sweep` / `combine` default to the CUDA kernels.

    Consistency across ranks: rank 0 alone reads the ledgers and broadcasts the finished set,
    so every rank works on the same `remaining` list; before combining, a per-segment
    contributor count is all-reduced and must be exactly 1 everywhere (else RuntimeError)."""
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
    done = _load_all(prefix, n, a, P.units, seg_units, sha) if (prefix and rank == 0) else {}
    loaded = set(done)
    # rank 0's view of the finished segments (and the run id for the claim counter) -> everyone
    run_id = 0
    if world > 1 and store is not None and rank == 0:
        run_id = int(store.add(f"permb200/run/{sha[:16]}/{a}", 1))
    msg = [sorted(loaded), run_id]
    if world > 1:
        dist.broadcast_object_list(msg, src=0, group=group)
    loaded_ids, run_id = set(msg[0]), msg[1]
    remaining = [k for k in range(len(segs)) if k not in loaded_ids]
    key = f"permb200/claim/{sha[:16]}/{a}/{run_id}"

    mine_k, mine_parts = [], []
    own = ledger_path(prefix, rank, tag) if prefix else None
    if own and os.path.exists(own):                      # keep what this rank already finished
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
        if world > 1 and store is not None:
            idx = int(store.add(key, 1)) - 1             # dynamic claim: fast ranks take more
        elif world > 1:
            idx = rank + world * next_local              # static round robin
            next_local += 1
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
        if own:
            Ledger(n, a, P.units, seg_units, sha, np.asarray(mine_k, np.int64),
                   np.concatenate(mine_parts, axis=0)).save(own)
        if on_segment is not None:
            on_segment(k, lo, hi)

    stop_any = torch.tensor([1 if stopped else 0], dtype=torch.int64)
    table = np.zeros((P.units, 4), np.float64)
    counts = np.zeros(len(segs), np.int64)
    # every unit gets exactly one contributor: the rank that computed it in this call, or
    # rank 0 for the units loaded from ledgers
    for k in computed_k + (sorted(loaded) if rank == 0 else []):
        lo, hi = segs[k]
        table[lo:hi] = done[k]
        counts[k] += 1
    if world > 1:
        dev = A.device if A.is_cuda and dist.get_backend(group) == "nccl" else torch.device("cpu")
        s = stop_any.to(dev)
        dist.all_reduce(s, op=dist.ReduceOp.MAX, group=group)
        if int(s.item()):
            return None, False
        c = torch.from_numpy(counts).to(dev)
        dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
        counts = c.cpu().numpy()
    elif stopped:
        return None, False
    if not np.all(counts == 1):
        bad = np.nonzero(counts != 1)[0][:8].tolist()
        raise RuntimeError(f"segment contributor counts must be exactly 1; segments {bad} have "
                           f"{counts[bad].tolist()}")
    if world > 1:
        t = torch.from_numpy(table).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)   # exact: one contributor per unit
        table_t = t.to(A.device)
    else:
        table_t = torch.from_numpy(table).to(A.device)
    val, _ = combine(table_t, n, a, scale=True)
    return val, True
