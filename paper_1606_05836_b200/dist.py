"""Multi-GPU paths.

One permanent partitioned over a process group (PAPER.md Alg. A1/A2,
P:217-219 contiguous per-process ranges, P:230/P:261 one ALLREDUCE, P:262 final factor).

Each rank sweeps a contiguous, aligned block of the canonical plan's units and reduces it to
its subtree root (double-double, unscaled).  ONE collective then gathers the roots: an
all_reduce(SUM) of a (world, 4) float64 buffer in which rank r fills only row r -- every
slot has exactly one non-zero contributor, so the sum is exact and order-independent (an
all-gather expressed as the single NCCL all-reduce the north_star names).  Every rank then
combines the roots with the same pairwise tree, so for world | units (powers of two) the
result is bit-identical to the single-GPU perm_glynn / perm_ryser.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def unit_range(units: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of units owned by `rank` (aligned subtree when world | units)."""
    return rank * units // world, (rank + 1) * units // world


def gather_roots(local_root: torch.Tensor, world: int, rank: int, group=None) -> torch.Tensor:
    """(4,) float64 root of this rank -> (world, 4) roots of all ranks via one all_reduce."""
    buf = torch.zeros((world, 4), dtype=torch.float64, device=local_root.device)
    buf[rank] = local_root
    if world > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def perm_dist(A: torch.Tensor, alg: str = "glynn", group=None,
              sweep: Optional[Callable] = None, combine: Optional[Callable] = None) -> torch.Tensor:
    """Perm(A) with the Gray-index range split over the ranks of `group` (default: WORLD).

    A must be the same n x n complex128 matrix on every rank (on that rank's GPU).  Returns
    the 0-d complex128 result on every rank.  `sweep` / `combine` default to the CUDA
    kernels (paper_1606_05836_b200.sweep_units / combine)."""
    import paper_1606_05836_b200 as pb
    sweep = sweep or pb.sweep_units
    combine = combine or pb.combine
    n = A.shape[0]
    a = pb._alg(alg)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    P = pb.plan(n, a)
    ulo, uhi = unit_range(P.units, world, rank)
    if uhi > ulo:
        root = combine(sweep(A, a, ulo, uhi), n, a, scale=False)[1]
    else:
        root = torch.zeros(4, dtype=torch.float64, device=A.device)
    roots = gather_roots(root, world, rank, group)
    val, _ = combine(roots, n, a, scale=True)
    return val


def batch_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of batch items owned by `rank`."""
    return rank * batch // world, (rank + 1) * batch // world


def batched_dist(As: torch.Tensor, group=None, fn: Optional[Callable] = None) -> torch.Tensor:
    """Batched permanents sharded over the ranks of `group` (boson-sampling
    probabilities need many independent permanents; no reduction, the items are
    independent).  Every rank passes the same (B, n, n) complex128 batch (on its GPU); rank r
    computes items batch_range(B, world, r) with perm_glynn_batched and ONE all_gather returns
    the (B,) permanents on every rank.  `fn` defaults to the CUDA kernel."""
    import paper_1606_05836_b200 as pb
    fn = fn or pb.glynn_batched
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B = As.shape[0]
    lo, hi = batch_range(B, world, rank)
    mine = fn(As[lo:hi])
    if world == 1:
        return mine
    per = (B + world - 1) // world                      # equal-size slots for all_gather
    buf = torch.zeros((per, 2), dtype=torch.float64, device=mine.device)
    buf[: hi - lo] = torch.view_as_real(mine)
    out = torch.empty((world * per, 2), dtype=torch.float64, device=mine.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    parts = [out[r * per: r * per + batch_range(B, world, r)[1] - batch_range(B, world, r)[0]] for r in range(world)]
    return torch.view_as_complex(torch.cat(parts).contiguous())
