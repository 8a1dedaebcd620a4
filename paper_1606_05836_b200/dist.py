"""Multi-GPU paths.

One permanent partitioned over a process group (PAPER.md Alg. A1/A2,
P:217-219 contiguous per-process ranges, P:230/P:261 one ALLREDUCE, P:262 final factor).

Each rank sweeps a contiguous, aligned block of the canonical plan's units and reduces it to
its subtree root (double-double, unscaled).  ONE collective then gathers the roots: an
all_reduce(SUM) of a (world, 4) float64 buffer in which rank r fills only row r -- every
slot has exactly one non-zero contributor, so the sum is exact and order-independent (an
all-gather expressed as the single NCCL all-reduce the north_star names).  Every rank then
combines the roots with the same pairwise tree, so for world | units (powers of two) the
result is bit-identical to the single-GPU perm_glynn / perm_ryser.  Other world sizes (3, 5,
6, 7 GPUs) gather the whole unit-partial table instead (reduce_partials): still one
collective, still bit-identical.
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


def subtree_aligned(units: int, world: int) -> bool:
    """True when every rank's contiguous unit block is one subtree of the canonical tree
    (world a power of two dividing `units`): then one root per rank suffices."""
    return world & (world - 1) == 0 and units % world == 0


def reduce_partials(parts: torch.Tensor, n: int, alg: int, units: int, ulo: int, uhi: int, world: int, rank: int,
                    group=None, combine: Optional[Callable] = None) -> torch.Tensor:
    """This rank's unit partials [ulo, uhi) -> the scaled permanent on every rank, with ONE
    collective and bit-identical to the single-GPU combine for ANY world size:

      world == 1        combine(parts) directly (no collective);
      subtree-aligned   each rank reduces its block to its subtree root, one all_reduce(SUM) of a
                        (world, 4) one-hot table gathers the roots exactly, combine(roots);
      otherwise         (3, 5, 6, 7 ... GPUs: blocks are not subtrees) one all_reduce(SUM) of the
                        (units, 4) table, each unit with exactly one non-zero contributor
                        (exact), then combine over all units -- units x 32 B (4 MiB at n = 40)."""
    import paper_1606_05836_b200 as pb
    combine = combine or pb.combine
    if world == 1:
        return combine(parts, n, alg, scale=True)[0]
    dev = parts.device
    if subtree_aligned(units, world):
        if uhi > ulo:
            root = combine(parts, n, alg, scale=False)[1]
        else:
            root = torch.zeros(4, dtype=torch.float64, device=dev)
        return combine(gather_roots(root, world, rank, group), n, alg, scale=True)[0]
    table = torch.zeros((units, 4), dtype=torch.float64, device=dev)
    if uhi > ulo:
        table[ulo:uhi] = parts
    dist.all_reduce(table, op=dist.ReduceOp.SUM, group=group)
    return combine(table, n, alg, scale=True)[0]


def perm_dist(A: torch.Tensor, alg: str = "glynn", group=None,
              sweep: Optional[Callable] = None, combine: Optional[Callable] = None) -> torch.Tensor:
    """Perm(A) with the Gray-index range split over the ranks of `group` (default: WORLD).

    A must be the same n x n complex128 matrix on every rank (on that rank's GPU).  Returns
    the 0-d complex128 result on every rank, bit-identical to the single-GPU perm_glynn /
    perm_ryser for any world size (reduce_partials).  `sweep` / `combine` default to the CUDA
    kernels (paper_1606_05836_b200.sweep_units / combine)."""
    import paper_1606_05836_b200 as pb
    sweep = sweep or pb.sweep_units
    n = A.shape[0]
    a = pb._alg(alg)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    P = pb.plan(n, a)
    ulo, uhi = unit_range(P.units, world, rank)
    parts = sweep(A, a, ulo, uhi) if uhi > ulo else torch.zeros((0, 4), dtype=torch.float64, device=A.device)
    return reduce_partials(parts, n, a, P.units, ulo, uhi, world, rank, group, combine)


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
