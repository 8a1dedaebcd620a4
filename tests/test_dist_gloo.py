"""Multi-process host logic of the partitioned permanent (paper_1606_05836_b200/dist.py) on
CPU with the gloo backend, world_size 2 (the N>1 path without GPUs): contiguous unit blocks,
the single all_reduce used as an exact gather, and the pairwise combine of the roots.  The
per-rank partial sums come from the oracle (CPU) in place of the CUDA sweep."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1606_05836_b200.dist import gather_roots, subtree_aligned, unit_range
from standins import oracle_sweep, tree_combine


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, units, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    A = synth.gaussian(n, 123)
    T = 1 << (n - 1)
    ut = T // units
    ulo, uhi = unit_range(units, world, rank)
    d, _ = oracle.glynn_partial(A, ulo * ut, uhi * ut, threads=1)
    root = torch.tensor(d.as4(), dtype=torch.float64)
    roots = gather_roots(root, world, rank)
    out_q.put((rank, root.numpy().copy(), roots.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_partition_and_exact_gather(world):
    n, units = 12, 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, units, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    locals_ = np.stack([r[1] for r in res])
    for _, _, roots in res:
        assert np.array_equal(roots, locals_)          # all_reduce of one-hot rows == exact gather
    import oracle
    import synth
    A = synth.gaussian(n, 123)
    acc = oracle.DD.from4(locals_[0])
    for k in range(1, world):
        acc = acc + oracle.DD.from4(locals_[k])
    full = oracle.glynn(A)
    got = acc.scaled(-(n - 1)).to_complex()
    assert abs(got - full.value) <= 1e-26 * full.l1 * 2 ** (n - 1) + 1e-30


def test_unit_range_tiles():
    for units in (1, 2, 8, 1 << 17):
        for world in (1, 2, 4, 8):
            spans = [unit_range(units, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == units
            for (a, b), (c, d) in zip(spans[:-1], spans[1:]):
                assert b == c
            if units % world == 0:
                assert len({b - a for a, b in spans}) == 1


def _oracle_batched(As):
    import oracle
    return torch.tensor([oracle.glynn(a).value for a in As.numpy()], dtype=torch.complex128)


def _batched_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_1606_05836_b200.dist import batched_dist
    As = torch.from_numpy(synth.haar_batch(7, 64, 8, 5, 6))      # 7 items: ragged over 2 ranks
    out = batched_dist(As, fn=_oracle_batched)
    out_q.put((rank, out.numpy().copy()))
    dist.destroy_process_group()


def test_gloo_batched_sharding_one_all_gather():
    """batch items sharded over ranks, one all_gather, ragged split (7 over 2)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batched_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    import synth
    As = synth.haar_batch(7, 64, 8, 5, 6)
    want = np.array([oracle.glynn(a).value for a in As])
    for _, out in res:
        assert out.shape == (7,)
        assert np.array_equal(out, want)


def _perm_dist_worker(rank, world, port, n, alg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_1606_05836_b200.dist import perm_dist
    A = torch.from_numpy(synth.gaussian(n, 99))
    v = perm_dist(A, alg, sweep=oracle_sweep, combine=tree_combine)
    out_q.put((rank, complex(v.item())))
    dist.destroy_process_group()


def _run_world(world, n, alg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_perm_dist_worker, args=(r, world, port, n, alg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [v for _, v in res]


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
def test_perm_dist_any_world_size_is_bit_identical(alg):
    """perm_dist on 2 ranks (subtree-aligned: one root per rank) and 3 ranks (not aligned: the
    whole unit table in one all_reduce) equals the single-process canonical combine bit for
    bit (world sizes that are not powers of two)."""
    import synth
    import paper_1606_05836_b200 as pb
    n = 14
    A = torch.from_numpy(synth.gaussian(n, 99))
    P = pb.plan(n, pb._alg(alg))
    one = complex(tree_combine(oracle_sweep(A, pb._alg(alg), 0, P.units), n, pb._alg(alg))[0].item())
    assert subtree_aligned(P.units, 2) and not subtree_aligned(P.units, 3)
    for world in (2, 3):
        vals = _run_world(world, n, alg)
        assert all(v == one for v in vals), (world, vals, one)
