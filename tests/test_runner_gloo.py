"""Checkpoint / resume and dynamic segment claims of paper_1606_05836_b200/runner.py on CPU
(gloo, world_size 2).  The per-unit partial sums come from the oracle in place
of the CUDA sweep and the canonical pairwise tree is done in Python with the oracle's dd
addition (the GPU versions are exercised by tests/test_gpu_runner.py); what is tested here is
the host logic: ledgers, resume, claims, the exact gather -- the result of an interrupted and
resumed 2-rank run must equal the uninterrupted single-process run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from standins import oracle_sweep, tree_combine

N = 20
SEG = 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, prefix, max_segments, out_q, use_store=False, tag=""):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_1606_05836_b200.runner import run_checkpointed
    store = dist.TCPStore("127.0.0.1", port + 1, world, rank == 0) if use_store else None
    A = torch.from_numpy(synth.gaussian(N, 321))
    val, complete = run_checkpointed(A, "glynn", prefix, segment_units=SEG, max_segments=max_segments,
                                     sweep=oracle_sweep, combine=tree_combine, store=store, tag=tag)
    out_q.put((rank, None if val is None else complex(val.item()), complete))
    dist.barrier()
    dist.destroy_process_group()


def _launch(world, prefix, max_segments, use_store=False, tag=""):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, prefix, max_segments, q, use_store, tag))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_interrupted_resumed_run_is_bit_identical(tmp_path):
    import synth
    import oracle
    from paper_1606_05836_b200.runner import Ledger, run_checkpointed
    prefix = str(tmp_path / "job")
    # phase 1: both ranks stop after one segment each (a simulated failure)
    res = _launch(2, prefix, 1)
    assert all(v is None and not c for _, v, c in res)
    ledgers = [Ledger.load(prefix + f".rank{r}.npz") for r in range(2)]
    assert sorted(int(k) for L in ledgers for k in L.seg_done) == sorted(set(int(k) for L in ledgers for k in L.seg_done))
    assert sum(len(L.seg_done) for L in ledgers) == 2
    # phase 2: resume; the remaining segments are claimed dynamically
    res = _launch(2, prefix, None)
    vals = [v for _, v, c in res]
    assert all(c for _, _, c in res) and vals[0] == vals[1]
    ledgers = [Ledger.load(prefix + f".rank{r}.npz") for r in range(2)]
    done = sorted(int(k) for L in ledgers for k in L.seg_done)
    assert done == list(range(-(-__import__("paper_1606_05836_b200").plan(N).units // SEG)))                      # every segment exactly once
    # reference: one process, no checkpoint
    A = torch.from_numpy(synth.gaussian(N, 321))
    ref, ok = run_checkpointed(A, "glynn", None, segment_units=SEG, sweep=oracle_sweep, combine=tree_combine)
    assert ok and complex(ref.item()) == vals[0]
    want = oracle.glynn(A.numpy()).value
    assert abs(vals[0] - want) <= 1e-24 * abs(want) + 1e-300


def test_ledger_of_another_job_is_rejected(tmp_path):
    import synth
    from paper_1606_05836_b200.runner import run_checkpointed
    prefix = str(tmp_path / "job")
    A = torch.from_numpy(synth.gaussian(N, 321))
    v, ok = run_checkpointed(A, "glynn", prefix, segment_units=SEG, max_segments=1, sweep=oracle_sweep,
                             combine=tree_combine)
    assert v is None and not ok
    B = torch.from_numpy(synth.gaussian(N, 322))
    with pytest.raises(ValueError):
        run_checkpointed(B, "glynn", prefix, segment_units=SEG, sweep=oracle_sweep, combine=tree_combine)


def _reference():
    import synth
    from paper_1606_05836_b200.runner import run_checkpointed
    A = torch.from_numpy(synth.gaussian(N, 321))
    ref, ok = run_checkpointed(A, "glynn", None, segment_units=SEG, sweep=oracle_sweep, combine=tree_combine)
    assert ok
    return complex(ref.item())


def test_dynamic_claims_through_a_store_and_session_ledgers(tmp_path):
    """Claims through an explicit TCPStore (no private accessor); two sessions, each writing its
    own per-session ledger (tag); the resumed result equals the uninterrupted one bit for bit."""
    from paper_1606_05836_b200.runner import Ledger, ledger_files
    prefix = str(tmp_path / "job")
    res = _launch(2, prefix, 2, use_store=True, tag="s1")
    assert all(v is None and not c for _, v, c in res)
    res = _launch(2, prefix, None, use_store=True, tag="s2")
    vals = [v for _, v, c in res]
    assert all(c for _, _, c in res) and vals[0] == vals[1] == _reference()
    files = ledger_files(prefix)
    assert len(files) == 4 and all((".s1." in f) or (".s2." in f) for f in files)
    segs = [int(k) for f in files for k in Ledger.load(f).seg_done]
    assert sorted(segs) == list(range(-(-__import__("paper_1606_05836_b200").plan(N).units // SEG)))              # every segment exactly once


def test_truncated_temporary_files_are_ignored(tmp_path):
    """A process killed while saving leaves a temporary file; resume must not read it."""
    import synth
    from paper_1606_05836_b200.runner import ledger_files, run_checkpointed
    prefix = str(tmp_path / "job")
    A = torch.from_numpy(synth.gaussian(N, 321))
    v, ok = run_checkpointed(A, "glynn", prefix, segment_units=SEG, max_segments=2, sweep=oracle_sweep,
                             combine=tree_combine)
    assert not ok
    for junk in (".tmp-job.rank0.npz", "job.rank0.npz.tmp.npz", "job.rank1.npz.tmp", "job.rank0.x.y.npz"):
        with open(tmp_path / junk, "wb") as f:
            f.write(b"PK\x03\x04 truncated")
    assert ledger_files(prefix) == [prefix + ".rank0.npz"]
    v, ok = run_checkpointed(A, "glynn", prefix, segment_units=SEG, sweep=oracle_sweep, combine=tree_combine)
    assert ok and complex(v.item()) == _reference()
