"""GPU: checkpointed / resumed sweeps (paper_1606_05836_b200/runner.py) through
the CUDA kernels reproduce the one-shot C-ABI result bit for bit, for every arithmetic mode."""
import numpy as np
import pytest
import torch

import synth
import paper_1606_05836_b200 as pb
from paper_1606_05836_b200.runner import Ledger, run_checkpointed

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.mark.parametrize("alg,n", [("glynn", 28), ("ryser", 24), ("glynn_dd", 22), ("ryser_plain", 22)])
def test_interrupt_resume_bit_identical(tmp_path, alg, n):
    A = torch.from_numpy(synth.gaussian(n, 77 + n)).to(DEV)
    a = pb._alg(alg)
    P = pb.plan(n, a)
    seg = max(1, P.units // 8)
    prefix = str(tmp_path / "job")
    v, ok = run_checkpointed(A, a, prefix, segment_units=seg, max_segments=3)
    assert v is None and not ok
    assert len(Ledger.load(prefix + ".rank0.npz").seg_done) == 3
    v, ok = run_checkpointed(A, a, prefix, segment_units=seg)
    assert ok
    one_shot = pb.perm_alg(A, a)
    assert complex(v.item()) == complex(one_shot.item())
    if alg == "glynn":
        assert complex(v.item()) == complex(pb.glynn(A).item())
    assert sorted(Ledger.load(prefix + ".rank0.npz").seg_done.tolist()) == list(range((P.units + seg - 1) // seg))


def test_batched_dist_shards_equal_full_batch():
    """§8(f)3 on one GPU: the per-rank shards of batched_dist, computed separately, are the
    full batch's values bit for bit (items are independent blocks)."""
    from paper_1606_05836_b200.dist import batch_range, batched_dist
    As = torch.from_numpy(synth.haar_batch(301, 256, 16, 16, 17)).to(DEV)
    full = pb.glynn_batched(As)
    assert torch.equal(batched_dist(As), full)
    for world in (2, 3, 8):
        parts = [pb.glynn_batched(As[slice(*batch_range(301, world, r))]) for r in range(world)]
        assert torch.equal(torch.cat(parts), full)
