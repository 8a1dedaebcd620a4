"""CUDA-graph capture of the C-ABI calls (paper_1606_05836_b200.PermGraph): replays on new
inputs give the eager calls' bits; the constant-slot path refuses capture loudly."""
import numpy as np
import pytest
import torch

import synth
import paper_1606_05836_b200 as pb

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(DEV)


@pytest.mark.parametrize("n,alg", [(20, "glynn"), (21, "ryser"), (14, "glynn_dd"), (18, "glynn_plain")])
def test_graph_replay_bit_identical(n, alg):
    g = pb.PermGraph(n, alg)
    for seed in range(3):
        A = T(synth.gaussian(n, 40 + seed))
        out = g(A).clone()
        want = pb.glynn_dd(A) if alg == "glynn_dd" else pb.perm_alg(A, alg)
        assert torch.equal(out, want), (alg, seed)


def test_graph_batched():
    As = T(synth.haar_batch(64, 64, 10, 3, 4))
    g = pb.PermGraph(10, "glynn", batch=64)
    assert torch.equal(g(As).clone(), pb.glynn_batched(As))


def test_constant_slot_path_refuses_capture():
    with pytest.raises(pb.PermError):
        pb.PermGraph(30, "glynn")
