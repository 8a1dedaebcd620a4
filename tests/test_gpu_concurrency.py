"""Re-entrancy of the C ABI (include/permb200.h "Concurrent calls on different streams /
devices are safe"): sweeps of the same n launched on different CUDA streams -- from one host
thread and from several -- must give the same bits as sequential calls, although they share
the translation unit's constant-memory column slot (fenced with events, perm_api.cu)."""
import threading

import numpy as np
import pytest
import torch

import synth
import paper_1606_05836_b200 as pb

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(DEV)


@pytest.mark.parametrize("n", [20, 30])
def test_two_streams_interleaved_bit_identical(n):
    mats = [T(synth.gaussian(n, 700 + k)) for k in range(6)]
    want = [complex(pb.glynn(A).item()) for A in mats]
    streams = [torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)]
    outs = []
    for k, A in enumerate(mats):
        with torch.cuda.stream(streams[k % 2]):
            outs.append(pb.glynn(A))
    torch.cuda.synchronize()
    assert [complex(o.item()) for o in outs] == want


def test_host_threads_on_own_streams_bit_identical():
    n = 28
    mats = [T(synth.gaussian(n, 800 + k)) for k in range(8)]
    want = [complex(pb.glynn(A).item()) for A in mats]
    got = [None] * len(mats)

    def work(idx):
        s = torch.cuda.Stream(DEV)
        with torch.cuda.stream(s):
            for k in idx:
                got[k] = pb.glynn(mats[k])
        s.synchronize()

    threads = [threading.Thread(target=work, args=(range(t, len(mats), 4),)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert [complex(g.item()) for g in got] == want


def test_mixed_modes_concurrently():
    """FP64 (constant slot), dd (no slot) and batched launches interleaved on two streams."""
    A = T(synth.gaussian(24, 5))
    As = T(np.stack([synth.gaussian(12, s) for s in range(64)]))
    w1, w2, w3 = complex(pb.glynn(A).item()), pb.glynn_dd(A).cpu(), pb.glynn_batched(As).cpu()
    w4 = complex(pb.ryser(A).item())
    s1, s2 = torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)
    res = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            res.append(("g", pb.glynn(A)))
            res.append(("b", pb.glynn_batched(As)))
        with torch.cuda.stream(s2):
            res.append(("d", pb.glynn_dd(A)))
            res.append(("r", pb.ryser(A)))
    torch.cuda.synchronize()
    for kind, v in res:
        if kind == "g":
            assert complex(v.item()) == w1
        elif kind == "r":
            assert complex(v.item()) == w4
        elif kind == "d":
            assert torch.equal(v.cpu(), w2)
        else:
            assert torch.equal(v.cpu(), w3)
