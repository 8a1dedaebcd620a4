"""CPU stand-ins for the two CUDA kernels of the canonical reduction, used by the multi-process
gloo tests of the host logic (dist.py, runner.py) where no GPU exists: the unit partials come
from the oracle's Gray walk over each unit's index range, and the canonical pairwise tree
(node = left + right, zero padding to a power of two -- the shape of combine_kernel) is done
with the oracle's double-double addition.  Test infrastructure only."""
import numpy as np
import torch


def oracle_sweep(A, alg, lo, hi):
    import oracle
    import paper_1606_05836_b200 as pb
    a = A.numpy()
    P = pb.plan(a.shape[0], alg)
    fn = oracle.glynn_partial if alg in (pb.ALG_GLYNN, "glynn") else oracle.ryser_partial
    out = [fn(a, u * P.unit_terms, (u + 1) * P.unit_terms, threads=1)[0].as4() for u in range(lo, hi)]
    return torch.from_numpy(np.stack(out)) if out else torch.zeros((0, 4), dtype=torch.float64)


def tree_combine(parts, n, alg, scale=True):
    import oracle
    import paper_1606_05836_b200 as pb
    v = [oracle.DD.from4(r) for r in parts.numpy()]
    size = 1
    while size < len(v):
        size *= 2
    v += [oracle.DD(0.0, 0.0, 0.0, 0.0)] * (size - len(v))
    while len(v) > 1:
        v = [v[i] + v[i + 1] for i in range(0, len(v), 2)]
    root = v[0]
    glynn = alg in (pb.ALG_GLYNN, "glynn")
    val = (root.scaled(-(n - 1)) if glynn else root).to_complex() if scale else None
    return (torch.tensor(val, dtype=torch.complex128) if scale else None), torch.from_numpy(root.as4())
