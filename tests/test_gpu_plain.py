"""GPU parity of the plain-accumulation mode (PERM_ALG_GLYNN_PLAIN / PERM_ALG_RYSER_PLAIN,
SURVEY §8(f)2): the FP64 sweep with the compensation removed (the paper's
"Perm = Perm +- delta"), used for the compensated-vs-plain discrepancy.

Tolerance (reading R15): the terms are the FP64 sweep's, bounded by class B; the
accumulation is a sequence of plain additions: a thread adds its K = 2^(c + leaf_bits) terms
(in 16-term blocks) and the block / grid trees add block_bits + unit_bits more levels, so
  |plain - oracle| <= bound_B + (2^(c+leaf_bits) + block_bits + unit_bits + 16) u L1.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_1606_05836_b200 as pb
from tolerance import check_B, plain_extra

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(DEV)


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
@pytest.mark.parametrize("n", [1, 3, 6, 12, 17, 20, 23])
def test_plain_vs_oracle(n, alg):
    A = synth.gaussian(n, 6000 + n)
    a = pb._alg(alg + "_plain")
    P = pb.plan(n, a)
    part = oracle.partial_ex(A, 0, P.terms, alg)
    scale = 2.0 ** -(n - 1) if alg == "glynn" else 1.0
    ref = part.dd.to_complex() * scale
    got = complex(pb.perm_alg(T(A), a).item())
    check_B(got, part, n, P.chunk_bits, scale, ref=ref, extra=plain_extra(part, P, scale), what=f"{alg}_plain n={n}")


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
def test_plain_equals_compensated_on_exact_inputs(alg):
    """Class E inputs: every term and every partial sum is an integer below 2^53, so plain and
    compensated accumulation give the same (exact) bits."""
    for A in (synth.ones(12), synth.ones_minus_eye(13), synth.bernoulli(12, 3), synth.diag_1pi(25)):
        ex = oracle.exact(A, alg)
        if not ex.fp64_exact_eligible():
            continue
        got = complex(pb.perm_alg(T(A), alg + "_plain").item())
        assert got == complex(float(ex.value[0]), float(ex.value[1]))


@pytest.mark.parametrize("n,alg", [(22, "glynn_plain"), (21, "ryser_plain")])
def test_plain_partition_bit_identical(n, alg):
    A = T(synth.gaussian(n, 4545))
    a = pb._alg(alg)
    P = pb.plan(n, a)
    full = pb.perm_alg(A, a)
    for world in (2, 4, 8):
        roots = [pb.combine(pb.sweep_units(A, a, r * P.units // world, (r + 1) * P.units // world), n, a,
                            scale=False)[1] for r in range(world)]
        val, _ = pb.combine(torch.stack(roots), n, a, scale=True)
        assert complex(val.item()) == complex(full.item()), world


def test_plain_partials_have_zero_low_parts():
    A = T(synth.gaussian(16, 1))
    parts = pb.sweep_units(A, pb.ALG_GLYNN_PLAIN, 0, pb.plan(16, pb.ALG_GLYNN_PLAIN).units).cpu().numpy()
    assert np.all(parts[:, 1] == 0) and np.all(parts[:, 3] == 0)
