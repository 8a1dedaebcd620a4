"""The warp-pair row-split sweep (paper_1606_05836_b200/csrc/perm_kernels_wsplit.cuh), the FP64
sweep of the canonical plan from n = 52 (4 terms per exchange up to n = 59, 2 from n = 60; Eq. (2), Eq. (1); SURVEY §8 a3/a4 "row
sums kept in registers for n <= 64"): each chunk's row sums live in lane l of a PAIR of warps and
the two half products meet through shared memory.

  * fast-path units anywhere in the Gray range vs the oracle, Glynn and Ryser, both parities of
    n (odd n: the two warps hold ceil(n/2) and floor(n/2) rows), c = 4 (the shortest fast
    chunk: 2 exchange iterations per half-walk) and c = 11;
  * a unit's partial does not depend on the launch it is part of (bit-identical);
  * a range with ragged ends around whole canonical units: the launcher's split into the
    one-lane generic kernel (ends) and the warp-pair kernel (interior) with the partials
    written at the right offsets -- the range value equals the canonical combination of its
    ragged ends (vs the oracle) and the interior units' partials.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_1606_05836_b200 as pb
from tolerance import check_B

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(DEV)


def _c(d):
    d = np.asarray(d)
    return complex(d[0] + d[1], d[2] + d[3])


@pytest.mark.parametrize("n,alg", [(52, "glynn"), (53, "glynn"), (53, "ryser"), (58, "glynn"), (59, "ryser"),
                                   (60, "glynn"), (63, "ryser"), (64, "glynn")])
def test_wsplit_fast_units_vs_oracle(n, alg):
    A = synth.gaussian(n, 9700 + n)
    dA = T(A)
    a = pb._alg(alg)
    P = pb.plan(n, a)
    assert P.lanes == 2 and P.block_bits == 6
    m = P.log2_terms
    for c in (4, 11):
        wb = 6
        lam = max(0, m - c - wb - 40)    # the custom-plan API allows at most 2^40 units
        units = 1 << (m - c - wb - lam)
        for u in (sorted({0, units // 3 + 1, units - 1}) if lam == 0 else (1, units - 1)):
            got = pb.sweep_units_custom(dA, a, c, lam, wb, u, u + 1).cpu().numpy()[0]
            lo, hi = u << (c + wb + lam), (u + 1) << (c + wb + lam)
            part = oracle.partial_ex(A, lo, hi, alg)
            check_B(_c(got), part, n, c, what=f"wsplit {alg} n={n} c={c} unit {u}")


def test_wsplit_unit_partials_independent_of_launch():
    n = 55
    A = T(synth.gaussian(n, 4455))
    c, lam, wb = 5, 3, 6                  # 2^(54 - 14) = 2^40 units: the custom-plan API's maximum
    whole = pb.sweep_units_custom(A, pb.ALG_GLYNN, c, lam, wb, 100, 164).cpu().numpy()
    for lo, hi in ((100, 101), (131, 164), (150, 151)):
        part = pb.sweep_units_custom(A, pb.ALG_GLYNN, c, lam, wb, lo, hi).cpu().numpy()
        assert np.array_equal(part, whole[lo - 100:hi - 100]), (lo, hi)
    # repeated launches: deterministic
    again = pb.sweep_units_custom(A, pb.ALG_GLYNN, c, lam, wb, 100, 164).cpu().numpy()
    assert np.array_equal(again, whole)


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
def test_wsplit_range_with_ragged_ends(alg):
    n = 52
    A = synth.gaussian(n, 5252)
    dA = T(A)
    a = pb._alg(alg)
    P = pb.plan(n, a)
    UT, chunk = P.unit_terms, 1 << P.chunk_bits
    u = 5
    lo, hi = u * UT - 3 * chunk - 5, (u + 2) * UT + 2 * chunk + 7
    fn = pb.glynn_range if alg == "glynn" else pb.ryser_range
    got = _c(fn(dA, lo, hi).cpu().numpy())
    left_d = fn(dA, lo, u * UT).cpu().numpy()
    right_d = fn(dA, (u + 2) * UT, hi).cpu().numpy()
    inner = pb.sweep_units(dA, a, u, u + 2).cpu().numpy()
    # the ragged ends against the oracle
    for (x, y), d in (((lo, u * UT), left_d), (((u + 2) * UT, hi), right_d)):
        part = oracle.partial_ex(A, x, y, alg)
        check_B(_c(d), part, n, P.chunk_bits, what=f"{alg} ragged [{x},{y})")
    # the range = its 4 unit partials (ragged, interior, interior, ragged), combined in dd
    terms = [_c(left_d), _c(inner[0]), _c(inner[1]), _c(right_d)]
    want = sum(terms)
    scale = sum(abs(t) for t in terms)
    assert abs(got - want) <= 1e-15 * scale, (got, want)
