"""GPU parity of the summation-order modes of the precision lab (the paper's
Table AV), of the batched |perm|^2 output and of the
library's launch counter.

  separate   PERM_ALG_*_SEP: even- and odd-index terms summed apart in plain FP64, subtracted
             once ("(0+2+4+6)-(1+3+5+7)").  Class E inputs: exact (each sum is an integer
             below 2^53).  Otherwise: class B for the terms plus the plain-accumulation allowance
             of reading R15 for each of the two sums, plus one rounding of the difference.
  original / random   perm_sum_ordered over the 32-term chunk partials of a plain-mode sweep,
             in index order / in a seeded random permutation: a sequential sum of K partials
             adds at most K u sum|partial| <= K u L1 to the chunk errors (class B with c = 5 +
             the 32-term plain block, reading R15).
  merge      perm_combine (canonical pairwise tree) over the same plain chunk partials.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_1606_05836_b200 as pb
from tolerance import U, check_B, check_R, plain_extra

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(DEV)


def cval(t) -> complex:
    return complex(t.item())


def _exact(A, alg):
    ex = oracle.exact(A, alg)
    return ex, complex(float(ex.value[0]), float(ex.value[1]))


# ----------------------------------------------------------------- separate addition
@pytest.mark.parametrize("alg", ["glynn", "ryser"])
@pytest.mark.parametrize("name,A", [("J8", synth.ones(8)), ("J12", synth.ones(12)), ("J-I13", synth.ones_minus_eye(13)),
                                    ("bern12", synth.bernoulli(12, 1)), ("diag1i9", synth.diag_1pi(9))],
                         ids=["J8", "J12", "J-I13", "bern12", "diag1i9"])
def test_separate_exact_on_class_E(name, A, alg):
    ex, want = _exact(A, alg)
    if not ex.fp64_exact_eligible():
        pytest.skip("exactness precondition not met")
    got = cval(pb.perm_alg(T(A), alg + "_sep"))
    assert got == want, (got, want)


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
@pytest.mark.parametrize("n", [1, 2, 5, 11, 17, 21, 24])
def test_separate_vs_oracle(n, alg):
    A = synth.gaussian(n, 6100 + n)
    a = pb._alg(alg + "_sep")
    P = pb.plan(n, a)
    part = oracle.partial_ex(A, 0, P.terms, alg)
    scale = 2.0 ** -(n - 1) if alg == "glynn" else 1.0
    ref = part.dd.to_complex() * scale
    got = cval(pb.perm_alg(T(A), a))
    # each of the two plain sums carries the R15 allowance; the final subtraction rounds once
    extra = 2 * plain_extra(part, P, scale) + U * abs(ref)
    check_B(got, part, n, P.chunk_bits, scale, ref=ref, extra=extra, what=f"{alg}_sep n={n}")


@pytest.mark.parametrize("n,alg", [(22, "glynn_sep"), (23, "ryser_sep")])
def test_separate_partition_bit_identical_and_partials(n, alg):
    """(even, odd) partials of any aligned partition combine to the one-call value bit for bit;
    the partial's slots are the even and odd sums (checked against the oracle on one unit)."""
    Ah = synth.gaussian(n, 4646)
    A = T(Ah)
    a = pb._alg(alg)
    P = pb.plan(n, a)
    full = cval(pb.perm_alg(A, a))
    for world in (2, 4):
        roots = [pb.combine(pb.sweep_units(A, a, r * P.units // world, (r + 1) * P.units // world), n, a,
                            scale=False)[1] for r in range(world)]
        assert cval(pb.combine(torch.stack(roots), n, a, scale=True)[0]) == full, world
    u = P.units // 3
    d = pb.sweep_units(A, a, u, u + 1).cpu().numpy()[0]
    lo, hi = u * P.unit_terms, (u + 1) * P.unit_terms
    base = alg.split("_")[0]
    # even - odd (times the Ryser sign) is the signed partial of the unit
    part = oracle.partial_ex(Ah, lo, hi, base)
    sgn = -1.0 if (base == "ryser" and n % 2) else 1.0      # Eq. (1)'s (-1)^n on even - odd
    signed = sgn * complex(d[0] - d[1], d[2] - d[3])
    check_B(signed, part, n, P.chunk_bits, extra=2 * plain_extra(part, P) + U * abs(part.dd.to_complex()),
            what=f"{alg} unit {u}")


# ----------------------------------------------------------------- original / random / merge
def _chunk_partials(A, alg_plain, n):
    P = pb.plan(n, pb._alg(alg_plain))
    count = P.terms >> 5
    return pb.sweep_units_custom(A, alg_plain, 5, 0, 0, 0, count), count


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
@pytest.mark.parametrize("n", [6, 13, 18])
def test_ordered_sums_vs_oracle(n, alg):
    Ah = synth.gaussian(n, 6200 + n)
    A = T(Ah)
    parts, count = _chunk_partials(A, alg + "_plain", n)
    P = pb.plan(n, pb._alg(alg))
    part = oracle.partial_ex(Ah, 0, P.terms, alg)
    scale = 2.0 ** -(n - 1) if alg == "glynn" else 1.0
    ref = part.dd.to_complex() * scale
    extra = U * (count + 32 + 16) * part.l1 * scale
    ident = torch.arange(count, dtype=torch.int64, device=DEV)
    rnd = torch.from_numpy(synth.permutation(count, 1606 + n)).to(DEV)
    for name, order in (("original", ident), ("random", rnd)):
        got = cval(pb.sum_ordered(parts, order, n, alg + "_plain"))
        check_B(got, part, n, 5, scale, ref=ref, extra=extra, what=f"{alg} {name} n={n}")
    merged = cval(pb.combine(parts, n, alg + "_plain")[0])
    check_B(merged, part, n, 5, scale, ref=ref, extra=extra, what=f"{alg} merge n={n}")


def test_ordered_sum_exact_on_class_E_and_order_matters():
    """Integer terms below 2^53: every order gives the exact value.  J_24 Ryser (terms up to
    24^24, far beyond 2^53): the identity and a random order give different roundings."""
    A = synth.ones(12)
    ex, want = _exact(A, "ryser")
    assert ex.fp64_exact_eligible()
    parts, count = _chunk_partials(T(A), "ryser_plain", 12)
    for seed in (1, 2):
        order = torch.from_numpy(synth.permutation(count, seed)).to(DEV)
        assert cval(pb.sum_ordered(parts, order, 12, "ryser_plain")) == want
    parts, count = _chunk_partials(T(synth.ones(24)), "ryser_plain", 24)
    ident = cval(pb.sum_ordered(parts, torch.arange(count, dtype=torch.int64, device=DEV), 24, "ryser_plain"))
    rnd = cval(pb.sum_ordered(parts, torch.from_numpy(synth.permutation(count, 3)).to(DEV), 24, "ryser_plain"))
    assert ident != rnd


def test_ordered_sum_bad_arguments():
    parts = torch.zeros((4, 4), dtype=torch.float64, device=DEV)
    with pytest.raises(TypeError):
        pb.sum_ordered(parts, torch.arange(3, dtype=torch.int64, device=DEV), 4, "glynn")
    with pytest.raises(TypeError):
        pb.sum_ordered(parts, torch.arange(4, dtype=torch.int32, device=DEV), 4, "glynn")


# ----------------------------------------------------------------- |perm|^2 (boson sampling)
def test_batched_abs2_vs_oracle_and_values():
    As = synth.haar_batch(512, 256, 16, 16, 17)
    dA = T(As)
    p2 = pb.glynn_batched_abs2(dA).cpu().numpy()
    vals = pb.glynn_batched(dA).cpu().numpy()
    assert np.allclose(p2, vals.real ** 2 + vals.imag ** 2, rtol=4 * U, atol=0)
    for b in range(0, 512, 37):
        ref = oracle.glynn(As[b]).value
        check_R(complex(p2[b]), abs(ref) ** 2, tol=3e-9, what=f"abs2 item {b}")
    host = pb.glynn_batched_abs2_host(As[:7])
    assert np.array_equal(host, p2[:7])
    assert pb.glynn_batched_abs2(torch.zeros((0, 5, 5), dtype=torch.complex128, device=DEV)).shape == (0,)


def test_batched_abs2_exact_on_integers():
    As = np.stack([synth.bernoulli(12, s) for s in range(4)] + [synth.ones(12), synth.ones_minus_eye(12)])
    p2 = pb.glynn_batched_abs2(T(As)).cpu().numpy()
    for b in range(As.shape[0]):
        ex = oracle.exact(As[b]).value
        assert p2[b] == float(ex[0]) ** 2 + float(ex[1]) ** 2


# ----------------------------------------------------------------- launch counter
def test_launch_count_matches_the_path():
    A = T(synth.gaussian(30, 1))
    torch.cuda.synchronize()
    k0 = pb.launch_count()
    pb.glynn(A)                      # 2^29 terms: column staging + sweep + combine
    assert pb.launch_count() - k0 == 3
    k0 = pb.launch_count()
    pb.glynn(T(synth.gaussian(16, 2)))   # small n: one fused cooperative launch
    assert pb.launch_count() - k0 == 1
    k0 = pb.launch_count()
    pb.glynn_batched(T(np.stack([synth.gaussian(8, s) for s in range(5)])))
    assert pb.launch_count() - k0 == 1


# ----------------------------------------------------------------- Table AV rows (Ryser on J_N)
@pytest.mark.parametrize("N", [8, 13, 14, 17, 20])
def test_table_av_J_N_all_orders_vs_oracle(N):
    """The four summation orders of Table AV on Ryser J_N against the exact N!
    (oracle.exact / int128 up to its range, else the oracle's dd walk): exact while every term
    and partial sum stays an integer below 2^53 (N <= 13), within the walk-aware bound plus the
    order's accumulation allowance beyond."""
    A = synth.ones(N)
    dA = T(A)
    P = pb.plan(N, pb.ALG_RYSER)
    part = oracle.partial_ex(A, 0, P.terms, "ryser")
    ref = float(math.factorial(N))
    assert abs(part.dd.to_complex() - ref) <= 1e-20 * ref        # the oracle walk itself: exact here
    parts, count = _chunk_partials(dA, "ryser_plain", N)
    rows = {
        "original": cval(pb.sum_ordered(parts, torch.arange(count, dtype=torch.int64, device=DEV), N, "ryser_plain")),
        "random": cval(pb.sum_ordered(parts, torch.from_numpy(synth.permutation(count, 977 + N)).to(DEV), N,
                                      "ryser_plain")),
        "merge": cval(pb.combine(parts, N, "ryser_plain")[0]),
        "separate": cval(pb.perm_alg(dA, "ryser_sep")),
    }
    Ps = pb.plan(N, pb.ALG_RYSER_SEP)
    for name, got in rows.items():
        if N <= 13:
            assert got == ref, (name, got)
            continue
        extra = U * (count + 48) * part.l1 if name != "separate" else 2 * plain_extra(part, Ps) + U * ref
        c = 5 if name != "separate" else Ps.chunk_bits
        check_B(got, part, N, c, ref=complex(ref), extra=extra, what=f"J_{N} {name}")
