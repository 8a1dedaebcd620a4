"""Pins for the CPU oracle (task rule ③): the oracle is checked against things other
than itself — hand values, brute force over permutations in exact Python arithmetic,
closed forms of the permanent, algebraic invariants, and the values the paper prints.

Each pin is chosen so a plausible oracle mistake (a dropped term, a wrong sign or
index, a transposed operand, a missing/doubled final factor) fails one of them.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- exact brute force
def _brute_exact(A):
    """Definition (PAPER.md:60 notation): sum over permutations, exact rationals."""
    n = A.shape[0]
    ent = [[(Fraction(float(A[i, j].real)), Fraction(float(A[i, j].imag))) for j in range(n)] for i in range(n)]
    tr, ti = Fraction(0), Fraction(0)
    for perm in itertools.permutations(range(n)):
        pr, pi = Fraction(1), Fraction(0)
        for i, j in enumerate(perm):
            ar, ai = ent[i][j]
            pr, pi = pr * ar - pi * ai, pr * ai + pi * ar
        tr += pr
        ti += pi
    return tr, ti


def _fr(x: float) -> Fraction:
    return Fraction(float(x))


def _dd_err(dd: oracle.DD, exact, scale=Fraction(1)):
    er, ei = dd.exact()
    return max(abs(er * scale - exact[0]), abs(ei * scale - exact[1]))


def _mag(exact):
    return float(abs(exact[0]) + abs(exact[1]))


# ----------------------------------------------------------------- hand values
def test_hand_values():
    # S:120 [[1,2],[3,4]] -> 1*4 + 2*3 = 10 ; [[2]] -> 2 ; [[1,2,3],[4,5,6],[7,8,9]] -> 450 by cofactor expansion
    assert oracle.naive([[1, 2], [3, 4]]).to_complex() == 10
    assert oracle.naive([[2]]).to_complex() == 2
    assert oracle.naive(np.arange(1, 10).reshape(3, 3)).to_complex() == 450
    for fn in (oracle.glynn, oracle.ryser):
        assert fn([[1, 2], [3, 4]]).value == 10
        assert fn(np.arange(1, 10).reshape(3, 3)).value == 450
        assert fn([[2 + 3j]]).value == 2 + 3j
    # perm of a 2x2 complex: a11 a22 + a12 a21
    a = np.array([[1 + 2j, 3 - 1j], [0.5j, -2 + 1j]])
    want = a[0, 0] * a[1, 1] + a[0, 1] * a[1, 0]
    assert abs(oracle.glynn(a).value - want) < 1e-15
    assert abs(oracle.ryser(a).value - want) < 1e-15


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (3, 2), (4, 3), (5, 4), (6, 5)])
def test_naive_vs_bruteforce_integer(n, seed):
    A = synth.random_int(n, seed)
    want = _brute_exact(A)
    got = oracle.naive(A).exact()
    assert got == want
    for alg in ("glynn", "ryser"):
        ex = oracle.exact(A, alg)
        assert ex.value == want


@pytest.mark.parametrize("n,seed", [(3, 10), (4, 11), (5, 12), (6, 13)])
def test_all_oracles_vs_bruteforce_float(n, seed):
    A = synth.random_complex_small(n, seed)
    want = _brute_exact(A)
    tol = 1e-28 * math.factorial(n) * 4 ** n  # dd rounding budget, far below fp64 noise
    assert _dd_err(oracle.naive(A), want) < tol
    n1 = n - 1
    assert _dd_err(oracle.glynn(A).dd, want) < tol
    assert _dd_err(oracle.glynn_faithful(A), want, Fraction(1, 1 << n1)) < tol
    assert _dd_err(oracle.ryser(A).dd, want) < tol
    assert _dd_err(oracle.ryser_faithful(A), want) < tol


# ----------------------------------------------------------------- closed forms, exact int oracle
def _derangements(n):
    d = [1, 0]
    for k in range(2, n + 1):
        d.append((k - 1) * (d[-1] + d[-2]))
    return d[n]


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
def test_exact_closed_forms(alg):
    for n in range(1, 19):
        assert oracle.exact(synth.ones(n), alg).value == (math.factorial(n), 0)      # P:136 perm(J_N) = N!
        assert oracle.exact(synth.eye(n), alg).value == (1, 0)
        assert oracle.exact(synth.ones_minus_eye(n), alg).value == (_derangements(n), 0)
        d = oracle.exact(synth.diag_1pi(n), alg).value                              # P:572 (1+i)^N
        z = (1 + 1j) ** n
        assert d == (int(z.real), int(z.imag))
    # D_20 = 895014631192902121 (odd, not representable in fp64: exact-int oracle only)
    assert oracle.exact(synth.ones_minus_eye(20), alg).value == (895014631192902121, 0)
    # menage numbers (OEIS A000179) for n = 3..8
    for n, u in zip(range(3, 9), [1, 2, 13, 80, 579, 4738]):
        assert oracle.exact(synth.menage(n), alg).value == (u, 0)
    # perm(J + xI) = sum_k C(n,k) D_{n-k} (1+x)^k
    for n in (5, 9, 12):
        for x in (1, 2, -3):
            want = sum(math.comb(n, k) * _derangements(n - k) * (1 + x) ** k for k in range(n + 1))
            assert oracle.exact(synth.x_eye_plus_ones(n, x), alg).value == (want, 0)


def test_exact_glynn_sign_and_term_count():
    """J_n: every Glynn term is (sum delta)^n with sign prod delta; l1 = sum_j C(n-1,j)|n-2j|^n
    and the numerator is 2^{n-1} n!. Fails for a wrong delta_1 convention, a missing sign,
    or a term counted twice / skipped."""
    for n in range(1, 17):
        ex = oracle.exact(synth.ones(n), "glynn")
        assert ex.numerator == (math.factorial(n) << (n - 1), 0)
        assert ex.l1 == sum(math.comb(n - 1, j) * abs(n - 2 * j) ** n for j in range(n))
        exr = oracle.exact(synth.ones(n), "ryser")
        assert exr.l1 == sum(math.comb(n, k) * k ** n for k in range(n + 1))


def test_exact_glynn_equals_ryser_bernoulli():
    for s in range(5):
        A = synth.bernoulli(12, s)
        g, r = oracle.exact(A, "glynn"), oracle.exact(A, "ryser")
        assert g.value == r.value
        assert g.fp64_exact_eligible() and r.fp64_exact_eligible()
    for s in range(3):
        A = synth.random_int(9, 100 + s)
        assert oracle.exact(A, "glynn").value == oracle.exact(A, "ryser").value


def test_exact_row_scaling_transpose_permutation():
    rng = np.random.default_rng(7)
    A = synth.random_int(8, 42)
    base = oracle.exact(A).value
    assert oracle.exact(A.T.copy()).value == base                       # S:162 transpose
    p = rng.permutation(8)
    assert oracle.exact(A[p].copy()).value == base                      # row permutation
    assert oracle.exact(A[:, p].copy()).value == base                   # column permutation
    B = A.copy()
    B[3] *= (2 - 1j)                                                    # S:163 row scaling by c
    br, bi = base
    assert oracle.exact(B).value == (br * 2 + bi * 1, bi * 2 - br * 1)


# ----------------------------------------------------------------- double-double oracle vs exact
@pytest.mark.parametrize("A", [synth.ones(20), synth.ones_minus_eye(20)], ids=["J20", "J20-I"])
def test_dd_glynn_exact_on_integer_20(A):
    ex = oracle.exact(A, "glynn")
    got = oracle.glynn(A).dd.exact()
    assert got == ex.value        # 20! and D_20 reproduced exactly in double-double


def test_dd_exact_on_bernoulli_and_int():
    for s in range(5):
        A = synth.bernoulli(12, s)
        ex = oracle.exact(A, "glynn").value
        assert oracle.glynn(A).dd.exact() == ex
        assert oracle.ryser(A).dd.exact() == ex
    for s in range(3):
        A = synth.random_int(11, 200 + s)
        ex = oracle.exact(A, "glynn").value
        assert oracle.glynn(A).dd.exact() == ex
        assert oracle.ryser(A).dd.exact() == ex


@pytest.mark.parametrize("n", [8, 11, 13])
def test_gray_walk_equals_faithful(n):
    """Gray-code walk (north_star order) vs Alg. A1/A2 literal loops (fresh sums per iter)."""
    A = synth.gaussian(n, 300 + n)
    g = oracle.glynn_partial(A, 0, 1 << (n - 1))[0]
    f = oracle.glynn_faithful(A)
    r = oracle.ryser_partial(A, 0, 1 << n)[0]
    rf = oracle.ryser_faithful(A)
    l1 = oracle.glynn(A).l1 * 2 ** (n - 1)
    assert abs(g.to_complex() - f.to_complex()) <= 1e-26 * l1
    assert abs(r.to_complex() - rf.to_complex()) <= 1e-24 * oracle.ryser(A).l1
    # an aligned Gray block [q 2^k, (q+1) 2^k) enumerates exactly the codes x with
    # x >> k == G(q) (G(g) >> k == G(g >> k)), i.e. the ascending iter block [G(q) 2^k, (G(q)+1) 2^k)
    k = 4
    for q in (1, 2, 5, (1 << (n - 1 - k)) - 1):
        gq = q ^ (q >> 1)
        gp = oracle.glynn_partial(A, q << k, (q + 1) << k)[0].to_complex()
        fp = oracle.glynn_faithful(A, gq << k, (gq + 1) << k).to_complex()
        assert abs(gp - fp) <= 1e-26 * l1


@pytest.mark.parametrize("n", [10, 16, 20])
def test_dd_glynn_vs_ryser_random(n):
    A = synth.gaussian(n, 500 + n)
    g = oracle.glynn(A)
    r = oracle.ryser(A)
    assert abs(g.value - r.value) <= 1e-24 * r.l1 + 1e-28 * g.l1
    assert abs(g.value - r.value) <= 1e-13 * abs(g.value)


def test_dd_matches_naive_n9():
    A = synth.gaussian(9, 77)
    nv = oracle.naive(A)
    assert abs(oracle.glynn(A).value - nv.to_complex()) <= 1e-15 * abs(nv.to_complex())
    assert abs(oracle.ryser(A).value - nv.to_complex()) <= 1e-15 * abs(nv.to_complex())


# ----------------------------------------------------------------- closed forms with complex values
@pytest.mark.parametrize("n", [6, 12, 16])
def test_rank1_closed_form(n):
    """perm(u v^T) = n! prod u_i prod v_j (every permutation contributes the same product)."""
    u, v = synth.rank1_factors(n, 900 + n)
    A = np.outer(u, v)
    mpmath.mp.prec = 200
    # the matrix actually stored is fl(u_i v_j); the closed form holds for the rounded entries
    # only approximately, so compare at the fp64-input-rounding scale: n! * 2n * u
    want = mpmath.factorial(n) * mpmath.fprod([mpmath.mpc(x) for x in u]) * mpmath.fprod([mpmath.mpc(x) for x in v])
    got = oracle.glynn(A).value
    assert abs(complex(want) - got) <= math.factorial(n) * 4 * n * 2 ** -53
    got_r = oracle.ryser(A).value
    assert abs(complex(want) - got_r) <= math.factorial(n) * 4 * n * 2 ** -53


def test_rank1_exact_integer():
    u = np.array([1, 2, -1, 3, 1, -2, 1, 1], dtype=complex)
    v = np.array([2, 1j, 1, -1, 1 + 1j, 1, -1j, 1], dtype=complex)
    A = np.outer(u, v)
    want = math.factorial(8) * np.prod(u) * np.prod(v)
    ex = oracle.exact(A).value
    assert ex == (int(want.real), int(want.imag))


@pytest.mark.parametrize("r", [1.0, 0.1, 0.2, 10.0, 1 + 1j, 10 + 10j])
def test_all_r_closed_form(r):
    """Tables AI-AIV: perm of the all-r matrix is r^N N!."""
    n = 14
    A = synth.all_r(n, r)
    rr = complex(A[0, 0])
    fr = (_fr(rr.real), _fr(rr.imag))
    # exact (r)^n for the stored r
    pr, pi = Fraction(1), Fraction(0)
    for _ in range(n):
        pr, pi = pr * fr[0] - pi * fr[1], pr * fr[1] + pi * fr[0]
    want = (pr * math.factorial(n), pi * math.factorial(n))
    assert _dd_err(oracle.glynn(A).dd, want) <= 1e-27 * _mag(want) * 2 ** n
    assert _dd_err(oracle.ryser(A).dd, want) <= 1e-27 * _mag(want) * 2 ** (2 * n)


def test_block_diagonal_product():
    A1 = synth.gaussian(6, 1)
    A2 = synth.gaussian(7, 2)
    A = synth.block_diag(A1, A2)
    want = oracle.naive(A1).to_complex() * oracle.naive(A2).to_complex()
    assert abs(oracle.glynn(A).value - want) <= 1e-14 * abs(want)
    assert abs(oracle.ryser(A).value - want) <= 1e-13 * abs(want)


def test_float_invariants():
    A = synth.gaussian(12, 5)
    base = oracle.glynn(A)
    tol = 1e-25 * base.l1
    p = np.random.default_rng(3).permutation(12)
    assert abs(oracle.glynn(A.T.copy()).value - base.value) <= tol + 1e-16 * abs(base.value)
    assert abs(oracle.glynn(A[p].copy()).value - base.value) <= tol + 1e-16 * abs(base.value)
    assert abs(oracle.glynn(A[:, p].copy()).value - base.value) <= tol + 1e-16 * abs(base.value)
    assert oracle.glynn(np.conj(A)).value == np.conj(base.value)
    assert oracle.glynn(-A).value == base.value                     # (-1)^12
    B = A.copy()
    B[4] *= 1j
    assert abs(oracle.glynn(B).value - 1j * base.value) <= tol + 1e-16 * abs(base.value)


def test_range_partition_complete():
    """every sign vector counted exactly once; sum of partials over any split == whole."""
    n = 15
    A = synth.gaussian(n, 9)
    T = 1 << (n - 1)
    whole = oracle.glynn_partial(A, 0, T)[0]
    cuts = [0, 1, 2, 777, 4096, 9999, T]
    acc = None
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        d = oracle.glynn_partial(A, lo, hi, threads=3)[0]
        acc = d if acc is None else acc + d
    assert abs(acc.to_complex() - whole.to_complex()) <= 1e-28 * oracle.glynn(A).l1 * T
    # an empty range contributes exactly zero
    assert oracle.glynn_partial(A, 5, 5)[0].to_complex() == 0
    # Ryser's empty set term is exactly 0: [0,1) sums to zero
    assert oracle.ryser_partial(A, 0, 1)[0].to_complex() == 0


def test_thread_count_does_not_change_value_materially():
    A = synth.gaussian(16, 11)
    a = oracle.glynn(A, threads=1)
    b = oracle.glynn(A, threads=7)
    assert abs(a.value - b.value) <= 1e-28 * a.l1 * 2 ** 15


# ----------------------------------------------------------------- values printed in the paper
def test_paper_table_values():
    """tests/golden/paper_values.json: Theor. Value columns of Table AI and
    the FIG. A3 diag(1+i) statement, to the printed 3 significant figures."""
    with open(os.path.join(GOLDEN, "paper_values.json")) as f:
        rows = json.load(f)["bbfg_all_r"]
    for row in rows:
        n, r, printed = row["N"], row["r"], row["theor"]
        if n > 20:
            continue
        got = oracle.glynn(synth.all_r(n, r)).value.real
        assert float(f"{got:.2E}") == printed, (n, r, got, printed)


def test_paper_diag_1pi_45_term_identity():
    """perm(diag(1+i)_45) = (1+i)^45 = -2^22 - 2^22 i.  The full walk (2^44 terms) is
    too long for the CPU, but every Glynn term of a diagonal matrix equals (1+i)^n, so any
    sub-range sums to (#terms) (1+i)^n exactly — checked here on a 4096-term window."""
    n = 45
    A = synth.diag_1pi(n)
    lo, hi = (1 << 40) + 12345, (1 << 40) + 12345 + 4096
    d = oracle.glynn_partial(A, lo, hi, threads=2)[0]
    assert d.exact() == (Fraction(-(hi - lo) * 2 ** 22), Fraction(-(hi - lo) * 2 ** 22))
    assert (1 + 1j) ** 45 == complex(-2 ** 22, -2 ** 22)


# ----------------------------------------------------------------- error scales L1 and L1c
# oracle.partial_ex returns, besides the value, the two error scales every class-B tolerance
# is built from (reading R10b; tests/tolerance.py):
#   L1  = sum over the walked terms of |term|
#   L1c = sum over the walked terms of |term| * sum_i (sum_j |a_ij|) / |s_i|
# (s_i the row sums of that term).  Pinned here against closed forms and an independent
# brute-force enumeration (ascending delta / subset order, numpy arithmetic, no Gray walk),
# so a mistake in them cannot silently loosen or tighten the GPU parity checks.

def _l1_closed_J(n: int, alg: str) -> tuple[int, Fraction]:
    """J_n: Glynn terms with k of delta_2..delta_n = -1 have every row sum n - 2k (C(n-1, k) of
    them); Ryser subsets of size k have every row sum k (C(n, k) of them).  Row abs sum = n."""
    l1, l1c = 0, Fraction(0)
    if alg == "glynn":
        for k in range(n):
            s = abs(n - 2 * k)
            l1 += math.comb(n - 1, k) * s ** n
            if s:
                l1c += math.comb(n - 1, k) * Fraction(s ** n * n * n, s)
    else:
        for k in range(1, n + 1):
            l1 += math.comb(n, k) * k ** n
            l1c += math.comb(n, k) * Fraction(k ** n * n * n, k)
    return l1, l1c


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
@pytest.mark.parametrize("n", [1, 2, 5, 9, 14, 20])
def test_error_scales_J_closed_form(n, alg):
    T = 1 << (n - 1 if alg == "glynn" else n)
    part = oracle.partial_ex(synth.ones(n), 0, T, alg)
    l1, l1c = _l1_closed_J(n, alg)
    tol = T * 2.0 ** -53 + 1e-14          # the scales are plain FP64 sums over T terms
    assert part.l1 == pytest.approx(float(l1), rel=tol)
    assert part.l1c == pytest.approx(float(l1c), rel=tol)
    if alg == "glynn" and n > 1:
        # the 2^-(n-1) scale is applied to L1 where glynn() applies it to the value
        assert oracle.glynn(synth.ones(n)).l1 == pytest.approx(float(l1) / 2 ** (n - 1), rel=tol)


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
@pytest.mark.parametrize("n", [1, 4, 11, 30])
def test_error_scales_diag_closed_form(n, alg):
    """diag(d), d_i != 0: Glynn row sums are delta_i d_i, every one of the 2^(n-1) terms has
    modulus prod |d_i| and kappa = sum_i |d_i| / |d_i| = n;  Ryser: only S = all columns gives a
    non-zero term.  So L1c = n L1 exactly in both."""
    rng = np.random.default_rng(n)
    d = (rng.uniform(0.5, 2.0, n) * np.exp(1j * rng.uniform(0, 2 * np.pi, n)))
    A = np.diag(d)
    T = 1 << (n - 1 if alg == "glynn" else n)
    lo, hi = 0, T
    if T > 1 << 20 and alg == "glynn":
        lo, hi = T - (1 << 16), T
    elif T > 1 << 20:
        # a window holding the full set for Ryser: Gray index g with G(g) = 2^n - 1
        g, code = 0, (1 << n) - 1
        while code:
            g ^= code
            code >>= 1
        lo, hi = max(0, g - (1 << 15)), min(T, g + (1 << 15))
    part = oracle.partial_ex(A, lo, hi, alg)
    prod = float(np.prod(np.abs(d)))
    want = (hi - lo) * prod if alg == "glynn" else prod
    assert part.l1 == pytest.approx(want, rel=1e-12)
    assert part.l1c == pytest.approx(n * want, rel=1e-12)


@pytest.mark.parametrize("A,alg", [(synth.ones_minus_eye(9), "glynn"), (synth.ones_minus_eye(9), "ryser"),
                                   (synth.bernoulli(12, 2), "glynn"), (synth.bernoulli(12, 2), "ryser"),
                                   (synth.random_int(10, 3, complex_=False), "glynn")],
                         ids=["J-I9g", "J-I9r", "bern12g", "bern12r", "rint10g"])
def test_error_scales_L1_equals_exact_int(A, alg):
    """On real integer matrices the exact-int128 oracle's L1 (sum |Re t| + |Im t|) is the
    walk's L1 (sum |t|), computed independently and exactly."""
    n = A.shape[0]
    T = 1 << (n - 1 if alg == "glynn" else n)
    part = oracle.partial_ex(A, 0, T, alg)
    ex = oracle.exact(A, alg)
    assert part.l1 == pytest.approx(float(ex.l1), rel=1e-13)


def _brute_scales(A, alg):
    """Independent enumeration (ascending delta / subset index, numpy complex arithmetic)."""
    n = A.shape[0]
    rowabs = np.abs(A).sum(axis=1)
    l1 = l1c = 0.0
    if alg == "glynn":
        for m in range(1 << (n - 1)):
            delta = np.array([1.0] + [-1.0 if (m >> (j - 1)) & 1 else 1.0 for j in range(1, n)])
            s = A @ delta
            t = abs(np.prod(s))
            l1 += t
            if t > 0:
                l1c += t * float(np.sum(rowabs / np.abs(s)))
    else:
        for m in range(1 << n):
            sel = np.array([1.0 if (m >> j) & 1 else 0.0 for j in range(n)])
            s = A @ sel
            t = abs(np.prod(s))
            l1 += t
            if t > 0:
                l1c += t * float(np.sum(rowabs / np.abs(s)))
    return l1, l1c


@pytest.mark.parametrize("alg", ["glynn", "ryser"])
@pytest.mark.parametrize("n,seed", [(3, 1), (6, 2), (9, 3)])
def test_error_scales_bruteforce(n, seed, alg):
    A = synth.gaussian(n, 700 + seed)
    T = 1 << (n - 1 if alg == "glynn" else n)
    part = oracle.partial_ex(A, 0, T, alg)
    l1, l1c = _brute_scales(A, alg)
    assert part.l1 == pytest.approx(l1, rel=1e-10)
    assert part.l1c == pytest.approx(l1c, rel=1e-10)
    # every row sum is bounded by its row's abs sum, so each kappa term is >= n
    assert part.l1c >= n * part.l1 * (1 - 1e-12)


def test_error_scales_additive_over_ranges():
    """L1 and L1c of a range are sums over its terms: additive over any split."""
    A = synth.gaussian(12, 5)
    full = oracle.partial_ex(A, 0, 1 << 11)
    a, b = oracle.partial_ex(A, 0, 777), oracle.partial_ex(A, 777, 1 << 11)
    assert a.l1 + b.l1 == pytest.approx(full.l1, rel=1e-13)
    assert a.l1c + b.l1c == pytest.approx(full.l1c, rel=1e-13)
