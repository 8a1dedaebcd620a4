"""GPU precision probes with closed-form values (SURVEY §8(c) class P, §8(f)2; PAPER.md
"Precision Performance" P:134-163, Tables AI-AIV): all-r matrices, perm = r^N N!
exactly (for the double nearest r).  The full sweep is tools/precision_lab.py
(profiles/r01_precision/); these are the pinned cases."""
import math
from fractions import Fraction

import pytest
import torch

import paper_1606_05836_b200 as pb

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def theor(r: complex, n: int) -> complex:
    re, im = Fraction(float(r.real)), Fraction(float(r.imag))
    pr, pi = Fraction(1), Fraction(0)
    for _ in range(n):
        pr, pi = pr * re - pi * im, pr * im + pi * re
    f = math.factorial(n)
    return complex(float(pr * f), float(pi * f))


def rel(a: complex, b: complex) -> float:
    return abs(a - b) / abs(b)


@pytest.mark.parametrize("r", [1.0, 0.1, 1 + 1j, 10 + 10j])
@pytest.mark.parametrize("n", [24, 30])
def test_all_r_glynn_fp64_and_dd(r, n):
    A = torch.full((n, n), complex(r), dtype=torch.complex128, device=DEV)
    t = theor(complex(r), n)
    assert rel(complex(pb.glynn(A).item()), t) <= 1e-9          # BB/FG is trustworthy
    assert rel(pb.dd_to_complex(pb.glynn_dd(A)), t) <= 1e-20


@pytest.mark.parametrize("r", [1.0, 1 + 1j])
def test_ryser_fp64_breaks_down_dd_does_not(r):
    """The paper's finding (FIG. 4): FP64 Ryser on J_N loses all accuracy by N ~ 32
    (paper: 100.95 % at N = 32) while BB/FG stays accurate; the dd mode restores Ryser."""
    n = 32
    A = torch.full((n, n), complex(r), dtype=torch.complex128, device=DEV)
    t = theor(complex(r), n)
    e_ryser = rel(complex(pb.ryser(A).item()), t)
    e_glynn = rel(complex(pb.glynn(A).item()), t)
    assert e_ryser > 1e-3 and e_glynn < 1e-10
    assert rel(pb.dd_to_complex(pb.ryser_dd(A)), t) <= 1e-12
