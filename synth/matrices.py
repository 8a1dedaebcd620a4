"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO permanent arithmetic: it only draws matrices.  It is the one
module both sides of the parity check may import (task rule ③).  Recipes follow
SURVEY.md §8(d) (the stand-ins for the paper's MATLAB-generated matrices,
PAPER.md:1045 "random unitary", "derived from a 100x100 matrix",
which are not available):

* ``gaussian(n, seed)``      iid (N(0,1) + i N(0,1)) / sqrt(2n)       (BASELINE configs 0, 2, 4)
* ``haar_unitary(m, seed)``  QR of a complex Gaussian, phase-fixed      (configs 1, 3)
* ``haar_submatrix``         first n columns, seeded random n rows       (configs 1, 3)
* 0/1 and structured families used as closed-form pins (PAPER.md:136 all-one,
  PAPER.md:572 diag(1+i), Bernoulli(0.5) 12x12 for the bit-exact class).

All matrices are returned as C-contiguous numpy complex128 (row-major, interleaved
re/im: the layout of ``perm_c128`` in include/permb200.h).
"""
from __future__ import annotations

import hashlib

import numpy as np

__all__ = [
    "gaussian", "haar_unitary", "haar_submatrix", "haar_batch", "ones", "ones_minus_eye",
    "eye", "bernoulli", "diag_1pi", "all_r", "rank1_factors", "block_diag", "menage",
    "x_eye_plus_ones", "random_int", "random_complex_small", "sha256", "workload",
    "WORKLOADS",
    "permutation",
]


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def gaussian(n: int, seed: int) -> np.ndarray:
    """A = (X + iY)/sqrt(2n), X then Y drawn with default_rng(seed).standard_normal((n, n))."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, n))
    y = rng.standard_normal((n, n))
    return _c128((x + 1j * y) / np.sqrt(2.0 * n))


def haar_unitary(m: int, seed: int) -> np.ndarray:
    """Haar-random m x m unitary: Z = (X+iY)/sqrt(2); Q,R = qr(Z); U = Q diag(R_kk/|R_kk|)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((m, m))
    y = rng.standard_normal((m, m))
    z = (x + 1j * y) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    d = np.diagonal(r)
    return _c128(q * (d / np.abs(d))[None, :])


def haar_submatrix(m: int, n: int, seed_u: int, seed_rows: int, u: np.ndarray | None = None) -> np.ndarray:
    """First n columns and n seeded random rows (order as drawn) of a Haar(m) unitary."""
    if u is None:
        u = haar_unitary(m, seed_u)
    rows = np.random.default_rng(seed_rows).choice(m, n, replace=False)
    return _c128(u[rows, :n])


def haar_batch(batch: int = 4096, m: int = 256, n: int = 16, seed_u: int = 16, seed_rows: int = 17) -> np.ndarray:
    """Config 1 (M2): ``batch`` n x n submatrices of one Haar(m) unitary; shape (batch, n, n)."""
    u = haar_unitary(m, seed_u)
    g = np.random.default_rng(seed_rows)
    out = np.empty((batch, n, n), dtype=np.complex128)
    for b in range(batch):
        rows = g.choice(m, n, replace=False)
        out[b] = u[rows, :n]
    return _c128(out)


def ones(n: int) -> np.ndarray:
    return _c128(np.ones((n, n)))


def ones_minus_eye(n: int) -> np.ndarray:
    return _c128(np.ones((n, n)) - np.eye(n))


def eye(n: int) -> np.ndarray:
    return _c128(np.eye(n))


def bernoulli(n: int, seed: int) -> np.ndarray:
    return _c128(np.random.default_rng(seed).integers(0, 2, (n, n)))


def diag_1pi(n: int) -> np.ndarray:
    return _c128(np.diag(np.full(n, 1 + 1j)))


def all_r(n: int, r: complex) -> np.ndarray:
    return _c128(np.full((n, n), r))


def rank1_factors(n: int, seed: int):
    """u, v with entries of modulus ~1 (unit-circle phases times 2^k-free scalars); A = outer(u, v)."""
    rng = np.random.default_rng(seed)
    u = np.exp(2j * np.pi * rng.random(n))
    v = np.exp(2j * np.pi * rng.random(n))
    return _c128(u), _c128(v)


def block_diag(a1: np.ndarray, a2: np.ndarray) -> np.ndarray:
    n1, n2 = a1.shape[0], a2.shape[0]
    out = np.zeros((n1 + n2, n1 + n2), dtype=np.complex128)
    out[:n1, :n1] = a1
    out[n1:, n1:] = a2
    return _c128(out)


def menage(n: int) -> np.ndarray:
    """J - I - P where P is the cyclic shift i -> i+1 (mod n)."""
    p = np.roll(np.eye(n), 1, axis=1)
    return _c128(np.ones((n, n)) - np.eye(n) - p)


def x_eye_plus_ones(n: int, x: int) -> np.ndarray:
    return _c128(np.ones((n, n)) + x * np.eye(n))


def random_int(n: int, seed: int, lo: int = -3, hi: int = 4, complex_: bool = True) -> np.ndarray:
    rng = np.random.default_rng(seed)
    re = rng.integers(lo, hi, (n, n))
    im = rng.integers(lo, hi, (n, n)) if complex_ else np.zeros((n, n), dtype=np.int64)
    return _c128(re + 1j * im)


def random_complex_small(n: int, seed: int) -> np.ndarray:
    """Entries uniform in [-1,1]^2 (SPEC.md:159 oracle-equivalence recipe)."""
    rng = np.random.default_rng(seed)
    return _c128(rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n)))


def permutation(count: int, seed: int) -> np.ndarray:
    """Seeded random permutation of [0, count) (int64): the "random order" of the summation-
    order experiments (Table AV) is an input, drawn here."""
    return np.random.default_rng(seed).permutation(count).astype(np.int64)


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# BASELINE.json configs -> (name, generator).  Only matrices; no permanents.
WORKLOADS = {
    "M1": dict(desc="n=20 Gaussian (N(0,1)+iN(0,1))/sqrt(2n), seed 20; Glynn+Ryser, 1 GPU", n=20,
               make=lambda: gaussian(20, 20)),
    "M2": dict(desc="4096 x (16x16) submatrices of Haar(256) (seed 16, rows seed 17); batched Glynn, 1 GPU", n=16,
               make=lambda: haar_batch(4096, 256, 16, 16, 17)),
    "M3": dict(desc="n=32 Gaussian, seed 32; Glynn+Ryser, 1 GPU", n=32, make=lambda: gaussian(32, 32)),
    "M4": dict(desc="n=40 submatrix of Haar(1600) (seed 40, rows seed 41); Glynn over 1/2/4/8 GPUs", n=40,
               make=lambda: haar_submatrix(1600, 40, 40, 41)),
    "M5": dict(desc="n=50 Gaussian, seed 50; Glynn+Ryser over 8 GPUs", n=50, make=lambda: gaussian(50, 50)),
}


def workload(name: str) -> np.ndarray:
    return WORKLOADS[name]["make"]()
