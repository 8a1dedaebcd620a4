"""CPU oracle for the permanent hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_1606_05836_b200`` never imports it and shares no code with it (task rule ③).

The arithmetic lives in ``oracle/perm_oracle.c`` (plain C, double-double, built with
``-ffp-contract=off``); this module only marshals arguments and applies the final
factor of Eq. (2) once (reading R3 in DESIGN.md).

Functions (PAPER.md line citations in perm_oracle.c):
  naive(A)                    definition, n <= 10
  glynn(A) / ryser(A)         Gray-code walk in double-double, threaded   (Eq. 2 / Eq. 1)
  glynn_partial / ryser_partial   unscaled signed sums over [lo, hi)
  glynn_faithful / ryser_faithful Alg. A2 / A1 loop bodies literally (O(2^n n^2))
  exact(A, alg)               exact Gaussian-integer value + exactness bounds (int128)

Pins: tests/test_oracle_pins.py.  Parity unpinned: none.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "perm_oracle.c")
_LIB = os.path.join(_HERE, "libperm_oracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared",
               "-pthread", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        dp, u64, i32, i64p = ctypes.POINTER(ctypes.c_double), ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)
        _lib.oracle_naive.argtypes = [dp, i32, dp]
        _lib.oracle_glynn_faithful.argtypes = [dp, i32, u64, u64, dp]
        _lib.oracle_ryser_faithful.argtypes = [dp, i32, u64, u64, dp]
        _lib.oracle_glynn_gray.argtypes = [dp, i32, u64, u64, i32, dp, dp]
        _lib.oracle_ryser_gray.argtypes = [dp, i32, u64, u64, i32, dp, dp]
        _lib.oracle_exact_int.argtypes = [i64p, i64p, i32, i32, i64p, i64p, i64p, dp]
        _lib.oracle_gray_ex.argtypes = [dp, i32, i32, u64, u64, i32, dp, dp, dp]
        _lib.oracle_dd_add.argtypes = [dp, dp, dp]
        _lib.oracle_dd_add.restype = None
    return _lib


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _mat(A) -> tuple[np.ndarray, int]:
    a = np.ascontiguousarray(np.asarray(A, dtype=np.complex128))
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("square matrix required")
    return a, a.shape[0]


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@dataclass
class DD:
    """Complex double-double (re_hi + re_lo) + i (im_hi + im_lo)."""
    re_hi: float
    re_lo: float
    im_hi: float
    im_lo: float

    @classmethod
    def from4(cls, v) -> "DD":
        return cls(float(v[0]), float(v[1]), float(v[2]), float(v[3]))

    def as4(self) -> np.ndarray:
        return np.array([self.re_hi, self.re_lo, self.im_hi, self.im_lo], dtype=np.float64)

    def scaled(self, e: int) -> "DD":
        """Multiply by 2^e (exact barring under/overflow)."""
        return DD(np.ldexp(self.re_hi, e), np.ldexp(self.re_lo, e), np.ldexp(self.im_hi, e), np.ldexp(self.im_lo, e))

    def to_complex(self) -> complex:
        return complex(self.re_hi + self.re_lo, self.im_hi + self.im_lo)

    def exact(self) -> tuple[Fraction, Fraction]:
        return (Fraction(self.re_hi) + Fraction(self.re_lo), Fraction(self.im_hi) + Fraction(self.im_lo))

    def __add__(self, other: "DD") -> "DD":
        out = np.zeros(4)
        a, b = self.as4(), other.as4()
        _L().oracle_dd_add(_dp(a), _dp(b), _dp(out))
        return DD.from4(out)


@dataclass
class Result:
    value: complex        # rounded to complex128
    dd: DD                # scaled double-double value
    l1: float             # sum |term| * final scale (approximate)


def naive(A) -> DD:
    a, n = _mat(A)
    out = np.zeros(4)
    if _L().oracle_naive(_dp(a), n, _dp(out)) != 0:
        raise ValueError("naive oracle requires 1 <= n <= 10")
    return DD.from4(out)


def _partial(fn, A, lo, hi, threads):
    a, n = _mat(A)
    out = np.zeros(4)
    l1 = ctypes.c_double(0.0)
    rc = fn(_dp(a), n, int(lo), int(hi), int(threads or default_threads()), _dp(out), ctypes.byref(l1))
    if rc != 0:
        raise ValueError(f"bad arguments n={n} lo={lo} hi={hi}")
    return DD.from4(out), l1.value


def glynn_partial(A, lo: int, hi: int, threads: int | None = None) -> tuple[DD, float]:
    """Unscaled sum over Gray indices [lo, hi) of Eq. (2)'s numerator; also sum |term|."""
    return _partial(_L().oracle_glynn_gray, A, lo, hi, threads)


def ryser_partial(A, lo: int, hi: int, threads: int | None = None) -> tuple[DD, float]:
    """Signed sum over Gray indices [lo, hi) of Eq. (1) terms (sign (-1)^{n-|S|}); also sum |term|."""
    return _partial(_L().oracle_ryser_gray, A, lo, hi, threads)


@dataclass
class Partial:
    dd: DD        # unscaled signed sum over the range
    l1: float     # sum |term|
    l1c: float    # sum |term| * sum_i (sum_j |a_ij|) / |s_i|  (componentwise error scale)


def partial_ex(A, lo: int, hi: int, alg: str = "glynn", threads: int | None = None) -> Partial:
    """Range partial with both error scales (reading R10b)."""
    a, n = _mat(A)
    out = np.zeros(4)
    l1 = ctypes.c_double(0.0)
    l1c = ctypes.c_double(0.0)
    rc = _L().oracle_gray_ex(_dp(a), n, 1 if alg == "ryser" else 0, int(lo), int(hi),
                             int(threads or default_threads()), _dp(out), ctypes.byref(l1), ctypes.byref(l1c))
    if rc != 0:
        raise ValueError(f"bad arguments n={n} lo={lo} hi={hi}")
    return Partial(DD.from4(out), l1.value, l1c.value)


def glynn(A, threads: int | None = None) -> Result:
    a, n = _mat(A)
    d, l1 = glynn_partial(a, 0, 1 << (n - 1), threads)
    d = d.scaled(-(n - 1))                      # Eq. (2): divide once, after the full sum
    return Result(d.to_complex(), d, float(np.ldexp(l1, -(n - 1))))


def ryser(A, threads: int | None = None) -> Result:
    a, n = _mat(A)
    d, l1 = ryser_partial(a, 0, 1 << n, threads)
    return Result(d.to_complex(), d, l1)


def glynn_faithful(A, lo: int = 0, hi: int | None = None) -> DD:
    a, n = _mat(A)
    hi = (1 << (n - 1)) if hi is None else hi
    out = np.zeros(4)
    if _L().oracle_glynn_faithful(_dp(a), n, int(lo), int(hi), _dp(out)) != 0:
        raise ValueError("bad arguments")
    return DD.from4(out)


def ryser_faithful(A, lo: int = 0, hi: int | None = None) -> DD:
    a, n = _mat(A)
    hi = (1 << n) if hi is None else hi
    out = np.zeros(4)
    if _L().oracle_ryser_faithful(_dp(a), n, int(lo), int(hi), _dp(out)) != 0:
        raise ValueError("bad arguments")
    return DD.from4(out)


@dataclass
class Exact:
    value: tuple[Fraction, Fraction]   # exact perm (re, im)
    numerator: tuple[int, int]         # unscaled signed sum (Glynn: 2^{n-1} perm)
    l1: int                            # sum over terms of |Re t| + |Im t| (unscaled)
    maxprod: float                     # bound on every partial product of row sums

    def fp64_exact_eligible(self) -> bool:
        """Bit-exact class E precondition: every partial product and every
        partial sum an integer below 2^53 in magnitude."""
        return self.maxprod < 2.0 ** 53 and self.l1 < 2 ** 53


def _i128(v) -> int:
    hi, lo = int(v[0]), int(v[1]) & 0xFFFFFFFFFFFFFFFF
    return (hi << 64) | lo


def exact(A, alg: str = "glynn") -> Exact:
    """Exact permanent of an integer (Gaussian-integer) matrix via Eq. (2) or Eq. (1) in int128."""
    a, n = _mat(A)
    re = np.ascontiguousarray(np.real(a))
    im = np.ascontiguousarray(np.imag(a))
    if not (np.all(re == np.round(re)) and np.all(im == np.round(im))):
        raise ValueError("exact oracle needs integer entries")
    re_i = re.astype(np.int64)
    im_i = im.astype(np.int64)
    outr = np.zeros(2, np.int64)
    outi = np.zeros(2, np.int64)
    l1 = np.zeros(2, np.int64)
    mp = ctypes.c_double(0)
    i64p = ctypes.POINTER(ctypes.c_int64)
    rc = _L().oracle_exact_int(re_i.ctypes.data_as(i64p), im_i.ctypes.data_as(i64p), n, 1 if alg == "ryser" else 0,
                               outr.ctypes.data_as(i64p), outi.ctypes.data_as(i64p), l1.ctypes.data_as(i64p),
                               ctypes.byref(mp))
    if rc == 2:
        raise OverflowError("int128 overflow")
    if rc != 0:
        raise ValueError("bad arguments")
    num = (_i128(outr), _i128(outi))
    scale = Fraction(1, 1 << (n - 1)) if alg == "glynn" else Fraction(1)
    return Exact((num[0] * scale, num[1] * scale), num, _i128(l1), mp.value)
