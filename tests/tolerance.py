"""Tolerance classes of the GPU parity tests (readings R10b, R14, R15),
in one place, with two guards that keep the class-B bound from going vacuous:

  * every class-B comparison is recorded (err / bound, bound / |ref|, the bound factor
    bound / (u L1)); conftest.py prints the worst ratios per test at the end of the session
    and writes them as JSON when PERMB200_TOL_REPORT names a file;
  * the bound is asserted below stated ceilings:
      - L1c <= L1C_MAX_PER_N * n * L1  (measured l1c / (n l1): 2 .. 16 on Gaussian inputs up to
        n = 50, tests/test_oracle_pins.py pins L1 and L1c themselves against closed forms),
      - bound / |ref| <= `rel_ceiling` where a test states one (full permanents: Glynn 1e-7,
        Ryser 1e-3 -- measured worst 1.1e-9 / 1.5e-5 for the test matrices).

Class B (reading R10b):  |gpu - oracle| <= u [ (sqrt(n) + 2^(c/2)) L1c + (3n + 16) L1 ] * scale
Class Rdd (R14):         the same with u -> 2 u_dd and 3n + 32.
Class plain (R15):       class B + (2^(c+leaf_bits) + block_bits + unit_bits + 16) u L1.
"""
from __future__ import annotations

import math
import os

U = 2.0 ** -53
U_DD = 2.0 ** -104
L1C_MAX_PER_N = 50.0

REPORT: list[dict] = []


def _current_test() -> str:
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]


def bound_B(part, n: int, c: int, scale: float = 1.0) -> float:
    return U * ((math.sqrt(n) + 2 ** (c / 2)) * part.l1c + (3 * n + 16) * part.l1) * scale


def bound_dd(part, n: int, c: int, scale: float = 1.0) -> float:
    return 2 * U_DD * ((math.sqrt(n) + 2 ** (c / 2)) * part.l1c + (3 * n + 32) * part.l1) * scale


def plain_extra(part, P, scale: float = 1.0) -> float:
    k = 2 ** (P.chunk_bits + P.leaf_bits) + P.block_bits + P.unit_bits + 16
    return U * k * part.l1 * scale


def _guard(part, n: int) -> None:
    if part.l1 > 0:
        assert part.l1c <= L1C_MAX_PER_N * n * part.l1, \
            f"L1c / (n L1) = {part.l1c / (n * part.l1):.1f} above the ceiling {L1C_MAX_PER_N}: vacuous bound?"


def record(kind: str, err: float, bound: float, ref: complex, part=None, n: int = 0, what: str = "",
           scale: float = 1.0) -> None:
    REPORT.append({"test": _current_test(), "kind": kind, "what": what, "n": n, "err": err, "bound": bound,
                   "err_over_bound": err / bound if bound > 0 else (0.0 if err == 0 else math.inf),
                   "bound_over_ref": bound / abs(ref) if ref != 0 else None,
                   "bound_factor": (bound / (U * part.l1 * scale)) if part is not None and part.l1 > 0 else None})


def check_B(got: complex, part, n: int, c: int, scale: float = 1.0, *, ref: complex | None = None,
            extra: float = 0.0, rel_ceiling: float | None = None, what: str = "", dd: bool = False) -> float:
    """Assert |got - ref| <= class-B (or Rdd when dd) bound (+ extra); ref defaults to the
    oracle partial scaled.  Records the ratios; returns err / bound."""
    _guard(part, n)
    if ref is None:
        ref = part.dd.to_complex() * scale
    bound = (bound_dd if dd else bound_B)(part, n, c, scale) + extra
    err = abs(got - ref)
    record("Rdd" if dd else "B", err, bound, ref, part, n, what, scale)
    if rel_ceiling is not None and ref != 0:
        assert bound <= rel_ceiling * abs(ref), f"bound / |ref| = {bound / abs(ref):.2e} > ceiling {rel_ceiling:.0e}"
    assert err <= bound + 1e-300, f"{what}: err {err:.3e} > bound {bound:.3e} (ratio {err / bound:.2f})"
    return err / bound if bound > 0 else 0.0


def rel(a: complex, b: complex) -> float:
    return abs(a - b) / abs(b)


def check_R(got: complex, ref: complex, tol: float = 1e-9, what: str = "") -> float:
    r = rel(got, ref)
    record("R", abs(got - ref), tol * abs(ref), ref, None, 0, what)
    assert r <= tol, f"{what}: relative error {r:.3e} > {tol:.0e}"
    return r
