"""ctypes binding of libpermb200.so (include/permb200.h).  Argument marshalling only: every
step of the permanent runs in the library's CUDA kernels.  There is no CPU fallback: if
the shared library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
# PERMB200_LIB selects another build of the same library (the bounds-checked debug build,
# libpermb200_checked.so); there is no fallback of any kind.
LIB_PATH = os.environ.get("PERMB200_LIB") or os.path.join(_HERE, "libpermb200.so")

PERM_OK, PERM_EINVAL, PERM_ECUDA, PERM_ENOTIMPL = 0, 1, 2, 3
ALG_GLYNN, ALG_RYSER, ALG_GLYNN_DD, ALG_RYSER_DD, ALG_GLYNN_PLAIN, ALG_RYSER_PLAIN = 0, 1, 2, 3, 4, 5
ALG_GLYNN_SEP, ALG_RYSER_SEP = 6, 7

# every symbol include/permb200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "perm_max_n", "perm_strerror", "perm_plan", "perm_glynn", "perm_ryser", "perm_sweep_units",
    "perm_glynn_range", "perm_ryser_range", "perm_combine", "perm_glynn_batched", "perm_glynn_host",
    "perm_ryser_host", "perm_glynn_batched_host", "perm_glynn_dd", "perm_ryser_dd", "perm_range", "perm_sweep_units_custom",
    "perm_glynn_batched_abs2", "perm_glynn_batched_abs2_host", "perm_sum_ordered", "perm_launch_count",
)


class PermError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} (status {code})")


class PlanT(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("alg", ctypes.c_int), ("log2_terms", ctypes.c_int),
                ("chunk_bits", ctypes.c_int), ("leaf_bits", ctypes.c_int), ("block_bits", ctypes.c_int),
                ("unit_bits", ctypes.c_int), ("lanes", ctypes.c_int), ("unit_terms", ctypes.c_uint64),
                ("units", ctypes.c_int64)]


@dataclass(frozen=True)
class Plan:
    n: int
    alg: int
    log2_terms: int
    chunk_bits: int
    leaf_bits: int
    block_bits: int
    unit_bits: int
    unit_terms: int
    units: int
    lanes: int = 1          # threads per leaf (row-split sweeps: 4 small n, 2 for n >= 52)

    @property
    def terms(self) -> int:
        return 1 << self.log2_terms


_lib = None


def lib() -> ctypes.CDLL:
    """Load libpermb200.so (raises OSError if it is missing: build it with
    `python -m paper_1606_05836_b200.build`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not found; run `python -m paper_1606_05836_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
        L.perm_max_n.restype = i32
        L.perm_max_n.argtypes = []
        L.perm_strerror.restype = ctypes.c_char_p
        L.perm_strerror.argtypes = [i32]
        L.perm_plan.argtypes = [i32, i32, ctypes.POINTER(PlanT)]
        L.perm_glynn.argtypes = [vp, i32, vp, vp]
        L.perm_ryser.argtypes = [vp, i32, vp, vp]
        L.perm_sweep_units.argtypes = [vp, i32, i32, i64, i64, vp, vp]
        L.perm_glynn_range.argtypes = [vp, i32, u64, u64, vp, vp]
        L.perm_ryser_range.argtypes = [vp, i32, u64, u64, vp, vp]
        L.perm_combine.argtypes = [vp, i64, i32, i32, vp, vp, vp]
        L.perm_glynn_batched.argtypes = [vp, i32, i64, vp, vp]
        L.perm_glynn_dd.argtypes = [vp, i32, vp, vp]
        L.perm_ryser_dd.argtypes = [vp, i32, vp, vp]
        L.perm_range.argtypes = [vp, i32, i32, u64, u64, vp, vp]
        L.perm_sweep_units_custom.argtypes = [vp, i32, i32, i32, i32, i32, i64, i64, vp, vp]
        L.perm_glynn_host.argtypes = [vp, i32, vp]
        L.perm_ryser_host.argtypes = [vp, i32, vp]
        L.perm_glynn_batched_host.argtypes = [vp, i32, i64, vp]
        L.perm_glynn_batched_abs2.argtypes = [vp, i32, i64, vp, vp]
        L.perm_glynn_batched_abs2_host.argtypes = [vp, i32, i64, vp]
        L.perm_sum_ordered.argtypes = [vp, i64, vp, i32, i32, vp, vp]
        L.perm_launch_count.argtypes = []
        for name in EXPORTS:
            if name not in ("perm_max_n", "perm_strerror", "perm_launch_count"):
                getattr(L, name).restype = i32
        L.perm_launch_count.restype = ctypes.c_longlong
        _lib = L
    return _lib


def strerror(code: int) -> str:
    return lib().perm_strerror(int(code)).decode()


def check(code: int, where: str) -> None:
    if code != PERM_OK:
        raise PermError(code, where)


def max_n() -> int:
    return int(lib().perm_max_n())


def plan(n: int, alg: int = ALG_GLYNN) -> Plan:
    p = PlanT()
    check(lib().perm_plan(int(n), int(alg), ctypes.byref(p)), "perm_plan")
    return Plan(p.n, p.alg, p.log2_terms, p.chunk_bits, p.leaf_bits, p.block_bits, p.unit_bits,
                int(p.unit_terms), int(p.units), int(p.lanes))


def launch_count() -> int:
    """Kernels libpermb200.so has launched since it was loaded (perm_launch_count)."""
    return int(lib().perm_launch_count())
