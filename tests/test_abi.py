"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol the
header declares, validates arguments before touching CUDA, and plans canonically."""
import ctypes
import os
import re

import pytest

import paper_1606_05836_b200 as pb
from paper_1606_05836_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "permb200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*)\s+(perm_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _declared()
    assert len(declared) >= 13
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib.EXPORTS)


def test_max_n_and_strerror():
    assert pb.max_n() == 64
    assert _lib.strerror(0) == "ok"
    assert "invalid" in _lib.strerror(1)
    assert _lib.strerror(3) == "not implemented"


def test_invalid_arguments_rejected_without_cuda():
    L = _lib.lib()
    buf = ctypes.create_string_buffer(64)
    assert L.perm_glynn(None, 4, buf, None) == _lib.PERM_EINVAL
    assert L.perm_glynn(buf, 0, buf, None) == _lib.PERM_EINVAL
    assert L.perm_ryser(buf, 65, buf, None) == _lib.PERM_EINVAL
    assert L.perm_glynn_batched(buf, 4, -1, buf, None) == _lib.PERM_EINVAL
    assert L.perm_glynn_batched(None, 4, 0, None, None) == _lib.PERM_OK     # empty batch: no-op
    assert L.perm_glynn_range(buf, 4, 5, 4, buf, None) == _lib.PERM_EINVAL   # lo > hi
    assert L.perm_glynn_range(buf, 4, 0, 9, buf, None) == _lib.PERM_EINVAL   # hi > 2^(n-1)
    assert L.perm_sweep_units(buf, 4, 8, 0, 1, buf, None) == _lib.PERM_EINVAL  # bad alg
    assert L.perm_sweep_units(buf, 41, _lib.ALG_GLYNN_SEP, 0, 1, buf, None) == _lib.PERM_EINVAL  # sep: n <= 40
    assert L.perm_glynn_batched_abs2(buf, 4, 3, None, None) == _lib.PERM_EINVAL   # null out
    assert L.perm_glynn_batched_abs2(None, 4, 0, None, None) == _lib.PERM_OK      # empty batch
    assert L.perm_sum_ordered(buf, 0, buf, 4, 0, buf, None) == _lib.PERM_EINVAL   # count < 1
    assert L.perm_sum_ordered(buf, 4, None, 4, 0, buf, None) == _lib.PERM_EINVAL  # null order
    assert L.perm_launch_count() == 0                                             # nothing launched
    assert L.perm_sweep_units(buf, 4, -1, 0, 1, buf, None) == _lib.PERM_EINVAL
    assert L.perm_range(buf, 4, 8, 0, 1, buf, None) == _lib.PERM_EINVAL
    assert L.perm_range(buf, 4, pb.ALG_RYSER_PLAIN, 0, 17, buf, None) == _lib.PERM_EINVAL
    assert L.perm_range(buf, 4, pb.ALG_RYSER_DD, 0, 17, buf, None) == _lib.PERM_EINVAL   # hi > 2^n
    assert L.perm_glynn_dd(None, 4, buf, None) == _lib.PERM_EINVAL
    assert L.perm_glynn_dd(buf, 4, None, None) == _lib.PERM_EINVAL
    assert L.perm_ryser_dd(buf, 64, buf, None) == _lib.PERM_EINVAL
    assert L.perm_combine(buf, 0, 4, 0, buf, buf, None) == _lib.PERM_EINVAL   # count < 1
    assert L.perm_glynn_host(None, 3, buf) == _lib.PERM_EINVAL
    with pytest.raises(pb.PermError):
        pb.plan(0)
    with pytest.raises(pb.PermError):
        pb.plan(64, pb.ALG_RYSER)                       # 2^64 Gray indices do not fit


@pytest.mark.parametrize("alg", [pb.ALG_GLYNN, pb.ALG_RYSER, pb.ALG_GLYNN_DD, pb.ALG_RYSER_DD,
                                 pb.ALG_GLYNN_PLAIN, pb.ALG_RYSER_PLAIN])
def test_plan_is_a_partition(alg):
    glynn = alg % 2 == 0
    for n in range(1, 65 if glynn else 64):
        P = pb.plan(n, alg)
        m = n - 1 if glynn else n
        assert P.log2_terms == m
        assert P.chunk_bits + P.leaf_bits + P.block_bits + P.unit_bits == m
        assert P.units * P.unit_terms == 1 << m
        assert 0 <= P.block_bits <= (6 if alg in (pb.ALG_GLYNN_DD, pb.ALG_RYSER_DD) else 7) and 0 <= P.chunk_bits <= 12
        if m >= 5:
            assert P.chunk_bits >= 5                       # fast path usable
        assert P.units <= 1 << 22 and (P.units <= 1 << 17 or P.unit_terms >= 1 << 29)


def test_plain_mode_plans_equal_fp64_plans():
    """The plain-accumulation mode walks exactly the FP64 plan (same terms, same order)."""
    for n in (5, 20, 40, 50):
        for a, p in ((pb.ALG_GLYNN, pb.ALG_GLYNN_PLAIN), (pb.ALG_RYSER, pb.ALG_RYSER_PLAIN)):
            x, y = pb.plan(n, a), pb.plan(n, p)
            assert (x.chunk_bits, x.leaf_bits, x.block_bits, x.unit_bits) == (y.chunk_bits, y.leaf_bits, y.block_bits, y.unit_bits)


def test_plan_large_n_shards_eight_ways():
    for n in (32, 40, 50):
        P = pb.plan(n)
        assert P.units % 8 == 0 and P.units >= 4096


def test_custom_plan_arguments_validated_without_cuda():
    L = _lib.lib()
    buf = ctypes.create_string_buffer(64)
    f = L.perm_sweep_units_custom
    assert f(buf, 20, 0, 3, 0, 7, 0, 1, buf, None) == _lib.PERM_EINVAL      # chunk_bits < 4 (kMinFastC)
    assert f(buf, 20, 0, 13, 0, 0, 0, 1, buf, None) == _lib.PERM_EINVAL     # chunk_bits > 12
    assert f(buf, 30, 0, 10, 0, 8, 0, 1, buf, None) == _lib.PERM_EINVAL     # block_bits > 7
    assert f(buf, 56, 0, 10, 0, 7, 0, 1, buf, None) == _lib.PERM_EINVAL     # 2-lane leaves: block_bits > 6
    assert f(buf, 20, 2, 10, 0, 7, 0, 1, buf, None) == _lib.PERM_EINVAL     # dd: block_bits > 6
    assert f(buf, 20, 0, 10, 5, 5, 0, 1, buf, None) == _lib.PERM_EINVAL     # c + lam + wb > 19
    assert f(buf, 20, 0, 10, 0, 5, 0, 17, buf, None) == _lib.PERM_EINVAL    # unit_hi > units (16)
    assert f(buf, 20, 0, 10, 0, 5, 0, 0, buf, None) == _lib.PERM_OK         # empty
