"""SASS guard (CPU, cuobjdump): the sweep kernels must read their Gray-step columns from
constant memory through UNIFORM registers (LDCU) -- no per-thread LDC of the column table --
and contain no tensor-core or legacy-HMMA instructions.  ptxas only produces this for a particular loop shape; this
test catches a change that silently falls back to per-thread loads + spills."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_1606_05836_b200", "_build")

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not available")


def _sass(obj):
    path = os.path.join(BUILD, obj)
    if not os.path.exists(path):
        from paper_1606_05836_b200 import build
        build.build()
    return subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout


def _kernel(sass, n, alg):
    out, on = [], False
    for line in sass.splitlines():
        if "Function : " in line:
            on = f"sweep_kernelILi{n}ELi{alg}E" in line
        elif on:
            out.append(line)
    assert out, f"sweep_kernel<{n},{alg}> not found"
    return "\n".join(out)


@pytest.mark.parametrize("obj,n,alg", [("perm_inst_glynn_b.o", 32, 0), ("perm_inst_glynn_c.o", 40, 0),
                                       ("perm_inst_glynn_c.o", 50, 0), ("perm_inst_ryser_b.o", 32, 1)])
def test_sweep_columns_are_uniform_operands(obj, n, alg):
    k = _kernel(_sass(obj), n, alg)
    ldcu = len(re.findall(r"\bLDCU", k))
    ldc_vec = len(re.findall(r"LDC(?:\.64)? R\d+, c\[0x3\]\[R", k))
    assert ldcu >= 10 * n, (ldcu, ldc_vec)
    assert ldc_vec <= 8, (ldcu, ldc_vec)
    assert "DFMA" in k and "DMUL" in k
    for bad in ("HMMA", "UTCHMMA", "DMMA"):
        assert bad not in k


@pytest.mark.parametrize("obj,n,alg", [("perm_inst_glynn_c.o", 40, 0), ("perm_inst_glynn_c.o", 48, 0),
                                       ("perm_inst_glynn_c.o", 50, 0), ("perm_inst_ryser_c.o", 50, 1),
                                       ("perm_inst_glynn_c.o", 51, 0)])
def test_hot_loop_has_no_spills_up_to_n51(obj, n, alg):
    """The register-budget choices (perm_kernels.cuh acc_in_smem / product_chains) keep the
    half-walk loop free of local-memory traffic up to n = 51."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from sass_loop_stats import loop_stats
    name, length, c = loop_stats(_sass(obj), f"sweep_kernelILi{n}ELi{alg}ELi0E")
    assert length > 0
    spills = sum(v for k, v in c.items() if k.startswith(("STL", "LDL")))
    assert spills == 0, (n, spills)
    assert c["IMAD.MOV.U32"] + c["MOV"] <= 16, (n, c["IMAD.MOV.U32"] + c["MOV"])
    assert c["DADD"] + c["DMUL"] + c["DFMA"] > 0


def _function(sass, want):
    for f in re.split(r"\n\s*Function : ", sass):
        if want in f.split("\n")[0]:
            return f
    raise AssertionError(f"{want} not found")


@pytest.mark.parametrize("obj,n,alg", [("perm_inst_wsplit_a.o", 52, 0), ("perm_inst_wsplit_a.o", 53, 1),
                                       ("perm_inst_wsplit_a.o", 54, 0), ("perm_inst_wsplit_b.o", 56, 0),
                                       ("perm_inst_wsplit_b.o", 59, 1), ("perm_inst_wsplit_b.o", 60, 0),
                                       ("perm_inst_wsplit_b.o", 63, 1), ("perm_inst_wsplit_b.o", 64, 0)])
def test_wsplit_columns_uniform_and_no_spills(obj, n, alg):
    """The warp-pair row split (perm_kernels_wsplit.cuh, n >= 52): the warp index reaches the
    K-branches through a shuffle so ptxas sees them as warp-uniform -- the columns must stay
    LDCU uniform operands (the plain (threadIdx.x >> 5) & 1 spelling fell back to per-thread LDC
    for every column) -- and the whole kernel (both half-walk copies) has no local memory."""
    f = _function(_sass(obj), f"wsplit_kernelILi{n}ELi{alg}ELi0E")
    ldcu = len(re.findall(r"\bLDCU", f))
    ldc_vec = len(re.findall(r"LDC(?:\.64)? R\d+, c\[0x3\]\[R", f))
    # per term n LDCU.64 (2 per row, n/2 rows, 2 warps' copies); 4 terms per loop body, 2 from n = 60
    assert ldcu >= (5 if n >= 60 else 10) * n and ldc_vec == 0, (ldcu, ldc_vec)
    assert not re.search(r"\b(STL|LDL)", f)
    assert "BAR.SYNC" in f or "BAR.SYNC.DEFER_BLOCKING" in f or "BAR " in f
