"""paper_1606_05836_b200 — B200-native BB/FG (Glynn) and Ryser permanents.

PAPER.md (arXiv 1606.05836): Eq. (2) BB/FG P:66-68 and Eq. (1) Ryser P:62-64, walked in
Gray-code order by hand-written sm_100a FP64 kernels (paper_1606_05836_b200/csrc).  This
module is the thin Python layer over the C ABI (include/permb200.h): it checks tensor
shapes/dtypes/devices, passes raw device pointers and the current CUDA stream, and raises
on any non-zero status.  PyTorch supplies device memory and streams only.

    glynn(A) / ryser(A)              permanent of one n x n complex128 CUDA matrix
    glynn_batched(As)                (B, n, n) -> (B,)  one permanent per thread block
    glynn_dd(A) / ryser_dd(A)        double-double precision mode: (re_hi, re_lo, im_hi, im_lo)
    glynn_range / ryser_range        unscaled double-double partial over Gray indices [lo, hi)
    range_partial(A, alg, lo, hi)    the same for any algorithm code (incl. the dd mode)
    perm_alg(A, alg)                 Perm(A) for any algorithm code (FP64 / dd / plain accumulation)
    PermGraph(n, alg)                a CUDA-graph replay of one call (launch-bound small n)
    sweep_units / combine            the two kernels of the canonical reduction (multi-GPU)
    glynn_host / ryser_host / glynn_batched_host   host-buffer C-ABI entry points
    dist.perm_dist                   one permanent partitioned over a process group (NCCL)
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _lib
from ._lib import (ALG_GLYNN, ALG_GLYNN_DD, ALG_GLYNN_PLAIN, ALG_GLYNN_SEP, ALG_RYSER, ALG_RYSER_DD,  # noqa: F401
                   ALG_RYSER_PLAIN, ALG_RYSER_SEP, Plan, PermError, launch_count, max_n, plan)

__all__ = ["glynn", "ryser", "glynn_batched", "glynn_range", "ryser_range", "sweep_units", "combine",
           "glynn_host", "ryser_host", "glynn_batched_host", "plan", "max_n", "Plan", "PermError",
           "ALG_GLYNN", "ALG_RYSER", "ALG_GLYNN_DD", "ALG_RYSER_DD", "ALG_GLYNN_PLAIN", "ALG_RYSER_PLAIN",
           "ALG_GLYNN_SEP", "ALG_RYSER_SEP", "glynn_dd", "ryser_dd", "range_partial", "perm_alg", "sweep_units_custom",
           "PermGraph", "dd_to_complex", "glynn_batched_abs2", "glynn_batched_abs2_host", "sum_ordered",
           "launch_count"]


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _square(A: torch.Tensor) -> int:
    if not isinstance(A, torch.Tensor) or A.dtype != torch.complex128 or not A.is_cuda:
        raise TypeError("expected a torch.complex128 CUDA tensor")
    if A.dim() != 2 or A.shape[0] != A.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {tuple(A.shape)}")
    return A.shape[0]


def _alg(alg) -> int:
    if alg in (ALG_GLYNN, "glynn"):
        return ALG_GLYNN
    if alg in (ALG_RYSER, "ryser"):
        return ALG_RYSER
    if alg in (ALG_GLYNN_DD, "glynn_dd"):
        return ALG_GLYNN_DD
    if alg in (ALG_RYSER_DD, "ryser_dd"):
        return ALG_RYSER_DD
    if alg in (ALG_GLYNN_PLAIN, "glynn_plain"):
        return ALG_GLYNN_PLAIN
    if alg in (ALG_RYSER_PLAIN, "ryser_plain"):
        return ALG_RYSER_PLAIN
    if alg in (ALG_GLYNN_SEP, "glynn_sep"):
        return ALG_GLYNN_SEP
    if alg in (ALG_RYSER_SEP, "ryser_sep"):
        return ALG_RYSER_SEP
    raise ValueError(f"unknown algorithm {alg!r}")


def _perm(fn, name: str, A: torch.Tensor) -> torch.Tensor:
    n = _square(A)
    A = A.contiguous()
    out = torch.empty((), dtype=torch.complex128, device=A.device)
    with torch.cuda.device(A.device):
        _lib.check(fn(A.data_ptr(), n, out.data_ptr(), _stream(A.device)), name)
    return out


def glynn(A: torch.Tensor) -> torch.Tensor:
    """Perm(A) by BB/FG / Glynn, Eq. (2) (0-d complex128 tensor on A's device)."""
    return _perm(_lib.lib().perm_glynn, "perm_glynn", A)


def ryser(A: torch.Tensor) -> torch.Tensor:
    """Perm(A) by Ryser, Eq. (1)."""
    return _perm(_lib.lib().perm_ryser, "perm_ryser", A)


def _perm_dd(fn, name: str, A: torch.Tensor) -> torch.Tensor:
    n = _square(A)
    A = A.contiguous()
    out = torch.empty(4, dtype=torch.float64, device=A.device)
    with torch.cuda.device(A.device):
        _lib.check(fn(A.data_ptr(), n, out.data_ptr(), _stream(A.device)), name)
    return out


def glynn_dd(A: torch.Tensor) -> torch.Tensor:
    """Perm(A) by Eq. (2) in the double-double mode: (4,) float64 (re_hi, re_lo, im_hi, im_lo),
    scaled by 2^-(n-1)."""
    return _perm_dd(_lib.lib().perm_glynn_dd, "perm_glynn_dd", A)


def ryser_dd(A: torch.Tensor) -> torch.Tensor:
    """Perm(A) by Eq. (1) in the double-double mode (4 float64, see glynn_dd)."""
    return _perm_dd(_lib.lib().perm_ryser_dd, "perm_ryser_dd", A)


def dd_to_complex(d) -> complex:
    """(re_hi, re_lo, im_hi, im_lo) -> complex128 (rounded)."""
    v = [float(x) for x in (d.tolist() if hasattr(d, "tolist") else d)]
    return complex(v[0] + v[1], v[2] + v[3])


def _batch(As: torch.Tensor) -> tuple[int, int]:
    if not isinstance(As, torch.Tensor) or As.dtype != torch.complex128 or not As.is_cuda:
        raise TypeError("expected a torch.complex128 CUDA tensor")
    if As.dim() != 3 or As.shape[1] != As.shape[2]:
        raise ValueError(f"expected (B, n, n), got {tuple(As.shape)}")
    return As.shape[0], As.shape[1]


def glynn_batched(As: torch.Tensor) -> torch.Tensor:
    """(B, n, n) complex128 CUDA -> (B,) permanents, one thread block per matrix."""
    B, n = _batch(As)
    As = As.contiguous()
    out = torch.empty((B,), dtype=torch.complex128, device=As.device)
    with torch.cuda.device(As.device):
        _lib.check(_lib.lib().perm_glynn_batched(As.data_ptr() if B else None, n, B, out.data_ptr() if B else None,
                                                 _stream(As.device)), "perm_glynn_batched")
    return out


def glynn_batched_abs2(As: torch.Tensor) -> torch.Tensor:
    """(B, n, n) complex128 CUDA -> (B,) float64 |Perm(A_b)|^2 (boson-sampling probability
    numerators), computed in the batched kernel."""
    B, n = _batch(As)
    As = As.contiguous()
    out = torch.empty((B,), dtype=torch.float64, device=As.device)
    with torch.cuda.device(As.device):
        _lib.check(_lib.lib().perm_glynn_batched_abs2(As.data_ptr() if B else None, n, B,
                                                      out.data_ptr() if B else None, _stream(As.device)),
                   "perm_glynn_batched_abs2")
    return out


def sum_ordered(partials: torch.Tensor, order: torch.Tensor, n: int, alg) -> torch.Tensor:
    """Sequential plain-FP64 sum of (count, 4) float64 CUDA partials in the order given by the
    int64 CUDA permutation `order`, finished like perm_combine (x 2^-(n-1) for Glynn): the
    paper's "original" / "random" summation orders (Table AV; perm_sum_ordered)."""
    if partials.dtype != torch.float64 or not partials.is_cuda or partials.dim() != 2 or partials.shape[1] != 4:
        raise TypeError("expected a (count, 4) float64 CUDA tensor")
    if order.dtype != torch.int64 or order.device != partials.device or order.shape != (partials.shape[0],):
        raise TypeError("order must be an int64 tensor of shape (count,) on the partials' device")
    partials, order = partials.contiguous(), order.contiguous()
    out = torch.empty((), dtype=torch.complex128, device=partials.device)
    with torch.cuda.device(partials.device):
        _lib.check(_lib.lib().perm_sum_ordered(partials.data_ptr(), partials.shape[0], order.data_ptr(), int(n),
                                               _alg(alg), out.data_ptr(), _stream(partials.device)),
                   "perm_sum_ordered")
    return out


def _range(fn, name, A, lo, hi) -> torch.Tensor:
    n = _square(A)
    A = A.contiguous()
    out = torch.empty(4, dtype=torch.float64, device=A.device)
    with torch.cuda.device(A.device):
        _lib.check(fn(A.data_ptr(), n, int(lo), int(hi), out.data_ptr(), _stream(A.device)), name)
    return out


def glynn_range(A: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """Unscaled Glynn partial over Gray indices [lo, hi) as (re_hi, re_lo, im_hi, im_lo) float64."""
    return _range(_lib.lib().perm_glynn_range, "perm_glynn_range", A, lo, hi)


def ryser_range(A: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """Signed Ryser partial over Gray indices [lo, hi) (double-double, 4 float64)."""
    return _range(_lib.lib().perm_ryser_range, "perm_ryser_range", A, lo, hi)


def range_partial(A: torch.Tensor, alg, lo: int, hi: int) -> torch.Tensor:
    """Unscaled partial over Gray indices [lo, hi) for any algorithm code (4 float64)."""
    n = _square(A)
    A = A.contiguous()
    out = torch.empty(4, dtype=torch.float64, device=A.device)
    with torch.cuda.device(A.device):
        _lib.check(_lib.lib().perm_range(A.data_ptr(), n, _alg(alg), int(lo), int(hi), out.data_ptr(),
                                         _stream(A.device)), "perm_range")
    return out


def perm_alg(A: torch.Tensor, alg) -> torch.Tensor:
    """Perm(A) for any algorithm code (FP64, double-double or plain-accumulation mode),
    rounded to a 0-d complex128 tensor: sweep_units over all units + combine (one call each)."""
    n = _square(A)
    a = _alg(alg)
    P = plan(n, a)
    val, _ = combine(sweep_units(A, a, 0, P.units), n, a, scale=True)
    return val


def sweep_units(A: torch.Tensor, alg, unit_lo: int, unit_hi: int) -> torch.Tensor:
    """Canonical unit partials for units [unit_lo, unit_hi) of plan(n, alg): (count, 4) float64."""
    n = _square(A)
    A = A.contiguous()
    a = _alg(alg)
    count = int(unit_hi) - int(unit_lo)
    out = torch.empty((max(count, 0), 4), dtype=torch.float64, device=A.device)
    with torch.cuda.device(A.device):
        _lib.check(_lib.lib().perm_sweep_units(A.data_ptr(), n, a, int(unit_lo), int(unit_hi),
                                               out.data_ptr() if count > 0 else None, _stream(A.device)),
                   "perm_sweep_units")
    return out


def sweep_units_custom(A: torch.Tensor, alg, chunk_bits: int, leaf_bits: int, block_bits: int,
                       unit_lo: int, unit_hi: int) -> torch.Tensor:
    """The sweep kernel on a non-canonical plan (profiling / experiments): (count, 4) float64."""
    n = _square(A)
    A = A.contiguous()
    count = int(unit_hi) - int(unit_lo)
    out = torch.empty((max(count, 0), 4), dtype=torch.float64, device=A.device)
    with torch.cuda.device(A.device):
        _lib.check(_lib.lib().perm_sweep_units_custom(A.data_ptr(), n, _alg(alg), int(chunk_bits), int(leaf_bits),
                                                      int(block_bits), int(unit_lo), int(unit_hi),
                                                      out.data_ptr() if count > 0 else None, _stream(A.device)),
                   "perm_sweep_units_custom")
    return out


def combine(partials: torch.Tensor, n: int, alg, scale: bool = True):
    """Canonical pairwise tree over (count, 4) float64 CUDA partials.  Returns (value, root_dd):
    value = root * 2^-(n-1) (Glynn) rounded to complex128 if scale else None."""
    if partials.dtype != torch.float64 or not partials.is_cuda or partials.dim() != 2 or partials.shape[1] != 4:
        raise TypeError("expected a (count, 4) float64 CUDA tensor")
    partials = partials.contiguous()
    a = _alg(alg)
    root = torch.empty(4, dtype=torch.float64, device=partials.device)
    val = torch.empty((), dtype=torch.complex128, device=partials.device) if scale else None
    with torch.cuda.device(partials.device):
        _lib.check(_lib.lib().perm_combine(partials.data_ptr(), partials.shape[0], int(n), a,
                                           val.data_ptr() if val is not None else None, root.data_ptr(),
                                           _stream(partials.device)), "perm_combine")
    return val, root


def _host(fn, name, A, n, batch) -> "object":
    import numpy as np
    a = np.ascontiguousarray(A, dtype=np.complex128)
    out = np.empty(1 if batch is None else max(batch, 1), dtype=np.complex128)
    if batch is None:
        _lib.check(fn(a.ctypes.data, n, out.ctypes.data), name)
    else:
        _lib.check(fn(a.ctypes.data, n, batch, out.ctypes.data), name)
    return out


def _host_square(A):
    import numpy as np
    a = np.ascontiguousarray(A, dtype=np.complex128)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < 1:
        raise ValueError(f"expected a square matrix, got shape {a.shape}")
    return a


def _host_batch(As):
    import numpy as np
    a = np.ascontiguousarray(As, dtype=np.complex128)
    if a.ndim != 3 or a.shape[1] != a.shape[2] or a.shape[1] < 1:
        raise ValueError(f"expected (B, n, n), got shape {a.shape}")
    return a


def glynn_host(A) -> complex:
    """Host-buffer entry point (C ABI perm_glynn_host): numpy in, complex out; copies inside."""
    a = _host_square(A)
    return complex(_host(_lib.lib().perm_glynn_host, "perm_glynn_host", a, a.shape[0], None)[0])


def ryser_host(A) -> complex:
    a = _host_square(A)
    return complex(_host(_lib.lib().perm_ryser_host, "perm_ryser_host", a, a.shape[0], None)[0])


def glynn_batched_host(As):
    a = _host_batch(As)
    B, n = a.shape[0], a.shape[1]
    return _host(_lib.lib().perm_glynn_batched_host, "perm_glynn_batched_host", a, n, B)[:B]


def glynn_batched_abs2_host(As):
    """Host-buffer |Perm(A_b)|^2 (C ABI perm_glynn_batched_abs2_host): (B,) float64."""
    import numpy as np
    a = _host_batch(As)
    B, n = a.shape[0], a.shape[1]
    out = np.empty(max(B, 1), dtype=np.float64)
    _lib.check(_lib.lib().perm_glynn_batched_abs2_host(a.ctypes.data, n, B, out.ctypes.data),
               "perm_glynn_batched_abs2_host")
    return out[:B]


class PermGraph:
    """One permanent call captured in a CUDA graph and replayed per input: for launch-bound
    sizes (M1: n = 20 is ~7 us of FP64 work against ~25 us of host-side submission per eager
    call).  Capturable: Glynn n <= 22 / Ryser n <= 21 (the small-n sweep), the dd modes, and
    batched calls (pass `batch`).  Larger FP64 sweeps use the constant-memory column slot and
    raise PermError at capture.

        g = PermGraph(20, "glynn")
        out = g(A)          # copies A into the graph's input, replays, returns g.out
    """

    def __init__(self, n: int, alg="glynn", batch: Optional[int] = None, device=None):
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        shape = (batch, n, n) if batch is not None else (n, n)
        self.A = torch.zeros(shape, dtype=torch.complex128, device=device)
        self.A[..., range(n), range(n)] = 1.0            # identity: a valid warm-up input
        if batch is not None:
            if alg not in ("glynn", ALG_GLYNN):
                raise ValueError("batched graphs are Glynn (perm_glynn_batched)")
            fn = glynn_batched
        else:
            a = _alg(alg)
            fn = {ALG_GLYNN: glynn, ALG_RYSER: ryser, ALG_GLYNN_DD: glynn_dd, ALG_RYSER_DD: ryser_dd}.get(a)
            if fn is None:
                fn = lambda X: perm_alg(X, a)           # noqa: E731
        s = torch.cuda.Stream(device)
        s.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(s):
            fn(self.A)                                  # warm-up (module load, pool) outside capture
        torch.cuda.current_stream(device).wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out = fn(self.A)

    def __call__(self, A: torch.Tensor) -> torch.Tensor:
        self.A.copy_(A)
        self.graph.replay()
        return self.out
