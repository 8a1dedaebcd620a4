"""bench.py's multi-GPU launch contract (VERDICT r01 "make multi-GPU driver-measurable"):
`python bench.py --gpus N` without torchrun re-launches itself as N ranks, fails loudly when
fewer than N GPUs are visible, and (gloo, ranks sharing one GPU) reports n_gpus = N with a
result bit-identical to the single-GPU permanent."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, env=env, timeout=timeout,
                          cwd=ROOT)


def _json_lines(out: str):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_too_few_gpus_fails_loudly():
    import torch
    have = torch.cuda.device_count()
    for n in sorted({have + 1, max(2, have + 1)}):          # the single-process and the self-launch paths
        r = _run(["--gpus", str(n), "--steps", "1", "--warmup", "3"])
        assert r.returncode != 0
        assert f"needs {n} visible GPUs" in r.stderr, r.stderr[-1000:]
        assert not _json_lines(r.stdout)


def test_reference_arm_self_launches_two_ranks():
    """--impl reference --gpus 2: two ranks via torch.distributed.run, rank 0 alone prints."""
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--cpu-seconds", "1",
              "--workload", "M1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    L = lines[0]
    assert L["impl"] == "reference" and L["n_gpus"] == 2 and L["value"] > 0
    assert L["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.gpu
def test_gloo_two_ranks_on_one_gpu_bit_identical():
    import numpy as np
    import torch
    import synth
    import paper_1606_05836_b200 as pb
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3", "--workload", "M3", "--no-cpu-baseline",
              "--e2e-steps", "1"], {"PERMB200_DIST_BACKEND": "gloo"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    L = lines[0]
    assert L["n_gpus"] == 2 and L["ranks_share_gpus"] is True
    assert len(L["clocks_per_rank"]) == 2
    assert L["gpu_launches"] >= 2 * 3 * 1          # per rank per step: staging + sweep + combine (+ combine)
    v = complex(pb.glynn(torch.from_numpy(synth.workload("M3")).cuda()).item())
    assert L["result"] == [v.real, v.imag]
    assert np.isfinite(L["value"]) and L["value"] > 0
