import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running (minutes) case")


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Worst err/bound per test for the tolerance-class checks (tests/tolerance.py)."""
    try:
        import tolerance
    except ImportError:
        return
    rep = tolerance.REPORT
    if not rep:
        return
    worst = {}
    for r in rep:
        k = r["test"]
        if k not in worst or r["err_over_bound"] > worst[k]["err_over_bound"]:
            worst[k] = r
    tr = terminalreporter
    tr.write_sep("-", f"tolerance checks: {len(rep)} comparisons, worst err/bound per test")
    for k, r in sorted(worst.items(), key=lambda kv: -kv[1]["err_over_bound"]):
        bf = r["bound_factor"]
        br = r["bound_over_ref"]
        tr.write_line(f"{r['kind']:>3} err/bound={r['err_over_bound']:.3e} "
                      f"bound/|ref|={'-' if br is None else f'{br:.2e}'} "
                      f"bound/(u L1)={'-' if bf is None else f'{bf:.0f}'}  {k}")
    path = os.environ.get("PERMB200_TOL_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump({"comparisons": len(rep), "worst_per_test": worst}, f, indent=1)
