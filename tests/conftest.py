import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Parity margins of every GPU check (tests/parity_util.MARGINS), printed even when all tests pass."""
    try:
        from tests.parity_util import MARGINS
    except Exception:  # pragma: no cover
        return
    if not MARGINS:
        return
    tr = terminalreporter
    tr.write_sep("-", "parity margins (quantity, value, bound)")
    for tag, q, v, b in MARGINS:
        tr.write_line(f"{tag}  {q} {v:.3e}" + (f" (bound {b:g})" if b is not None else " (per-pixel rules only)"))
    errs = [v for _, q, v, _ in MARGINS if q == "max_norm_err"]
    agr = [v for _, q, v, b in MARGINS if q == "label_agreement"]
    if errs:
        tr.write_line(f"worst max normalised error {max(errs):.3e} of 1e-4 over {len(errs)} checks; "
                      f"lowest label agreement {min(agr) if agr else float('nan'):.6f}")
