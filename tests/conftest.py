import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built libmom.so")
    config.addinivalue_line("markers", "slow: long-running (full-size oracle) test")


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda:0")


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Print every gated parity comparison of the session (tests/parity.RECORDS): the measured
    normwise errors against their gate and regression bound, and the argmax top-2 gaps."""
    try:
        from tests.parity import RECORDS
    except Exception:  # pragma: no cover
        return
    if not RECORDS:
        return
    tr = terminalreporter
    tr.section("parity records")
    for rec in RECORDS:
        if rec[0] == "close":
            _, what, e, rmax, tol, reg = rec
            tr.write_line(f"close  {e:.3e} (worst row {rmax:.3e}) tol {tol:.0e} reg {reg or '-'}  {what}")
        else:
            _, what, rel, gap, got, best = rec
            tr.write_line(f"argmax {got} == {best}  top-2 gap {gap:.3e} ({rel:.2e} of max)  {what}")
