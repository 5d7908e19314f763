import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build_oracle

    build_oracle(with_ref=True)
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Ref()


@pytest.fixture(scope="session")
def verifier():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_11016_b200 import Verifier

    return Verifier(0)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Mismatch counts of the parity campaign (tests/parity.py log_parity):
    every token mismatch is explained by |u - threshold| < 1e-6 or the test fails."""
    try:
        from tests.parity import PARITY_LOG
    except Exception:
        return
    if not PARITY_LOG:
        return
    tr = terminalreporter
    tr.section("parity campaign: explained token mismatches (|u - threshold| < 1e-6); unexplained = 0")
    tot_r = tot_m = 0
    for label, rows, mism, note in PARITY_LOG:
        tr.write_line(f"{label:<58} rows={rows:<7} explained_mismatches={mism:<3} {note}")
        tot_r += rows
        tot_m += mism
    tr.write_line(f"{'TOTAL':<58} rows={tot_r:<7} explained_mismatches={tot_m}")
