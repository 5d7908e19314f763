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
