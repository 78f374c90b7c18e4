import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _ensure_oracle():
    from oracle import oracle as O
    if not O.restatement_available() or (not O.reference_available()
                                         and os.path.isdir("/root/reference/proj")):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=True)


@pytest.fixture(scope="session")
def restate():
    _ensure_oracle()
    from oracle.oracle import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def ref():
    _ensure_oracle()
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return O.Reference()


@pytest.fixture(scope="session")
def prof():
    from oracle.oracle import default_profile
    return default_profile()


@pytest.fixture(scope="session")
def gsb():
    """The product library on cuda:0 (GPU tests only)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_16449_b200 import api
    return api.Engine(device=0)
