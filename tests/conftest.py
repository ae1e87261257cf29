import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")
    # build the native artefacts if they are missing (incremental make)
    if not os.path.exists(os.path.join(ROOT, "paper_1708_07271_b200", "libcmvg.so")):
        subprocess.check_call(["make", "-j8", "-C", os.path.join(ROOT, "paper_1708_07271_b200", "csrc")])
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libcmv_oracle.so")):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle")])


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
