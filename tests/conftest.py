import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size check")


def _built():
    need = ["paper_2008_12441_b200/libhmat.so", "oracle/liboracle.so", "gen/libhgen.so", "gen/libhgen_dev.so"]
    return all(os.path.exists(os.path.join(ROOT, p)) for p in need)


def pytest_sessionstart(session):
    # Build the in-tree native artefacts if a fresh checkout lacks them.
    if not _built():
        subprocess.run(["make", "-s", "-j8", "-C", ROOT], check=False)


@pytest.fixture(scope="session")
def has_gpu():
    import torch
    return torch.cuda.is_available()
