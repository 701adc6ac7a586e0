import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1410_0759_b200", "libdnnp.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j8", "-C",
                        os.path.join(ROOT, "paper_1410_0759_b200", "csrc")], check=True)
    orc = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(orc):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def golden_conv():
    return np.load(os.path.join(GOLDEN, "conv.npz"))


@pytest.fixture(scope="session")
def golden_nnops():
    return np.load(os.path.join(GOLDEN, "nnops.npz"))


@pytest.fixture(scope="session")
def golden_info():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture
def rng():
    return np.random.default_rng(20140101)


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
