import os
import sys
from pathlib import Path

# before any CUDA context exists: one hardware queue per stream, so the
# loopback tests' thread-ranks (each with its own streams on one GPU) never
# queue a kernel behind another rank's spinning device barrier
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtenvec_b200.so")


def load_golden(name: str):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture(scope="session")
def oracle():
    import tenvec_oracle

    return tenvec_oracle


@pytest.fixture(scope="session")
def tv_host():
    """The product package for host-only logic (no device needed)."""
    import paper_2501_03121_b200 as pkg

    return pkg


@pytest.fixture(scope="session")
def tv():
    """The product package with its CUDA library loaded (GPU tests only)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_03121_b200 as pkg
    from paper_2501_03121_b200 import _lib, build

    build.build()
    _lib.load()
    return pkg
