"""Shared pytest configuration: marker registration, golden loader, oracle handle."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def load_golden(name: str):
    return np.load(GOLDEN / f"{name}.npz")


@pytest.fixture(scope="session")
def oracle():
    from oracle import d360_oracle

    d360_oracle.build()
    return d360_oracle


def golden_group(oracle, z, top_k=None):
    """Oracle Group from a hot_* golden file (reference is frame 1, neighbours 0 and 2)."""
    imgs, rot, tr = z["images"], z["rotations"], z["translations"]
    return oracle.Group(imgs[1], [imgs[0], imgs[2]], (rot[1], tr[1]), [(rot[0], tr[0]), (rot[2], tr[2])],
                        int(z["half_window"]), int(z["sample_stride"]), float(z["trunc"]), top_k=top_k)
