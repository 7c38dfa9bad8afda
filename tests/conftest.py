import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Native libraries are built in-tree; build whatever is missing (CPU-only
    build: nvcc cross-compiles sm_100a without a GPU)."""
    from paper_2504_04670_b200 import build as B
    B.build()
    from oracle import oracle as O
    O.build(ref=os.path.isdir(os.environ.get("HG_REF_DIR", "/root/reference/proj")))
    yield


def has_gpu() -> bool:
    try:
        from paper_2504_04670_b200 import hgs
        return hgs.device_count() > 0
    except Exception:
        return False
