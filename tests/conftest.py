import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

REF_SRC = Path("/root/reference/proj")
ORACLE_SO = ROOT / "oracle" / "_ref" / "libepp_ref.so"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def planner():
    from paper_2509_21275_b200 import planner as P
    return P


@pytest.fixture(scope="session")
def ref_api():
    """The compiled reference planner (oracle/_ref), or skip."""
    if not ORACLE_SO.exists():
        pytest.skip("oracle/_ref/libepp_ref.so not built")
    from paper_2509_21275_b200 import planner as P
    return P._Api(ORACLE_SO, prefix="epp_ref_")
