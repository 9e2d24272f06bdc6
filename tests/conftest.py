"""Shared test fixtures.  `-m gpu` tests need a B200 (they call the C-ABI
library through the public API); everything else runs on CPU."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def soe8():
    from paper_2403_01521_b200.soe import build_soe_contour
    return build_soe_contour(8)


@pytest.fixture(scope="session")
def soe16():
    from paper_2403_01521_b200.soe import build_soe_contour
    return build_soe_contour(16)


@pytest.fixture(scope="session")
def soe24():
    from paper_2403_01521_b200.soe import build_soe_contour
    return build_soe_contour(24)
