"""pytest configuration: markers, import paths, golden-vector fixtures."""

import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

from fgs_testlib import GOLDEN_CASES, GoldenCase  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session", params=GOLDEN_CASES)
def golden(request):
    return GoldenCase(request.param)


@pytest.fixture(scope="session")
def golden_c1():
    return GoldenCase("c1_mixed10k_256")
