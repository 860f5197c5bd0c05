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


def _gpu_ready():
    """A CUDA device and the built library: what every gpu-marked test needs."""
    try:
        import torch
        if not torch.cuda.is_available():
            return False, "no CUDA device"
    except Exception as e:            # pragma: no cover
        return False, f"torch unavailable: {e}"
    from paper_2408_07967_b200 import _capi
    if not os.path.exists(_capi.LIB_PATH):
        return False, f"{_capi.LIB_PATH} not built"
    return True, ""


def pytest_collection_modifyitems(config, items):
    """gpu-marked tests are skipped (not failed) on a box without a GPU or the library, so
    the plain `pytest tests/` run is green on a CPU box too.  The product itself still
    raises there -- tests/test_host_cpu.py checks that."""
    ok, why = _gpu_ready()
    if ok:
        return
    skip = pytest.mark.skip(reason=f"needs the GPU path: {why}")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", params=GOLDEN_CASES)
def golden(request):
    return GoldenCase(request.param)


@pytest.fixture(scope="session")
def golden_c1():
    return GoldenCase("c1_mixed10k_256")
