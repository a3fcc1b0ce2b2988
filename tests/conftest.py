"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; the CPU suite
(``-m "not gpu"``) covers the oracle against golden vectors, the policy
drop-in API, host logic and the C-ABI exports."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (run -m gpu on the B200 box)")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "moesim_golden.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle import tensor_oracle

    tensor_oracle.build()
    return tensor_oracle


@pytest.fixture(scope="session")
def native():
    from paper_2510_10302_b200 import _native

    return _native.load(build_if_missing=True)
