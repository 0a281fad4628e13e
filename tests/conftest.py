"""Shared pytest configuration.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu`` on the GPU box); every
other test runs on CPU in the build container.
"""

import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "decisions.json").read_text())


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
