"""Shared test configuration.

Markers: ``gpu`` tests need a B200 and the built libwidemod_b200.so; they are
the parity tests proper and go through the C ABI.  Everything else runs on
CPU (oracle pinning, host logic, ABI symbol checks, gloo multi-process)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libwidemod_b200.so")


def load_golden(name: str):
    return json.loads((GOLDEN / f"{name}.json").read_text())


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture(scope="session")
def cuda():
    """The GPU tests' gate: on a GPU box a missing device or library is an
    error, never a skip (no silent CPU fallback)."""
    import torch
    assert torch.cuda.is_available(), "gpu test run without a CUDA device"
    from paper_2501_07535_b200 import _lib
    _lib.load()
    return torch
