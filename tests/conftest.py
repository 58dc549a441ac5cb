"""Shared pytest configuration.

Markers:
  gpu  -- needs a CUDA device (B200); run with ``pytest -m gpu`` on the GPU host.
Everything unmarked runs on the GPU-less build host.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (B200)")
    config.addinivalue_line("markers", "reference: requires the read-only reference checkout")


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    cuda = has_cuda()
    ref = REFERENCE_SRC.exists()
    for item in items:
        if "gpu" in item.keywords and not cuda:
            item.add_marker(pytest.mark.skip(reason="no CUDA device"))
        if "reference" in item.keywords and not ref:
            item.add_marker(pytest.mark.skip(reason="reference checkout not present"))
