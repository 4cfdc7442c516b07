"""Shared test plumbing.

* registers the ``gpu`` marker (tests that need a B200; the CPU suite runs
  with ``-m "not gpu"``);
* puts the repo root on sys.path so ``oracle`` (test infrastructure) and the
  product package import the same way here and on the GPU box;
* ``golden(name)`` loads a committed fixture from tests/golden/.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def grid_of(d: dict, prefix: str = "grid"):
    return d[f"{prefix}_lo"], d[f"{prefix}_hi"], tuple(int(r) for r in d[f"{prefix}_res"])


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
