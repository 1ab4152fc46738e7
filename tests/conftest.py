"""Shared test configuration.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU.  Hypothesis runs
derandomized, like the reference suite (pkg/tests/conftest.py:15-16).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

try:
    from hypothesis import settings

    settings.register_profile("deterministic", derandomize=True, deadline=None)
    settings.load_profile("deterministic")
except ImportError:  # pragma: no cover
    pass

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cb2():
    from paper_2505_18231_b200.codebook import default_codebook

    return default_codebook("2b")


@pytest.fixture(scope="session")
def cb1():
    from paper_2505_18231_b200.codebook import default_codebook

    return default_codebook("1b")


def codebook_for(bit_mode: int):
    from paper_2505_18231_b200.codebook import default_codebook

    return default_codebook(f"{bit_mode}b")
