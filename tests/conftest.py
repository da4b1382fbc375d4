"""Shared test configuration.

Markers: `gpu` tests need a CUDA device (run on the B200 box with
`pytest -m gpu`); everything else runs on CPU.  Hypothesis uses the
reference's deterministic profile (pkg/tests/conftest.py:10-16).
"""

import os
import sys
from pathlib import Path

import hypothesis
import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

hypothesis.settings.register_profile("deterministic", derandomize=True, deadline=None,
                                     max_examples=25)
hypothesis.settings.load_profile("deterministic")

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test needs a CUDA device (run with -m 'not gpu' on CPU)")
    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def reference():
    """The live reference from oracle/_ref (None when not built)."""
    from oracle import import_reference

    return import_reference()
