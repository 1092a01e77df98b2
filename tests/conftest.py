"""Shared fixtures.  GPU tests are marked `gpu`; CPU tests run anywhere."""

import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def load_golden(name):
    with gzip.open(os.path.join(GOLDEN, name), "rb") as fh:
        return json.loads(fh.read())


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def to_workers(a):
    """ShardAssignment -> golden-vector form [[[pos, start, end], ...], ...]."""
    return [[[p, r.start, r.end] for p, r in w] for w in a.workers]
