"""Shared test fixtures.

Markers: ``gpu`` -- needs a CUDA device (B200); run with ``-m gpu``.
Everything else runs on CPU (``-m "not gpu"``).
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def small_golden():
    d = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    names = sorted({k.split("/")[0] for k in d.files})
    cases = {}
    for n in names:
        cases[n] = {k.split("/", 1)[1]: d[k] for k in d.files if k.startswith(n + "/")}
    return cases


@pytest.fixture(scope="session")
def config_golden():
    import json
    d = np.load(os.path.join(GOLDEN, "configs.npz"))
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        index = json.load(f)
    out = {}
    for meta in index["configs"]:
        n = meta["name"]
        out[n] = {"meta": meta,
                  **{k.split("/", 1)[1]: d[k] for k in d.files if k.startswith(n + "/")}}
    return out


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
