"""Shared fixtures: golden vectors from the live reference, GPU marker."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs (set GRIDOT_FULL=1)")


def _load(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    index = json.loads(str(z["index"]))
    cases = []
    for entry in index:
        tag = entry["tag"]
        pre = tag + "/"
        data = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
        data.update(entry)
        data["dims"] = tuple(int(x) for x in data["dims"])
        data["kappa"] = int(data["kappa"])
        data["p"] = float(data["p"])
        cases.append(data)
    return cases


@pytest.fixture(scope="session")
def small_cases():
    return _load("small_cases.npz")


@pytest.fixture(scope="session")
def config_cases():
    return _load("configs.npz")


def case_ids(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    return [e["tag"] for e in json.loads(str(z["index"]))]


def rel_close(a, b, tol):
    return abs(a - b) <= tol * max(1.0, abs(a), abs(b))


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
