"""Shared fixtures. GPU tests carry @pytest.mark.gpu; everything else runs on CPU."""
from __future__ import annotations

import functools
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run through gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def T():
    import paper_1601_05871_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def oracle():
    from checkers import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=None)
def analyzed(name: str):
    """(raw matrix, analysis) of a golden case, built with this repo's host analysis."""
    import paper_1601_05871_b200 as T
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        g = json.load(f)[name]
    kind, p0, p1, seed = g["generator"]
    a = T.generate(kind, p0, p1, seed)
    an = T.analyze(a, level=g["level"], leaf_size=g["leaf_size"])
    return a, an


@functools.lru_cache(maxsize=None)
def planned(name: str):
    import paper_1601_05871_b200 as T
    _, an = analyzed(name)
    return T.Plan(an.a_permuted, an.pattern, an.ranges)


def bitwise_equal(x: np.ndarray, y: np.ndarray) -> bool:
    return x.shape == y.shape and np.array_equal(x.view(np.int64), y.view(np.int64))


def max_rel_diff(x: np.ndarray, ref: np.ndarray) -> float:
    """Reference verify formula (tools/taskchol.cpp:209-214)."""
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(x - ref) / (np.abs(ref) + 1e-300)))
