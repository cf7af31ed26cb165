"""Shared test plumbing: the ``gpu`` marker, golden-fixture loading, oracle import."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
# a single-request CUDA-graph capture that fails is a test failure, not a silent step-by-step
# fallback (paper_2511_14881_b200/fastpath.py)
os.environ.setdefault("FB_GRAPH_STRICT", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


def load_npz(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)


def load_json(name: str):
    return json.loads((GOLDEN / name).read_text())


def json_to_expr(j):
    """Golden JSON expr -> package AST."""
    from paper_2511_14881_b200.filter_query import And, Leaf, Not, Or
    kind = j[0]
    if kind == "leaf":
        return Leaf(int(j[1]), int(j[2]))
    if kind == "not":
        return Not(json_to_expr(j[1]))
    cls = And if kind == "and" else Or
    return cls(tuple(json_to_expr(c) for c in j[1]))


def json_to_oracle_expr(j):
    kind = j[0]
    if kind == "leaf":
        return ("leaf", int(j[1]), int(j[2]))
    if kind == "not":
        return ("not", json_to_oracle_expr(j[1]))
    return (kind, [json_to_oracle_expr(c) for c in j[1]])


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_14881_b200 import _native
    _native.lib()  # loud failure if the sm_100a library is missing
    return torch.device("cuda:0")
