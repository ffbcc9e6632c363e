"""Shared test setup.

``-m gpu`` tests run the CUDA path (through the C ABI) against the golden
fixtures / the CPU oracle; everything else runs on CPU.  /root/reference is
never read here: the reference's outputs travel as tests/golden/ fixtures.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: config-scale case (minutes of CPU or large HBM)")


class SmallCase:
    def __init__(self, name, data):
        self.name = name
        p = f"{name}/"
        self.n = int(data[p + "n"])
        self.pairs = data[p + "pairs"]
        self.row = data[p + "row_offsets"]
        self.nb = data[p + "neighbors"]
        self.eu = data[p + "edge_u"]
        self.ev = data[p + "edge_v"]
        self.level = data[p + "level"]
        self.parent = data[p + "parent"]
        self.edge_class = data[p + "edge_class"]
        self.components = int(data[p + "components"])
        self.max_level = int(data[p + "max_level"])
        self.cover = data[p + "cover"]
        self.ratio = float(data[p + "ratio"])
        self.T = int(data[p + "T"])
        self.c1 = int(data[p + "c1"])
        self.c2 = int(data[p + "c2"])
        self.deg_row = data[p + "deg_row_offsets"]
        self.deg_nb = data[p + "deg_neighbors"]
        self.fe_forward = bool(data[p + "fe_forward"])

    @property
    def m(self):
        return len(self.eu)

    def __repr__(self):
        return f"SmallCase({self.name})"


def _load_small():
    data = np.load(GOLDEN / "small_cases.npz")
    return [SmallCase(str(n), data) for n in data["_names"]]


SMALL_CASES = _load_small()
SMALL_IDS = [c.name for c in SMALL_CASES]


def config_goldens() -> dict:
    p = GOLDEN / "configs.json"
    return json.loads(p.read_text()) if p.exists() else {}


@pytest.fixture(scope="session")
def small_cases():
    return SMALL_CASES


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
