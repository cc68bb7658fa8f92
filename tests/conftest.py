"""Shared fixtures.  Tests marked ``gpu`` need a B200 (run with -m gpu);
everything else runs on CPU (-m "not gpu")."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


class Golden:
    """Access to one golden npz: cases are '<key>__<field>' entries."""

    def __init__(self, name):
        self.z = np.load(GOLDEN / f"{name}.npz")

    def keys(self, suffix):
        return sorted({k.rsplit("__", 1)[0] for k in self.z.files if k.endswith("__" + suffix)})

    def case(self, key):
        pre = key + "__"
        out = {}
        for k in self.z.files:
            if k.startswith(pre):
                f = k[len(pre):]
                v = self.z[k]
                out[f] = json.loads(bytes(v).decode()) if f == "spec" else v
        return out


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]
    return get


def oracle_cover(case):
    """Oracle covering rebuilt from a golden case's root + paths."""
    from oracle import gis_oracle as O

    lo, hi = O.boxes_from_paths(case["root_lo"], case["root_hi"], case["depths"], case["bits"])
    return O.Cover(case["root_lo"], case["root_hi"], case["depths"], case["bits"], lo, hi,
                   presorted=True)


def peeling_fixed_point(n_vertices, edges):
    """tests/conftest.py:75-89 of the reference (zero-out-degree peeling)."""
    alive = np.ones(n_vertices, dtype=bool)
    if not edges:
        return alive & False
    src = np.array([e[0] for e in edges], dtype=np.int64)
    dst = np.array([e[1] for e in edges], dtype=np.int64)
    while True:
        live = alive[src] & alive[dst]
        dead = alive & (np.bincount(src[live], minlength=n_vertices) == 0)
        if not dead.any():
            return alive
        alive &= ~dead


def grid_boxes(nx, ny, width=1.0):
    lo = np.array([(c * width, r * width) for r in range(ny) for c in range(nx)], dtype=float)
    return lo, lo + width
