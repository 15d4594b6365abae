from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


# Worked example of the reference tests (pkg/tests/conftest.py:21-22).
GT_EDGES = [(0, 1), (0, 2), (1, 3), (2, 3), (3, 4), (4, 5), (5, 3)]
GT_VERTICES = 6


class Golden:
    """Lazy access to the committed fixtures (made by golden/make_golden.py)."""

    def __init__(self):
        self._npz = {}
        self._json = {}

    def npz(self, name):
        if name not in self._npz:
            self._npz[name] = np.load(GOLDEN / f"{name}.npz")
        return self._npz[name]

    def meta(self, name):
        if name not in self._json:
            self._json[name] = json.loads((GOLDEN / f"{name}.json").read_text())
        return self._json[name]

    def kernel_case(self, case):
        z = self.npz("kernels")
        p = case["id"]
        gid = str(z[f"{p}/graph"])
        src = z[f"{gid}/src"].astype(np.int64)
        dst = z[f"{gid}/dst"].astype(np.int64)
        w = z[f"{gid}/w"].astype(np.int64) if f"{gid}/w" in z.files else None
        out = dict(src=src, dst=dst, w=w)
        for k in ("prev", "out", "wedge", "frontier"):
            if f"{p}/{k}" in z.files:
                out[k] = z[f"{p}/{k}"]
        if f"{p}/chg_idx" in z.files:
            nxt = out["prev"].copy()
            nxt[z[f"{p}/chg_idx"]] = z[f"{p}/chg_val"]
            out["nxt"] = nxt
        return out


@pytest.fixture(scope="session")
def golden():
    return Golden()


def kern_of(app):
    import oracle
    return oracle.kern_of(app)
