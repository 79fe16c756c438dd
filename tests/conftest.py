import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_kernels.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: longer CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN, allow_pickle=False))


def golden_scene(g, name):
    p = f"ev_{name}_"
    return {k[len(p):]: v for k, v in g.items() if k.startswith(p)}


def golden_domain(g, which="unit"):
    return tuple(g[f"dom_{which}_{k}"] for k in ("dv", "dc", "dp", "dt", "dlp", "dlv"))


OUT_KEYS = ("status", "vol", "ksur", "cent", "ipt", "m2", "fcount", "ftag", "farea", "fh",
            "fnrm", "fcent")
