import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def rng_for(seed):
    return np.random.Generator(np.random.Philox(seed))


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz"))
        return cache[name]

    return load


def instances(store):
    """(key, dims, data, lam, factors, [G_k]) for every packed instance."""
    keys = sorted({k.split("/")[0] for k in store if "/" in k})
    out = []
    for key in keys:
        dims = tuple(int(x) for x in store[f"{key}/dims"])
        d = len(dims)
        out.append((key, dims, store[f"{key}/data"], store[f"{key}/lam"],
                    [store[f"{key}/A{j}"] for j in range(d)], [store[f"{key}/G{k}"] for k in range(d)]))
    return out
