"""Sharded driver on the device (world 1 here; the collectives are covered by
the gloo tests in test_sharded.py): DeviceOps must reproduce cp_als."""

import numpy as np
import pytest
import torch

import paper_2510_14891_b200 as ck
from oracle import gen, oracle
from paper_2510_14891_b200 import sharded

pytestmark = pytest.mark.gpu


def test_device_ops_world1_matches_cp_als():
    dims = (40, 36, 34)
    rng = np.random.Generator(np.random.Philox(4))
    y = ck.DenseTensor(dims, rng.random(int(np.prod(dims))))
    cfg = ck.AlsConfig(rank=12, tol=0.0, max_iters=5, seed=1)
    _, tr_ref = ck.cp_als(y, cfg)
    part = sharded.partition_for(dims, 1)
    model, tr = sharded.cp_als_sharded(y, part, cfg)
    assert np.max(np.abs(np.asarray(tr.fits) - np.asarray(tr_ref.fits))) <= 1e-12
    _, _, fits_o = oracle.cp_als(y.data, dims, 12, max_iters=5, tol=0.0, seed=1)
    assert np.max(np.abs(np.asarray(tr.fits) - np.asarray(fits_o))) <= 1e-10
    assert len(tr.sweep_seconds) == 5


def test_uniform_slab_matches_cpu_twin():
    dims = (9, 7, 6)
    part = sharded.partition_for(dims, 3, 0)
    full = gen.splitmix_uniform(int(np.prod(dims)), seed=5).reshape(dims, order="F")
    for r in range(3):
        lo, hi = part.bounds(r)
        sl = sharded.uniform_slab(part, r, seed=5)
        got = sl.data.cpu().numpy().reshape(sl.dims, order="F")
        assert np.array_equal(got, full[lo:hi])
    t = ck.DenseTensor.uniform(dims, seed=5)
    assert np.array_equal(t.data.cpu().numpy(), full.ravel(order="F"))
