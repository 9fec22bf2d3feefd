"""Sharded CP-ALS protocol under gloo, world sizes 2 and 3, on CPU.

The driver (paper_2510_14891_b200.sharded) is run with a CPU oracle compute
backend (test-only) so the partition, the collectives and the fit assembly
are checked without a GPU: every rank must reproduce the single-process
oracle cp_als trajectory (cpals.py:92-171 restated in oracle/)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2510_14891_b200 import sharded
from paper_2510_14891_b200.cpals import AlsConfig
from paper_2510_14891_b200.dtensor import DenseTensor


class NumpyOps:
    """Test-only compute backend for the sharded protocol (the oracle)."""

    def prepare_tensor(self, y):
        return np.asarray(y.data if isinstance(y, DenseTensor) else y, dtype=np.float64).ravel()

    def asarray(self, a):
        return np.array(a, dtype=np.float64)

    def ones(self, r):
        return np.ones(r)

    def copy(self, a):
        return a.copy()

    def all_finite(self, y):
        return bool(np.all(np.isfinite(y)))

    def sumsq(self, y):
        return np.array([float(y @ y)])

    def mttkrp(self, y, local_dims, factors, k):
        return oracle.mttkrp_ref(y, local_dims, k, factors)

    def gram(self, a):
        return oracle.gram(a) if a.shape[0] else np.zeros((a.shape[1], a.shape[1]))

    def hadamard(self, grams, skip):
        out = np.ones_like(grams[0])
        for m, g in enumerate(grams):
            if m != skip:
                out = out * g
        return out

    def solve(self, gamma, g):
        return oracle._solve_normal(gamma, g) if g.shape[0] else g

    def colnorms_sq(self, a):
        return np.sum(a * a, axis=0)

    def scale_columns(self, a, nsq):
        nrm = np.sqrt(nsq)
        nz = nrm > 0
        a[:, nz] /= nrm[nz]
        return np.where(nz, nrm, 0.0)

    def fit_terms(self, h, lam, g, a):
        return np.array([float(lam @ h @ lam), float(np.sum((g * lam) * a))])

    def to_host(self, x):
        return np.asarray(x)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, rank_r, mode, iters, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.Philox(42))
        data = rng.random(int(np.prod(dims)))
        part = sharded.partition_for(dims, world, mode)
        y_local = sharded.local_slab(DenseTensor(dims, data), part, rank)
        model, tr = sharded.cp_als_sharded(y_local, part, AlsConfig(rank=rank_r, tol=0.0, max_iters=iters, seed=3),
                                           sharded.Comm(), NumpyOps())
        out_q.put((rank, tr.fits, [np.asarray(a) for a in model.factors], np.asarray(model.weights), tr.comm_bytes))
    finally:
        dist.destroy_process_group()


def _run(world, dims, rank_r, mode, iters):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, rank_r, mode, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


@pytest.mark.parametrize(
    "world,dims,mode",
    [(2, (9, 6, 5), None), (3, (7, 8, 5), 1), (2, (6, 5, 4, 3), 3), (3, (10, 4, 3, 2), 0)],
)
def test_sharded_protocol_matches_single_process(world, dims, mode):
    rank_r, iters = 3, 6
    rng = np.random.Generator(np.random.Philox(42))
    data = rng.random(int(np.prod(dims)))
    lam_ref, f_ref, fits_ref = oracle.cp_als(data, dims, rank_r, max_iters=iters, tol=0.0, seed=3, mttkrp="ref")
    res = _run(world, dims, rank_r, mode, iters)
    for rank, fits, factors, lam, nbytes in res:
        assert np.max(np.abs(np.asarray(fits) - np.asarray(fits_ref))) <= 1e-10, rank
        assert oracle.rel_err(lam, lam_ref) <= 1e-9
        for a, b in zip(factors, f_ref):
            assert a.shape == b.shape
            assert oracle.rel_err(a, b) <= 1e-9
        assert nbytes > 0
    # every rank holds the same model
    for r in res[1:]:
        assert r[1] == res[0][1]


def test_partition_bounds_cover_the_mode():
    for n, world in [(4096, 8), (10, 3), (7, 7), (5, 2)]:
        part = sharded.partition_for((n, 3), world, 0)
        spans = [part.bounds(r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    assert sharded.partition_for((4096, 2048, 2048), 8).mode == 0
    assert sharded.partition_for((5, 9, 9), 2).mode == 1
    with pytest.raises(Exception):
        sharded.partition_for((2, 2), 3, 0)


def test_local_slab_is_the_mode_block():
    dims = (4, 6, 5)
    data = np.arange(120, dtype=np.float64)
    full = data.reshape(dims, order="F")
    part = sharded.partition_for(dims, 3, 1)
    for r in range(3):
        lo, hi = part.bounds(r)
        sl = sharded.local_slab(DenseTensor(dims, data), part, r)
        assert sl.dims == part.local_dims(r)
        assert np.array_equal(np.asarray(sl.data).reshape(sl.dims, order="F"), full[:, lo:hi, :])
