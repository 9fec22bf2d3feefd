"""Sharded CP-ALS protocol under gloo, world sizes 2 and 3, on CPU.

The driver (paper_2510_14891_b200.sharded) is run with a CPU oracle compute
backend (test-only) so the partition, the collectives and the fit assembly
are checked without a GPU: every rank must reproduce the single-process
oracle cp_als trajectory (cpals.py:92-171 restated in oracle/)."""

import os
import socket
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2510_14891_b200 import als_sweep, sharded
from paper_2510_14891_b200.cpals import AlsConfig
from paper_2510_14891_b200.dtensor import DenseTensor


class _Clock:
    def record(self):
        self.t = time.perf_counter()

    def seconds_to(self, other):
        return other.t - self.t

    def synchronize(self):
        pass


class CpuOracleBackend:
    """Test-only backend for als_sweep.run_sweeps: torch CPU tensors, the
    oracle's kernels (oracle/, restating cpals.py / kruskal.py / _kernels.py).
    Same interface as als_sweep.DeviceBackend, so the engine and its
    collectives are the production ones."""

    graphable = False

    def __init__(self, y, run_dims):
        self.y = torch.as_tensor(np.asarray(y.data if isinstance(y, DenseTensor) else y, dtype=np.float64)).ravel()
        self.dims = tuple(run_dims)
        self._chol = None

    def tensor(self, *shape, dtype=torch.float64):
        return torch.zeros(shape, dtype=dtype)

    def upload(self, a):
        return torch.from_numpy(np.array(a, dtype=np.float64))

    def host_buffer(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def stamp(self):
        return _Clock()

    def sumsq(self, x, out):
        v = x.numpy()
        out[0] = float(v @ v)

    def gram(self, a, out):
        out.copy_(torch.from_numpy(oracle.gram(a.numpy())))

    def hadamard(self, grams, skip, out):
        h = np.ones(tuple(out.shape))
        for m, g in enumerate(grams):
            if m != skip:
                h = h * g.numpy()
        out.copy_(torch.from_numpy(h))

    def mttkrp(self, factors, k, out):
        out.copy_(torch.from_numpy(oracle.mttkrp_ref(self.y.numpy(), self.dims, k, [f.numpy() for f in factors])))

    def factor_spec(self, gamma, info_k):
        from scipy.linalg import cho_factor

        try:
            self._chol = cho_factor(gamma.numpy().copy(), check_finite=False)
            info_k[0] = 0
        except np.linalg.LinAlgError:
            self._chol = None
            info_k[0] = 1

    def apply_spec(self, g, info_k):
        from scipy.linalg import cho_solve

        if int(info_k[0]) == 0:
            g.copy_(torch.from_numpy(cho_solve(self._chol, g.numpy().T, check_finite=False).T.copy()))

    def solve_ladder(self, gamma, g):
        g.copy_(torch.from_numpy(np.ascontiguousarray(oracle._solve_normal(gamma.numpy(), g.numpy()))))

    def colnorms_sq(self, a, out):
        v = a.numpy()
        out.copy_(torch.from_numpy(np.sum(v * v, axis=0)))

    def scale_columns(self, a, normsq, lam):
        nrm = np.sqrt(normsq.numpy())
        nz = nrm > 0
        v = a.numpy()
        v[:, nz] /= nrm[nz]
        lam.copy_(torch.from_numpy(np.where(nz, nrm, 0.0)))

    def fit_terms(self, h, lam, g, a, out):
        lv = lam.numpy()
        out[0] = float(lv @ h.numpy() @ lv)
        out[1] = float(np.sum((g.numpy() * lv) * a.numpy()))

    # dimension tree (als_sweep.tree_split): W_G from the oracle's MTTKRP of
    # the merged view, the in-group contraction in numpy
    def tree_budget(self):
        return 1 << 40

    def setup_tree(self, p):
        self.tree_p = p
        self.tree_groups = als_sweep.tree_groups(len(self.dims), p)
        self.tree_w = [None, None]

    def tree_mttkrp(self, gi, factors):
        p, grp = self.tree_p, self.tree_groups[gi]
        ig = int(np.prod([self.dims[m] for m in grp]))
        r = factors[0].shape[1]
        fs = [f.numpy() for f in factors]
        if gi == 0:
            vdims, vf, k = (ig,) + self.dims[p:], [np.zeros((ig, r))] + fs[p:], 0
        else:
            vdims, vf, k = self.dims[:p] + (ig,), fs[:p] + [np.zeros((ig, r))], p
        self.tree_w[gi] = oracle.mttkrp_ref(self.y.numpy(), vdims, k, vf)

    def tree_contract(self, gi, factors, j, out):
        grp = self.tree_groups[gi]
        g, ext = len(grp), [self.dims[m] for m in grp]
        r = out.shape[1]
        t = self.tree_w[gi].reshape(tuple(reversed(ext)) + (r,))  # first-mode-fastest rows
        for l, m in enumerate(grp):
            if l != j:
                shape = [1] * g + [r]
                shape[g - 1 - l] = ext[l]
                t = t * factors[m].numpy().reshape(shape)
        out.copy_(torch.from_numpy(np.ascontiguousarray(t.sum(axis=tuple(g - 1 - l for l in range(g) if l != j)))))

    def readback(self, src, dst):
        dst.copy_(src)

    def synchronize(self):
        pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, rank_r, mode, iters, out_q, tree=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.Philox(42))
        data = rng.random(int(np.prod(dims)))
        part = sharded.partition_for(dims, world, mode)
        y_local = sharded.local_slab(DenseTensor(dims, data), part, rank)
        be = CpuOracleBackend(y_local, part.local_dims(rank))
        cfg = AlsConfig(rank=rank_r, tol=0.0, max_iters=iters, seed=3, dimtree=tree)
        model, tr = sharded.cp_als_sharded(y_local, part, cfg, sharded.Comm(), backend=be)
        out_q.put((rank, tr.fits, [np.asarray(a) for a in model.factors], np.asarray(model.weights), tr.comm_bytes,
                   tr.comm_calls, tr.tree_split))
    finally:
        dist.destroy_process_group()


def _run(world, dims, rank_r, mode, iters, tree=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, rank_r, mode, iters, q, tree))
             for r in range(world)]
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
    d = len(dims)
    for rank, fits, factors, lam, nbytes, calls, _ in res:
        assert np.max(np.abs(np.asarray(fits) - np.asarray(fits_ref))) <= 1e-10, rank
        assert oracle.rel_err(lam, lam_ref) <= 1e-9
        for a, b in zip(factors, f_ref):
            assert a.shape == b.shape
            assert oracle.rel_err(a, b) <= 1e-9
        assert nbytes > 0
        # per sweep: d-1 partial G_k, the shard Gram and column norms, the
        # stats vector; plus ||Y||^2 and the initial shard Gram
        assert calls == 2 + iters * (d + 2), calls
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


def test_strict_comm_rejects_host_tensors():
    """A communicator bound to a CUDA device raises on anything but a CUDA
    tensor on that device -- before NCCL sees it (an NCCL group has no CPU
    backend; round 1's numpy flag died there)."""
    from paper_2510_14891_b200.errors import DeviceError

    comm = sharded.Comm(device=torch.device("cuda", 0))
    with pytest.raises(DeviceError):
        comm.allreduce_(torch.zeros(2, dtype=torch.float64))
    with pytest.raises(DeviceError):
        comm.allreduce_(np.zeros(2))
    with pytest.raises(DeviceError):
        comm.allgather_rows(torch.zeros((2, 2)), [(0, 2)])
    # the CPU test communicator accepts host tensors (world 1: a no-op)
    t = torch.ones(3, dtype=torch.float64)
    assert sharded.Comm().allreduce_(t) is t


def _graph_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims = (6, 5, 4)
        data = np.random.Generator(np.random.Philox(1)).random(120)
        part = sharded.partition_for(dims, world)
        y_local = sharded.local_slab(DenseTensor(dims, data), part, rank)
        be = CpuOracleBackend(y_local, part.local_dims(rank))
        try:
            sharded.cp_als_sharded(y_local, part, AlsConfig(rank=2, max_iters=2), sharded.Comm(), backend=be,
                                   graph=True)
            out_q.put((rank, "no error"))
        except Exception as exc:  # noqa: BLE001
            out_q.put((rank, type(exc).__name__))
    finally:
        dist.destroy_process_group()


def test_graph_replay_is_single_rank_only():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_graph_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, "ParameterError"), (1, "ParameterError")]


def test_tree_split_choices():
    """als_sweep.tree_split: the split with the least W_G traffic that fits,
    multi-mode groups holding the shard mode, off when it does not pay."""
    ts = als_sweep.tree_split
    assert ts((4096, 2048, 2048), 512) == 1  # W = I_1 I_2 x R (17 GB), not I_0 I_1 x R
    assert ts((4096, 2048, 2048), 512, shard_mode=0) == 2  # the left group holds mode 0
    assert ts((4096, 2048, 2048), 512, shard_mode=2) == 1
    assert ts((128,) * 4, 256) == 2
    assert ts((1024,) * 3, 2000) == 1
    assert ts((4096, 2048, 2048), 512, budget_bytes=1 << 30) is None
    assert ts((8, 9), 4) is None and ts((8, 9), 4, force=True) is None  # two modes: nothing to share
    # R far above the other group's extents: W_G outweighs the saved pass
    assert ts((36, 20, 28), 70) is None and ts((36, 20, 28), 70, force=True) == 1
    for d in range(3, 8):
        dims = (5,) * d
        for s in range(d):
            p = ts(dims, 3, shard_mode=s, force=True)
            assert p is not None
            assert all(s in g for g in als_sweep.tree_groups(d, p) if len(g) > 1)


@pytest.mark.parametrize("dims,rank", [((9, 6, 5), 3), ((6, 5, 4, 3), 4), ((4, 3, 5, 2, 3), 2),
                                        ((3, 4, 2, 3, 2, 3), 3)])
def test_tree_sweep_matches_oracle(dims, rank):
    """The dimension-tree sweep (W_G + in-group contraction) on the oracle
    backend follows the oracle's per-mode cp_als trajectory."""
    rng = np.random.Generator(np.random.Philox(9))
    data = rng.random(int(np.prod(dims)))
    be = CpuOracleBackend(data, dims)
    res = als_sweep.run_sweeps(be, dims, rank, 3, 5, 0.0, be.y, tree=True)
    assert res.tree_split is not None
    lam_ref, f_ref, fits_ref = oracle.cp_als(data, dims, rank, max_iters=5, tol=0.0, seed=3, mttkrp="ref")
    assert np.max(np.abs(np.asarray(res.fits) - np.asarray(fits_ref))) <= 1e-10
    assert oracle.rel_err(res.lam.numpy(), lam_ref) <= 1e-9
    for a, b in zip(res.factors, f_ref):
        assert oracle.rel_err(a.numpy(), b) <= 1e-9


@pytest.mark.parametrize("world,dims,mode", [(2, (9, 6, 5), 0), (3, (7, 8, 5), 2), (2, (6, 5, 4, 3), 1)])
def test_sharded_tree_protocol_matches_single_process(world, dims, mode):
    """Sharded dimension tree: the split keeps every W_G rank-local, the
    collectives are the per-mode sweep's, every rank ends on the oracle
    trajectory."""
    rank_r, iters = 3, 5
    data = np.random.Generator(np.random.Philox(42)).random(int(np.prod(dims)))
    lam_ref, f_ref, fits_ref = oracle.cp_als(data, dims, rank_r, max_iters=iters, tol=0.0, seed=3, mttkrp="ref")
    res = _run(world, dims, rank_r, mode, iters, tree=True)
    d = len(dims)
    for rank, fits, factors, lam, nbytes, calls, split in res:
        assert split is not None
        assert all(mode in g for g in als_sweep.tree_groups(d, split) if len(g) > 1)
        assert np.max(np.abs(np.asarray(fits) - np.asarray(fits_ref))) <= 1e-10, rank
        assert oracle.rel_err(lam, lam_ref) <= 1e-9
        for a, b in zip(factors, f_ref):
            assert oracle.rel_err(a, b) <= 1e-9
        assert calls == 2 + iters * (d + 2), calls
