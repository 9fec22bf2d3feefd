"""Sharded driver on the device.  World 1 is the cp_als engine itself (bitwise);
world 2-3 runs as several processes on the one GPU with gloo carrying CUDA
tensors through the strict communicator (NCCL refuses two ranks on one GPU,
so this is the closest the one-GPU box gets to the production data plane:
every collective must see a device tensor or the Comm raises)."""

import numpy as np
import pytest
import torch

import paper_2510_14891_b200 as ck
from oracle import gen, oracle
from paper_2510_14891_b200 import als_sweep, sharded

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tree", [None, True])
@pytest.mark.parametrize("dims", [(40, 36, 34), (41, 10, 6, 12)])
def test_world1_sharded_is_cp_als_bitwise(dims, tree):
    rng = np.random.Generator(np.random.Philox(4))
    y = ck.DenseTensor(dims, rng.random(int(np.prod(dims))))
    cfg = ck.AlsConfig(rank=12, tol=0.0, max_iters=5, seed=1, dimtree=tree)
    ref, tr_ref = ck.cp_als(y, cfg, graph=False)
    part = sharded.partition_for(dims, 1)
    model, tr = sharded.cp_als_sharded(y, part, cfg)
    assert tr.fits == tr_ref.fits
    assert torch.equal(model.weights, ref.weights)
    for a, b in zip(model.factors, ref.factors):
        assert torch.equal(a, b)
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


def _gpu_worker(rank, world, port, dims, rank_r, iters, dten, out_q, tree=None):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # gloo with CUDA tensors: every rank on cuda:0 (one GPU here); the
    # kernels, partition, collectives and fit assembly are the real path
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        part = sharded.partition_for(dims, world)
        if dten:
            y_local = sharded.dten_slab(dten, part, rank, device="cuda")
        else:
            y_local = sharded.uniform_slab(part, rank, seed=7)
        comm = sharded.Comm(device=torch.device("cuda", 0))  # strict: CUDA tensors only
        model, tr = sharded.cp_als_sharded(y_local, part, ck.AlsConfig(rank=rank_r, tol=0.0, max_iters=iters,
                                                                       seed=3, dimtree=tree), comm)
        out_q.put((rank, tr.fits, [a.cpu().numpy() for a in model.factors], model.weights.cpu().numpy(),
                   tr.comm_calls, tr.tree_split))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,dten,tree", [(2, (40, 36, 34), False, None), (3, (30, 20, 8, 6), False, None),
                                                  (2, (33, 24, 18), True, None), (2, (40, 36, 34), False, True),
                                                  (3, (30, 20, 8, 6), False, True)])
def test_multi_process_device_path_matches_single_process(tmp_path, world, dims, dten, tree):
    """world 2-3 processes, each running the sm_100a kernels on its slab
    (generated on device, or read from a DTEN file), gloo collectives:
    every rank ends with the single-process trajectory and model."""
    import socket

    import torch.multiprocessing as mp

    full = gen.splitmix_uniform(int(np.prod(dims)), seed=7)
    path = None
    if dten:
        path = str(tmp_path / "y.dten")
        ck.write_dten(path, ck.DenseTensor(dims, full))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, dims, 6, 4, path, q, tree)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, tr_ref = ck.cp_als(ck.DenseTensor(dims, full), ck.AlsConfig(rank=6, tol=0.0, max_iters=4, seed=3))
    part = sharded.partition_for(dims, world)
    for rank, fits, factors, lam, calls, split in res:
        if tree:  # the dimension tree on the slabs: every multi-mode group holds the shard mode
            assert split is not None
            assert all(part.mode in g for g in als_sweep.tree_groups(len(dims), split) if len(g) > 1)
        assert np.max(np.abs(np.asarray(fits) - np.asarray(tr_ref.fits))) <= 1e-10, rank
        assert calls == 2 + 4 * (len(dims) + 2)
        assert [a.shape for a in factors] == [(n, 6) for n in dims]
        assert np.array_equal(factors[1], res[0][2][1]) and np.array_equal(lam, res[0][3])  # replicated


class _CountingBackend(sharded.DeviceBackend):
    readbacks = 0

    def readback(self, src, dst):
        type(self).readbacks += 1
        super().readback(src, dst)


def test_one_readback_and_no_torch_sync_per_sweep():
    """The loop's only device->host traffic is one stats readback per sweep:
    no torch op inside the sweeps synchronizes.  Sync debug mode counts every
    synchronizing torch call as a warning (the setup's ||Y||^2 readback and
    pageable factor uploads are some); the count must not grow with the
    number of sweeps."""
    import warnings

    from paper_2510_14891_b200 import als_sweep

    dims, r = (40, 36, 34), 8
    y = ck.DenseTensor.uniform(dims, seed=2, device="cuda")

    def syncs_for(iters):
        be = _CountingBackend(y.device_data(), dims, r, ck.MttkrpPlan(ck.Variant.B200, 0))
        _CountingBackend.readbacks = 0
        torch.cuda.synchronize()
        torch.cuda.set_sync_debug_mode("warn")
        try:
            with warnings.catch_warnings(record=True) as w:
                warnings.simplefilter("always")
                res = als_sweep.run_sweeps(be, dims, r, 0, iters, 0.0, y.device_data(), graph=False)
        finally:
            torch.cuda.set_sync_debug_mode(0)
        assert _CountingBackend.readbacks == iters and res.rollbacks == 0
        return len([x for x in w if "synchroniz" in str(x.message)])

    assert syncs_for(6) == syncs_for(2)
