"""Sharded multi-GPU CP-ALS: block partition along the longest mode, NCCL.

The reference runs on one CPU process; the paper's distributed
GenTen CP-ALS redistributes the tensor and all-reduces.
This driver needs no redistribution: each rank (one process per GPU,
torchrun) holds one contiguous slab of the tensor along mode s, generated or
loaded straight into its own HBM, and runs the same sweep as cp_als
(cpals.py:118-159) -- literally: both drivers run als_sweep.run_sweeps --
with these exchange steps, all on device tensors, stream-ordered:

* mode k != s: the local MTTKRP of the slab is a partial sum of G_k
  (I_k x R); one allreduce makes G_k whole, and the (replicated) solve,
  normalization and Gram then run bit-identically on every rank;
* mode k == s: the local MTTKRP gives exactly this rank's rows of G_s (no
  communication); the solve updates the local rows; the column norms and the
  Gram of A_s are sums over rows -> one allreduce of R values and one of
  R x R;
* once per sweep, the (2 + d)-scalar stats vector (fit terms + Cholesky
  flags) with replicated terms masked to rank 0's copy: <Y, M> is a sum over
  rows when the last mode is the shard mode, and every rank sees the same
  flags, so a speculative-solve rollback is taken by all ranks or none.
  ||Y||^2 is reduced once.

Per sweep that is (d-1) allreduces of I_k x R, one R x R, one R-vector and
one (2 + d)-vector: ~18 MiB at config 5 (R = 512), against ~0.15 s of MTTKRP
per mode per GPU at 8 GPUs.  The communicator is strict (Comm(device=...)):
a CPU tensor reaching a collective raises instead of failing inside NCCL.

The compute backend is injectable (`backend`): DeviceBackend runs the sm_100a
C-ABI kernels (the only production backend); tests drive the same engine
with a CPU oracle backend under gloo to check the collective logic.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
import importlib

mt = importlib.import_module(".mttkrp", __package__)  # the submodule (the package re-exports a function of the same name)
from ._device import require_cuda, stream_ptr
from .als_sweep import Comm, DeviceBackend, Shard, run_sweeps  # noqa: F401  (Comm is part of this module's API)
from .cpals import AlsConfig, AlsTrace
from .dtensor import DenseTensor, check_dims, num_elements
from .errors import ParameterError, ShapeError
from .kruskal import KruskalTensor


# --------------------------------------------------------------- partition
@dataclass(frozen=True)
class Partition:
    """Block partition of `dims` along `mode` over `world` ranks; the first
    (I_s mod world) ranks get one extra slice."""

    dims: tuple
    mode: int
    world: int

    def bounds(self, rank: int) -> tuple:
        n = self.dims[self.mode]
        base, rem = divmod(n, self.world)
        lo = rank * base + min(rank, rem)
        return lo, lo + base + (1 if rank < rem else 0)

    def local_dims(self, rank: int) -> tuple:
        lo, hi = self.bounds(rank)
        return tuple(hi - lo if m == self.mode else e for m, e in enumerate(self.dims))


def partition_for(dims, world: int, mode: int | None = None) -> Partition:
    """Partition along `mode`, default the longest mode (lowest on ties)."""
    dims = check_dims(dims)
    if world < 1:
        raise ParameterError(f"world size must be >= 1, got {world}")
    if mode is None:
        mode = max(range(len(dims)), key=lambda m: (dims[m], -m))
    if not 0 <= mode < len(dims):
        raise ParameterError(f"shard mode {mode} out of range")
    if dims[mode] < world:
        raise ShapeError(f"cannot split extent {dims[mode]} of mode {mode} over {world} ranks")
    return Partition(dims, int(mode), int(world))


# ------------------------------------------------------------------ driver
@dataclass
class ShardedTrace(AlsTrace):
    sweep_seconds: list = None
    comm_seconds: float = 0.0
    comm_bytes: int = 0
    comm_calls: int = 0
    world: int = 1
    shard_mode: int = 0
    rollbacks: int = 0


def local_slab(y: DenseTensor, part: Partition, rank: int) -> DenseTensor:
    """This rank's slab of a full tensor (host or device payload)."""
    lo, hi = part.bounds(rank)
    s = part.mode
    pre = num_elements(part.dims[:s])
    post = num_elements(part.dims[s + 1:])
    data = y.data
    if isinstance(data, torch.Tensor):
        v = data.view(post, part.dims[s], pre)[:, lo:hi, :].contiguous().view(-1)
    else:
        v = np.ascontiguousarray(np.asarray(data).reshape(post, part.dims[s], pre)[:, lo:hi, :]).ravel()
    return DenseTensor(part.local_dims(rank), v)


def uniform_slab(part: Partition, rank: int, seed: int = 0, device=None) -> DenseTensor:
    """This rank's slab of the synthetic splitmix tensor, generated on its GPU."""
    dev = require_cuda(device)
    lo, hi = part.bounds(rank)
    local = part.local_dims(rank)
    buf = torch.empty(num_elements(local), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().cpk_fill_uniform_slab_f64(buf.data_ptr(), len(part.dims), _lib.i64_array(part.dims),
                                                     part.mode, lo, hi, int(seed), stream_ptr(dev)), "fill slab")
    return DenseTensor(local, buf)


def dten_slab(path, part: Partition, rank: int, device=None) -> DenseTensor:
    """This rank's slab of a DTEN file, read straight into its GPU
    (cpk_dten_load_slab_f64): only rows [lo, hi) of the partition mode are
    read from disk, so ingest needs no redistribution."""
    from .dtensor import read_dten, read_dten_header

    if tuple(read_dten_header(path)) != tuple(part.dims):
        raise ShapeError(f"{path} holds {read_dten_header(path)}, partition is for {part.dims}")
    lo, hi = part.bounds(rank)
    return read_dten(path, device=require_cuda(device), mode=part.mode, lo=lo, hi=hi)


def cp_als_sharded(y_local, part: Partition, config: AlsConfig, comm: Comm | None = None, backend=None,
                   gather: bool = True, graph: bool | None = None):
    """CP-ALS over a row-partitioned tensor; every rank returns the same
    (lam, factors) model (shard factor gathered when `gather`) and trace.

    The sweep is als_sweep.run_sweeps -- the single-GPU engine (speculative
    side-stream solves, one host sync per sweep) -- with the exchange steps
    of the module doc.  `backend` defaults to the sm_100a DeviceBackend on
    the current device; `graph` (CUDA-graph replay) is for world 1 only.
    """
    config.validate()
    if comm is None:
        comm = Comm(device=require_cuda() if backend is None else None)
    if comm.world != part.world:
        raise ParameterError(f"partition is for {part.world} ranks, communicator has {comm.world}")
    rank = comm.rank
    s, dims = part.mode, part.dims
    lo, hi = part.bounds(rank)
    local_dims = part.local_dims(rank)
    d, r = len(dims), config.rank
    t_start = time.perf_counter()
    pad = False
    if backend is None:
        dev = require_cuda()
        if comm.device is None:
            comm.device = dev
        if isinstance(y_local, DenseTensor):
            if tuple(y_local.dims) != tuple(local_dims):
                raise ShapeError(f"local slab has dims {y_local.dims}, partition gives {local_dims}")
            y_t = y_local
        else:
            y_t = DenseTensor(local_dims, y_local.to(dev, dtype=torch.float64).reshape(-1))
        # an odd local I_0 runs on the zero-padded even copy, as in cp_als
        pad = mt._pad_first_mode(y_t, mt.plan_for_mode(config.plan, local_dims, 0), dev) and d >= 2
        run_dims = ((local_dims[0] + 1,) + local_dims[1:]) if pad else local_dims
        y_src = y_t.device_data(dev)
        backend = DeviceBackend(y_t.even_device_data(dev) if pad else y_src, run_dims, r, config.plan, dev)
    else:
        y_src = backend.y
    shard = Shard(s, lo, hi) if comm.world > 1 else None
    res = run_sweeps(backend, dims, r, config.seed, config.max_iters, config.tol, y_src, comm=comm, shard=shard,
                     graph=graph, pad_first=pad, tree=config.dimtree)
    total = time.perf_counter() - t_start
    factors = res.factors
    if pad:
        factors[0] = factors[0][: local_dims[0]]
    if gather and comm.world > 1:
        factors[s] = comm.allgather_rows(factors[s].contiguous(), [part.bounds(q) for q in range(comm.world)])
    model = KruskalTensor(res.lam, factors, validate=False)
    trace = ShardedTrace(fits=res.fits, mttkrp_seconds=res.mttkrp_seconds, other_seconds=res.other_seconds,
                         total_seconds=total, iterations=len(res.fits), converged=res.converged,
                         sweep_seconds=res.sweep_seconds, comm_seconds=comm.seconds, comm_bytes=comm.bytes,
                         comm_calls=comm.calls, world=comm.world, shard_mode=s, rollbacks=res.rollbacks,
                         tree_split=res.tree_split)
    return model, trace
