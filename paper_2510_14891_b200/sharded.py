"""Sharded multi-GPU CP-ALS: block partition along the longest mode, NCCL.

The reference runs on one CPU process; the paper's distributed
GenTen CP-ALS redistributes the tensor and all-reduces.
This driver needs no redistribution: each rank (one process per GPU,
torchrun) holds one contiguous slab of the tensor along mode s, generated or
loaded straight into its own HBM, and runs the same sweep as cp_als
(cpals.py:118-159) with three collectives:

* mode k != s: the local MTTKRP of the slab is a partial sum of G_k
  (I_k x R); one allreduce makes G_k whole, and the (replicated) solve,
  normalization and Gram then run bit-identically on every rank;
* mode k == s: the local MTTKRP gives exactly this rank's rows of G_s (no
  communication); the solve updates the local rows; the column norms and the
  Gram of A_s are sums over rows -> one allreduce of R values and one of
  R x R;
* fit: <Y, M> uses the last mode's G; it is a local partial only when the
  last mode is the shard mode.  ||Y||^2 is reduced once.

Per sweep that is (d-1) allreduces of I_k x R, one R x R and one R-vector:
~18 MiB at config 5 (R = 512), against ~1 s of MTTKRP per mode per GPU.

The compute backend is injectable (`ops`): DeviceOps runs the sm_100a C-ABI
kernels (the only production backend); tests drive the same protocol with a
CPU oracle backend under gloo to check the collective logic.
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
from ._device import EventTimer, require_cuda, stream_ptr, workspace
from .cpals import AlsConfig, AlsTrace, _Solver, init_factors
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


# -------------------------------------------------------------------- comm
class Comm:
    """torch.distributed plumbing (NCCL on GPUs, gloo for CPU tests);
    world 1 without an initialized process group is a no-op."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.seconds = 0.0
        self.bytes = 0

    def allreduce_(self, x):
        """Sum in place across ranks; numpy arrays are wrapped zero-copy."""
        if self.world == 1:
            return x
        t = torch.from_numpy(x) if isinstance(x, np.ndarray) else x
        t0 = time.perf_counter()
        self.dist.all_reduce(t, group=self.group)
        self.seconds += time.perf_counter() - t0
        self.bytes += t.numel() * t.element_size()
        return x

    def allgather_rows(self, local, part: Partition):
        """Concatenate each rank's rows of a row-partitioned factor."""
        if self.world == 1:
            return local
        is_np = isinstance(local, np.ndarray)
        t = torch.from_numpy(np.ascontiguousarray(local)) if is_np else local.contiguous()
        r = t.shape[1]
        rows = max(part.bounds(q)[1] - part.bounds(q)[0] for q in range(self.world))
        pad = torch.zeros((rows, r), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        full = torch.cat([o[: part.bounds(q)[1] - part.bounds(q)[0]] for q, o in enumerate(outs)])
        return full.numpy() if is_np else full


# --------------------------------------------------------------- device ops
class DeviceOps:
    """The sm_100a C-ABI kernels, on the current CUDA device and stream."""

    def __init__(self, device=None, plan: mt.MttkrpPlan | None = None):
        self.dev = require_cuda(device)
        self.plan = plan or mt.MttkrpPlan(mt.Variant.B200, 0)
        self.lib = _lib.load()
        self._solver = None
        self.mttkrp_timers = []

    def sp(self):
        return stream_ptr(self.dev)

    def asarray(self, a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.dev)

    def ones(self, r):
        return torch.ones(r, dtype=torch.float64, device=self.dev)

    def copy(self, a):
        return a.clone()

    def all_finite(self, y_local) -> bool:
        # a NaN/Inf anywhere makes the sum of squares non-finite; no N-sized
        # temporaries (c5 is 137 GB)
        return bool(torch.isfinite(self.sumsq(y_local)).item())

    def sumsq(self, y_local):
        out = torch.empty(1, dtype=torch.float64, device=self.dev)
        work = workspace(self.dev, 8 * _lib.CPK_SUMSQ_PARTIALS, tag="sumsq")
        _lib.check(self.lib.cpk_sumsq_f64(y_local.data_ptr(), y_local.numel(), work.data_ptr(), out.data_ptr(),
                                          self.sp()), "sumsq")
        return out

    def mttkrp(self, y_local, local_dims, factors, k):
        plan = mt.plan_for_mode(self.plan, local_dims, k)
        g, _, timer = mt.mttkrp_device(y_local, local_dims, factors, k, None, plan)
        self.mttkrp_timers.append(timer)
        return g

    def gram(self, a):
        r = a.shape[1]
        out = torch.empty((r, r), dtype=torch.float64, device=self.dev)
        if a.shape[0] == 0:
            return out.zero_()
        _lib.check(self.lib.cpk_gram_f64(a.data_ptr(), a.shape[0], r, a.stride(0), out.data_ptr(), self.sp()),
                   "gram")
        return out

    def hadamard(self, grams, skip):
        from .kruskal import hadamard

        return hadamard(grams, skip)

    def prepare_tensor(self, y_local):
        if isinstance(y_local, DenseTensor):
            return y_local.device_data(self.dev)
        return y_local.to(self.dev, dtype=torch.float64).reshape(-1)

    def solve(self, gamma, g):
        if self._solver is None:
            self._solver = _Solver(self.dev, 1, gamma.shape[0])
        if g.shape[0] == 0:
            return g
        return self._solver(gamma, g)

    def colnorms_sq(self, a):
        r = a.shape[1]
        out = torch.zeros(r, dtype=torch.float64, device=self.dev)
        if a.shape[0] > 0:
            _lib.check(self.lib.cpk_colnorms_sq_f64(a.data_ptr(), a.shape[0], r, a.stride(0), out.data_ptr(),
                                                    self.sp()), "colnorms")
        return out

    def scale_columns(self, a, normsq):
        r = a.shape[1]
        lam = torch.empty(r, dtype=torch.float64, device=self.dev)
        # lam is written by the row-0 thread; a shard with no rows still needs it
        lam.copy_(torch.sqrt(normsq))
        if a.shape[0] > 0:
            _lib.check(self.lib.cpk_scale_columns_f64(a.data_ptr(), a.shape[0], r, a.stride(0), normsq.data_ptr(),
                                                      lam.data_ptr(), self.sp()), "scale")
        return lam

    def fit_terms(self, h, lam, g, a):
        out = torch.empty(2, dtype=torch.float64, device=self.dev)
        _lib.check(self.lib.cpk_fit_terms_f64(h.data_ptr(), lam.data_ptr(), g.data_ptr(), a.data_ptr(), g.shape[0],
                                              h.shape[0], out.data_ptr(), self.sp()), "fit terms")
        return out

    def to_host(self, x):
        return x.cpu().numpy()

    def sync(self):
        torch.cuda.synchronize(self.dev)


# ------------------------------------------------------------------ driver
@dataclass
class ShardedTrace(AlsTrace):
    sweep_seconds: list = None
    comm_seconds: float = 0.0
    comm_bytes: int = 0
    world: int = 1
    shard_mode: int = 0


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


def cp_als_sharded(y_local, part: Partition, config: AlsConfig, comm: Comm | None = None, ops=None,
                   gather: bool = True):
    """CP-ALS over a row-partitioned tensor; every rank returns the same
    (lam, factors) model (shard factor gathered when `gather`) and trace."""
    config.validate()
    comm = comm or Comm()
    ops = ops or DeviceOps()
    if comm.world != part.world:
        raise ParameterError(f"partition is for {part.world} ranks, communicator has {comm.world}")
    rank = comm.rank
    s, dims = part.mode, part.dims
    lo, hi = part.bounds(rank)
    local_dims = part.local_dims(rank)
    d, r = len(dims), config.rank
    y_dev = ops.prepare_tensor(y_local)

    bad = np.array([0.0 if ops.all_finite(y_dev) else 1.0])
    comm.allreduce_(bad)
    if bad[0] > 0:
        raise ParameterError("tensor has non-finite entries")
    sq = ops.sumsq(y_dev)
    comm.allreduce_(sq)
    norm_y = math.sqrt(float(ops.to_host(sq).ravel()[0]))
    if norm_y == 0.0:
        raise ParameterError("cannot fit an all-zero tensor (fit is undefined)")

    t_start = time.perf_counter()
    init = init_factors(dims, r, config.seed)  # replicated Philox stream (cpals.py:108-109)
    init[s] = init[s][lo:hi]
    factors = [ops.asarray(a) for a in init]
    grams = [ops.gram(a) for a in factors]
    comm.allreduce_(grams[s])
    lam = ops.ones(r)

    fits, mttkrp_seconds, other_seconds, sweep_seconds = [], [], [], []
    converged = False
    if hasattr(ops, "sync"):
        ops.sync()
    for _ in range(config.max_iters):
        t_sweep = time.perf_counter()
        sweep_mt = []
        g_last = None
        for k in range(d):
            t0 = time.perf_counter()
            g = ops.mttkrp(y_dev, local_dims, factors, k)
            if k != s:
                comm.allreduce_(g)
            if hasattr(ops, "mttkrp_timers") and ops.mttkrp_timers:
                sweep_mt.append(ops.mttkrp_timers[-1])
            else:
                sweep_mt.append(time.perf_counter() - t0)
            gamma = ops.hadamard(grams, k)
            if k == d - 1:
                g_last = ops.copy(g)
            a_hat = ops.solve(gamma, g)
            nsq = ops.colnorms_sq(a_hat)
            if k == s:
                comm.allreduce_(nsq)
            lam = ops.scale_columns(a_hat, nsq)
            factors[k] = a_hat
            grams[k] = ops.gram(a_hat)
            if k == s:
                comm.allreduce_(grams[k])
        h = ops.hadamard(grams, -1)
        terms = ops.fit_terms(h, lam, g_last, factors[d - 1])
        if d - 1 == s:
            # <Y, M> is a sum over the rows of the shard mode
            part_ip = terms[1:2].clone() if isinstance(terms, torch.Tensor) else terms[1:2].copy()
            comm.allreduce_(part_ip)
            terms[1:2] = part_ip
        norm_m_sq, iprod = (float(v) for v in ops.to_host(terms).ravel()[:2])
        resid_sq = max(0.0, norm_y ** 2 - 2.0 * iprod + norm_m_sq)
        fit = 1.0 - math.sqrt(resid_sq) / norm_y
        fits.append(float(fit))
        sweep_seconds.append(time.perf_counter() - t_sweep)  # the fit readback synchronized
        mt_s = [t.seconds if isinstance(t, EventTimer) else float(t) for t in sweep_mt]
        mttkrp_seconds.append(mt_s)
        other_seconds.append(max(0.0, time.perf_counter() - t_sweep - sum(mt_s)))
        if len(fits) >= 2 and abs(fits[-1] - fits[-2]) < config.tol:
            converged = True
            break

    if hasattr(ops, "sync"):
        ops.sync()
    total = time.perf_counter() - t_start
    if gather:
        factors[s] = comm.allgather_rows(factors[s], part)
    model = KruskalTensor(lam, factors, validate=False)
    trace = ShardedTrace(fits=fits, mttkrp_seconds=mttkrp_seconds, other_seconds=other_seconds, total_seconds=total,
                         iterations=len(fits), converged=converged, sweep_seconds=sweep_seconds,
                         comm_seconds=comm.seconds, comm_bytes=comm.bytes,
                         world=comm.world, shard_mode=s)
    return model, trace
