"""The CP-ALS sweep engine shared by `cp_als` (one GPU) and `cp_als_sharded`.

One implementation of the reference sweep (cpals.py:118-159) for every
world size, so the sharded driver runs exactly the single-GPU machinery:

* fixed buffers: mode k's MTTKRP is written straight into A_k's buffer (A_k
  is not read by its own MTTKRP) and solved in place; Grams, Gamma, lam and
  the fit terms live in preallocated device tensors;
* speculative solves: Gamma_k depends only on the Grams, so its Cholesky runs
  on a side stream while mode k's MTTKRP runs on the main stream; the
  factorization flags stay on the device, and the only host sync per sweep
  is one (2 + d)-scalar readback (fit terms + flags) for the stopping rule
  (cpals.py:157).  A flag restores the sweep's snapshot and reruns it through
  the full eps ladder (cpals.py:78-89), so the trajectory is the ladder's;
* optional CUDA-graph replay of sweeps 2.. (world 1);
* dimension tree (`tree_split`): the modes split into a left group
  {0..p-1} and a right group {p..d-1}; one MTTKRP over a view of the tensor
  with the group merged into one mode gives W_G (I_G x R, the contraction
  with every factor outside the group), and each mode of the group reads its
  MTTKRP out of W_G (cpk_dimtree_contract_f64).  A sweep then runs 2 tensor
  passes instead of d; the factors each mode sees are the reference's
  (cpals.py:118-135: a group's outside factors are unchanged until the group
  is done), so only the summation order differs.

Sharding (world > 1, `Shard`): the tensor is a block of rows [lo, hi) of
mode s, and A_s holds only those rows.  The exchange steps are the ones the
math needs and nothing else, all on device tensors, stream-ordered:

* k != s: allreduce of the partial G_k (I_k x R), then a replicated solve;
* k == s: G_s rows are local; allreduce of the column norms (R) between the
  two halves of the normalization, and of the local Gram A_s^T A_s (R x R);
* once per sweep: allreduce of the stats vector, where every rank's replicated
  terms are masked to rank 0's copy, so the fit is exact and every rank takes
  the same rollback decision.

The compute backend is injectable: `DeviceBackend` (below) runs the sm_100a
C-ABI kernels and is the only production backend; the tests drive the same
engine with a CPU oracle backend under gloo to check the protocol at world
2-3 without a GPU.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
import importlib

mt = importlib.import_module(".mttkrp", __package__)  # the submodule (the package re-exports a function of the same name)
from ._device import require_cuda, stream_ptr
from .errors import DeviceError, ParameterError


@dataclass(frozen=True)
class Shard:
    """This rank's block [lo, hi) of mode `mode` (the partition mode)."""

    mode: int
    lo: int
    hi: int


def init_factors(dims, rank: int, seed: int) -> list:
    """Philox(seed) uniform [0,1) factors in mode order (cpals.py:108-109)."""
    rng = np.random.Generator(np.random.Philox(seed))
    return [rng.random((i_k, rank)) for i_k in dims]


# FP64 issue rate and HBM bandwidth of a B200 (MEASURED_PEAKS.json /
# cpk_fp64_peak_probe), only their ratio matters for the tree decision
_TREE_FLOPS = 37.1e12
_TREE_BW = 6.5e12


def tree_split(dims, rank: int, shard_mode: int = -1, budget_bytes: int | None = None, force: bool = False):
    """Dimension-tree split point p (left group {0..p-1}, right {p..d-1}) for a
    CP-ALS sweep over `dims` at `rank`, or None when no split pays.

    A group of one mode is its plain MTTKRP; a group G of two or more keeps
    W_G (prod I_G x R doubles), written once and read once per mode of G.
    Sharded (`shard_mode` >= 0): every multi-mode group must hold the shard
    mode, so W_G is rank-local (a group without it would need W_G summed
    over ranks).  Among the splits whose largest W_G fits `budget_bytes`,
    the one with the least W_G traffic; it is used when that traffic costs
    less than half of the (d - 2) tensor passes the tree saves (`force`:
    whenever one fits).
    """
    d = len(dims)
    if d < 3:
        return None
    n = math.prod(dims)
    best = None
    for p in range(1, d):
        big = [g for g in (range(p), range(p, d)) if len(g) >= 2]
        if shard_mode >= 0 and any(shard_mode not in g for g in big):
            continue
        wbytes = [math.prod(dims[m] for m in g) * rank * 8 for g in big]
        if budget_bytes is not None and max(wbytes) > budget_bytes:
            continue
        traffic = sum((1 + len(g)) * b for g, b in zip(big, wbytes))
        if best is None or traffic < best[0]:
            best = (traffic, p)
    if best is None:
        return None
    pass_s = max(8.0 * n / _TREE_BW, 2.0 * n * rank / _TREE_FLOPS)
    if not force and best[0] / _TREE_BW >= 0.5 * (d - 2) * pass_s:
        return None
    return best[1]


def tree_groups(d: int, p: int):
    return (tuple(range(p)), tuple(range(p, d)))


# W_G up to this size is taken without asking the driver for free memory
# (cudaMemGetInfo costs milliseconds on a busy device)
TREE_SMALL_BYTES = 1 << 30


def tree_peak_bytes(dims, rank: int, p: int) -> int:
    """The largest W_G of split p (bytes; 0 when both groups are single modes)."""
    return max([math.prod(dims[m] for m in g) * rank * 8 for g in tree_groups(len(dims), p) if len(g) > 1] or [0])


def choose_tree(dims, rank: int, shard_mode: int, want, budget_fn):
    """Split point for `want` (None: when it pays, True: whenever it fits);
    `budget_fn()` (free device bytes for W_G) is only called for large W_G."""
    force = bool(want)
    p = tree_split(dims, rank, shard_mode, None, force=force)
    if p is None or tree_peak_bytes(dims, rank, p) <= TREE_SMALL_BYTES:
        return p
    return tree_split(dims, rank, shard_mode, budget_fn(), force=force)


# -------------------------------------------------------------------- comm
class Comm:
    """torch.distributed plumbing for the sharded sweep.

    With a CUDA `device` the communicator is strict: every collective must get
    a CUDA tensor on that device (an NCCL group has no CPU backend; a CPU
    tensor here is a protocol bug, raised as DeviceError before it reaches
    the backend).  Collectives are stream-ordered; their time is taken with
    CUDA events on the current stream (read lazily), not with host clocks.
    World 1 without an initialized process group is a no-op.
    """

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.device = torch.device(device) if device is not None else None
        self.bytes = 0
        self.calls = 0
        self._events = []
        self._host_seconds = 0.0

    def _check(self, t):
        if not isinstance(t, torch.Tensor):
            raise DeviceError(f"collective on a {type(t).__name__}: the sharded sweep passes torch tensors only")
        if self.device is not None and self.device.type == "cuda" and (not t.is_cuda or t.device != self.device):
            raise DeviceError(f"collective on a {t.device} tensor; this communicator is strict to {self.device}")
        if not t.is_contiguous():
            raise ParameterError("collectives need contiguous tensors")

    def allreduce_(self, t, op=None):
        """Sum (or `op`) in place across ranks."""
        self._check(t)
        if self.world == 1:
            return t
        kw = {} if op is None else {"op": op}
        if t.is_cuda:
            s = torch.cuda.current_stream(t.device)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            self.dist.all_reduce(t, group=self.group, **kw)
            b.record(s)
            self._events.append((a, b))
        else:
            t0 = time.perf_counter()
            self.dist.all_reduce(t, group=self.group, **kw)
            self._host_seconds += time.perf_counter() - t0
        self.bytes += t.numel() * t.element_size()
        self.calls += 1
        return t

    def allgather_rows(self, local, bounds):
        """Concatenate each rank's rows of a row-partitioned factor;
        `bounds[q]` = rank q's (lo, hi)."""
        self._check(local)
        if self.world == 1:
            return local
        r = local.shape[1]
        rows = max(hi - lo for lo, hi in bounds)
        pad = torch.zeros((rows, r), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        return torch.cat([o[: hi - lo] for o, (lo, hi) in zip(outs, bounds)])

    @property
    def seconds(self) -> float:
        """Time spent in collectives (CUDA events; synchronizes on first read)."""
        for a, b in self._events:
            b.synchronize()
            self._host_seconds += a.elapsed_time(b) * 1e-3
        self._events.clear()
        return self._host_seconds

    def reset(self):
        self.seconds  # drain
        self._host_seconds = 0.0
        self.bytes = 0
        self.calls = 0


# ----------------------------------------------------------- device backend
class _Stamp:
    """A CUDA timing event, external so that a replayed graph re-records it."""

    def __init__(self):
        self.ev = torch.cuda.Event(enable_timing=True, external=True)

    def record(self):
        self.ev.record()

    def seconds_to(self, other: "_Stamp") -> float:
        return self.ev.elapsed_time(other.ev) * 1e-3

    def synchronize(self):
        self.ev.synchronize()


class DeviceBackend:
    """The sm_100a C-ABI kernels on one CUDA device (the production backend).

    Holds the tensor, the per-mode plans and a private MTTKRP workspace (no
    process-global scratch is shared with other callers), the solver
    workspace and the side stream the speculative factorization runs on.
    """

    graphable = True

    def __init__(self, y_dev, run_dims, rank, plan: mt.MttkrpPlan, device=None):
        self.dev = require_cuda(device if device is not None else y_dev.device)
        self.lib = _lib.load()
        self.y = y_dev
        self.dims = tuple(run_dims)
        self.rank = rank
        base = plan
        # The Cholesky of Gamma_k runs on a side stream during mode k's
        # MTTKRP and needs a free SM: an automatic plan fills one SM fewer
        # with split-K waves (c3: ~0.2 ms per mode off the critical path)
        if base.splits == 0 and base.sm_count == 0 and base.tile_volume is None:
            base = replace(base, sm_count=max(1, torch.cuda.get_device_properties(self.dev).multi_processor_count - 1))
        d = len(self.dims)
        self._base = base
        self.plans = [mt.plan_for_mode(base, self.dims, k) for k in range(d)]
        nb = 0
        for k in range(d):
            req = mt._plan_request(self.plans[k])
            n = _lib.C.c_size_t(0)
            _lib.check(self.lib.cpk_mttkrp_workspace_bytes(d, _lib.i64_array(self.dims), k, rank, req,
                                                            _lib.C.byref(n)), "workspace")
            nb = max(nb, n.value)
        self.mt_ws = torch.empty(max(1, (nb + 7) // 8), dtype=torch.float64, device=self.dev)
        n = _lib.C.c_size_t(0)
        _lib.check(self.lib.cpk_solve_workspace_bytes(max(self.dims), rank, _lib.C.byref(n)), "solve workspace")
        self.solve_ws = torch.empty(max(1, (n.value + 7) // 8), dtype=torch.float64, device=self.dev)
        self.solve_bytes = n.value
        self.sumsq_ws = torch.empty(_lib.CPK_SUMSQ_PARTIALS, dtype=torch.float64, device=self.dev)
        self.side = torch.cuda.Stream(self.dev)
        self._ev_gamma, self._ev_factor = torch.cuda.Event(), torch.cuda.Event()

    # buffers --------------------------------------------------------------
    def tensor(self, *shape, dtype=torch.float64):
        return torch.zeros(shape, dtype=dtype, device=self.dev)

    def upload(self, a: np.ndarray) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.dev)

    def host_buffer(self, n: int) -> torch.Tensor:
        return torch.zeros(n, dtype=torch.float64, pin_memory=True)

    def stamp(self) -> _Stamp:
        return _Stamp()

    def sp(self):
        return stream_ptr(self.dev)

    # kernels --------------------------------------------------------------
    def sumsq(self, x, out):
        _lib.check(self.lib.cpk_sumsq_f64(x.data_ptr(), x.numel(), self.sumsq_ws.data_ptr(), out.data_ptr(),
                                          self.sp()), "sumsq")

    def gram(self, a, out):
        _lib.check(self.lib.cpk_gram_f64(a.data_ptr(), a.shape[0], a.shape[1], a.stride(0), out.data_ptr(),
                                         self.sp()), "gram")

    def hadamard(self, grams, skip, out):
        ptrs = _lib.ptr_array([g.data_ptr() if m != skip else 0 for m, g in enumerate(grams)])
        _lib.check(self.lib.cpk_hadamard_f64(ptrs, len(grams), int(skip), out.shape[0], out.data_ptr(), self.sp()),
                   "hadamard")

    def mttkrp(self, factors, k, out):
        mt.mttkrp_device(self.y, self.dims, factors, k, None, self.plans[k], out=out, workspace_buf=self.mt_ws)

    # dimension tree ----------------------------------------------------------
    def tree_budget(self) -> int:
        """Bytes the tree's W_G may take: the free device memory less a margin."""
        free = torch.cuda.mem_get_info(self.dev)[0]
        return max(0, free - max(2 << 30, free // 4))

    def setup_tree(self, p: int) -> None:
        """Views, plans and W_G buffers for split p (als_sweep.tree_split)."""
        d = len(self.dims)
        self.tree_p = p
        self.tree_groups = tree_groups(d, p)
        self.tree_views, self.tree_w = [], []
        nb = self.mt_ws.numel() * 8
        for gi, grp in enumerate(self.tree_groups):
            if len(grp) < 2:
                self.tree_views.append(None)
                self.tree_w.append(None)
                continue
            ig = math.prod(self.dims[m] for m in grp)
            vdims, vmode = ((ig,) + self.dims[p:], 0) if gi == 0 else (self.dims[:p] + (ig,), p)
            plan = mt.plan_for_mode(self._base, vdims, vmode)
            n = _lib.C.c_size_t(0)
            _lib.check(self.lib.cpk_mttkrp_workspace_bytes(len(vdims), _lib.i64_array(vdims), vmode, self.rank,
                                                            mt._plan_request(plan), _lib.C.byref(n)),
                       "workspace (tree view)")
            nb = max(nb, n.value)
            self.tree_views.append((vdims, vmode, plan))
            self.tree_w.append(torch.empty((ig, self.rank), dtype=torch.float64, device=self.dev))
        if nb > self.mt_ws.numel() * 8:
            self.mt_ws = torch.empty((nb + 7) // 8, dtype=torch.float64, device=self.dev)

    def tree_mttkrp(self, gi: int, factors) -> None:
        """W_G: the MTTKRP of the view with group gi merged into one mode."""
        vdims, vmode, plan = self.tree_views[gi]
        p = self.tree_p
        vf = [None] + list(factors[p:]) if gi == 0 else list(factors[:p]) + [None]
        mt.mttkrp_device(self.y, vdims, vf, vmode, None, plan, out=self.tree_w[gi], workspace_buf=self.mt_ws)

    def tree_contract(self, gi: int, factors, j: int, out) -> None:
        """Mode j of group gi: its MTTKRP out of W_G (cpk_dimtree_contract_f64)."""
        grp = self.tree_groups[gi]
        mt.dimtree_contract(self.tree_w[gi], [self.dims[m] for m in grp], j, [factors[m] for m in grp], out,
                            self.rank)

    def tree_keep(self) -> list:
        return [w for w in getattr(self, "tree_w", []) if w is not None]

    def factor_spec(self, gamma, info_k):
        """Cholesky of Gamma (rung 0) on the side stream, after the main
        stream's Gamma is ready; the flag stays on the device."""
        main = torch.cuda.current_stream(self.dev)
        self._ev_gamma.record(main)
        self.side.wait_event(self._ev_gamma)
        _lib.check(self.lib.cpk_solve_factor_spec_f64(gamma.data_ptr(), gamma.shape[0], self.solve_ws.data_ptr(),
                                                      self.solve_bytes, info_k.data_ptr(), self.side.cuda_stream),
                   "solve factor (speculative)")
        self._ev_factor.record(self.side)

    def apply_spec(self, g, info_k):
        torch.cuda.current_stream(self.dev).wait_event(self._ev_factor)
        _lib.check(self.lib.cpk_solve_apply_spec_f64(g.data_ptr(), g.shape[0], g.shape[1], self.solve_ws.data_ptr(),
                                                     self.solve_bytes, info_k.data_ptr(), self.sp()),
                   "solve apply (speculative)")

    def solve_ladder(self, gamma, g):
        """X Gamma = G in place through the full eps ladder (host syncs)."""
        rc = self.lib.cpk_solve_normal_f64(gamma.data_ptr(), g.data_ptr(), g.shape[0], g.shape[1],
                                           self.solve_ws.data_ptr(), self.solve_bytes, self.sp())
        if rc == _lib.CPK_ERR_NOT_PD:
            # last rung of cpals.py:89: minimum-norm least squares,
            # lstsq(Gamma, G^T)^T == G pinv(Gamma) for symmetric Gamma
            g.copy_(g @ torch.linalg.pinv(gamma))
            return
        _lib.check(rc, "solve")

    def colnorms_sq(self, a, out):
        _lib.check(self.lib.cpk_colnorms_sq_f64(a.data_ptr(), a.shape[0], a.shape[1], a.stride(0), out.data_ptr(),
                                                self.sp()), "colnorms")

    def scale_columns(self, a, normsq, lam):
        _lib.check(self.lib.cpk_scale_columns_f64(a.data_ptr(), a.shape[0], a.shape[1], a.stride(0),
                                                  normsq.data_ptr(), lam.data_ptr(), self.sp()), "scale columns")

    def fit_terms(self, h, lam, g, a, out):
        _lib.check(self.lib.cpk_fit_terms_f64(h.data_ptr(), lam.data_ptr(), g.data_ptr(), a.data_ptr(), g.shape[0],
                                              h.shape[0], out.data_ptr(), self.sp()), "fit terms")

    def readback(self, src, dst):
        dst.copy_(src, non_blocking=True)

    def synchronize(self):
        torch.cuda.synchronize(self.dev)

    # graph capture ---------------------------------------------------------
    def capture(self, fn, keep):
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(self.dev)  # not `side`: the sweep forks onto that one
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        # capture_begin/end directly: torch.cuda.graph() would also
        # gc.collect() and empty the allocator cache on entry
        with torch.cuda.stream(cap):
            g.capture_begin()
            try:
                fn()
            finally:
                g.capture_end()
        torch.cuda.current_stream(self.dev).wait_stream(cap)
        g.keep = keep
        return g


# ------------------------------------------------------------------ engine
@dataclass
class SweepResult:
    lam: object
    factors: list
    fits: list
    mttkrp_seconds: list
    other_seconds: list
    sweep_seconds: list
    converged: bool
    rollbacks: int
    tree_split: int | None = None


# Capturing a sweep costs ~6 ms once and saves ~0.5 ms of host gaps per
# sweep (c3: 17.5 ms eager vs 17.0 replayed; 10 sweeps break even,
# profiles/r01_bench.jsonl), so the auto mode captures runs that may go
# longer than that.
GRAPH_MIN_ITERS = 12


def run_sweeps(be, dims, rank: int, seed: int, max_iters: int, tol: float, norm_src, comm: Comm | None = None,
               shard: Shard | None = None, graph: bool | None = None, pad_first: bool = False,
               tree: bool | None = None) -> SweepResult:
    """CP-ALS sweeps (cpals.py:92-171) over backend `be`.

    `dims` are the global extents; `be.dims` the extents the kernels run on
    (this rank's block of the shard mode, and I_0 + 1 when `pad_first`: the
    extra A_0 row stays exactly zero).  `norm_src` is the unpadded local
    tensor ||Y||^2 is summed over.  `tree`: None runs the dimension tree when
    `tree_split` finds a split that pays and fits, True whenever a split fits,
    False never (d tensor passes per sweep, the reference's structure).
    """
    world = comm.world if comm is not None else 1
    sharded = world > 1
    if sharded and shard is None:
        raise ParameterError("a communicator of more than one rank needs a Shard")
    if graph is None:
        graph = (max_iters >= GRAPH_MIN_ITERS) and not sharded and be.graphable
    if graph and (sharded or not be.graphable):
        raise ParameterError("graph replay is for single-rank device sweeps")
    d, r = len(dims), rank
    run_dims = be.dims
    s = shard.mode if sharded else -1

    # ||Y||^2: local sum of squares, one allreduce, the run's one early sync;
    # a NaN/Inf anywhere makes it non-finite
    sq = be.tensor(1)
    be.sumsq(norm_src, sq)
    if sharded:
        comm.allreduce_(sq)
    norm_y = math.sqrt(float(sq.cpu()[0]))
    if not math.isfinite(norm_y):
        raise ParameterError("tensor has non-finite entries")
    if norm_y == 0.0:
        raise ParameterError("cannot fit an all-zero tensor (fit is undefined)")

    tree_p = None
    if tree is not False and hasattr(be, "setup_tree"):
        tree_p = choose_tree(run_dims, r, s, tree, be.tree_budget)
        if tree_p is not None:
            be.setup_tree(tree_p)
    elif tree:
        raise ParameterError("this backend has no dimension-tree sweep")
    groups = tree_groups(d, tree_p) if tree_p is not None else None

    init = init_factors(dims, r, seed)  # replicated Philox stream (cpals.py:108-109)
    if sharded:
        init[s] = init[s][shard.lo:shard.hi]
    if pad_first:
        init[0] = np.concatenate([init[0], np.zeros((1, r))])
    factors = [be.upload(a) for a in init]
    grams = [be.tensor(r, r) for _ in range(d)]
    for m in range(d):
        be.gram(factors[m], grams[m])
    if sharded:
        comm.allreduce_(grams[s])
    lam = be.tensor(r)
    lam.fill_(1.0)
    gamma, h = be.tensor(r, r), be.tensor(r, r)
    normsq = be.tensor(r)
    g_last = be.tensor(run_dims[d - 1], r)
    stats = be.tensor(2 + d)  # fit terms, Cholesky flags
    info = be.tensor(d, dtype=torch.int32)
    stats_host = be.host_buffer(2 + d)
    mask = None
    if sharded:
        # replicated terms count once (rank 0); <Y, M> is a sum over the
        # shard mode's rows when the last mode is the shard mode
        m = np.ones(2 + d)
        if comm.rank != 0:
            m[0] = 0.0
            if s != d - 1:
                m[1] = 0.0
        mask = be.upload(m)
    st_mt = [(be.stamp(), be.stamp()) for _ in range(d)]
    st_sweep = (be.stamp(), be.stamp())

    def sweep(spec: bool) -> None:
        st_sweep[0].record()
        for k in range(d):
            be.hadamard(grams, k, gamma)
            if spec:
                be.factor_spec(gamma, info[k:k + 1])
            st_mt[k][0].record()
            grp = None if groups is None else groups[0 if k < tree_p else 1]
            if grp is None or len(grp) == 1:
                be.mttkrp(factors, k, factors[k])
            else:
                gi = 0 if k < tree_p else 1
                if k == grp[0]:  # W_G, from the factors outside the group
                    be.tree_mttkrp(gi, factors)
                be.tree_contract(gi, factors, k - grp[0], factors[k])
            st_mt[k][1].record()
            if sharded and k != s:
                comm.allreduce_(factors[k])  # partial G_k -> G_k on every rank
            if k == d - 1:  # the fit needs the last mode's G itself
                g_last.copy_(factors[k])
            if spec:
                be.apply_spec(factors[k], info[k:k + 1])
            else:
                be.solve_ladder(gamma, factors[k])
            be.colnorms_sq(factors[k], normsq)
            if sharded and k == s:
                comm.allreduce_(normsq)  # column norms of the row-partitioned A_s
            be.scale_columns(factors[k], normsq, lam)
            be.gram(factors[k], grams[k])
            if sharded and k == s:
                comm.allreduce_(grams[k])
        be.hadamard(grams, -1, h)
        # g_last is the unit-weight mode-(d-1) MTTKRP and A_{d-1} was solved from it
        be.fit_terms(h, lam, g_last, factors[d - 1], stats[0:2])
        stats[2:].copy_(info)
        if sharded:
            stats.mul_(mask)
            comm.allreduce_(stats)
        be.readback(stats, stats_host)
        st_sweep[1].record()  # after the readback: waiting on it makes stats_host valid

    saved = [torch.empty_like(t) for t in factors + grams + [lam]]

    def snapshot():  # one multi-tensor copy launch, not 2d + 1
        torch._foreach_copy_(saved, factors + grams + [lam])

    def restore():
        torch._foreach_copy_(factors + grams + [lam], saved)

    def spec_sweep():
        snapshot()
        info.zero_()
        sweep(spec=True)

    captured = None
    fits, mttkrp_seconds, other_seconds, sweep_seconds = [], [], [], []
    converged = False
    rollbacks = 0
    for it in range(max_iters):
        if it == 0 or not graph:
            spec_sweep()  # eager: one host sync per sweep
        else:
            if captured is None:
                captured = be.capture(spec_sweep, keep=[be.mt_ws, be.solve_ws, be.sumsq_ws] + be.tree_keep())
            captured.replay()
        st_sweep[1].synchronize()
        if bool((stats_host[2:] != 0).any()):
            # a speculative Cholesky failed: roll the sweep back and rerun it
            # through the ladder (cpals.py:78-88)
            rollbacks += 1
            restore()
            info.zero_()
            sweep(spec=False)
            st_sweep[1].synchronize()
        norm_m_sq, iprod = float(stats_host[0]), float(stats_host[1])
        resid_sq = max(0.0, norm_y ** 2 - 2.0 * iprod + norm_m_sq)
        fits.append(float(1.0 - math.sqrt(resid_sq) / norm_y))
        mts = [a.seconds_to(b) for a, b in st_mt]
        total = st_sweep[0].seconds_to(st_sweep[1])
        mttkrp_seconds.append(mts)
        other_seconds.append(max(0.0, total - sum(mts)))
        sweep_seconds.append(total)
        if len(fits) >= 2 and abs(fits[-1] - fits[-2]) < tol:
            converged = True
            break
    be.synchronize()
    return SweepResult(lam=lam, factors=factors, fits=fits, mttkrp_seconds=mttkrp_seconds,
                       other_seconds=other_seconds, sweep_seconds=sweep_seconds, converged=converged,
                       rollbacks=rollbacks, tree_split=tree_p)
