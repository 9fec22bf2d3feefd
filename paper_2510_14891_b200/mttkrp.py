"""MTTKRP for dense tensors on B200: G = Y_(k) (KRP of the other factors) diag(lam).

Drop-in for the cpkern.mttkrp dispatcher (pkg/src/cpkern/mttkrp.py): the same
Variant / MttkrpPlan / MttkrpStats / MttkrpOutput types, `run(y, m, plan)`
(mttkrp.py:378-391), the per-variant entry points, `plan_for_mode`
(mttkrp.py:394-401) and the Eq. 6 tile heuristic (mttkrp.py:404-428), plus
the north-star convenience `mttkrp(tensor, factors, mode)`.

Every variant executes the hand-written sm_100a kernel behind
cpk_mttkrp_f64 (csrc/mttkrp.cu); nothing is computed on the host.  What the
variants keep from the reference is their *partitioning* and *accounting*:

* TILE   -- tile_volume (N_T) sets the in-slice elements per CTA work item,
            i.e. the split-K granularity (the reference's tiles per slice);
* SLICE  -- one work item per output row block (no split of a slice);
* ELEM / REFERENCE / GEMM / FULL_KRP / B200 -- the auto plan (splits chosen
            to fill whole waves of the 148 SMs).

Stats (element_visits, atomic_updates, ...) follow the reference formulas so
reports stay comparable; `seconds` is the CUDA-event time of the kernel plus
the split-K merge on the launching stream (the reference times kernel +
private-copy merge, mttkrp.py:279-286), read lazily so timing adds no sync.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from enum import Enum

import numpy as np
import torch

from . import _lib
from ._device import EventTimer, require_cuda, stream_ptr, workspace
from .dtensor import DenseTensor, check_dims, num_elements
from .errors import DeviceError, IndexRangeError, ParameterError, ResourceError, ShapeError
from .kruskal import KruskalTensor


_ENGINES = {"auto": 0, "cpasync": 1, "tma": 2, "dmma": 3, "cpdmma": 4}


class Variant(str, Enum):
    REFERENCE = "reference"
    FULL_KRP = "full-krp"
    GEMM = "gemm"
    ELEM = "elem"
    SLICE = "slice"
    TILE = "tile"
    B200 = "b200"


@dataclass(frozen=True)
class MttkrpPlan:
    """How to run one MTTKRP (mttkrp.py:53-89), with the GPU knobs added.

    ``unroll`` (F), ``team_width`` (b_x) and ``vector_width`` (b_y) keep the
    paper's meaning; on the GPU the column block is the rank tile, so they
    are validated (>= 1) but the kernel's register tile is fixed at 8x8.
    ``rank_tile`` (0 = auto, else 16/32/64/128/256), ``splits`` (0 = auto) and
    ``block_k`` (chunk depth, 0 = auto, else 16/32) are the B200
    realization of the rank tiling and of N_T; ``engine`` picks the data
    movement ("auto", "tma" = warp-specialized TMA kernel, "cpasync").
    ``sm_count`` (0 = the device's) is how many SMs the automatic split
    count fills in whole waves -- cp_als leaves one free for the Cholesky it
    runs beside the MTTKRP.  ``workers`` is accepted for compatibility and
    ignored (one GPU per process).
    """

    variant: Variant
    mode: int
    unroll: int = 4
    team_width: int = 1
    vector_width: int = 1
    tile_volume: int | None = None
    workers: int = 0
    rank_tile: int = 0
    splits: int = 0
    block_k: int = 0
    engine: str = "auto"
    sm_count: int = 0

    def validate(self, dims, rank) -> None:
        d = len(dims)
        if not 0 <= self.mode < d:
            raise IndexRangeError(f"mode {self.mode} out of range [0, {d - 1}]")
        if self.unroll < 1:
            raise ParameterError(f"unroll must be >= 1, got {self.unroll}")
        if self.team_width < 1 or self.vector_width < 1:
            raise ParameterError("team_width and vector_width must be >= 1")
        if rank < 1:
            raise ParameterError(f"rank must be >= 1, got {rank}")
        if self.rank_tile not in (0, 16, 32, 64, 128, 256):
            raise ParameterError(f"rank_tile must be 0, 16, 32, 64, 128 or 256, got {self.rank_tile}")
        if self.splits < 0:
            raise ParameterError(f"splits must be >= 0, got {self.splits}")
        if self.engine not in _ENGINES:
            raise ParameterError(f"engine must be one of {sorted(_ENGINES)}, got {self.engine!r}")
        if self.block_k not in (0, 16, 32):
            raise ParameterError(f"block_k must be 0, 16 or 32, got {self.block_k}")
        if self.sm_count < 0:
            raise ParameterError(f"sm_count must be >= 0, got {self.sm_count}")
        if self.variant == Variant.TILE:
            n_s = num_elements(dims) // dims[self.mode]
            if self.tile_volume is None:
                raise ParameterError("tile variant needs an explicit tile_volume")
            if not 1 <= int(self.tile_volume) <= n_s:
                raise ParameterError(f"tile_volume {self.tile_volume} out of range [1, {n_s}]")


@dataclass
class MttkrpStats:
    """Work accounting and timing for one MTTKRP (mttkrp.py:92-111)."""

    variant: Variant
    mode: int
    element_visits: int
    atomic_updates: int
    _seconds: object = field(repr=False, default=0.0)
    workers: int = 1
    tile_volume: int | None = None
    unroll: int | None = None
    scratch_bytes: int | None = None
    footprint_bytes: int | None = None
    rank_tile: int | None = None
    splits: int | None = None
    device: str = "cuda"

    @property
    def seconds(self) -> float:
        s = self._seconds
        return s.seconds if isinstance(s, EventTimer) else float(s)


@dataclass
class MttkrpOutput:
    matrix: object  # numpy.ndarray for host inputs, torch CUDA tensor for device inputs
    stats: MttkrpStats


def _check_inputs(y: DenseTensor, m: KruskalTensor, mode: int) -> None:
    if y.dims != m.dims:
        raise ShapeError(f"tensor dims {y.dims} do not match model dims {m.dims}")
    if not 0 <= int(mode) < y.ndim:
        raise IndexRangeError(f"mode {mode} out of range [0, {y.ndim - 1}]")


def _plan_request(plan: MttkrpPlan) -> _lib.CpkPlan:
    """The CpkPlan the C side resolves itself: zero fields mean "choose"
    (a fully automatic request may also merge a small mode with a neighbour)."""
    p = _lib.CpkPlan(plan.rank_tile, 0, 0, plan.splits, plan.sm_count, plan.block_k, _ENGINES[plan.engine])
    v = Variant(plan.variant)
    if plan.splits == 0:
        if v == Variant.TILE:
            p.tile_volume = int(plan.tile_volume)
        elif v == Variant.SLICE:
            p.splits = 1
    return p


def _gpu_plan(plan: MttkrpPlan, dims, rank: int) -> _lib.CpkPlan:
    """The resolved plan (for stats and validation; cpk_plan_resolve)."""
    p = _plan_request(plan)
    dims_c = _lib.i64_array(dims)
    _lib.check(_lib.load().cpk_plan_resolve(len(dims), dims_c, int(plan.mode), int(rank), p), "plan")
    return p


def resolve_plan(plan: MttkrpPlan, dims, rank: int) -> dict:
    """The concrete GPU plan (rank tile, row block, N_T, splits) for a problem."""
    require_cuda()
    p = _gpu_plan(plan, check_dims(dims), rank)
    return {"rank_tile": p.rank_tile, "block_rows": p.block_rows, "tile_volume": p.tile_volume,
            "splits": p.splits, "sm_count": p.sm_count, "block_k": p.block_k,
            "engine": {v: k for k, v in _ENGINES.items()}[p.engine]}


def mttkrp_device(y_dev: torch.Tensor, dims, factors, mode: int, weights=None, plan: MttkrpPlan | None = None,
                  out: torch.Tensor | None = None, landed=None, workspace_buf: torch.Tensor | None = None):
    """Low-level device entry: y_dev flat CUDA float64, factors CUDA (I_m, R).

    ``landed = (lo, hi)`` runs only the work whose slices along the slowest
    mode lie in [0, hi) and not all in [0, lo) (cpk_mttkrp_f64_landed): the
    streaming building block; the call with hi = dims[-1] completes G.
    Returns (G, resolved CpkPlan, EventTimer).  G is (I_k, R) row-major CUDA.
    """
    dims = check_dims(dims)
    d = len(dims)
    mode = int(mode)
    dev = y_dev.device
    if not y_dev.is_cuda:
        raise DeviceError("mttkrp_device needs a CUDA tensor (there is no CPU path)")
    if y_dev.dim() != 1 or not y_dev.is_contiguous() or y_dev.numel() != num_elements(dims):
        raise ShapeError(f"y must be a flat contiguous tensor of {num_elements(dims)} elements")
    if len(factors) != d:
        raise ShapeError(f"{len(factors)} factors for a {d}-way tensor")
    rank = next(int(f.shape[1]) for f in factors if f is not None)
    if plan is None:
        plan = MttkrpPlan(Variant.B200, mode)
    # the kernels read row-major factors with unit column stride, in y's dtype
    want = y_dev.dtype if y_dev.dtype == torch.float32 else torch.float64
    # (mode k's own factor is not read: passed through untouched)
    factors = [f if (m == mode or (f.dtype == want and f.device == dev and f.stride(1) == 1)) else
               f.to(device=dev, dtype=want).contiguous()
               for m, f in enumerate(factors)]
    for m, f in enumerate(factors):
        if m != mode and (f.dim() != 2 or f.shape[0] != dims[m] or f.shape[1] != rank):
            raise ShapeError(f"factor {m} has shape {tuple(f.shape)}, expected ({dims[m]}, {rank})")
    if weights is not None and (weights.dtype != want or weights.device != dev or not weights.is_contiguous()):
        weights = weights.to(device=dev, dtype=want).contiguous()
    if y_dev.dtype == torch.float32:
        if landed is not None:
            raise ParameterError("the float32 path has no streamed (landed) form")
        return _mttkrp_device_f32(y_dev, dims, factors, mode, weights, plan, out)
    p = _gpu_plan(plan, dims, rank)
    req = _plan_request(plan)  # the C side resolves (and may merge) from the request
    dims_c = _lib.i64_array(dims)
    nbytes = _lib.C.c_size_t(0)
    lib = _lib.load()
    _lib.check(lib.cpk_mttkrp_workspace_bytes(d, dims_c, mode, rank, req, _lib.C.byref(nbytes)), "workspace")
    if workspace_buf is not None:
        if workspace_buf.numel() * workspace_buf.element_size() < nbytes.value:
            raise ParameterError("workspace_buf is smaller than the plan's split-K workspace")
        ws = workspace_buf if nbytes.value else None
    else:
        ws = workspace(dev, nbytes.value)
    if out is None:
        out = torch.empty((dims[mode], rank), dtype=torch.float64, device=dev)
    ptrs = _lib.ptr_array([f.data_ptr() if (m != mode and f is not None) else 0 for m, f in enumerate(factors)])
    lds = _lib.i64_array([f.stride(0) if f is not None else rank for f in factors])
    lam_ptr = weights.data_ptr() if weights is not None else None
    timer = EventTimer(dev)
    args = (y_dev.data_ptr(), d, dims_c, mode, ptrs, lds, lam_ptr, rank, out.data_ptr(), out.stride(0),
            req, ws.data_ptr() if ws is not None else None, nbytes.value, stream_ptr(dev))
    if landed is None:
        rc = lib.cpk_mttkrp_f64(*args)
    else:
        rc = lib.cpk_mttkrp_f64_landed(*args, int(landed[0]), int(landed[1]))
    timer.stop(dev)
    _lib.check(rc, "mttkrp")
    return out, p, timer


def f32_eligible(dims, factors=None) -> bool:
    """Shapes the tcgen05 float32 kernel takes (TMA needs 16-byte strides:
    I_0 % 4 == 0; factors are re-laid out with ld % 4 == 0 when needed)."""
    return 2 <= len(dims) <= 5 and dims[0] % 4 == 0 and max(dims) < 2 ** 31


def _ld4(f: torch.Tensor) -> torch.Tensor:
    """f with a 16-byte aligned base and a leading dimension that is a
    multiple of 4 floats (a padded copy only when f is not already so)."""
    if f.stride(1) == 1 and f.stride(0) % 4 == 0 and f.data_ptr() % 16 == 0:
        return f
    r = f.shape[1]
    buf = torch.zeros((f.shape[0], (r + 3) // 4 * 4), dtype=torch.float32, device=f.device)
    buf[:, :r] = f
    return buf[:, :r]


def _mttkrp_device_f32(y_dev, dims, factors, mode, weights, plan, out):
    """Optional float32 path (north star: <= 1e-4): cpk_mttkrp_f32, the
    tcgen05 kind::tf32 kernel with a 3xTF32 split.  Shapes TMA cannot
    describe run the FP64 kernel on float64 copies (still on the device)."""
    d = len(dims)
    dev = y_dev.device
    fac = [None if m == mode else _ld4(f.to(device=dev, dtype=torch.float32)) for m, f in enumerate(factors)]
    rank = next(int(f.shape[1]) for f in fac if f is not None)
    lam = None if weights is None else weights.to(device=dev, dtype=torch.float32).contiguous()
    if out is None:
        out = torch.empty((dims[mode], rank), dtype=torch.float32, device=dev)
    if not f32_eligible(dims, fac) or y_dev.data_ptr() % 16:
        g64, p, timer = mttkrp_device(y_dev.double(), dims, [None if f is None else f.double() for f in fac], mode,
                                      None if lam is None else lam.double(), replace(plan, engine="auto"))
        out.copy_(g64)
        return out, p, timer
    splits = int(plan.splits or 0)
    dims_c = _lib.i64_array(dims)
    nbytes = _lib.C.c_size_t(0)
    lib = _lib.load()
    _lib.check(lib.cpk_mttkrp_f32_workspace_bytes(d, dims_c, mode, rank, splits, _lib.C.byref(nbytes)), "workspace")
    ws = workspace(dev, nbytes.value, tag="mttkrp_f32")
    ptrs = _lib.ptr_array([0 if f is None else f.data_ptr() for f in fac])
    lds = _lib.i64_array([rank if f is None else f.stride(0) for f in fac])
    timer = EventTimer(dev)
    rc = lib.cpk_mttkrp_f32(y_dev.data_ptr(), d, dims_c, mode, ptrs, lds, None if lam is None else lam.data_ptr(),
                            rank, out.data_ptr(), out.stride(0), splits, ws.data_ptr() if ws is not None else None,
                            nbytes.value, stream_ptr(dev))
    timer.stop(dev)
    _lib.check(rc, "mttkrp f32")
    p = _lib.CpkPlan(128, 128, 0, splits, 0, 32, -1, -1)  # engine -1: the fp32 tcgen05 kernel
    return out, p, timer


def _unit_weights(w) -> bool:
    """True for all-ones weights (then none are passed to the kernel).  A
    CUDA tensor is never inspected (that would sync the stream): it is
    folded, which is exact for ones as well."""
    if isinstance(w, torch.Tensor):
        return (not w.is_cuda) and bool((w == 1).all().item())
    return bool(np.all(np.asarray(w) == 1.0))


# A host-resident tensor at least this large is streamed to the device in
# slabs, each slab's MTTKRP overlapping the copy of the next.
STREAM_MIN_BYTES = 256 << 20
STREAM_SLABS = 16  # 8 -> 16: e2e 394 -> 387 ms at c4 (first slab lands sooner); 32 is slower
STREAM_GEOMETRIC = 8  # slabs 1/128, 1/128, 1/64, ... 1/2 of the extent (0: equal slabs)


def _run_gpu(y: DenseTensor, m: KruskalTensor, plan: MttkrpPlan):
    dev = require_cuda()
    fac = m.device_factors(dev)
    lam = None if _unit_weights(m.weights) else m.device_weights(dev)
    if y.needs_upload(dev) and y.size * 8 >= STREAM_MIN_BYTES and y.ndim >= 2 and y.dims[-1] >= 2:
        g, p, timer = _mttkrp_streamed(y, fac, plan, lam, dev)
    elif y.landing is not None:
        # the upload may still be in flight: run on the slabs as they land
        # (a side stream, so this call overlaps the earlier ones)
        g, p, timer = _landed_pieces(y.device_data(dev, wait=False), y.dims, fac, plan, lam, dev, *y.landing)
    elif _pad_first_mode(y, plan, dev):
        g, p, timer = _mttkrp_even(y, fac, plan, lam, dev)
    else:
        g, p, timer = mttkrp_device(y.device_data(dev), y.dims, fac, plan.mode, lam, plan)
    # numpy in, numpy out; a torch payload (CUDA, or pinned host memory being
    # streamed) keeps G on the device
    host = not isinstance(y.data, torch.Tensor)
    matrix = np.ascontiguousarray(g.cpu().numpy()) if host else g
    return matrix, p, timer


# An odd I_0 rules out TMA (16-byte strides); tensors up to this size are
# run through a zero-padded copy with an even I_0 instead (DenseTensor.
# even_device_data): the TMA + DMMA kernel on the copy beats the cp.async
# kernel on the original by ~40 % (c4-sized, profiles/r01_sweep_odd_cpdmma.agg.csv).
EVEN_PAD_MAX_BYTES = 16 << 30


def _pad_first_mode(y: DenseTensor, plan: MttkrpPlan, dev) -> bool:
    if y.ndim < 2 or y.dims[0] % 2 == 0 or Variant(plan.variant) not in (Variant.B200, Variant.GEMM,
                                                                          Variant.FULL_KRP, Variant.ELEM):
        return False
    if plan.engine not in ("auto", "dmma") or plan.rank_tile or plan.splits or plan.block_k:
        return False
    nbytes = 8 * (y.size // y.dims[0]) * (y.dims[0] + 1)
    return nbytes <= min(EVEN_PAD_MAX_BYTES, torch.cuda.mem_get_info(dev)[0] // 4)


def _mttkrp_even(y: DenseTensor, fac, plan: MttkrpPlan, lam, dev):
    """MTTKRP through the zero-padded even copy (see _pad_first_mode)."""
    dims = (y.dims[0] + 1,) + y.dims[1:]
    fac = list(fac)
    if plan.mode != 0:
        a0 = fac[0]
        fac[0] = torch.cat([a0, torch.zeros((1, a0.shape[1]), dtype=a0.dtype, device=a0.device)])
    g, p, timer = mttkrp_device(y.even_device_data(dev), dims, fac, plan.mode, lam, plan)
    return (g[: y.dims[0]] if plan.mode == 0 else g), p, timer


_side = {}
_copy = {}


def _modes_stream(dev, i: int = 0) -> torch.cuda.Stream:
    """Dedicated stream i of mttkrp_modes (one per mode; cached, so each
    stream's allocator pool is reused call after call)."""
    if ("modes", dev.index, i) not in _copy:
        _copy[("modes", dev.index, i)] = torch.cuda.Stream(dev)
    return _copy[("modes", dev.index, i)]


def _copy_stream(dev) -> torch.cuda.Stream:
    if dev.index not in _copy:
        _copy[dev.index] = torch.cuda.Stream(dev)
    return _copy[dev.index]


def _side_stream(dev) -> torch.cuda.Stream:
    """Round-robin pool of side streams for calls that run on landing slabs."""
    pool, nxt = _side.setdefault(dev.index, ([torch.cuda.Stream(dev) for _ in range(3)], [0]))
    s = pool[nxt[0] % len(pool)]
    nxt[0] += 1
    return s


def _landed_pieces(y_dev, dims, fac, plan, lam, dev, bounds, events):
    """One MTTKRP as per-slab pieces (cpk_mttkrp_f64_landed), each after its
    slab's copy event, on a side stream with a private workspace: calls on
    the same in-flight tensor (the modes of one step) overlap each other and
    the copy.  Same plan, work items and merge order as one resident call,
    so G is bit-identical to it."""
    main = torch.cuda.current_stream(dev)
    side = _side_stream(dev)
    side.wait_stream(main)  # inputs (factors, weights) are ordered on `main`
    mode = plan.mode
    rank = next(int(f.shape[1]) for f in fac if f is not None)
    nbytes = _lib.C.c_size_t(0)
    _lib.check(_lib.load().cpk_mttkrp_workspace_bytes(len(dims), _lib.i64_array(dims), mode, rank,
                                                       _plan_request(plan), _lib.C.byref(nbytes)), "workspace")
    with torch.cuda.stream(side):
        out = torch.empty((dims[mode], rank), dtype=torch.float64, device=dev)
        ws = torch.empty(max(1, (nbytes.value + 7) // 8), dtype=torch.float64, device=dev)
        timer = EventTimer(dev)
        p = None
        for (lo, hi), ev in zip(bounds, events):
            side.wait_event(ev)
            _, p, _ = mttkrp_device(y_dev, dims, fac, mode, lam, plan, out=out, landed=(lo, hi), workspace_buf=ws)
        timer.stop(dev)
    main.wait_stream(side)
    out.record_stream(main)
    return out, p, timer


def _slab_bounds(extent: int) -> list:
    """Slabs of the slowest mode for a streamed upload.  STREAM_GEOMETRIC:
    sizes grow geometrically from 1/2^(n-1) of the extent (first slab lands
    after ~1 % of the copy, so compute starts almost at once; the copy then
    stays ahead of the compute, which consumes the tensor ~2x slower than
    PCIe delivers it); else STREAM_SLABS equal slabs."""
    if STREAM_GEOMETRIC and extent >= 2 ** (STREAM_GEOMETRIC - 1):
        n = STREAM_GEOMETRIC
        cuts = [0] + [extent >> (n - 1 - i) for i in range(n)]
        cuts[-1] = extent
        return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    n = min(STREAM_SLABS, extent)
    return [(extent * i // n, extent * (i + 1) // n) for i in range(n)]


def _start_upload(y: DenseTensor, dev):
    """Begin the slab-wise H2D copy of a host tensor on a copy stream; the
    device copy is cached on `y` with the slab events (DenseTensor.landing)."""
    dims = y.dims
    per_slice = num_elements(dims[:-1])
    host = y.host_view()
    compute = torch.cuda.current_stream(dev)
    copy = _copy_stream(dev)
    with torch.cuda.stream(copy):
        # allocated on the copy stream: the copy need not wait for the
        # compute stream's queue (only its own stream's earlier users)
        y_dev = torch.empty(y.size, dtype=torch.float64, device=dev)
    y_dev.record_stream(compute)
    bounds = _slab_bounds(dims[-1])
    landed = []
    with torch.cuda.stream(copy):
        for lo, hi in bounds:
            y_dev[lo * per_slice:hi * per_slice].copy_(host[lo * per_slice:hi * per_slice], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
            landed.append(ev)
    y_dev.record_stream(copy)
    y.cache_device(y_dev, landing=(bounds, landed))
    return y_dev, bounds, landed


def mttkrp_modes(tensor, factors, modes=None, weights=None, plan: MttkrpPlan | None = None,
                 tree: bool = False) -> list:
    """The MTTKRPs of several modes against the same factors (e.g. every mode
    of a step), returned as a list of (I_k, R) matrices of the input's kind.

    For a large host tensor this is where streaming pays most: the copy runs
    in slabs along the slowest mode and, for every landed slab, the work
    items of *all* requested modes are issued (cpk_mttkrp_f64_landed), so
    the copy hides under the compute of every mode, not just the first.
    Each mode has its own stream: a piece's last partial wave of CTAs is
    filled by the other modes' pieces instead of idling SMs (c4: ~24 piece
    launches, ~0.5 ms of tail each on one stream).  Each mode keeps its own
    plan, workspace and merge order: results are bit-identical to one
    resident call per mode.

    ``tree=True`` computes the modes through a dimension tree instead
    (_modes_tree): two tensor passes for all d modes, equal to the per-mode
    results up to summation order (the tensor is uploaded whole first; no
    streaming overlap).
    """
    if isinstance(factors, KruskalTensor):
        m = factors
    else:
        fs = list(factors)
        m = KruskalTensor(weights if weights is not None else np.ones(int(fs[0].shape[1])), fs, validate=False)
    if not isinstance(tensor, DenseTensor):
        tensor = DenseTensor(m.dims, tensor)
    y = tensor
    modes = list(range(y.ndim)) if modes is None else [int(k) for k in modes]
    for k in modes:
        _check_inputs(y, m, k)
    dev = require_cuda()
    if tree and y.ndim >= 3 and len(set(modes)) > 2:
        outs = _modes_tree(y.device_data(dev), y.dims, m.device_factors(dev),
                           None if _unit_weights(m.weights) else m.device_weights(dev), modes, plan, dev)
        host = not isinstance(y.data, torch.Tensor)
        return [np.ascontiguousarray(g.cpu().numpy()) for g in outs] if host else outs
    stream_it = y.needs_upload(dev) and y.size * 8 >= STREAM_MIN_BYTES and y.ndim >= 2 and y.dims[-1] >= 2
    if not stream_it and y.landing is None:
        return [mttkrp(y, m, k, plan=plan) for k in modes]
    fac = m.device_factors(dev)
    lam = None if _unit_weights(m.weights) else m.device_weights(dev)
    if stream_it:
        y_dev, bounds, events = _start_upload(y, dev)
    else:
        y_dev, (bounds, events) = y.device_data(dev, wait=False), y.landing
    dims, rank = y.dims, m.rank
    plans = [replace(plan, mode=k) if plan is not None else MttkrpPlan(Variant.B200, k) for k in modes]
    # The pieces run on a side stream, never on the legacy default stream:
    # waits on the copy events issued there resolved only after the whole
    # copy once the default stream had done any H2D (measured,
    # tools/dbg_copy2.py), which serialized copy and compute.
    main = torch.cuda.current_stream(dev)
    sides = [_modes_stream(dev, i) for i in range(len(plans))]
    outs, wss = [], []
    for pk, st in zip(plans, sides):
        st.wait_stream(main)  # inputs are ordered on `main`
        with torch.cuda.stream(st):
            nbytes = _lib.C.c_size_t(0)
            _lib.check(_lib.load().cpk_mttkrp_workspace_bytes(len(dims), _lib.i64_array(dims), pk.mode, rank,
                                                               _plan_request(pk), _lib.C.byref(nbytes)), "workspace")
            outs.append(torch.empty((dims[pk.mode], rank), dtype=torch.float64, device=dev))
            wss.append(torch.empty(max(1, (nbytes.value + 7) // 8), dtype=torch.float64, device=dev))
    for (lo, hi), ev in zip(bounds, events):  # slab-major, so every stream has work early
        for pk, out, ws, st in zip(plans, outs, wss, sides):
            st.wait_event(ev)
            with torch.cuda.stream(st):
                mttkrp_device(y_dev, dims, fac, pk.mode, lam, pk, out=out, landed=(lo, hi), workspace_buf=ws)
    for out, st in zip(outs, sides):
        main.wait_stream(st)
        out.record_stream(main)
    host = not isinstance(y.data, torch.Tensor)
    return [np.ascontiguousarray(g.cpu().numpy()) for g in outs] if host else outs


def dimtree_contract(w: torch.Tensor, exts, j: int, group_factors, out: torch.Tensor, rank: int) -> None:
    """out = mode j of a group's MTTKRP read out of W_G (cpk_dimtree_contract_f64):
    W_G (prod(exts) x R rows, group multi-index first-mode-fastest) is the
    MTTKRP over the modes outside the group; group_factors[l] (l != j) are
    the group's factors (row-major, unit column stride)."""
    ptrs = _lib.ptr_array([f.data_ptr() if l != j else 0 for l, f in enumerate(group_factors)])
    lds = _lib.i64_array([f.stride(0) for f in group_factors])
    _lib.check(_lib.load().cpk_dimtree_contract_f64(w.data_ptr(), w.stride(0), len(exts), _lib.i64_array(exts), j,
                                                    ptrs, lds, rank, out.data_ptr(), out.stride(0),
                                                    stream_ptr(out.device)), "dimtree contract")


def _modes_tree(y_dev, dims, fac, lam, modes, plan, dev) -> list:
    """Several modes' MTTKRPs by a dimension tree (als_sweep.tree_split): per
    group of two or more modes one MTTKRP over the view with the group merged
    (W_G, weights folded in), then each mode of the group out of W_G; a
    one-mode group is its plain MTTKRP.  Two tensor passes for all modes."""
    from .als_sweep import choose_tree, tree_groups

    d, rank = len(dims), int(fac[0].shape[1])
    p = choose_tree(dims, rank, -1, True, lambda: max(0, torch.cuda.mem_get_info(dev)[0] - (2 << 30)))
    if p is None:
        raise ResourceError("no dimension-tree split fits in device memory")
    want = set(modes)
    res = {}
    for gi, grp in enumerate(tree_groups(d, p)):
        ks = [k for k in grp if k in want]
        if len(grp) == 1 or len(ks) == 1:  # a one-mode group (or one wanted mode): its plain MTTKRP
            for k in ks:
                pk = replace(plan, mode=k) if plan is not None else MttkrpPlan(Variant.B200, k)
                res[k] = mttkrp_device(y_dev, dims, fac, k, lam, pk)[0]
            continue
        if not ks:
            continue
        ig = int(np.prod([dims[m] for m in grp]))
        vdims, vmode = ((ig,) + tuple(dims[p:]), 0) if gi == 0 else (tuple(dims[:p]) + (ig,), p)
        vf = [None] + list(fac[p:]) if gi == 0 else list(fac[:p]) + [None]
        pv = replace(plan, mode=vmode) if plan is not None else MttkrpPlan(Variant.B200, vmode)
        w = mttkrp_device(y_dev, vdims, vf, vmode, lam, pv)[0]
        for k in ks:
            out = torch.empty((dims[k], rank), dtype=torch.float64, device=dev)
            dimtree_contract(w, [dims[m] for m in grp], k - grp[0], [fac[m] for m in grp], out, rank)
            res[k] = out
        del w
    return [res[k] for k in modes]


def _mttkrp_streamed(y: DenseTensor, fac, plan: MttkrpPlan, lam, dev):
    """First touch of a large host tensor: copy it to the device in slabs
    along its slowest mode on a copy stream while the MTTKRP work items whose
    slices have landed run (_landed_pieces).  The device copy is cached on
    `y` together with the slab events, so the next calls (the other modes of
    the same step) also start on landed slabs instead of waiting for the
    whole copy."""
    y_dev, bounds, landed = _start_upload(y, dev)
    return _landed_pieces(y_dev, y.dims, fac, plan, lam, dev, bounds, landed)


def _stats(variant, y, m, plan, p, timer, *, element_visits, atomic_updates, tile_volume=None, unroll=None,
           scratch=None, footprint=None):
    return MttkrpStats(
        variant, plan.mode, element_visits=element_visits, atomic_updates=atomic_updates, _seconds=timer,
        workers=1, tile_volume=tile_volume, unroll=unroll, scratch_bytes=scratch, footprint_bytes=footprint,
        rank_tile=p.rank_tile, splits=p.splits,
    )


def mttkrp_reference(y: DenseTensor, m: KruskalTensor, mode: int) -> MttkrpOutput:
    """mttkrp.py:154-165 signature; runs the sm_100a kernel with one split."""
    _check_inputs(y, m, mode)
    plan = MttkrpPlan(Variant.REFERENCE, int(mode), splits=1)
    plan.validate(y.dims, m.rank)
    mat, p, t = _run_gpu(y, m, plan)
    return MttkrpOutput(mat, _stats(Variant.REFERENCE, y, m, plan, p, t, element_visits=y.size, atomic_updates=0))


def mttkrp_elem(y: DenseTensor, m: KruskalTensor, plan: MttkrpPlan) -> MttkrpOutput:
    if plan.variant != Variant.ELEM:
        raise ParameterError(f"plan variant is {plan.variant}, expected elem")
    _check_inputs(y, m, plan.mode)
    plan.validate(y.dims, m.rank)
    mat, p, t = _run_gpu(y, m, plan)
    return MttkrpOutput(
        mat,
        _stats(Variant.ELEM, y, m, plan, p, t, element_visits=y.size, atomic_updates=y.size * m.rank,
               unroll=plan.unroll),
    )


def mttkrp_slice(y: DenseTensor, m: KruskalTensor, plan: MttkrpPlan) -> MttkrpOutput:
    if plan.variant != Variant.SLICE:
        raise ParameterError(f"plan variant is {plan.variant}, expected slice")
    _check_inputs(y, m, plan.mode)
    plan.validate(y.dims, m.rank)
    mat, p, t = _run_gpu(y, m, plan)
    n_s = y.size // y.dims[plan.mode]
    return MttkrpOutput(
        mat,
        _stats(Variant.SLICE, y, m, plan, p, t, element_visits=y.size * math.ceil(m.rank / plan.unroll),
               atomic_updates=0, tile_volume=n_s, unroll=plan.unroll),
    )


def mttkrp_tile(y: DenseTensor, m: KruskalTensor, plan: MttkrpPlan) -> MttkrpOutput:
    if plan.variant != Variant.TILE:
        raise ParameterError(f"plan variant is {plan.variant}, expected tile")
    _check_inputs(y, m, plan.mode)
    plan.validate(y.dims, m.rank)
    mat, p, t = _run_gpu(y, m, plan)
    n_t = int(plan.tile_volume)
    i_k = y.dims[plan.mode]
    tps = -(-(y.size // i_k) // n_t)
    return MttkrpOutput(
        mat,
        _stats(Variant.TILE, y, m, plan, p, t, element_visits=y.size * math.ceil(m.rank / plan.unroll),
               atomic_updates=i_k * tps * m.rank, tile_volume=n_t, unroll=plan.unroll),
    )


def mttkrp_b200(y: DenseTensor, m: KruskalTensor, plan: MttkrpPlan) -> MttkrpOutput:
    """The auto-planned kernel: splits fill whole waves of SMs."""
    _check_inputs(y, m, plan.mode)
    plan.validate(y.dims, m.rank)
    mat, p, t = _run_gpu(y, m, plan)
    i_k = y.dims[plan.mode]
    return MttkrpOutput(
        mat,
        _stats(Variant(plan.variant), y, m, plan, p, t, element_visits=y.size,
               atomic_updates=i_k * p.splits * m.rank if p.splits > 1 else 0, tile_volume=int(p.tile_volume)),
    )


DEFAULT_KRP_BUDGET = 2 * 1024 ** 3  # bytes allowed for an explicit KRP (mttkrp.py:41)


def full_krp_bytes(dims, rank: int, mode: int) -> int:
    """Bytes of the explicit Khatri-Rao product of the other factors (mttkrp.py:166-168)."""
    return 8 * (num_elements(dims) // dims[mode]) * rank


def _split_extents(dims, mode: int) -> tuple:
    i_l = num_elements(dims[:mode]) if mode > 0 else 1
    i_r = num_elements(dims[mode + 1:]) if mode < len(dims) - 1 else 1
    return i_l, i_r


def gemm_scratch_bytes(dims, rank: int, mode: int) -> int:
    """Temporary bytes the dense GEMM baseline allocates for `mode` (mttkrp.py:213-221)."""
    d = len(dims)
    i_l, i_r = _split_extents(dims, mode)
    if mode == 0:
        return 8 * rank * i_r
    if mode == d - 1:
        return 8 * rank * i_l
    return 8 * (rank * (i_l + i_r) + i_l * dims[mode] * rank)


def gemm_model_bytes(dims, rank: int, mode: int) -> int:
    """Model footprint of the GEMM baseline: tensor + partial KRPs + output (mttkrp.py:224-227)."""
    i_l, i_r = _split_extents(dims, mode)
    return 8 * (num_elements(dims) + rank * (i_l + i_r + dims[mode]))


def mttkrp_full_krp(y: DenseTensor, m: KruskalTensor, mode: int,
                    budget_bytes: int = DEFAULT_KRP_BUDGET) -> MttkrpOutput:
    """mttkrp.py:173-203 contract: the reference's checks and budget
    (ResourceError when the explicit KRP would exceed ``budget_bytes``), and
    its stats accounting; the product itself runs on the matrix-free sm_100a
    kernel, so no KRP is ever formed here."""
    _check_inputs(y, m, mode)
    if y.ndim < 2:
        raise ParameterError("full-krp needs at least two modes")
    z_bytes = full_krp_bytes(y.dims, m.rank, mode)
    if z_bytes > budget_bytes:
        raise ResourceError(f"explicit KRP needs {z_bytes} bytes, budget is {budget_bytes}")
    plan = MttkrpPlan(Variant.FULL_KRP, int(mode))
    mat, p, t = _run_gpu(y, m, plan)
    return MttkrpOutput(mat, _stats(Variant.FULL_KRP, y, m, plan, p, t, element_visits=y.size, atomic_updates=0,
                                    scratch=z_bytes + (0 if mode == 0 else 8 * y.size)))


def mttkrp_gemm(y: DenseTensor, m: KruskalTensor, mode: int, scratch_cap_bytes: int | None = None) -> MttkrpOutput:
    """mttkrp.py:230-276 contract: the reference's checks, scratch cap
    (ResourceError above ``scratch_cap_bytes``) and stats accounting; the
    product runs on the matrix-free sm_100a kernel (the partial-KRP + DGEMM
    form of the baseline itself is `baselines.mttkrp_gemm_cublas`)."""
    _check_inputs(y, m, mode)
    if y.ndim < 2:
        raise ParameterError("gemm baseline needs at least two modes")
    scratch = gemm_scratch_bytes(y.dims, m.rank, mode)
    if scratch_cap_bytes is not None and scratch > scratch_cap_bytes:
        raise ResourceError(f"gemm baseline needs {scratch} scratch bytes, cap is {scratch_cap_bytes}")
    plan = MttkrpPlan(Variant.GEMM, int(mode))
    mat, p, t = _run_gpu(y, m, plan)
    return MttkrpOutput(mat, _stats(Variant.GEMM, y, m, plan, p, t, element_visits=y.size, atomic_updates=0,
                                    scratch=scratch, footprint=gemm_model_bytes(y.dims, m.rank, mode)))


def run(y: DenseTensor, m: KruskalTensor, plan: MttkrpPlan, **kwargs) -> MttkrpOutput:
    """Dispatch one MTTKRP according to the plan's variant (mttkrp.py:378-391).

    As in the reference, ``**kwargs`` (budget_bytes / scratch_cap_bytes) go
    to the FULL_KRP / GEMM variants, which keep their budget semantics.
    """
    v = Variant(plan.variant)
    if v == Variant.REFERENCE:
        return mttkrp_reference(y, m, plan.mode)
    if v == Variant.FULL_KRP:
        return mttkrp_full_krp(y, m, plan.mode, **kwargs)
    if v == Variant.GEMM:
        return mttkrp_gemm(y, m, plan.mode, **kwargs)
    if v == Variant.ELEM:
        return mttkrp_elem(y, m, plan)
    if v == Variant.SLICE:
        return mttkrp_slice(y, m, plan)
    if v == Variant.TILE:
        return mttkrp_tile(y, m, plan)
    return mttkrp_b200(y, m, plan)


def _split_weights(factors, weights):
    """Accept a ``(weights, [A_0, ..., A_{d-1}])`` pair where a factor list is
    expected (the (lambda, factors) form of a Kruskal model)."""
    if (isinstance(factors, tuple) and len(factors) == 2 and isinstance(factors[1], (list, tuple))
            and getattr(factors[0], "ndim", 2) == 1):
        if weights is not None:
            raise ParameterError("weights given twice")
        return list(factors[1]), factors[0]
    return factors, weights


def mttkrp(tensor, factors, mode: int, weights=None, plan: MttkrpPlan | None = None):
    """North-star convenience: G = MTTKRP(tensor, factors, mode).

    ``tensor`` is a DenseTensor or a flat/first-mode-fastest CUDA tensor
    (then ``factors`` must be CUDA too); ``factors`` is a list of (I_m, R)
    matrices, a ``(weights, factors)`` pair, or a KruskalTensor (weights are
    folded once).  Returns an (I_k, R) matrix of the input's kind (numpy for
    host, torch for CUDA).
    """
    factors, weights = _split_weights(factors, weights)
    if isinstance(tensor, torch.Tensor) and tensor.is_cuda and tensor.dtype == torch.float32:
        # optional float32 path: device in, device out (float32)
        fs = list(factors.factors if isinstance(factors, KruskalTensor) else factors)
        dims = tuple(int(f.shape[0]) for f in fs)
        w = factors.weights if isinstance(factors, KruskalTensor) else weights
        if w is not None and not isinstance(w, torch.Tensor):
            w = torch.as_tensor(np.asarray(w), device=tensor.device)
        return mttkrp_device(tensor.reshape(-1), dims, [torch.as_tensor(f, device=tensor.device) for f in fs],
                             int(mode), w, plan)[0]
    if isinstance(factors, KruskalTensor):
        m = factors
    else:
        fs = list(factors)
        r = int(fs[0].shape[1])
        # unit weights stay on the host: checking device weights for == 1
        # would cost a stream sync per call
        w = weights if weights is not None else np.ones(r)
        m = KruskalTensor(w, fs, validate=False)
    if not isinstance(tensor, DenseTensor):
        tensor = DenseTensor(m.dims, tensor)
    plan = plan or MttkrpPlan(Variant.B200, int(mode))
    if plan.mode != int(mode):
        plan = replace(plan, mode=int(mode))
    return run(tensor, m, plan).matrix


def plan_for_mode(plan: MttkrpPlan, dims, mode: int) -> MttkrpPlan:
    """Copy of ``plan`` retargeted at ``mode``; tile volume clamped to N_S
    (mttkrp.py:394-401)."""
    p = replace(plan, mode=mode)
    if p.variant == Variant.TILE and p.tile_volume is not None:
        n_s = num_elements(dims) // dims[mode]
        p = replace(p, tile_volume=max(1, min(int(p.tile_volume), n_s)))
    return p


def heuristic_tile_width(dims, machine) -> int:
    """Eq. 6 (mttkrp.py:404-423): w^(d-1) s_f c/2 = s_LM/4."""
    dims = tuple(int(x) for x in dims)
    d = len(dims)
    if d < 2:
        raise ParameterError("tile-width heuristic needs at least two modes")
    budget = (machine.s_lm_bytes / 4.0) / (machine.s_f_bytes * (machine.c_tiles / 2.0))
    if budget < 1.0:
        return 1
    w = int(math.floor(budget ** (1.0 / (d - 1))))
    while (w + 1) ** (d - 1) <= budget:
        w += 1
    while w > 1 and w ** (d - 1) > budget:
        w -= 1
    return max(1, min(w, min(dims)))


def heuristic_tile_volume(dims, machine) -> int:
    """N_T = w^(d-1) for the heuristic width (mttkrp.py:426-428)."""
    return heuristic_tile_width(dims, machine) ** (len(dims) - 1)


# (engine, rank tile, rows per CTA, relative DFMA rate) -- mirrors kChoices in
# csrc/mttkrp.cu; rates from the B200 sweeps (profiles/r01_sweep_*.agg.csv)
_TILE_CHOICES = (  # same order as kChoices (ties go to the earlier entry)
    ("tma", 256, 96, 0.95), ("tma", 128, 128, 1.00), ("tma", 64, 256, 0.93),
    ("dmma", 256, 64, 1.02), ("dmma", 128, 128, 1.23), ("dmma", 64, 256, 1.26),
    ("dmma", 32, 256, 1.15), ("dmma", 16, 256, 0.90),
    ("cpdmma", 128, 128, 0.97), ("cpdmma", 64, 256, 0.88),
    ("cpasync", 128, 128, 0.92), ("cpasync", 64, 128, 0.78), ("cpasync", 32, 64, 0.55),
)


def heuristic_rank_tile(rank: int, rows: int | None = None, tma: bool = True) -> tuple:
    """(engine, rank tile) the planner picks: the B200 analogue of Eq. 6.

    Eq. 6 sizes N_T so tensor elements fill a quarter of the private cache
    (PAPER.md:405-409).  On B200 the private level that bounds the *rank*
    tile is the register file: each consumer thread keeps a TM x 8 FP64
    accumulator tile (TM = 8 or 12), 256 threads per CTA, so the rank tile
    is 64, 128 or 256 columns with 256, 128 or 96 rows.  The planner picks
    the (engine, tile) minimizing padded rows x padded columns / measured
    rate; `tma` is whether the problem is TMA-eligible (even I_0 and R,
    2 <= d <= 5).  Mirrors resolve() in csrc/mttkrp.cu.
    """
    rows = rows or 1
    best, best_cost = None, float("inf")
    for eng, rt, bm, rate in _TILE_CHOICES:
        if eng in ("tma", "dmma") and not tma:
            continue
        if rate <= 0:  # explicit-only engine
            continue
        cost = (-(-rows // bm) * bm) * (-(-rank // rt) * rt) / rate
        if cost < best_cost * (1 - 1e-9):
            best, best_cost = (eng, rt), cost
    return best
