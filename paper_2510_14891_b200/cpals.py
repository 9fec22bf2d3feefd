"""CP-ALS on the device, on top of the sm_100a MTTKRP.

Drop-in for cpkern.cpals (pkg/src/cpkern/cpals.py:27-171): same AlsConfig /
AlsTrace / cp_als contract, same sweep (modes in order; Gamma = (*) of the
other Grams in ascending m; solve X Gamma = G with the eps ladder; column
norms folded into lam, which is *replaced* each mode; fit through the
factored identity with the last mode's unit-weight MTTKRP), same Philox
initialization order, so a fixed seed gives the reference's trajectory up to
floating-point reassociation.

Everything between two MTTKRPs stays on the device (Gram, Hadamard,
Cholesky via cuSOLVER, normalization, fit terms), in fixed buffers: the
MTTKRP of mode k is written straight into A_k's buffer (mode k's own factor
is not read by its MTTKRP) and solved in place.  Every sweep is
speculative: a snapshot of (factors, Grams, lam), the d modes with a rung-0
solve whose Cholesky flags stay on the device, and the fit terms; the only
host sync per sweep is one 2 + d scalar readback (fit terms + flags) for
the stopping rule (cpals.py:157).  If a flag shows a failed Cholesky, the
snapshot is restored and that sweep reruns through the full regularization
ladder (cpals.py:78-88; a host sync per mode), so the trajectory is the
ladder's either way.  With ``graph`` sweeps 2.. are one CUDA-graph replay
each (no per-launch host work at all).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib
import importlib

mt = importlib.import_module(".mttkrp", __package__)  # the submodule (the package re-exports a function of the same name)
from ._device import require_cuda, stream_ptr, workspace
from .dtensor import DenseTensor
from .errors import ParameterError
from .kruskal import KruskalTensor, gram, hadamard

_INITS = ("random-uniform",)


@dataclass(frozen=True)
class AlsConfig:
    """Rank, stopping rule, seed and the MTTKRP plan template (cpals.py:27-54)."""

    rank: int
    max_iters: int = 100
    tol: float = 1e-4
    seed: int = 0
    plan: mt.MttkrpPlan = field(default=mt.MttkrpPlan(variant=mt.Variant.B200, mode=0))
    init: str = "random-uniform"

    def validate(self) -> None:
        if self.rank < 1:
            raise ParameterError(f"rank must be >= 1, got {self.rank}")
        if self.max_iters < 1:
            raise ParameterError(f"max_iters must be >= 1, got {self.max_iters}")
        if not self.tol >= 0:
            raise ParameterError(f"tol must be >= 0, got {self.tol}")
        if self.init not in _INITS:
            raise ParameterError(f"unknown init {self.init!r}; choose from {_INITS}")


@dataclass
class AlsTrace:
    """Per-sweep fits and timing (cpals.py:57-72); times are CUDA-event seconds."""

    fits: list
    mttkrp_seconds: list
    other_seconds: list
    total_seconds: float
    iterations: int
    converged: bool


def init_factors(dims, rank: int, seed: int) -> list:
    """Philox(seed) uniform [0,1) factors in mode order (cpals.py:108-109)."""
    rng = np.random.Generator(np.random.Philox(seed))
    return [rng.random((i_k, rank)) for i_k in dims]


class _Solver:
    """Normal-equation solve X Gamma = G in place (cpals._solve_normal)."""

    def __init__(self, dev, max_rows: int, rank: int):
        self.dev = dev
        nbytes = _lib.C.c_size_t(0)
        _lib.check(_lib.load().cpk_solve_workspace_bytes(max_rows, rank, _lib.C.byref(nbytes)), "solve workspace")
        self.work = workspace(dev, nbytes.value, tag="solve")
        self.nbytes = nbytes.value

    def __call__(self, gamma: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
        rows, r = g.shape
        rc = _lib.load().cpk_solve_normal_f64(
            gamma.data_ptr(), g.data_ptr(), rows, r, self.work.data_ptr(), self.nbytes, stream_ptr(self.dev)
        )
        if rc == _lib.CPK_ERR_NOT_PD:
            # last rung of cpals.py:89: minimum-norm least squares,
            # lstsq(Gamma, G^T)^T == G pinv(Gamma) for symmetric Gamma
            return g @ torch.linalg.pinv(gamma)
        _lib.check(rc, "solve")
        return g


def _factor_spec(solver: "_Solver", gamma: torch.Tensor, info: torch.Tensor, stream) -> None:
    """First half of the speculative solve: Cholesky of Gamma into the solver
    workspace (cpk_solve_factor_spec_f64), on ``stream``."""
    r = gamma.shape[0]
    _lib.check(
        _lib.load().cpk_solve_factor_spec_f64(gamma.data_ptr(), r, solver.work.data_ptr(), solver.nbytes,
                                              info.data_ptr(), stream.cuda_stream),
        "solve factor (speculative)",
    )


def _apply_spec(solver: "_Solver", g: torch.Tensor, info: torch.Tensor) -> None:
    """Second half: X Gamma = G in place with the factor (skipped on a flag)."""
    rows, r = g.shape
    _lib.check(
        _lib.load().cpk_solve_apply_spec_f64(g.data_ptr(), rows, r, solver.work.data_ptr(), solver.nbytes,
                                             info.data_ptr(), stream_ptr(solver.dev)),
        "solve apply (speculative)",
    )


def _solve_spec(solver: "_Solver", gamma: torch.Tensor, g: torch.Tensor, info: torch.Tensor) -> None:
    rows, r = g.shape
    _lib.check(
        _lib.load().cpk_solve_normal_spec_f64(gamma.data_ptr(), g.data_ptr(), rows, r, solver.work.data_ptr(),
                                              solver.nbytes, info.data_ptr(), stream_ptr(solver.dev)),
        "solve (speculative)",
    )


# Capturing a sweep costs ~6 ms once and saves ~0.5 ms of host gaps per
# sweep (c3: 17.5 ms eager vs 17.0 replayed; 10 sweeps break even,
# profiles/r01_bench.jsonl), so the auto mode captures runs that may go
# longer than that.
GRAPH_MIN_ITERS = 12


def cp_als(y: DenseTensor, config: AlsConfig, graph: bool | None = None) -> tuple:
    """Run CP-ALS; returns (KruskalTensor with CUDA factors, AlsTrace).

    ``graph``: True replays sweeps 2.. as one captured CUDA graph (see the
    module doc); False runs every sweep eagerly with the ladder solve; None
    (default) captures when max_iters >= GRAPH_MIN_ITERS.
    """
    config.validate()
    if graph is None:
        graph = config.max_iters >= GRAPH_MIN_ITERS
    dev = require_cuda()
    norm_y = y.norm()
    if not math.isfinite(norm_y):  # NaN/Inf anywhere make ||y|| non-finite
        raise ParameterError("tensor has non-finite entries")
    if norm_y == 0.0:
        raise ParameterError("cannot fit an all-zero tensor (fit is undefined)")
    r = config.rank
    d = y.ndim
    dims = y.dims
    lib = _lib.load()

    t_start = time.perf_counter()
    # an odd I_0 runs on the zero-padded even copy (mttkrp._pad_first_mode):
    # A_0 then carries one extra row, which stays exactly zero (its MTTKRP
    # row is a sum over zeros, and solve / normalize / Gram keep it at zero)
    pad = mt._pad_first_mode(y, mt.plan_for_mode(config.plan, dims, 0), dev) and d >= 2
    run_dims = ((dims[0] + 1,) + dims[1:]) if pad else dims
    y_dev = y.even_device_data(dev) if pad else y.device_data(dev)
    # fixed buffers: every sweep (eager or replayed) reads and writes these
    factors = [torch.from_numpy(a).to(dev) for a in init_factors(dims, r, config.seed)]
    if pad:
        factors[0] = torch.cat([factors[0], torch.zeros((1, r), dtype=torch.float64, device=dev)])
    grams = [gram(a) for a in factors]
    lam = torch.ones(r, dtype=torch.float64, device=dev)
    solver = _Solver(dev, max(run_dims), r)
    gamma = torch.empty((r, r), dtype=torch.float64, device=dev)
    h = torch.empty((r, r), dtype=torch.float64, device=dev)
    normsq = torch.empty(r, dtype=torch.float64, device=dev)
    g_last = torch.empty((run_dims[d - 1], r), dtype=torch.float64, device=dev)
    stats = torch.zeros(2 + d, dtype=torch.float64, device=dev)  # fit terms, Cholesky flags
    info = torch.zeros(d, dtype=torch.int32, device=dev)
    stats_host = torch.zeros(2 + d, dtype=torch.float64, pin_memory=True)
    # The Cholesky of mode k's Gamma needs only the Grams, so speculative
    # sweeps factor it on a side stream while the MTTKRP runs; an automatic
    # plan then fills one SM fewer with split-K waves, leaving the SM the
    # one-CTA factorization takes (c3: ~0.2 ms per mode off the critical path)
    base = config.plan
    if base.splits == 0 and base.sm_count == 0 and base.tile_volume is None:
        base = replace(base, sm_count=max(1, torch.cuda.get_device_properties(dev).multi_processor_count - 1))
    plans = [mt.plan_for_mode(base, run_dims, k) for k in range(d)]
    ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(d + 2)]
    side = torch.cuda.Stream(dev)
    ev_gamma, ev_factor = torch.cuda.Event(), torch.cuda.Event()

    def sweep(spec: bool) -> None:
        sp = stream_ptr(dev)
        main = torch.cuda.current_stream(dev)
        ev[0].record()
        for k in range(d):
            hadamard(grams, skip=k, out=gamma)
            if spec:
                ev_gamma.record(main)
                side.wait_event(ev_gamma)
                _factor_spec(solver, gamma, info[k:k + 1], side)
                ev_factor.record(side)
            mt.mttkrp_device(y_dev, run_dims, factors, k, None, plans[k], out=factors[k])
            ev[k + 1].record()
            if k == d - 1:  # the fit needs the last mode's G itself
                g_last.copy_(factors[k])
            if spec:
                main.wait_event(ev_factor)
                _apply_spec(solver, factors[k], info[k:k + 1])
            else:
                x = solver(gamma, factors[k])
                if x is not factors[k]:  # least-squares last rung
                    factors[k].copy_(x)
            _lib.check(
                lib.cpk_normalize_columns_f64(factors[k].data_ptr(), run_dims[k], r, factors[k].stride(0),
                                              lam.data_ptr(), normsq.data_ptr(), sp),
                "normalize",
            )
            gram(factors[k], out=grams[k])
        hadamard(grams, skip=-1, out=h)
        # g_last is the unit-weight mode-(d-1) MTTKRP and A_{d-1} was solved from it
        _lib.check(
            lib.cpk_fit_terms_f64(h.data_ptr(), lam.data_ptr(), g_last.data_ptr(), factors[d - 1].data_ptr(),
                                  run_dims[d - 1], r, stats.data_ptr(), sp),
            "fit terms",
        )
        stats[2:].copy_(info)
        stats_host.copy_(stats, non_blocking=True)
        ev[d + 1].record()  # after the readback: waiting on it makes stats_host valid

    saved = [torch.empty_like(t) for t in factors + grams + [lam]]
    captured = None

    def snapshot():  # one multi-tensor copy launch, not 2d + 1
        torch._foreach_copy_(saved, factors + grams + [lam])

    def restore():
        torch._foreach_copy_(factors + grams + [lam], saved)

    fits, mttkrp_seconds, other_seconds = [], [], []
    converged = False
    for it in range(config.max_iters):
        if it == 0 or not graph:
            # eager: the same speculative sweep, one host sync per sweep
            snapshot()
            info.zero_()
            sweep(spec=True)
        else:
            if captured is None:
                keep = list(_device_workspaces(dev))  # captured pointers stay alive
                captured = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream(dev)  # not `side`: sweep() forks onto that one
                cap.wait_stream(torch.cuda.current_stream(dev))
                # capture_begin/end directly: torch.cuda.graph() would also
                # gc.collect() and empty the allocator cache on entry
                with torch.cuda.stream(cap):
                    captured.capture_begin()
                    try:
                        snapshot()
                        info.zero_()
                        sweep(spec=True)
                    finally:
                        captured.capture_end()
                torch.cuda.current_stream(dev).wait_stream(cap)
                captured.keep = keep
            captured.replay()
        ev[d + 1].synchronize()
        if bool((stats_host[2:] != 0).any()):
            # a speculative Cholesky failed: roll the sweep back, rerun it
            # through the ladder (cpals.py:78-88)
            restore()
            info.zero_()
            sweep(spec=False)
            ev[d + 1].synchronize()
        norm_m_sq, iprod = float(stats_host[0]), float(stats_host[1])
        resid_sq = max(0.0, norm_y ** 2 - 2.0 * iprod + norm_m_sq)
        fit = 1.0 - math.sqrt(resid_sq) / norm_y

        fits.append(float(fit))
        mts = [ev[k].elapsed_time(ev[k + 1]) * 1e-3 for k in range(d)]
        mttkrp_seconds.append(mts)
        other_seconds.append(ev[0].elapsed_time(ev[d + 1]) * 1e-3 - sum(mts))
        if len(fits) >= 2 and abs(fits[-1] - fits[-2]) < config.tol:
            converged = True
            break

    torch.cuda.synchronize(dev)
    total = time.perf_counter() - t_start
    if pad:
        factors[0] = factors[0][: dims[0]]
    model = KruskalTensor(lam.clone(), factors, validate=False)
    trace = AlsTrace(
        fits=fits,
        mttkrp_seconds=mttkrp_seconds,
        other_seconds=other_seconds,
        total_seconds=total,
        iterations=len(fits),
        converged=converged,
    )
    return model, trace


def _device_workspaces(dev):
    from . import _device

    with _device._ws_lock:
        return [t for (idx, _), t in _device._workspaces.items() if idx == dev.index]
