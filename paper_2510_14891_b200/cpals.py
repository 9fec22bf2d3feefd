"""CP-ALS on the device, on top of the sm_100a MTTKRP.

Drop-in for cpkern.cpals (pkg/src/cpkern/cpals.py:27-171): same AlsConfig /
AlsTrace / cp_als contract, same sweep (modes in order; Gamma = (*) of the
other Grams in ascending m; solve X Gamma = G with the eps ladder; column
norms folded into lam, which is *replaced* each mode; fit through the
factored identity with the last mode's unit-weight MTTKRP), same Philox
initialization order, so a fixed seed gives the reference's trajectory up to
floating-point reassociation.

Everything between two MTTKRPs stays on the device (Gram, Hadamard,
Cholesky via cuSOLVER, normalization, fit terms).  Host syncs per sweep: one
per mode for the Cholesky info flag (the regularization ladder branches on
it, cpals.py:78-88) and one for the two fit scalars (the stopping rule needs
them on the host, cpals.py:157).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
import importlib

mt = importlib.import_module(".mttkrp", __package__)  # the submodule (the package re-exports a function of the same name)
from ._device import EventTimer, require_cuda, stream_ptr, workspace
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


def cp_als(y: DenseTensor, config: AlsConfig) -> tuple:
    """Run CP-ALS; returns (KruskalTensor with CUDA factors, AlsTrace)."""
    config.validate()
    dev = require_cuda()
    y_dev = y.device_data(dev)
    norm_y = y.norm()
    if not math.isfinite(norm_y):  # NaN/Inf anywhere make ||y|| non-finite
        raise ParameterError("tensor has non-finite entries")
    if norm_y == 0.0:
        raise ParameterError("cannot fit an all-zero tensor (fit is undefined)")
    r = config.rank
    d = y.ndim
    dims = y.dims
    lib = _lib.load()
    sp = stream_ptr(dev)

    t_start = time.perf_counter()
    factors = [torch.from_numpy(a).to(dev) for a in init_factors(dims, r, config.seed)]
    grams = [gram(a) for a in factors]
    lam = torch.ones(r, dtype=torch.float64, device=dev)
    solver = _Solver(dev, max(dims), r)
    gamma = torch.empty((r, r), dtype=torch.float64, device=dev)
    h = torch.empty((r, r), dtype=torch.float64, device=dev)
    normsq = torch.empty(r, dtype=torch.float64, device=dev)
    terms = torch.empty(2, dtype=torch.float64, device=dev)

    fits, mttkrp_seconds, other_seconds = [], [], []
    converged = False
    for _ in range(config.max_iters):
        sweep_timers, other_timers = [], []
        g = None
        for k in range(d):
            plan_k = mt.plan_for_mode(config.plan, dims, k)
            g, _, timer = mt.mttkrp_device(y_dev, dims, factors, k, None, plan_k)
            sweep_timers.append(timer)
            t_other = EventTimer(dev)
            hadamard(grams, skip=k, out=gamma)
            # the solve is in place; the fit needs the last mode's G itself
            a_hat = solver(gamma, g.clone() if k == d - 1 else g)
            _lib.check(
                lib.cpk_normalize_columns_f64(a_hat.data_ptr(), a_hat.shape[0], r, a_hat.stride(0),
                                              lam.data_ptr(), normsq.data_ptr(), sp),
                "normalize",
            )
            factors[k] = a_hat
            grams[k] = gram(a_hat)
            other_timers.append(t_other.stop(dev))

        t_fit = EventTimer(dev)
        hadamard(grams, skip=-1, out=h)
        # g is the unit-weight mode-(d-1) MTTKRP and A_{d-1} was solved from it
        _lib.check(
            lib.cpk_fit_terms_f64(h.data_ptr(), lam.data_ptr(), g.data_ptr(), factors[d - 1].data_ptr(),
                                  g.shape[0], r, terms.data_ptr(), sp),
            "fit terms",
        )
        other_timers.append(t_fit.stop(dev))
        norm_m_sq, iprod = (float(v) for v in terms.cpu().tolist())
        resid_sq = max(0.0, norm_y ** 2 - 2.0 * iprod + norm_m_sq)
        fit = 1.0 - math.sqrt(resid_sq) / norm_y

        fits.append(float(fit))
        mttkrp_seconds.append([t.seconds for t in sweep_timers])
        other_seconds.append(sum(t.seconds for t in other_timers))
        if len(fits) >= 2 and abs(fits[-1] - fits[-2]) < config.tol:
            converged = True
            break

    torch.cuda.synchronize(dev)
    total = time.perf_counter() - t_start
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
