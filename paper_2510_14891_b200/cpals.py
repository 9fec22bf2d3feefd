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
from .als_sweep import GRAPH_MIN_ITERS, DeviceBackend, init_factors, run_sweeps  # noqa: F401
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
    # B200 extension: dimension-tree sweep (als_sweep.tree_split) -- None:
    # when it pays and its W_G fits; True: whenever it fits; False: d
    # tensor passes per sweep like the reference
    dimtree: bool | None = None

    def validate(self) -> None:
        if self.rank < 1:
            raise ParameterError(f"rank must be >= 1, got {self.rank}")
        if self.max_iters < 1:
            raise ParameterError(f"max_iters must be >= 1, got {self.max_iters}")
        if not self.tol >= 0:
            raise ParameterError(f"tol must be >= 0, got {self.tol}")
        if self.init not in _INITS:
            raise ParameterError(f"unknown init {self.init!r}; choose from {_INITS}")
        if self.dimtree not in (None, True, False):
            raise ParameterError(f"dimtree must be None, True or False, got {self.dimtree!r}")


@dataclass
class AlsTrace:
    """Per-sweep fits and timing (cpals.py:57-72); times are CUDA-event seconds."""

    fits: list
    mttkrp_seconds: list
    other_seconds: list
    total_seconds: float
    iterations: int
    converged: bool
    tree_split: int | None = None  # B200: the dimension-tree split point, None = per-mode sweep


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


def cp_als(y: DenseTensor, config: AlsConfig, graph: bool | None = None) -> tuple:
    """Run CP-ALS; returns (KruskalTensor with CUDA factors, AlsTrace).

    ``graph``: True replays sweeps 2.. as one captured CUDA graph (see the
    module doc); False runs every sweep eagerly; None (default) captures when
    max_iters >= GRAPH_MIN_ITERS.  The sweep itself is als_sweep.run_sweeps,
    the same engine the sharded driver runs at world > 1.
    """
    config.validate()
    dev = require_cuda()
    r = config.rank
    d = y.ndim
    dims = y.dims

    t_start = time.perf_counter()
    # an odd I_0 runs on the zero-padded even copy (mttkrp._pad_first_mode):
    # A_0 then carries one extra row, which stays exactly zero (its MTTKRP
    # row is a sum over zeros, and solve / normalize / Gram keep it at zero)
    pad = mt._pad_first_mode(y, mt.plan_for_mode(config.plan, dims, 0), dev) and d >= 2
    run_dims = ((dims[0] + 1,) + dims[1:]) if pad else dims
    y_src = y.device_data(dev)
    y_dev = y.even_device_data(dev) if pad else y_src
    be = DeviceBackend(y_dev, run_dims, r, config.plan, dev)
    res = run_sweeps(be, dims, r, config.seed, config.max_iters, config.tol, y_src, graph=graph, pad_first=pad,
                     tree=config.dimtree)
    torch.cuda.synchronize(dev)
    total = time.perf_counter() - t_start
    factors = res.factors
    if pad:
        factors[0] = factors[0][: dims[0]]
    model = KruskalTensor(res.lam.clone(), factors, validate=False)
    trace = AlsTrace(
        fits=res.fits,
        mttkrp_seconds=res.mttkrp_seconds,
        other_seconds=res.other_seconds,
        total_seconds=total,
        iterations=len(res.fits),
        converged=res.converged,
        tree_split=res.tree_split,
    )
    return model, trace
