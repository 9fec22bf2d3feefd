"""Library baselines on the same GPU, for comparison only (never the product
path): the reference's dense GEMM MTTKRP (`mttkrp_gemm`, mttkrp.py:230-276,
Phan et al.'s partial Khatri-Rao products) written the way
a user of the vendor library would: partial KRPs materialized in HBM with
torch elementwise ops, the contraction on cuBLAS DGEMM.  The paper's Fig. 4
compares MTTKRP-TILE against exactly this baseline.
"""

from __future__ import annotations

import torch

from .dtensor import num_elements


def _krp(mats) -> torch.Tensor:
    """Khatri-Rao product with the FIRST matrix's row index fastest:
    row (i_0 + I_0 i_1 + ...) = mats[0][i_0] * mats[1][i_1] * ...  (the
    column order of the first-mode-fastest unfolding; dtensor.py:305-331
    builds the same rows with the last factor fastest in its argument list)."""
    z = mats[0]
    for a in mats[1:]:
        z = (a[:, None, :] * z[None, :, :]).reshape(-1, z.shape[1])
    return z


def gemm_scratch_bytes(dims, rank: int, mode: int) -> int:
    """Temporary bytes of this baseline for `mode` (mttkrp.py:213-221)."""
    d = len(dims)
    i_l = num_elements(dims[:mode]) if mode > 0 else 1
    i_r = num_elements(dims[mode + 1:]) if mode < d - 1 else 1
    if mode == 0:
        return 8 * rank * i_r
    if mode == d - 1:
        return 8 * rank * i_l
    return 8 * (rank * (i_l + i_r) + i_l * dims[mode] * rank)


def mttkrp_gemm_cublas(y_dev: torch.Tensor, dims, factors, mode: int, weights=None) -> torch.Tensor:
    """G = Y_(k) (KRP of the other factors) diag(lam) via partial KRPs + DGEMM.

    y_dev: flat first-mode-fastest CUDA float64; factors: CUDA (I_m, R).
    Mode 0 / d-1: one GEMM against the right / left partial KRP; interior
    modes: C = Y[(I_L I_k), I_R] Z_R, then G[n, j] = sum_l C[l, n, j] Z_L[l, j]
    (mttkrp.py:257-265).  The weights are folded once into Z_R (or Z_L).
    """
    d = len(dims)
    i_k = dims[mode]
    i_l = num_elements(dims[:mode]) if mode > 0 else 1
    i_r = num_elements(dims[mode + 1:]) if mode < d - 1 else 1
    # column-major views of the flat buffer: Y[(i_l, i_k, i_r)] with i_l fastest
    y3 = y_dev.view(i_r, i_k, i_l)  # row-major view of the same memory
    if mode == 0:
        z_r = _krp(factors[1:])
        if weights is not None:
            z_r = z_r * weights
        return y3.reshape(i_r, i_k).t() @ z_r  # (i_k, i_r) @ (i_r, R)
    if mode == d - 1:
        z_l = _krp(factors[:-1])
        if weights is not None:
            z_l = z_l * weights
        return y3.reshape(i_k, i_l) @ z_l  # (i_k, i_l) @ (i_l, R)
    z_r = _krp(factors[mode + 1:])
    if weights is not None:
        z_r = z_r * weights
    c = y3.reshape(i_r, i_k * i_l).t() @ z_r  # (i_k i_l, R), i_l fastest in the row index
    z_l = _krp(factors[:mode])
    return torch.einsum("klj,lj->kj", c.view(i_k, i_l, -1), z_l)


def mttkrp_elem_atomic(y_dev: torch.Tensor, dims, factors, mode: int, weights=None) -> torch.Tensor:
    """The paper's baseline matrix-free GPU kernel, MTTKRP-ELEM: N R FP64
    atomics into G (cpk_mttkrp_elem_f64).  Comparison only."""
    from . import _lib
    from ._device import stream_ptr

    d = len(dims)
    rank = next(int(f.shape[1]) for f in factors if f is not None)
    out = torch.empty((dims[mode], rank), dtype=torch.float64, device=y_dev.device)
    ptrs = _lib.ptr_array([f.data_ptr() if m != mode else 0 for m, f in enumerate(factors)])
    lds = _lib.i64_array([f.stride(0) for f in factors])
    _lib.check(_lib.load().cpk_mttkrp_elem_f64(
        y_dev.data_ptr(), d, _lib.i64_array(dims), int(mode), ptrs, lds,
        weights.data_ptr() if weights is not None else None, rank, out.data_ptr(), out.stride(0),
        stream_ptr(y_dev.device)), "mttkrp elem")
    return out
