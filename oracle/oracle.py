"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the reference's MTTKRP / CP-ALS path:

* ctypes access to oracle/liboracle.so (mttkrp_ref.c): the serial reference
  kernel (_kernels.py:39-57), the TILE kernel with private-copy merge
  (_kernels.py:96-174, mttkrp.py:279-286) and a row-restricted reference.
* `mttkrp_gemm`: numpy restatement of the Phan partial-KRP baseline
  (mttkrp.py:230-276, dtensor.py:305-331) -- the fast oracle at c2/c3 sizes.
* `cp_als`: numpy/scipy restatement of cpals.cp_als (cpals.py:75-171).
"""

from __future__ import annotations

import ctypes as C
import math
import subprocess
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lock = threading.Lock()
_lib = None


def build() -> Path:
    """Compile liboracle.so with the committed Makefile (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not LIB.exists() or LIB.stat().st_mtime < (HERE / "mttkrp_ref.c").stat().st_mtime:
                build()
            L = C.CDLL(str(LIB))
            P, I64 = C.c_void_p, C.c_int64
            L.orc_mttkrp_ref.argtypes = [P, C.c_int, P, C.c_int, P, P, I64, P]
            L.orc_mttkrp_tile.argtypes = [P, C.c_int, P, C.c_int, P, P, I64, I64, I64, C.c_int, P]
            L.orc_mttkrp_rows.argtypes = [P, C.c_int, P, C.c_int, P, P, I64, P, I64, P]
            L.orc_max_threads.argtypes = []
            for fn in (L.orc_mttkrp_ref, L.orc_mttkrp_tile, L.orc_mttkrp_rows, L.orc_max_threads):
                fn.restype = C.c_int
            _lib = L
    return _lib


def _prep(data, dims, factors, lam):
    data = np.ascontiguousarray(data, dtype=np.float64).ravel()
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    facs = [np.ascontiguousarray(a, dtype=np.float64) for a in factors]
    ptrs = (C.c_void_p * len(facs))(*[a.ctypes.data for a in facs])
    lam_a = None if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
    return data, dims_a, facs, ptrs, lam_a


def mttkrp_ref(data, dims, k, factors, lam=None) -> np.ndarray:
    """Serial reference, canonical order (_kernels.py:39-57)."""
    data, dims_a, facs, ptrs, lam_a = _prep(data, dims, factors, lam)
    r = facs[0].shape[1]
    out = np.zeros((int(dims[k]), r))
    rc = lib().orc_mttkrp_ref(data.ctypes.data, len(dims), dims_a.ctypes.data, int(k), ptrs,
                              None if lam_a is None else lam_a.ctypes.data, r, out.ctypes.data)
    assert rc == 0
    return out


def mttkrp_tile(data, dims, k, factors, lam=None, f_cols=16, n_t=None, workers=0) -> tuple:
    """TILE kernel + private-copy merge; returns (G, workers used)."""
    data, dims_a, facs, ptrs, lam_a = _prep(data, dims, factors, lam)
    r = facs[0].shape[1]
    n_s = data.size // int(dims[k])
    n_t = n_s if n_t is None else max(1, min(int(n_t), n_s))
    out = np.zeros((int(dims[k]), r))
    w = lib().orc_mttkrp_tile(data.ctypes.data, len(dims), dims_a.ctypes.data, int(k), ptrs,
                              None if lam_a is None else lam_a.ctypes.data, r, int(f_cols), n_t, int(workers),
                              out.ctypes.data)
    assert w > 0
    return out, w


def mttkrp_rows(data, dims, k, factors, rows, lam=None) -> np.ndarray:
    """Rows `rows` of G, each bit-equal to the serial reference."""
    data, dims_a, facs, ptrs, lam_a = _prep(data, dims, factors, lam)
    r = facs[0].shape[1]
    rows_a = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((rows_a.size, r))
    rc = lib().orc_mttkrp_rows(data.ctypes.data, len(dims), dims_a.ctypes.data, int(k), ptrs,
                               None if lam_a is None else lam_a.ctypes.data, r, rows_a.ctypes.data, rows_a.size,
                               out.ctypes.data)
    assert rc == 0
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ------------------------------------------------------------------ numpy


def khatri_rao(a, b):
    """Column-wise Kronecker, first factor slowest (dtensor.py:305-319)."""
    return (a[:, None, :] * b[None, :, :]).reshape(a.shape[0] * b.shape[0], a.shape[1])


def khatri_rao_chain(mats):
    out = np.array(mats[0], dtype=np.float64)
    for m in mats[1:]:
        out = khatri_rao(out, m)
    return out


def mttkrp_gemm(data, dims, k, factors, lam=None) -> np.ndarray:
    """Phan partial-KRP GEMM baseline (mttkrp.py:230-276), lam applied once."""
    dims = tuple(int(x) for x in dims)
    d = len(dims)
    r = factors[0].shape[1]
    lam = np.ones(r) if lam is None else np.asarray(lam, dtype=np.float64)
    data = np.asarray(data, dtype=np.float64).ravel()
    i_l = int(np.prod(dims[:k])) if k > 0 else 1
    i_r = int(np.prod(dims[k + 1:])) if k < d - 1 else 1
    i_k = dims[k]
    if d == 1:
        return data[:, None] * lam[None, :]
    if k == 0:
        z_r = khatri_rao_chain([factors[m] for m in range(d - 1, 0, -1)]) * lam
        out = data.reshape((i_k, i_r), order="F") @ z_r
    elif k == d - 1:
        z_l = khatri_rao_chain([factors[m] for m in range(d - 2, -1, -1)]) * lam
        out = data.reshape((i_l, i_k), order="F").T @ z_l
    else:
        z_r = khatri_rao_chain([factors[m] for m in range(d - 1, k, -1)]) * lam
        c = data.reshape((i_l * i_k, i_r), order="F") @ z_r
        c3 = c.reshape((i_l, i_k, r), order="F")
        z_l = khatri_rao_chain([factors[m] for m in range(k - 1, -1, -1)])
        out = np.einsum("qlj,qj->lj", c3, z_l)
    return np.ascontiguousarray(out)


def rel_err(got, ref) -> float:
    ref = np.asarray(ref)
    denom = float(np.linalg.norm(ref))
    diff = float(np.linalg.norm(np.asarray(got) - ref))
    if denom == 0.0:
        return 0.0 if diff == 0.0 else math.inf
    return diff / denom


def gram(a):
    """A^T A symmetrized exactly (kruskal.py:110-114)."""
    g = a.T @ a
    return np.triu(g) + np.triu(g, 1).T


def _solve_normal(gamma, g):
    """cpals._solve_normal (cpals.py:75-89)."""
    from numpy.linalg import LinAlgError
    from scipy.linalg import cho_factor, cho_solve

    r = gamma.shape[0]
    try:
        return cho_solve(cho_factor(gamma, check_finite=False), g.T, check_finite=False).T
    except LinAlgError:
        pass
    eps = 1e-12
    for _ in range(5):
        reg = gamma + (eps * np.trace(gamma) / r) * np.eye(r)
        try:
            return cho_solve(cho_factor(reg, check_finite=False), g.T, check_finite=False).T
        except LinAlgError:
            eps *= 1e3
    return np.linalg.lstsq(gamma, g.T, rcond=None)[0].T


def cp_als(data, dims, rank, max_iters=100, tol=1e-4, seed=0, mttkrp="gemm"):
    """cpals.cp_als (cpals.py:92-171) restated; returns (lam, factors, fits)."""
    dims = tuple(int(x) for x in dims)
    data = np.asarray(data, dtype=np.float64).ravel()
    norm_y = float(np.linalg.norm(data))
    d = len(dims)
    rng = np.random.Generator(np.random.Philox(seed))
    factors = [rng.random((i_k, rank)) for i_k in dims]
    grams = [gram(a) for a in factors]
    lam = np.ones(rank)
    fits = []
    mt = {"gemm": mttkrp_gemm, "ref": mttkrp_ref}[mttkrp]
    for _ in range(max_iters):
        g = None
        for k in range(d):
            g = mt(data, dims, k, factors)
            gamma = np.ones((rank, rank))
            for m in range(d):
                if m != k:
                    gamma *= grams[m]
            a_hat = _solve_normal(gamma, g)
            nrm = np.linalg.norm(a_hat, axis=0)
            nz = nrm > 0
            a_hat[:, nz] /= nrm[nz]
            lam = np.where(nz, nrm, 0.0)
            factors[k] = np.ascontiguousarray(a_hat)
            grams[k] = gram(factors[k])
        h = np.ones((rank, rank))
        for m in range(d):
            h *= grams[m]
        norm_m_sq = float(lam @ h @ lam)
        iprod = float(np.sum((g * lam) * factors[d - 1]))
        resid_sq = max(0.0, norm_y ** 2 - 2.0 * iprod + norm_m_sq)
        fits.append(float(1.0 - np.sqrt(resid_sq) / norm_y))
        if len(fits) >= 2 and abs(fits[-1] - fits[-2]) < tol:
            break
    return lam, factors, fits
