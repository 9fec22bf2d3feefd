"""The CP-ALS normal-equation solve X Gamma = G (cpals._solve_normal,
cpals.py:75-89) on the device: the small-rank Cholesky kernels (default for
R <= 256; csrc/als.cu chol_small_kernel / chol_rows_kernel, CPK_SOLVE=kernel
forces them up to R = 512), the multi-CTA sweep (default above 256;
csrc/sweep_inv.cu: Gamma^-1 by a blocked Gauss-Jordan sweep with DMMA tile
updates, then X = G Gamma^-1 on the MTTKRP kernel; CPK_SOLVE=sweep forces it)
and the cuSOLVER path (CPK_SOLVE=cusolver) against the oracle's scipy
cho_factor / cho_solve.

Bar: relative Frobenius error <= 1e-10 on well-conditioned Gamma (observed
~1e-14); the non-positive-definite pivot flag matches LAPACK's column.
"""

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2510_14891_b200 import cpals

pytestmark = pytest.mark.gpu
TOL = 1e-10


def spd(r, rng, cond_shift=0.5):
    a = rng.standard_normal((max(2 * r, 4), r))
    return a.T @ a + cond_shift * np.eye(r)


def run_spec(gamma, g):
    dev = torch.device("cuda", 0)
    gam = torch.from_numpy(gamma).to(dev)
    gt = torch.from_numpy(np.ascontiguousarray(g)).to(dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    solver = cpals._Solver(dev, max(g.shape[0], 1), gamma.shape[0])
    cpals._solve_spec(solver, gam, gt, info)
    torch.cuda.synchronize()
    return gt.cpu().numpy(), int(info.item())


def run_ladder(gamma, g):
    dev = torch.device("cuda", 0)
    gam = torch.from_numpy(gamma).to(dev)
    gt = torch.from_numpy(np.ascontiguousarray(g)).to(dev)
    solver = cpals._Solver(dev, max(g.shape[0], 1), gamma.shape[0])
    x = solver(gam, gt)
    torch.cuda.synchronize()
    return x.cpu().numpy()


@pytest.mark.parametrize("path", ["kernel", "sweep", "cusolver"])
@pytest.mark.parametrize("r", [1, 5, 31, 32, 33, 64, 100, 256, 300, 512, 1000, 2000])
def test_spd_solve_matches_cho_solve(monkeypatch, path, r):
    if path == "kernel" and r > 512:
        pytest.skip("the one-CTA kernels stop at R = 512")
    monkeypatch.setenv("CPK_SOLVE", path)  # force the path (default: kernel for R <= 256, sweep above)
    rng = np.random.Generator(np.random.Philox(r))
    gamma = spd(r, rng)
    for rows in (1, 7, 33, 128, 1000) if r <= 512 else (1, 130, 1024):
        g = rng.standard_normal((rows, r))
        want = oracle._solve_normal(gamma, g)
        got, info = run_spec(gamma, g)
        assert info == 0
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= TOL, (path, r, rows, err)
        got2 = run_ladder(gamma, g)
        err2 = np.linalg.norm(got2 - want) / np.linalg.norm(want)
        assert err2 <= TOL, (path, r, rows, err2)


@pytest.mark.parametrize("r", [256, 512, 2000])
def test_paths_agree_on_a_cp_als_gamma(monkeypatch, r):
    # a Hadamard product of Grams, as the sweep builds it (cond ~1e4)
    rng = np.random.Generator(np.random.Philox(7))
    grams = [(lambda a: a.T @ a)(rng.random((128, r))) for _ in range(3)]
    gamma = grams[0] * grams[1] * grams[2]
    g = rng.random((128, r))
    want = oracle._solve_normal(gamma, g)
    scale = np.linalg.norm(want)
    monkeypatch.setenv("CPK_SOLVE", "cusolver")
    x_lib, info = run_spec(gamma, g)
    assert info == 0
    for path in ("kernel", "sweep") if r <= 512 else ("sweep",):
        monkeypatch.setenv("CPK_SOLVE", path)
        x, info = run_spec(gamma, g)
        assert info == 0
        assert np.linalg.norm(x - want) / scale <= TOL, path
        assert np.linalg.norm(x - x_lib) / scale <= TOL, path


@pytest.mark.parametrize("path", ["kernel", "sweep"])
@pytest.mark.parametrize("r,bad", [(1, 0), (40, 17), (256, 100), (256, 255), (500, 480), (2000, 1999), (700, 33)])
def test_not_positive_definite_flags_the_lapack_column(monkeypatch, path, r, bad):
    if path == "kernel" and r > 512:
        pytest.skip("the one-CTA kernels stop at R = 512")
    monkeypatch.setenv("CPK_SOLVE", path)
    gamma = np.eye(r) * 2.0
    gamma[bad, bad] = -1.0
    g = np.ones((5, r))
    _, info = run_spec(gamma, g)
    assert info == bad + 1  # potrf's 1-based column of the failed pivot
    # the ladder cannot fix a negative eigenvalue either: last rung = lstsq
    x = run_ladder(gamma, g)
    want = oracle._solve_normal(gamma, g)
    assert np.allclose(x, want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("r", [8, 300])
def test_nan_gamma_is_flagged(monkeypatch, r):
    monkeypatch.delenv("CPK_SOLVE", raising=False)
    gamma = np.eye(r)
    gamma[3, 3] = np.nan
    _, info = run_spec(gamma, np.ones((2, r)))
    assert info == 4


@pytest.mark.parametrize("r", [64, 320])
def test_singular_gamma_takes_a_regularized_rung(monkeypatch, r):
    # PSD Gamma with an exactly zero block (zero factor columns): rung 0 hits
    # a zero pivot, rung 1 (eps = 1e-12) succeeds; the blocks decouple, so
    # each is compared on its own scale
    monkeypatch.delenv("CPK_SOLVE", raising=False)
    rng = np.random.Generator(np.random.Philox(3))
    a = rng.standard_normal((2 * r, r))
    a[:, 20:] = 0.0
    gamma = a.T @ a
    g = rng.standard_normal((9, r))
    _, info = run_spec(gamma, g)
    assert info == 21
    x = run_ladder(gamma, g)
    want = oracle._solve_normal(gamma, g)
    for blk in (slice(0, 20), slice(20, r)):
        err = np.linalg.norm(x[:, blk] - want[:, blk]) / np.linalg.norm(want[:, blk])
        assert err <= TOL, (blk, err)


@pytest.mark.parametrize("path", ["kernel", "sweep"])
@pytest.mark.parametrize("cond", [1e6, 1e10])
def test_ill_conditioned_gamma_residual_matches_cusolver(monkeypatch, path, cond):
    """Near-collinear factors make Gamma ill-conditioned; the kernels' block
    inverses must not cost accuracy against cuSOLVER's substitutions: the
    residual ||X Gamma - G|| / ||G|| stays within a small factor of it (and of
    scipy's cho_solve)."""
    rng = np.random.Generator(np.random.Philox(int(np.log10(cond))))
    r = 256
    q, _ = np.linalg.qr(rng.standard_normal((r, r)))
    gamma = (q * np.logspace(0, -np.log10(cond), r)) @ q.T
    gamma = (gamma + gamma.T) / 2
    g = rng.standard_normal((64, r))

    def resid(x):
        return np.linalg.norm(x @ gamma - g) / np.linalg.norm(g)

    monkeypatch.setenv("CPK_SOLVE", path)
    xk, ik = run_spec(gamma, g)
    monkeypatch.setenv("CPK_SOLVE", "cusolver")
    xc, ic = run_spec(gamma, g)
    assert ik == 0 and ic == 0
    rs = resid(oracle._solve_normal(gamma, g))
    print(path, cond, "resid", resid(xk), resid(xc), rs)
    if path == "kernel":
        assert resid(xk) <= 10 * max(resid(xc), rs, 1e-15), (resid(xk), resid(xc), rs)
    else:
        # X = G Gamma^-1 through the explicit inverse: the residual grows
        # like cond * eps (not backward stable), the forward error -- what
        # parity with the reference's X measures -- stays cond-limited as for
        # every method (below)
        assert resid(xk) <= 100 * cond * 1e-16 + 10 * max(resid(xc), rs), (resid(xk), resid(xc), rs)
    want = oracle._solve_normal(gamma, g)
    # forward error is cond-limited for every method; the kernel's is no worse
    ek = np.linalg.norm(xk - want) / np.linalg.norm(want)
    ec = np.linalg.norm(xc - want) / np.linalg.norm(want)
    print(path, cond, "forward", ek, ec)
    assert ek <= 10 * max(ec, 1e-15), (ek, ec)
