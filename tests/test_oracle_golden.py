"""Pin the CPU oracle (oracle/) against golden outputs of the reference itself.

The goldens in tests/golden were produced by the reference package
(tests/golden/make_golden.py).  The C restatement of ref_kernel must match
them BIT FOR BIT (same evaluation order, no FMA contraction, as numba's
default), the TILE restatement and the numpy GEMM restatement to 1e-12.
"""

import numpy as np
import pytest

from conftest import instances
from oracle import gen, oracle


def test_ref_restatement_is_bit_exact_on_small_goldens(golden):
    store = golden("small")
    n = 0
    for key, dims, data, lam, factors, gs in instances(store):
        for k in range(len(dims)):
            got = oracle.mttkrp_ref(data, dims, k, factors, lam)
            assert np.array_equal(got, gs[k]), (key, k)
            n += 1
    assert n > 150


@pytest.mark.parametrize("workers", [1, 3])
def test_tile_restatement_matches_goldens(golden, workers):
    store = golden("small")
    for key, dims, data, lam, factors, gs in instances(store):
        for k in range(len(dims)):
            ns = data.size // dims[k]
            for nt in (1, min(5, ns), ns):
                got, _ = oracle.mttkrp_tile(data, dims, k, factors, lam, f_cols=4, n_t=nt, workers=workers)
                assert oracle.rel_err(got, gs[k]) <= 1e-12, (key, k, nt)
                if workers == 1 and nt == ns:
                    # one worker, one tile per slice = the canonical order
                    # except for the column-block split of the products
                    assert oracle.rel_err(got, gs[k]) <= 1e-15


def test_rows_restatement_is_bit_exact(golden):
    store = golden("small")
    for key, dims, data, lam, factors, gs in instances(store)[:20]:
        for k in range(len(dims)):
            rows = np.arange(dims[k])[::-1].copy()
            got = oracle.mttkrp_rows(data, dims, k, factors, rows, lam)
            assert np.array_equal(got, gs[k][rows]), (key, k)


def test_gemm_restatement_matches_goldens(golden):
    store = golden("small")
    for key, dims, data, lam, factors, gs in instances(store):
        if len(dims) < 2:
            continue
        for k in range(len(dims)):
            got = oracle.mttkrp_gemm(data, dims, k, factors, lam)
            assert oracle.rel_err(got, gs[k]) <= 1e-12, (key, k)


def test_c1_golden_and_cli_recipe(golden):
    c1 = golden("c1")
    dims = tuple(int(x) for x in c1["dims"])
    rank = int(c1["rank"])
    y = gen.philox_tensor(dims, 0)
    fs = gen.bench_factors(dims, rank, 0)
    for k in range(3):
        got = oracle.mttkrp_ref(y, dims, k, fs)
        assert np.array_equal(got, c1[f"G{k}"])


@pytest.mark.slow
def test_c2_sampled_rows_pin_gemm_golden(golden):
    c2 = golden("c2")
    dims = tuple(int(x) for x in c2["dims"])
    rank = int(c2["rank"])
    y = gen.philox_tensor(dims, 0)
    fs = gen.bench_factors(dims, rank, 0)
    for k in range(3):
        rows = c2[f"rows{k}"]
        # the reference's own serial kernel on single-slice sub-tensors ...
        assert np.array_equal(oracle.mttkrp_rows(y, dims, k, fs, rows), c2[f"Grows{k}"])
        # ... agrees with the GEMM golden at those rows
        assert oracle.rel_err(c2[f"G{k}"][rows], c2[f"Grows{k}"]) <= 1e-12


def test_cp_als_restatement_matches_reference_trajectories(golden):
    als = golden("als")
    for key in sorted({k.split("/")[0] for k in als if k.startswith("planted")}):
        dims = tuple(int(x) for x in als[f"{key}/dims"])
        rank = int(key.split("_r")[1])
        ref = als[f"{key}/fits_reference"]
        lam, _, fits = oracle.cp_als(als[f"{key}/data"], dims, rank, max_iters=len(ref), tol=0.0, seed=0)
        assert len(fits) == len(ref)
        assert np.max(np.abs(np.asarray(fits) - ref)) <= 1e-8, key
    lam, factors, fits = oracle.cp_als(als["rand765/data"], (7, 6, 5), 3, max_iters=20, tol=0.0, seed=2)
    assert np.max(np.abs(np.asarray(fits) - als["rand765/fits"])) <= 1e-12
    assert oracle.rel_err(lam, als["rand765/lam"]) <= 1e-10


def test_splitmix_twin_slices():
    dims = (3, 4, 5, 2)
    full = gen.splitmix_uniform(120, seed=7).reshape(dims, order="F")
    assert np.all((full >= 0) & (full < 1))
    for k in range(4):
        for n in range(dims[k]):
            s = gen.splitmix_slice(dims, k, n, seed=7)
            assert np.array_equal(s, np.take(full, n, axis=k).ravel(order="F"))
    # offset windows compose
    a = gen.splitmix_uniform(50, seed=1, offset=0)
    b = gen.splitmix_uniform(20, seed=1, offset=30)
    assert np.array_equal(a[30:], b)


def test_oracle_single_mode_update_matches_reference(golden):
    """SURVEY 8(c) plan (i): the oracle's Gram / Gamma / _solve_normal /
    normalization (cpals.py:122-140) reproduce the reference's single mode
    update (tests/golden/step.npz) -- the MTTKRP too at the rank-512 case."""
    st = golden("step")
    for name in ("c3", "r512"):
        dims = tuple(int(x) for x in st[f"{name}/dims"])
        rank = st[f"{name}/A{[k for k in range(len(dims)) if f'{name}/A{k}' in st][0]}"].shape[1]
        rng = np.random.Generator(np.random.Philox(0))
        factors = [rng.random((i, rank)) for i in dims]
        grams = [oracle.gram(a) for a in factors]
        y = np.random.Generator(np.random.Philox(0)).random(int(np.prod(dims))) if name == "r512" else None
        for k in range(len(dims)):
            if f"{name}/A{k}" not in st:
                continue
            g = st[f"{name}/G{k}"]
            if y is not None:
                assert oracle.rel_err(oracle.mttkrp_gemm(y, dims, k, factors), g) <= 1e-13
            gamma = np.ones((rank, rank))
            for m in range(len(dims)):
                if m != k:
                    gamma *= grams[m]
            a = oracle._solve_normal(gamma, g.copy())
            nrm = np.linalg.norm(a, axis=0)
            a[:, nrm > 0] /= nrm[nrm > 0]
            assert oracle.rel_err(a, st[f"{name}/A{k}"]) <= 1e-13
            assert oracle.rel_err(np.where(nrm > 0, nrm, 0.0), st[f"{name}/lam{k}"]) <= 1e-13
