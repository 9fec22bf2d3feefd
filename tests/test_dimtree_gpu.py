"""Dimension-tree CP-ALS on the device (als_sweep.tree_split,
cpk_dimtree_contract_f64): the in-group contraction against numpy, whole
sweeps against the oracle's per-mode cp_als (cpals.py:92-171) and against
the device's per-mode sweep."""

import numpy as np
import pytest
import torch

import paper_2510_14891_b200 as ck
from conftest import rng_for
from oracle import gen, oracle
from paper_2510_14891_b200 import _lib

pytestmark = pytest.mark.gpu


def _contract_np(w, ext, j, fs):
    g, r = len(ext), w.shape[1]
    t = w.reshape(tuple(reversed(ext)) + (r,))
    for l in range(g):
        if l != j:
            shape = [1] * g + [r]
            shape[g - 1 - l] = ext[l]
            t = t * fs[l].reshape(shape)
    return t.sum(axis=tuple(g - 1 - l for l in range(g) if l != j))


@pytest.mark.parametrize("ext,rank", [((7, 9), 5), ((40, 3), 33), ((3, 50), 70), ((5, 4, 6), 17),
                                      ((3, 2, 4, 5), 64), ((128, 128), 256), ((300, 70), 96), ((2, 500), 2)])
def test_contract_matches_numpy(ext, rank):
    """Every group mode j, ragged rank chunks, padded leading dimensions."""
    rng = rng_for(sum(ext) + rank)
    lib = _lib.load()
    rows = int(np.prod(ext))
    # odd leading dimensions (scalar lanes), and even ones (two columns per lane)
    for ldw, lda, ldo in ((rank + 3, rank + 1, rank + 5), (rank, rank, rank), (rank + 2, rank + 4, rank + 1)):
        _check_contract(lib, rng, ext, rank, rows, ldw, lda, ldo)


def _check_contract(lib, rng, ext, rank, rows, ldw, lda, ldo):
    w = torch.from_numpy(rng.random((rows, ldw))).cuda()
    fs = [torch.from_numpy(rng.random((n, lda))).cuda() for n in ext]
    for j in range(len(ext)):
        out = torch.full((ext[j], ldo), -7.0, dtype=torch.float64, device="cuda")
        ptrs = _lib.ptr_array([f.data_ptr() if l != j else 0 for l, f in enumerate(fs)])
        rc = lib.cpk_dimtree_contract_f64(w.data_ptr(), ldw, len(ext), _lib.i64_array(ext), j, ptrs,
                                          _lib.i64_array([lda] * len(ext)), rank, out.data_ptr(), ldo, None)
        assert rc == 0, _lib.load().cpk_last_error()
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        ref = _contract_np(w.cpu().numpy()[:, :rank], ext, j, [f.cpu().numpy()[:, :rank] for f in fs])
        assert oracle.rel_err(got[:, :rank], ref) <= 1e-13, j
        assert np.all(got[:, rank:] == -7.0)  # padding columns untouched


def test_contract_rejects_bad_arguments():
    # 3 = CPK_ERR_PARAM, 1 = CPK_ERR_SHAPE (include/cpk_b200.h)
    lib = _lib.load()
    ext = _lib.i64_array([4, 4])
    ptrs = _lib.ptr_array([0, 0])
    lds = _lib.i64_array([4, 4])
    buf = torch.zeros(64, dtype=torch.float64, device="cuda")
    p = buf.data_ptr()
    assert lib.cpk_dimtree_contract_f64(p, 4, 1, ext, 0, ptrs, lds, 4, p, 4, None) == 3
    assert lib.cpk_dimtree_contract_f64(p, 4, 2, ext, 2, ptrs, lds, 4, p, 4, None) == 3
    assert lib.cpk_dimtree_contract_f64(p, 4, 2, ext, 0, ptrs, lds, 4, p, 4, None) == 3  # NULL A_1
    assert lib.cpk_dimtree_contract_f64(p, 3, 2, ext, 0, _lib.ptr_array([0, p]), lds, 4, p, 4, None) \
        == 1
    assert lib.cpk_dimtree_contract_f64(None, 4, 2, ext, 0, ptrs, lds, 4, p, 4, None) == 3


@pytest.mark.parametrize("dims,rank", [((40, 36, 34), 24), ((41, 30, 28), 17), ((20, 12, 16, 10), 33),
                                       ((9, 8, 7), 4), ((12, 6, 8, 5, 6), 16), ((5, 4, 3, 6, 2, 3), 4),
                                       ((64, 48, 40), 130)])
def test_tree_sweeps_follow_the_oracle(dims, rank):
    """Forced tree (3- to 6-way, odd I_0 on the padded copy, rank tails):
    fits and weights at the oracle's per-mode trajectory."""
    y = rng_for(sum(dims) + rank).random(int(np.prod(dims)))
    model, tr = ck.cp_als(ck.DenseTensor(dims, y), ck.AlsConfig(rank=rank, tol=0.0, max_iters=4, seed=2,
                                                                dimtree=True))
    assert tr.tree_split is not None
    ref_lam, ref_f, ref_fits = oracle.cp_als(y, dims, rank, max_iters=4, tol=0.0, seed=2)
    assert np.max(np.abs(np.asarray(tr.fits) - np.asarray(ref_fits))) <= 1e-8
    assert oracle.rel_err(model.weights.cpu().numpy(), ref_lam) <= 1e-6
    assert [tuple(a.shape) for a in model.factors] == [(n, rank) for n in dims]


def test_tree_and_per_mode_sweeps_agree():
    """Same run with and without the tree: the sums differ in order only."""
    dims, rank = (48, 40, 36, 20), 24
    y = ck.DenseTensor(dims, rng_for(7).random(int(np.prod(dims))))
    m_t, t_t = ck.cp_als(y, ck.AlsConfig(rank=rank, tol=0.0, max_iters=6, seed=1, dimtree=True))
    m_p, t_p = ck.cp_als(y, ck.AlsConfig(rank=rank, tol=0.0, max_iters=6, seed=1, dimtree=False))
    assert t_t.tree_split == 2 and t_p.tree_split is None
    assert np.max(np.abs(np.asarray(t_t.fits) - np.asarray(t_p.fits))) <= 1e-12
    for a, b in zip(m_t.factors, m_p.factors):
        assert oracle.rel_err(a.cpu().numpy(), b.cpu().numpy()) <= 1e-10


def test_tree_graph_replay_matches_eager_bitwise():
    dims, rank = (30, 20, 24, 10), 12
    y = ck.DenseTensor(dims, rng_for(3).random(int(np.prod(dims))))
    cfg = ck.AlsConfig(rank=rank, tol=0.0, max_iters=6, seed=3, dimtree=True)
    m_g, t_g = ck.cp_als(y, cfg, graph=True)
    m_e, t_e = ck.cp_als(y, cfg, graph=False)
    assert t_g.fits == t_e.fits
    for a, b in zip(m_g.factors, m_e.factors):
        assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())


def test_c3_tree_sweeps_match_reference(golden):
    """BASELINE config 3 (128^4, R = 256, 10 sweeps): the automatic plan runs
    the tree (split 2: two tensor passes per sweep instead of four) and stays
    on the reference's trajectory."""
    als = golden("als")
    dims = (128, 128, 128, 128)
    y = ck.DenseTensor(dims, gen.philox_tensor(dims, 0))
    model, tr = ck.cp_als(y, ck.AlsConfig(rank=256, tol=0.0, max_iters=10, seed=0))
    assert tr.tree_split == 2
    assert np.max(np.abs(np.asarray(tr.fits) - als["c3/fits"])) <= 1e-12
    assert oracle.rel_err(model.weights.cpu().numpy(), als["c3/lam"]) <= 1e-10


@pytest.mark.parametrize("dims,rank,modes", [((40, 36, 34), 24, None), ((20, 12, 16, 10), 33, None),
                                             ((12, 6, 8, 5, 6), 16, (4, 0, 2, 1)), ((41, 30, 28), 17, (2, 0, 1)),
                                             ((20, 12, 16, 10), 8, (0, 1, 3))])
def test_mttkrp_modes_tree_matches_per_mode(dims, rank, modes):
    """mttkrp_modes(tree=True): every requested mode (any order, subsets,
    weights, host or device input) at the per-mode result and the oracle."""
    rng = rng_for(sum(dims) + rank)
    y = rng.random(int(np.prod(dims)))
    fs = [rng.random((n, rank)) for n in dims]
    lam = rng.random(rank) + 0.5
    ks = list(range(len(dims))) if modes is None else list(modes)
    got = ck.mttkrp_modes(ck.DenseTensor(dims, y), ck.KruskalTensor(lam, fs), modes, tree=True)
    assert all(isinstance(g, np.ndarray) for g in got)  # host in, host out
    for k, g in zip(ks, got):
        assert oracle.rel_err(g, oracle.mttkrp_ref(y, dims, k, fs, lam)) <= 1e-12, k
    yd = torch.from_numpy(y).cuda()
    fd = [torch.from_numpy(a).cuda() for a in fs]
    got_d = ck.mttkrp_modes(yd, fd, modes, tree=True)
    per = ck.mttkrp_modes(yd, fd, modes)
    for a, b in zip(got_d, per):
        assert a.is_cuda and oracle.rel_err(a.cpu().numpy(), b.cpu().numpy()) <= 1e-13


def test_tree_rollback_on_singular_gamma_matches_per_mode():
    """Rank above the extents (every Gamma_k of a 2x2x2 tensor at R = 5 has
    rank <= 4): the speculative Cholesky fails inside tree sweeps (eager and
    replayed), the sweep is rolled back and rerun through the ladder; the
    trajectory follows the per-mode run's."""
    from paper_2510_14891_b200 import als_sweep

    dims, r = (2, 2, 2), 5
    y = torch.from_numpy(rng_for(17).random(8)).cuda()
    plan = ck.MttkrpPlan(ck.Variant.B200, 0)
    ref = als_sweep.run_sweeps(als_sweep.DeviceBackend(y, dims, r, plan), dims, r, 1, 8, 0.0, y, graph=False,
                               tree=False)
    assert ref.rollbacks > 0
    for graph in (False, True):
        res = als_sweep.run_sweeps(als_sweep.DeviceBackend(y, dims, r, plan), dims, r, 1, 8, 0.0, y, graph=graph,
                                   tree=True)
        assert res.tree_split is not None and res.rollbacks > 0
        assert np.all(np.isfinite(res.fits))
        # an exact fit (residual ~0): fit = 1 - sqrt(resid)/||Y|| turns the
        # 1e-16 summation-order difference into ~1e-8, hence 1e-6 here
        assert np.max(np.abs(np.asarray(res.fits) - np.asarray(ref.fits))) <= 1e-6
