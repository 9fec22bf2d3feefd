"""GPU parity of the sm_100a MTTKRP against the oracle and the reference goldens.

Bar: relative Frobenius error <= 1e-10 in float64 (north star, BASELINE.json);
observed ~1e-15.  Every case goes through the public drop-in API (run /
mttkrp), i.e. through the C ABI into the CUDA kernel.
"""

import numpy as np
import pytest
import torch

import paper_2510_14891_b200 as ck
from conftest import instances, rng_for
from oracle import gen, oracle
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, mttkrp_device

pytestmark = pytest.mark.gpu
TOL = 1e-10


def model_of(lam, factors):
    return ck.KruskalTensor(lam, factors)


def test_small_goldens_all_variants(golden):
    store = golden("small")
    worst = 0.0
    for key, dims, data, lam, factors, gs in instances(store):
        y = ck.DenseTensor(dims, data)
        m = model_of(lam, factors)
        for k in range(len(dims)):
            ns = data.size // dims[k]
            for plan in [
                MttkrpPlan(Variant.B200, k),
                MttkrpPlan(Variant.SLICE, k),
                MttkrpPlan(Variant.TILE, k, tile_volume=min(5, ns)),
                MttkrpPlan(Variant.TILE, k, tile_volume=ns),
                MttkrpPlan(Variant.ELEM, k),
                MttkrpPlan(Variant.REFERENCE, k),
            ]:
                out = ck.run(y, m, plan)
                assert isinstance(out.matrix, np.ndarray)
                assert out.matrix.shape == (dims[k], m.rank) and out.matrix.flags["C_CONTIGUOUS"]
                err = oracle.rel_err(out.matrix, gs[k])
                worst = max(worst, err)
                assert err <= TOL, (key, k, plan)
    assert worst < 1e-13


@pytest.mark.parametrize("rank_tile", [32, 64, 128])
def test_every_rank_tile_and_layout(rank_tile):
    # odd I_0 forces the 8-byte cp.async path; even I_0 the 16-byte path
    for dims in [(7, 9, 5), (8, 6, 10), (6, 5, 4, 3), (4, 3, 2, 5, 2), (33, 17)]:
        for rank in (1, 5, 33, 130):
            y = rng_for(sum(dims) + rank).random(int(np.prod(dims)))
            fs = [rng_for(rank + j).random((n, rank)) for j, n in enumerate(dims)]
            lam = rng_for(3).random(rank) + 0.5
            m = ck.KruskalTensor(lam, fs)
            t = ck.DenseTensor(dims, y)
            for k in range(len(dims)):
                ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
                for splits in (0, 1, 3):
                    got = ck.run(t, m, MttkrpPlan(Variant.B200, k, rank_tile=rank_tile, splits=splits)).matrix
                    assert oracle.rel_err(got, ref) <= TOL, (dims, rank, k, splits)


def test_order_one_and_two():
    y = rng_for(1).random(7)
    m = ck.KruskalTensor(np.array([2.0, 0.5]), [rng_for(2).random((7, 2))])
    got = ck.run(ck.DenseTensor((7,), y), m, MttkrpPlan(Variant.B200, 0)).matrix
    assert np.allclose(got, y[:, None] * np.array([2.0, 0.5])[None, :], rtol=0, atol=0)
    # matrix case, reference test_reference_matrix_case (test_mttkrp.py:40-48)
    r = rng_for(2)
    y2 = r.random((5, 7))
    a2 = r.random((7, 3))
    lam = r.random(3) + 0.5
    m = ck.KruskalTensor(lam, [r.random((5, 3)), a2])
    got = ck.mttkrp_reference(ck.DenseTensor.from_ndarray(y2), m, 0).matrix
    np.testing.assert_allclose(got, y2 @ (a2 * lam), rtol=1e-13)


def test_zero_tensor_and_stats():
    dims = (3, 4, 2)
    m = ck.KruskalTensor(np.ones(3), [rng_for(1).random((n, 3)) for n in dims])
    out = ck.mttkrp_reference(ck.DenseTensor.zeros(dims), m, 1)
    assert np.array_equal(out.matrix, np.zeros((4, 3)))
    assert out.stats.element_visits == 24 and out.stats.atomic_updates == 0
    assert out.stats.seconds > 0
    # TILE atomic-count accounting follows mttkrp.py:365-375 exactly
    dims = (5, 4, 6)
    y = ck.DenseTensor(dims, rng_for(17).random(120))
    m = ck.KruskalTensor(np.ones(7), [rng_for(18).random((n, 7)) for n in dims])
    for k, i_k in enumerate(dims):
        n_s = 120 // i_k
        for nt in (1, 5, 7, n_s):
            st = ck.run(y, m, MttkrpPlan(Variant.TILE, k, tile_volume=nt)).stats
            assert st.atomic_updates == i_k * (-(-n_s // nt)) * 7
            assert st.tile_volume == nt
        st = ck.run(y, m, MttkrpPlan(Variant.ELEM, k)).stats
        assert st.atomic_updates == 120 * 7


def test_bit_reproducible_and_inputs_untouched():
    dims = (40, 24, 30)
    y = rng_for(5).random(int(np.prod(dims)))
    fs = [rng_for(6 + j).random((n, 37)) for j, n in enumerate(dims)]
    before = [a.copy() for a in fs], y.copy()
    t = ck.DenseTensor(dims, y)
    m = ck.KruskalTensor(np.ones(37), fs)
    for k in range(3):
        a = ck.run(t, m, MttkrpPlan(Variant.B200, k)).matrix
        b = ck.run(t, m, MttkrpPlan(Variant.B200, k)).matrix
        assert np.array_equal(a, b)
    assert np.array_equal(y, before[1]) and all(np.array_equal(a, b) for a, b in zip(fs, before[0]))


def test_device_tensors_in_device_tensors_out():
    dims = (16, 12, 10)
    dev = torch.device("cuda")
    y = torch.rand(int(np.prod(dims)), dtype=torch.float64, device=dev)
    fs = [torch.rand((n, 24), dtype=torch.float64, device=dev) for n in dims]
    for k in range(3):
        g = ck.mttkrp(y, fs, k)
        assert isinstance(g, torch.Tensor) and g.is_cuda and g.shape == (dims[k], 24)
        ref = oracle.mttkrp_ref(y.cpu().numpy(), dims, k, [f.cpu().numpy() for f in fs])
        assert oracle.rel_err(g.cpu().numpy(), ref) <= TOL


def test_errors_match_reference_classes():
    dims = (4, 5, 6)
    y = ck.DenseTensor(dims, rng_for(31).random(120))
    m = ck.KruskalTensor(np.ones(2), [rng_for(32).random((n, 2)) for n in dims])
    with pytest.raises(ck.IndexRangeError):
        ck.run(y, m, MttkrpPlan(Variant.SLICE, 3))
    with pytest.raises(ck.ParameterError):
        ck.run(y, m, MttkrpPlan(Variant.SLICE, 0, unroll=0))
    with pytest.raises(ck.ParameterError):
        ck.run(y, m, MttkrpPlan(Variant.TILE, 0))
    with pytest.raises(ck.ParameterError):
        ck.run(y, m, MttkrpPlan(Variant.TILE, 0, tile_volume=31))
    with pytest.raises(ck.ParameterError):
        ck.mttkrp_elem(y, m, MttkrpPlan(Variant.SLICE, 0))
    with pytest.raises(ck.ShapeError):
        ck.run(ck.DenseTensor((4, 5), rng_for(1).random(20)), m, MttkrpPlan(Variant.SLICE, 0))


def _config(golden, name):
    g = golden(name)
    dims = tuple(int(x) for x in g["dims"])
    rank = int(g["rank"])
    y = gen.philox_tensor(dims, 0)
    fs = gen.bench_factors(dims, rank, 0)
    return g, dims, rank, y, fs


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_baseline_configs_full_output(golden, name):
    g, dims, rank, y, fs = _config(golden, name)
    t = ck.DenseTensor(dims, y)
    m = ck.KruskalTensor(np.ones(rank), fs, validate=False)
    for k in range(len(dims)):
        got = ck.run(t, m, MttkrpPlan(Variant.B200, k)).matrix
        err = oracle.rel_err(got, g[f"G{k}"])
        assert err <= TOL, (name, k, err)


def test_c2_rank_tile_sweep_parity(golden):
    g, dims, rank, y, fs = _config(golden, "c2")
    t = ck.DenseTensor(dims, y)
    m = ck.KruskalTensor(np.ones(rank), fs, validate=False)
    for rt in (16, 32, 64, 128):
        for k in range(3):
            got = ck.run(t, m, MttkrpPlan(Variant.B200, k, rank_tile=rt)).matrix
            assert oracle.rel_err(got, g[f"G{k}"]) <= TOL


def test_c4_row_sampled_parity():
    """config 4 (1024^3, R=2000) on device; rows checked against the serial
    oracle on single-slice sub-tensors."""
    dims, rank, seed = (1024, 1024, 1024), 2000, 0
    t = ck.DenseTensor.uniform(dims, seed=seed)
    fs = gen.bench_factors(dims, rank, 0)
    m = ck.KruskalTensor(np.ones(rank), fs, validate=False)
    inner = []
    for k in range(3):
        got = ck.run(t, m, MttkrpPlan(Variant.B200, k)).matrix.cpu().numpy()
        inner.append((got * fs[k]).sum(axis=0))  # the same vector for every mode
        # first/last rows, both sides of the 256-row tile boundaries, one inside
        for n in (0, 255, 256, 517, 767, 768, 1023):
            ys = gen.splitmix_slice(dims, k, n, seed)
            sub_dims = tuple(1 if j == k else e for j, e in enumerate(dims))
            sub_f = [a[n:n + 1] if j == k else a for j, a in enumerate(fs)]
            # the TILE restatement on the single-slice sub-tensor, all host cores
            ref = oracle.mttkrp_tile(ys, sub_dims, k, sub_f, f_cols=16, n_t=16384)[0][0]
            assert oracle.rel_err(got[n], ref) <= TOL, (k, n)
    assert oracle.rel_err(inner[1], inner[0]) <= 1e-12 and oracle.rel_err(inner[2], inner[0]) <= 1e-12


@pytest.mark.parametrize("engine", ["tma", "dmma"])
@pytest.mark.parametrize("rank_tile", [64, 128, 256])
@pytest.mark.parametrize("dims", [(40, 36, 34), (130, 66, 3), (34, 40, 70, 6), (6, 4, 8, 10, 4), (64, 2)])
def test_tma_engine_parity(dims, rank_tile, engine):
    """The warp-specialized TMA kernels (forced; DFMA and DMMA consumers) on
    ragged shapes: I_k not a multiple of the row tile, chunk tails, rank
    tails, d = 2..5, splits."""
    for rank in (2, 130, 300):
        y = rng_for(sum(dims) * rank).random(int(np.prod(dims)))
        fs = [rng_for(rank + 7 * j).random((n, rank)) for j, n in enumerate(dims)]
        lam = rng_for(11).random(rank) + 0.5
        m = ck.KruskalTensor(lam, fs)
        t = ck.DenseTensor(dims, y)
        for k in range(len(dims)):
            ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
            for splits in (0, 1, 5):
                plan = MttkrpPlan(Variant.B200, k, rank_tile=rank_tile, splits=splits, engine=engine)
                got = ck.run(t, m, plan).matrix
                assert oracle.rel_err(got, ref) <= TOL, (dims, rank, k, splits)


@pytest.mark.parametrize("rank_tile", [16, 32])
@pytest.mark.parametrize("dims", [(40, 36, 34), (300, 66, 3), (34, 40, 70, 6), (6, 4, 8, 10, 4), (64, 2)])
def test_narrow_dmma_tiles_parity(dims, rank_tile):
    """The 16- and 32-column DMMA tiles (low-rank end): ragged rows (I_k not a
    multiple of 256), rank tails inside a fragment, several rank tiles,
    d = 2..5, splits; mode 0 exercises the permuted M-major fragment rows."""
    for rank in (2, 10, 24, 40):
        y = rng_for(sum(dims) * rank + 1).random(int(np.prod(dims)))
        fs = [rng_for(rank + 5 * j).random((n, rank)) for j, n in enumerate(dims)]
        lam = rng_for(13).random(rank) + 0.5
        m = ck.KruskalTensor(lam, fs)
        t = ck.DenseTensor(dims, y)
        for k in range(len(dims)):
            ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
            for splits in (0, 1, 5):
                plan = MttkrpPlan(Variant.B200, k, rank_tile=rank_tile, splits=splits, engine="dmma")
                got = ck.run(t, m, plan).matrix
                assert oracle.rel_err(got, ref) <= TOL, (dims, rank, k, splits)


@pytest.mark.parametrize("engine", ["dmma", "tma", "cpasync", "cpdmma"])
@pytest.mark.parametrize("dims", [(300, 66, 34), (34, 40, 70, 6), (6, 4, 8, 10, 4)])
def test_split_chain_is_bit_identical_to_partial_copies(monkeypatch, dims, engine):
    """The split-K chain (CPK_SPLIT_CHAIN=1: splits accumulate into G in
    order, common.cuh) and the partial-copy merge (splitk_reduce_f64) add the
    same numbers in the same order: identical bits, and both at the oracle.
    sm_count = 1 makes the planner chain any split plan (tiles >= sm_count /
    2); the chain waits are then real (every split of a tile is resident at
    once)."""
    rank = 40
    y = rng_for(sum(dims) + 3).random(int(np.prod(dims)))
    fs = [rng_for(rank + 9 * j).random((n, rank)) for j, n in enumerate(dims)]
    lam = rng_for(17).random(rank) + 0.5
    m = ck.KruskalTensor(lam, fs)
    t = ck.DenseTensor(dims, y)
    rt = 64 if engine != "cpasync" else 32
    for k in range(len(dims)):
        ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
        for splits in (2, 7):
            kw = dict(rank_tile=rt, splits=splits, engine=engine)
            monkeypatch.setenv("CPK_SPLIT_CHAIN", "1")
            chained = ck.run(t, m, MttkrpPlan(Variant.B200, k, sm_count=1, **kw)).matrix
            monkeypatch.delenv("CPK_SPLIT_CHAIN")
            copies = ck.run(t, m, MttkrpPlan(Variant.B200, k, sm_count=1, **kw)).matrix
            assert np.array_equal(np.asarray(chained), np.asarray(copies)), (dims, k, splits)
            assert oracle.rel_err(chained, ref) <= TOL, (dims, k, splits)


def test_engines_agree_bitwise_on_c2_mode1(golden):
    """Both engines produce the golden to 1e-10; each is bit-reproducible."""
    g, dims, rank, y, fs = _config(golden, "c2")
    t = ck.DenseTensor(dims, y)
    m = ck.KruskalTensor(np.ones(rank), fs, validate=False)
    for engine in ("tma", "cpasync", "dmma"):
        plan = MttkrpPlan(Variant.B200, 1, rank_tile=128, block_k=32, engine=engine)
        a = ck.run(t, m, plan).matrix
        b = ck.run(t, m, plan).matrix
        assert np.array_equal(a, b)
        assert oracle.rel_err(a, g["G1"]) <= TOL


@pytest.mark.parametrize("dims", [(30, 20, 17), (8, 6, 10, 9), (64, 9), (40, 36, 34, 4)])
def test_streamed_host_tensor(monkeypatch, dims):
    """First MTTKRP of a host tensor streams it in slabs along the slowest
    mode (copy overlapped with the work items whose slices have landed);
    the result is bit-identical to the call on the resident tensor, matches
    the oracle, and later modes reuse the cached device copy."""
    import importlib

    mt = importlib.import_module("paper_2510_14891_b200.mttkrp")  # the module, not the re-exported function
    monkeypatch.setattr(mt, "STREAM_MIN_BYTES", 0)
    rank = 70
    y = rng_for(5).random(int(np.prod(dims)))
    fs = [rng_for(9 + j).random((n, rank)) for j, n in enumerate(dims)]
    lam = rng_for(3).random(rank) + 0.5
    m = ck.KruskalTensor(lam, fs)
    for k in range(len(dims)):
        for plan in (MttkrpPlan(Variant.B200, k), MttkrpPlan(Variant.SLICE, k),
                     MttkrpPlan(Variant.B200, k, engine="cpasync", rank_tile=32)):
            t = ck.DenseTensor(dims, y)  # fresh: nothing cached
            assert t.needs_upload()
            got = ck.run(t, m, plan).matrix
            assert not t.needs_upload()
            again = ck.run(t, m, plan).matrix  # resident copy, one launch
            assert np.array_equal(got, again), (dims, k, plan)
            assert oracle.rel_err(got, oracle.mttkrp_ref(y, dims, k, fs, lam)) <= TOL, (dims, k, plan.variant)
    pinned = torch.from_numpy(y).pin_memory()
    t = ck.DenseTensor(dims, pinned)
    got = ck.mttkrp(t, [torch.from_numpy(a).cuda() for a in fs], 0)
    assert got.is_cuda
    assert oracle.rel_err(got.cpu().numpy(), oracle.mttkrp_ref(y, dims, 0, fs, None)) <= TOL


@pytest.mark.parametrize("dims", [(34, 30, 29), (64, 9), (9, 64), (6, 5, 4, 11), (50,)])
def test_landed_pieces_are_bit_identical(dims):
    """cpk_mttkrp_f64_landed over arbitrary (even empty) landed ranges covers
    every work item exactly once: bit-identical to one cpk_mttkrp_f64."""
    from paper_2510_14891_b200.mttkrp import mttkrp_device

    rank = 66
    dev = torch.device("cuda", 0)
    y = torch.from_numpy(rng_for(1).random(int(np.prod(dims)))).to(dev)
    fs = [torch.from_numpy(rng_for(2 + j).random((n, rank))).to(dev) for j, n in enumerate(dims)]
    last = dims[-1]
    cuts = sorted({0, last, *rng_for(7).integers(0, last + 1, size=4).tolist()})
    cuts = [0] + cuts  # an empty first piece
    for k in range(len(dims)):
        for plan in (MttkrpPlan(Variant.B200, k), MttkrpPlan(Variant.B200, k, splits=7),
                     MttkrpPlan(Variant.B200, k, engine="cpasync")):
            ref, _, _ = mttkrp_device(y, dims, fs, k, None, plan)
            out = torch.full_like(ref, float("nan"))
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                mttkrp_device(y, dims, fs, k, None, plan, out=out, landed=(lo, hi))
            assert torch.equal(out, ref), (dims, k, plan)


@pytest.mark.parametrize("dims", [(12, 7, 9), (5, 6, 4, 7), (9, 13)])
def test_cublas_gemm_baseline_parity(dims):
    """The library comparison baseline (partial KRPs + cuBLAS DGEMM,
    mttkrp.py:230-276) is itself checked against the oracle."""
    from paper_2510_14891_b200.baselines import mttkrp_elem_atomic, mttkrp_gemm_cublas

    rank = 11
    y = rng_for(21).random(int(np.prod(dims)))
    fs = [rng_for(22 + j).random((n, rank)) for j, n in enumerate(dims)]
    lam = rng_for(23).random(rank) + 0.5
    yd = torch.from_numpy(y).cuda()
    fd = [torch.from_numpy(a).cuda() for a in fs]
    for k in range(len(dims)):
        ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
        got = mttkrp_gemm_cublas(yd, dims, fd, k, torch.from_numpy(lam).cuda()).cpu().numpy()
        assert oracle.rel_err(got, ref) <= TOL, (dims, k)
        got = mttkrp_elem_atomic(yd, dims, fd, k, torch.from_numpy(lam).cuda()).cpu().numpy()
        assert oracle.rel_err(got, ref) <= TOL, (dims, k, "elem")


@pytest.mark.parametrize("dims", [(41, 23, 3, 17), (300, 3, 40), (6, 50, 7, 2, 9), (17, 19, 2)])
def test_small_modes_merge_with_a_neighbour(dims):
    """Modes far smaller than the row tile run as the merged (d-1)-way
    problem plus a contraction; results match the oracle, weights folded
    once, for resident and streamed (landed) tensors."""
    from paper_2510_14891_b200.mttkrp import mttkrp_device

    rank = 33
    y = rng_for(31).random(int(np.prod(dims)))
    fs = [rng_for(32 + j).random((n, rank)) for j, n in enumerate(dims)]
    lam = rng_for(30).random(rank) + 0.5
    m = ck.KruskalTensor(lam, fs)
    dev = torch.device("cuda", 0)
    yd = torch.from_numpy(y).to(dev)
    fd = [torch.from_numpy(a).to(dev) for a in fs]
    lamd = torch.from_numpy(lam).to(dev)
    for k in range(len(dims)):
        ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
        got = ck.run(ck.DenseTensor(dims, y), m, MttkrpPlan(Variant.B200, k)).matrix
        assert oracle.rel_err(got, ref) <= TOL, (dims, k)
        whole, _, _ = mttkrp_device(yd, dims, fd, k, lamd)
        out = torch.full_like(whole, float("nan"))
        cuts = [0, 1, dims[-1] // 2, dims[-1]]
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            mttkrp_device(yd, dims, fd, k, lamd, out=out, landed=(lo, hi))
        assert torch.equal(out, whole), (dims, k)


@pytest.mark.parametrize("rank_tile", [64, 128])
@pytest.mark.parametrize("dims", [(41, 36, 34), (131, 66, 3), (33, 40, 70, 7), (7, 5, 8, 9, 3), (65, 3)])
def test_cpasync_dmma_engine_parity(dims, rank_tile):
    """cp.async + DMMA tiles (engine "cpdmma", the path for tensors TMA
    cannot describe, e.g. odd I_0): ragged shapes, rank tails, splits."""
    for rank in (2, 67, 300):
        y = rng_for(sum(dims) * rank + 1).random(int(np.prod(dims)))
        fs = [rng_for(rank + 11 * j).random((n, rank)) for j, n in enumerate(dims)]
        lam = rng_for(12).random(rank) + 0.5
        m = ck.KruskalTensor(lam, fs)
        t = ck.DenseTensor(dims, y)
        for k in range(len(dims)):
            ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
            for splits in (0, 1, 5):
                plan = MttkrpPlan(Variant.B200, k, rank_tile=rank_tile, splits=splits, engine="cpdmma")
                got = ck.run(t, m, plan).matrix
                assert oracle.rel_err(got, ref) <= TOL, (dims, rank, k, splits)


def test_modes_of_a_streaming_tensor_overlap_and_match(monkeypatch):
    """All modes issued back to back on a host tensor whose upload is still
    in flight run on the landed slabs (side streams, private workspaces) and
    are bit-identical to the same calls on a resident tensor."""
    import importlib

    mt = importlib.import_module("paper_2510_14891_b200.mttkrp")
    monkeypatch.setattr(mt, "STREAM_MIN_BYTES", 0)
    dims, rank = (64, 48, 40, 12), 96
    y = rng_for(41).random(int(np.prod(dims)))
    fs = [rng_for(42 + j).random((n, rank)) for j, n in enumerate(dims)]
    m = ck.KruskalTensor(np.ones(rank), fs, validate=False)
    pinned = torch.from_numpy(y).pin_memory()
    t = ck.DenseTensor(dims, pinned)
    streamed = [ck.run(t, m, MttkrpPlan(Variant.B200, k)).matrix for k in range(len(dims))]
    resident = ck.DenseTensor(dims, torch.from_numpy(y).cuda())
    for k in range(len(dims)):
        ref = ck.run(resident, m, MttkrpPlan(Variant.B200, k)).matrix
        assert torch.equal(streamed[k], ref), k
        assert oracle.rel_err(ref.cpu().numpy(), oracle.mttkrp_ref(y, dims, k, fs)) <= TOL


@pytest.mark.parametrize("dims", [(64, 48, 40, 12), (30, 20, 17)])
def test_mttkrp_modes_streams_all_modes_bit_identically(monkeypatch, dims):
    """ck.mttkrp_modes on a host tensor: slab-major issue of every mode's
    landed work; each result equals the resident single-mode call bitwise."""
    import importlib

    mt = importlib.import_module("paper_2510_14891_b200.mttkrp")
    monkeypatch.setattr(mt, "STREAM_MIN_BYTES", 0)
    rank = 70
    y = rng_for(51).random(int(np.prod(dims)))
    fs = [rng_for(52 + j).random((n, rank)) for j, n in enumerate(dims)]
    lam = rng_for(50).random(rank) + 0.5
    m = ck.KruskalTensor(lam, fs)
    for payload in (y, torch.from_numpy(y).pin_memory()):
        t = ck.DenseTensor(dims, payload)
        got = ck.mttkrp_modes(t, m)
        resident = ck.DenseTensor(dims, torch.from_numpy(y).cuda())
        for k, g in enumerate(got):
            ref = ck.run(resident, m, MttkrpPlan(Variant.B200, k)).matrix.cpu().numpy()
            g = g.cpu().numpy() if torch.is_tensor(g) else g
            assert np.array_equal(g, ref), (dims, k)
            assert oracle.rel_err(g, oracle.mttkrp_ref(y, dims, k, fs, lam)) <= TOL


@pytest.mark.parametrize("dims", [(41, 36, 34), (7, 5, 8, 9), (65, 3), (129, 20, 3)])
def test_odd_first_extent_runs_through_the_even_copy(dims):
    """Odd I_0 (no 16-byte TMA strides): auto plans run on a zero-padded
    copy with an even I_0 -- same G for every mode (first I_0 rows for
    mode 0), weights folded once."""
    rank = 45
    y = rng_for(61).random(int(np.prod(dims)))
    fs = [rng_for(62 + j).random((n, rank)) for j, n in enumerate(dims)]
    lam = rng_for(60).random(rank) + 0.5
    m = ck.KruskalTensor(lam, fs)
    t = ck.DenseTensor(dims, y)
    for k in range(len(dims)):
        got = ck.run(t, m, MttkrpPlan(Variant.B200, k)).matrix
        assert got.shape == (dims[k], rank)
        assert oracle.rel_err(got, oracle.mttkrp_ref(y, dims, k, fs, lam)) <= TOL, (dims, k)


def test_device_entry_normalizes_factor_layouts_and_checks_shapes():
    """mttkrp_device with column-major (transposed-view) or float32 factors
    and a float64 tensor: the factors are re-laid out, not misread; wrong
    shapes and CPU tensors raise the reference's classes."""
    from paper_2510_14891_b200.mttkrp import mttkrp_device

    dims, rank = (20, 18, 16), 24
    y = rng_for(71).random(int(np.prod(dims)))
    fs = [rng_for(72 + j).random((n, rank)) for j, n in enumerate(dims)]
    yd = torch.from_numpy(y).cuda()
    for k in range(3):
        ref = oracle.mttkrp_ref(y, dims, k, fs)
        col_major = [torch.from_numpy(np.asfortranarray(a)).cuda() for a in fs]  # stride(1) != 1
        assert col_major[0].stride(1) != 1
        g, _, _ = mttkrp_device(yd, dims, col_major, k)
        assert oracle.rel_err(g.cpu().numpy(), ref) <= TOL
        g32f, _, _ = mttkrp_device(yd, dims, [torch.from_numpy(a.astype(np.float32)).cuda() for a in fs], k)
        assert g32f.dtype == torch.float64
        ref32f = oracle.mttkrp_ref(y, dims, k, [a.astype(np.float32).astype(np.float64) for a in fs])
        assert oracle.rel_err(g32f.cpu().numpy(), ref32f) <= TOL
    with pytest.raises(ck.ShapeError):
        mttkrp_device(yd, dims, [torch.from_numpy(a).cuda() for a in fs[:2]], 0)
    with pytest.raises(ck.ShapeError):
        mttkrp_device(yd, (20, 18, 15), [torch.from_numpy(a).cuda() for a in fs], 0)
    with pytest.raises(ck.DeviceError):
        mttkrp_device(torch.from_numpy(y), dims, [torch.from_numpy(a) for a in fs], 0)


def test_c5_full_size_row_sampled_parity():
    """BASELINE config 5 at full size on one GPU (4096 x 2048 x 2048 float64,
    137 GB, R = 512; int64 indexing well past 2^31 elements): rows of every
    mode's G against the oracle's TILE restatement on single-slice
    sub-tensors."""
    dims, rank, seed = (4096, 2048, 2048), 512, 0
    free = torch.cuda.mem_get_info()[0]
    if free < 8 * int(np.prod(dims)) + (8 << 30):
        pytest.skip(f"needs ~146 GB of free device memory, has {free / 1e9:.0f} GB")
    t = ck.DenseTensor.uniform(dims, seed=seed)
    fs = gen.bench_factors(dims, rank, 0)
    m = ck.KruskalTensor(np.ones(rank), fs, validate=False)
    inner = []
    try:
        for k in range(3):
            got = ck.run(t, m, MttkrpPlan(Variant.B200, k)).matrix.cpu().numpy()
            # size-independent identity: sum_n G_k[n, :] * A_k[n, :] = <Y, a_0j o a_1j o a_2j>
            # is the same vector for every mode k
            inner.append((got * fs[k]).sum(axis=0))
            for n in (0, 255, 256, dims[k] - 1):
                ys = gen.splitmix_slice(dims, k, n, seed)
                sub_dims = tuple(1 if j == k else e for j, e in enumerate(dims))
                sub_f = [a[n:n + 1] if j == k else a for j, a in enumerate(fs)]
                ref = oracle.mttkrp_tile(ys, sub_dims, k, sub_f, f_cols=16, n_t=65536)[0][0]
                assert oracle.rel_err(got[n], ref) <= TOL, (k, n)
        for k in (1, 2):
            assert oracle.rel_err(inner[k], inner[0]) <= 1e-12, k
    finally:
        del t
        torch.cuda.empty_cache()


def test_mttkrp_accepts_weights_factors_pair():
    """ck.mttkrp(tensor, (weights, factors), mode) == the KruskalTensor form."""
    dims, rank = (12, 10, 8), 9
    y = rng_for(81).random(int(np.prod(dims)))
    fs = [rng_for(82 + j).random((n, rank)) for j, n in enumerate(dims)]
    lam = rng_for(80).random(rank) + 0.5
    t = ck.DenseTensor(dims, y)
    for k in range(3):
        a = ck.mttkrp(t, (lam, fs), k)
        b = ck.mttkrp(t, ck.KruskalTensor(lam, fs), k)
        assert np.array_equal(a, b)
        assert oracle.rel_err(a, oracle.mttkrp_ref(y, dims, k, fs, lam)) <= TOL


def test_random_shapes_every_mode_fuzz():
    """Seeded fuzz over orders 2-5, extents 1-40 (odd and even), ranks 1-70
    and weights: every mode through the auto plan (TMA + DMMA with o-group
    TMEM accumulation, Khatri-Rao merges for d >= 4, small-mode merges, the
    cp.async kernels for odd shapes) against the oracle's serial kernel."""
    rng = np.random.Generator(np.random.Philox(2024))
    worst = 0.0
    for case in range(40):
        d = int(rng.integers(2, 6))
        dims = tuple(int(x) for x in rng.integers(1, 41 if d <= 3 else 13, size=d))
        r = int(rng.integers(1, 71))
        data = rng.random(int(np.prod(dims)))
        fs = [rng.random((n, r)) for n in dims]
        lam = rng.random(r) + 0.5
        y, m = ck.DenseTensor(dims, data), ck.KruskalTensor(lam, fs)
        for k in range(d):
            got = ck.run(y, m, MttkrpPlan(Variant.B200, k)).matrix
            err = oracle.rel_err(got, oracle.mttkrp_ref(data, dims, k, fs, lam))
            worst = max(worst, err)
            assert err <= TOL, (case, dims, r, k, err)
    assert worst < 1e-13


def test_device_caches_follow_the_payloads():
    """Reassigning or mutating factors / the tensor payload after a first GPU
    call is seen by the next call (the reference objects hold no cache)."""
    dims, r = (12, 10, 8), 5
    rng = np.random.Generator(np.random.Philox(21))
    y = rng.random(int(np.prod(dims)))
    fs = [rng.random((n, r)) for n in dims]
    t = ck.DenseTensor(dims, y.copy())
    m = ck.KruskalTensor(np.ones(r), [f.copy() for f in fs])
    ck.run(t, m, MttkrpPlan(Variant.B200, 0))
    # numpy factor: reassigned, then written in place
    m.factors[1] = fs[1] * 2.0
    got = ck.run(t, m, MttkrpPlan(Variant.B200, 0)).matrix
    assert oracle.rel_err(got, oracle.mttkrp_ref(y, dims, 0, [fs[0], fs[1] * 2.0, fs[2]])) <= 1e-12
    m.factors[2][:] = 0.5
    got = ck.run(t, m, MttkrpPlan(Variant.B200, 0)).matrix
    assert oracle.rel_err(got, oracle.mttkrp_ref(y, dims, 0, [fs[0], fs[1] * 2.0, np.full_like(fs[2], 0.5)])) <= 1e-12
    # torch factors: an in-place write bumps the version counter
    tf = [torch.from_numpy(f.copy()) for f in fs]
    mt_ = ck.KruskalTensor(np.ones(r), tf)
    ck.run(t, mt_, MttkrpPlan(Variant.B200, 1))
    mt_.factors[0].mul_(3.0)
    got = ck.run(t, mt_, MttkrpPlan(Variant.B200, 1)).matrix
    assert oracle.rel_err(got, oracle.mttkrp_ref(y, dims, 1, [fs[0] * 3.0, fs[1], fs[2]])) <= 1e-12
    # tensor payload reassigned (host) and mutated in place (torch host payload)
    t.data = y * 2.0
    got = ck.run(t, m, MttkrpPlan(Variant.B200, 2)).matrix
    ref_f = [fs[0], fs[1] * 2.0, np.full_like(fs[2], 0.5)]
    assert oracle.rel_err(got, oracle.mttkrp_ref(y * 2.0, dims, 2, ref_f)) <= 1e-12
    th = ck.DenseTensor(dims, torch.from_numpy(y.copy()))
    ck.run(th, m, MttkrpPlan(Variant.B200, 2))
    th.data.mul_(-1.0)
    got = ck.run(th, m, MttkrpPlan(Variant.B200, 2)).matrix.cpu().numpy()
    assert oracle.rel_err(got, oracle.mttkrp_ref(-y, dims, 2, ref_f)) <= 1e-12


def test_workspaces_are_per_stream():
    """Concurrent MTTKRPs on two streams do not share split-K scratch: both
    results are bit-identical to the serial ones."""
    from paper_2510_14891_b200._device import workspace

    dev = torch.device("cuda", 0)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    with torch.cuda.stream(s1):
        a = workspace(dev, 1 << 20)
    with torch.cuda.stream(s2):
        b = workspace(dev, 1 << 20)
    assert a.data_ptr() != b.data_ptr()
    dims, r = (64, 48, 40), 24
    y = ck.DenseTensor.uniform(dims, seed=3, device=dev)
    fs = [torch.rand((n, r), dtype=torch.float64, device=dev) for n in dims]
    plan = MttkrpPlan(Variant.B200, 1, splits=4)
    ref = [mttkrp_device(y.data, dims, fs, 1, None, plan)[0].clone() for _ in range(2)]
    torch.cuda.synchronize()
    outs = []
    for s in (s1, s2):
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            outs.append(mttkrp_device(y.data, dims, fs, 1, None, plan)[0])
    torch.cuda.synchronize()
    assert torch.equal(outs[0], ref[0]) and torch.equal(outs[1], ref[1])


def test_gemm_and_full_krp_names_keep_reference_budgets():
    """mttkrp_gemm / mttkrp_full_krp (mttkrp.py:173-276): same names, checks,
    ResourceError budgets and stats accounting as the reference; the product
    is the matrix-free kernel's (<= 1e-10 vs the oracle)."""
    dims, r = (14, 9, 11, 6), 7
    rng = np.random.Generator(np.random.Philox(8))
    y = rng.random(int(np.prod(dims)))
    fs = [rng.random((n, r)) for n in dims]
    lam = rng.random(r) + 0.5
    t, m = ck.DenseTensor(dims, y), ck.KruskalTensor(lam, fs)
    for k in range(4):
        ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
        g = ck.mttkrp_gemm(t, m, k)
        assert oracle.rel_err(g.matrix, ref) <= TOL and g.stats.variant == Variant.GEMM
        n_s = t.size // dims[k]
        i_l, i_r = int(np.prod(dims[:k])), int(np.prod(dims[k + 1:]))
        want = 8 * r * i_r if k == 0 else 8 * r * i_l if k == 3 else 8 * (r * (i_l + i_r) + i_l * dims[k] * r)
        assert g.stats.scratch_bytes == want
        f = ck.run(t, m, MttkrpPlan(Variant.FULL_KRP, k))
        assert oracle.rel_err(f.matrix, ref) <= TOL
        assert f.stats.scratch_bytes == 8 * n_s * r + (0 if k == 0 else 8 * t.size)
    with pytest.raises(ck.ResourceError, match="explicit KRP needs"):
        ck.run(t, m, MttkrpPlan(Variant.FULL_KRP, 0), budget_bytes=100)
    with pytest.raises(ck.ResourceError, match="scratch bytes, cap is"):
        ck.mttkrp_gemm(t, m, 1, scratch_cap_bytes=10)
    with pytest.raises(ck.ParameterError):
        ck.mttkrp_gemm(ck.DenseTensor((5,), np.ones(5)), ck.KruskalTensor(np.ones(2), [np.ones((5, 2))]), 0)


def test_tall_mode_beyond_the_grid_y_limit():
    """A mode with more row blocks than gridDim.y allows (65535 x 256 rows):
    the launch is cut into several along the rows (both kernel families)."""
    dims, rank = (16_800_002, 2), 4
    y = rng_for(77).random(int(np.prod(dims)))
    fs = [rng_for(78 + j).random((n, rank)) for j, n in enumerate(dims)]
    m = ck.KruskalTensor(np.ones(rank), fs, validate=False)
    t = ck.DenseTensor(dims, y)
    ref = oracle.mttkrp_ref(y, dims, 0, fs, None)
    for engine in ("auto", "cpasync"):
        got = ck.run(t, m, MttkrpPlan(Variant.B200, 0, engine=engine, rank_tile=0 if engine == "auto" else 32)).matrix
        assert oracle.rel_err(got, ref) <= TOL, engine


@pytest.mark.parametrize("dims", [(4, 3, 5, 2, 3, 4), (6, 2, 4, 2, 3, 2, 3), (2, 3, 2, 2, 3, 2, 2, 3),
                                  (5, 4, 3, 6, 2, 3), (2, 2, 3, 2, 2, 2, 3, 2, 2, 2, 2, 2)])
def test_orders_six_to_twelve_merge_o_modes(dims):
    """Orders the kernels cannot take directly (more than three o-modes):
    pairs of adjacent o-modes are merged into materialized Khatri-Rao
    factors until three remain (choose_order_merge), for every mode, with
    explicit reference-style plans too."""
    for rank in (5, 33):
        y = rng_for(sum(dims) + rank).random(int(np.prod(dims)))
        fs = [rng_for(rank + 3 * j).random((n, rank)) for j, n in enumerate(dims)]
        lam = rng_for(19).random(rank) + 0.5
        m = ck.KruskalTensor(lam, fs)
        t = ck.DenseTensor(dims, y)
        for k in range(len(dims)):
            ref = oracle.mttkrp_ref(y, dims, k, fs, lam)
            for plan in (MttkrpPlan(Variant.B200, k), MttkrpPlan(Variant.TILE, k, tile_volume=64)):
                got = ck.run(t, m, plan).matrix
                assert oracle.rel_err(got, ref) <= TOL, (dims, rank, k, plan.variant)


@pytest.mark.parametrize("dims", [(32, 20, 24, 6), (16, 40, 12, 10, 4), (48, 30, 20, 8)])
def test_khatri_rao_fold_for_a_middle_mode(dims):
    """Mode 1 of a d >= 4 tensor (k between the fastest non-k mode and the
    first o-mode): the automatic plan folds KR(A_0, A_2) into the factor
    rows (CPK_MERGE_KR_FOLD) -- against the oracle, against the unfolded
    plan, with weights, and round-tripped through the resolved plan."""
    for rank in (6, 40, 130):
        y = rng_for(sum(dims) * rank).random(int(np.prod(dims)))
        fs = [rng_for(rank + 11 * j).random((n, rank)) for j, n in enumerate(dims)]
        lam = rng_for(23).random(rank) + 0.5
        m = ck.KruskalTensor(lam, fs)
        t = ck.DenseTensor(dims, y)
        ref = oracle.mttkrp_ref(y, dims, 1, fs, lam)
        folded = ck.run(t, m, MttkrpPlan(Variant.B200, 1)).matrix
        plain = ck.run(t, m, MttkrpPlan(Variant.B200, 1, engine="dmma", rank_tile=64)).matrix
        assert oracle.rel_err(folded, ref) <= TOL, (dims, rank)
        assert oracle.rel_err(plain, ref) <= TOL, (dims, rank)
