"""C ABI: the library loads, exports every symbol of include/cpk_b200.h, and
its host-side planning / validation logic behaves (no GPU needed)."""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2510_14891_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "cpk_b200.h").read_text()
    return sorted(set(re.findall(r"\b(cpk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    # the Python binding declares a prototype for each of them
    assert sorted(_lib.exported_symbols()) == syms


def test_library_is_sm100a(tmp_path):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_version_and_error_string():
    lib = _lib.load()
    assert b"sm_100a" in lib.cpk_version()
    assert lib.cpk_last_error() is not None


def plan(dims, mode, rank, **kw):
    p = _lib.CpkPlan(kw.get("rank_tile", 0), 0, kw.get("tile_volume", 0), kw.get("splits", 0), 148)
    rc = _lib.load().cpk_plan_resolve(len(dims), _lib.i64_array(dims), mode, rank, p)
    return rc, p


def test_plan_resolution_fills_waves():
    # c4: 1024^3, R=2000: DMMA tile 256 x 64 -> 4 row tiles x 32 rank tiles =
    # 128 tiles; the split count the time model picks fills >= 99 % of its
    # waves
    rc, p = plan((1024, 1024, 1024), 0, 2000)
    assert rc == 0
    assert p.rank_tile == 64 and p.block_rows == 256 and p.engine == 3
    ctas = 4 * 32 * p.splits
    assert ctas / (148 * -(-ctas // 148)) >= 0.99
    # c2: R=64 -> rank tile 64
    rc, p = plan((512, 512, 512), 1, 64)
    assert rc == 0 and p.rank_tile == 64
    # low rank -> the narrow 16-column DMMA tile (256-row blocks; the small
    # mode 0 is merged with its neighbour into 4096 rows)
    rc, p = plan((64, 64, 64), 0, 16)
    assert rc == 0 and p.rank_tile == 16 and p.block_rows == 256 and p.engine == 3
    # R = 24 and 96 -> 32-wide tiles; 40 -> one 64-wide tile
    for r, rt in ((24, 32), (96, 32), (40, 64)):
        rc, p = plan((512, 512, 512), 1, r)
        assert rc == 0 and p.rank_tile == rt, (r, p.rank_tile)


def test_tiny_tile_volume_is_capped():
    # paper tensor A with N_T = 2^3: one chunk per split would be 78k splits;
    # the partial copies are capped like the auto plan's (<= 4096, <= 2 GiB)
    rc, p = plan((401, 201, 12, 501), 0, 32, tile_volume=8)
    assert rc == 0 and 1 <= p.splits <= 4096
    assert p.splits * 401 * 32 * 8 <= 2 * 2 ** 30


def test_plan_tile_volume_maps_to_splits():
    # N_S = 4096 in-slice elements, chunk = 16 of them: N_T = 256 -> 16 chunks/split
    rc, p = plan((64, 64, 64), 0, 16, tile_volume=256)
    assert rc == 0
    assert p.splits == 4096 // 256
    assert p.tile_volume == 256
    rc, p = plan((64, 64, 64), 0, 16, splits=1)
    assert rc == 0 and p.splits == 1 and p.tile_volume == 4096


@pytest.mark.parametrize(
    "dims,mode,rank,kw,code",
    [
        ((4, 5, 6), 3, 2, {}, 2),          # IndexRangeError
        ((4, 5, 6), -1, 2, {}, 2),
        ((4, 0, 6), 0, 2, {}, 1),          # ShapeError
        ((4, 5, 6), 0, 0, {}, 3),          # ParameterError: rank
        ((4, 5, 6), 0, 2, {"rank_tile": 48}, 3),
        ((4, 5, 6), 0, 2, {"tile_volume": 31}, 3),  # N_S = 30
    ],
)
def test_plan_errors_map_to_reference_exceptions(dims, mode, rank, kw, code):
    rc, _ = plan(dims, mode, rank, **kw)
    assert rc == code
    exc = _lib._CODE_TO_EXC[code]
    with pytest.raises(exc):
        _lib.check(rc, "plan")


def test_workspace_bytes(monkeypatch):
    p = _lib.CpkPlan(0, 0, 0, 0, 148)
    nb = C.c_size_t(0)
    rc = _lib.load().cpk_mttkrp_workspace_bytes(3, _lib.i64_array((1024, 1024, 1024)), 0, 2000, p, C.byref(nb))
    assert rc == 0
    rc2, q = plan((1024, 1024, 1024), 0, 2000)
    assert nb.value == q.splits * 1024 * 2000 * 8  # partial copies (default merge)
    p1 = _lib.CpkPlan(0, 0, 0, 1, 148)
    rc = _lib.load().cpk_mttkrp_workspace_bytes(3, _lib.i64_array((64, 64, 64)), 0, 16, p1, C.byref(nb))
    assert rc == 0 and nb.value == 0
    # CPK_SPLIT_CHAIN=1: c4's 128 output tiles >= 148 / 2 -> one counter per
    # tile instead of the partial copies; c2 (2 tiles) keeps the copies
    monkeypatch.setenv("CPK_SPLIT_CHAIN", "1")
    rc = _lib.load().cpk_mttkrp_workspace_bytes(3, _lib.i64_array((1024, 1024, 1024)), 0, 2000, p, C.byref(nb))
    assert rc == 0 and nb.value == 512
    rc = _lib.load().cpk_mttkrp_workspace_bytes(3, _lib.i64_array((512, 512, 512)), 1, 64, p, C.byref(nb))
    rc2, q = plan((512, 512, 512), 1, 64)
    assert rc == 0 and nb.value == q.splits * 512 * 64 * 8


def test_mttkrp_rejects_bad_arguments_before_touching_the_device():
    lib = _lib.load()
    dims = _lib.i64_array((4, 5, 6))
    ptrs = _lib.ptr_array([0, 0, 0])
    rc = lib.cpk_mttkrp_f64(None, 3, dims, 0, ptrs, None, None, 2, None, 2, None, None, 0, None)
    assert rc == 3  # NULL tensor -> ParameterError
    rc = lib.cpk_mttkrp_f64(None, 3, dims, 5, ptrs, None, None, 2, None, 2, None, None, 0, None)
    assert rc == 2


def test_small_mode_merge_is_reported_and_round_trips():
    # paper tensor A, mode 2 (I = 12): merged with a neighbour; the resolved
    # plan says which and describes the merged problem, and resolving the
    # resolved plan again is a fixed point
    rc, p = plan((401, 201, 12, 501), 2, 32)
    assert rc == 0 and p.merge in (1, 2)
    q = _lib.CpkPlan(p.rank_tile, p.block_rows, p.tile_volume, p.splits, p.sm_count, p.block_k, p.engine, p.merge)
    assert _lib.load().cpk_plan_resolve(4, _lib.i64_array((401, 201, 12, 501)), 2, 32, q) == 0
    assert (q.rank_tile, q.block_rows, q.splits, q.merge) == (p.rank_tile, p.block_rows, p.splits, p.merge)
    # big modes stay unmerged; impossible forced merges are rejected
    rc, p = plan((1024, 1024, 1024), 0, 2000)
    assert rc == 0 and p.merge == -1
    bad = _lib.CpkPlan(0, 0, 0, 0, 148, 0, 0, 1)  # PREV of mode 0
    assert _lib.load().cpk_plan_resolve(3, _lib.i64_array((8, 8, 8)), 0, 4, bad) == 3


def test_khatri_rao_merge_is_reported_sized_and_round_trips():
    # config 3 (128^4, R = 256): modes 0, 2, 3 merge their two fastest non-k
    # modes into one Khatri-Rao mode (CPK_MERGE_KR = 3); mode 1 cannot (k sits
    # between them) and folds KR(A_0, A_2) into its factor rows instead
    # (CPK_MERGE_KR_FOLD = 4); the workspace includes the 128 * 128 x 256
    # factor; the resolved plan is a fixed point; 3-way problems never merge
    dims = (128, 128, 128, 128)
    for k, want in ((0, 3), (1, 4), (2, 3), (3, 3)):
        rc, p = plan(dims, k, 256)
        assert rc == 0 and p.merge == want, (k, p.merge)
    rc, p = plan(dims, 0, 256)
    q = _lib.CpkPlan(p.rank_tile, p.block_rows, p.tile_volume, p.splits, p.sm_count, p.block_k, p.engine, p.merge)
    assert _lib.load().cpk_plan_resolve(4, _lib.i64_array(dims), 0, 256, q) == 0
    assert (q.rank_tile, q.block_rows, q.splits, q.merge) == (p.rank_tile, p.block_rows, p.splits, 3)
    nbytes = _lib.C.c_size_t(0)
    req = _lib.CpkPlan(0, 0, 0, 0, 148, 0, 0)
    assert _lib.load().cpk_mttkrp_workspace_bytes(4, _lib.i64_array(dims), 0, 256, req, _lib.C.byref(nbytes)) == 0
    assert nbytes.value >= 128 * 128 * 256 * 8
    rc, p = plan((1024, 1024, 1024), 1, 2000)
    assert rc == 0 and p.merge == -1
    forced = _lib.CpkPlan(0, 0, 0, 0, 148, 0, 0, 3)  # KR for mode 1: impossible
    assert _lib.load().cpk_plan_resolve(4, _lib.i64_array(dims), 1, 256, forced) == 3
    # the fold round-trips and sizes W (128 * 128 x 256) plus the ones rows
    rc, p = plan(dims, 1, 256)
    q = _lib.CpkPlan(p.rank_tile, p.block_rows, p.tile_volume, p.splits, p.sm_count, p.block_k, p.engine, p.merge)
    assert _lib.load().cpk_plan_resolve(4, _lib.i64_array(dims), 1, 256, q) == 0 and q.merge == 4
    assert _lib.load().cpk_mttkrp_workspace_bytes(4, _lib.i64_array(dims), 1, 256, req, _lib.C.byref(nbytes)) == 0
    assert nbytes.value >= 128 * 128 * 256 * 8 + 128 * 256 * 8
    # 3-way problems never fold (the fold would be the whole Khatri-Rao matrix)
    rc, p = plan((64, 64, 64), 1, 64)
    assert rc == 0 and p.merge != 4


def test_split_count_time_model():
    # the dimension tree's c3 view (16384 x 128 x 128, R = 256): 256 tiles of
    # 1024 chunks; 4 splits (98.8 % wave fill) measured 3.3 % faster than the
    # 15 (99.8 %) the first-wave-filling rule took (profiles/r02n_plan_ab.log)
    for dims, mode in (((16384, 128, 128), 0), ((128, 128, 16384), 2)):
        rc, p = plan(dims, mode, 256)
        assert rc == 0 and p.rank_tile == 64 and p.block_rows == 256 and p.splits == 4, (dims, p.splits)
    # c4 keeps its 128 splits (<= 512 chunks per CTA, 2 GiB workspace cap)
    for mode in range(3):
        rc, p = plan((1024, 1024, 1024), mode, 2000)
        assert rc == 0 and p.splits == 128
