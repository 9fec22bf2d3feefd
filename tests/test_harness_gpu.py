"""The sweep harness (cpkern `sweep`, cli.py:343-464) on the GPU: the
reference's CSV schema and aggregation rules, every row from a verified run."""

import csv

import numpy as np
import pytest

import paper_2510_14891_b200 as ck
from paper_2510_14891_b200 import harness

pytestmark = pytest.mark.gpu


def test_sweep_csv_schema_and_best_marks(tmp_path):
    dims = (20, 18, 16)
    y = ck.DenseTensor(dims, np.random.Generator(np.random.Philox(0)).random(int(np.prod(dims))))
    out = tmp_path / "s.csv"
    res = harness.sweep(y, ranks=[8, 40], variants=["tile", "slice", "elem", "b200"], tile_widths=[2, 5, 30],
                        reps=2, warmup=1, out=str(out))
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0]) == harness.COLUMNS + harness.B200_COLUMNS
    # tile: 2 ranks x 3 widths x 3 modes x 2 reps; the rest 2 x 3 x 2 each
    assert len(rows) == res["rows"] == 2 * 3 * 3 * 2 + 3 * (2 * 3 * 2)
    assert {r["mode"] for r in rows} == {"1", "2", "3"}
    tile = [r for r in rows if r["variant"] == "tile" and r["tile_width"] == "30"]
    assert all(int(r["N_T"]) == min(30 ** 2, 20 * 18 * 16 // dims[int(r["mode"]) - 1]) for r in tile)
    assert all(float(r["gflops"]) > 0 and float(r["time_s"]) > 0 for r in rows)
    agg = list(csv.DictReader(open(res["agg_out"])))
    assert list(agg[0]) == harness.AGG_COLUMNS
    for key in {(a["variant"], a["rank"]) for a in agg}:
        grp = [a for a in agg if (a["variant"], a["rank"]) == key]
        assert sum(int(a["best"]) for a in grp) == 1
        best = max(grp, key=lambda a: float(a["gflops"]))
        assert best["best"] == "1"


def test_cli_entry(tmp_path):
    out = tmp_path / "c.csv"
    assert harness.main(["sweep", "--shape", "12,10,8", "--ranks", "5", "--tile-widths", "3,4", "--reps", "1",
                         "--out", str(out)]) == 0
    assert len(list(csv.DictReader(open(out)))) == 2 * 3
