"""Rank-tile / chunk-depth / split sweep of the B200 MTTKRP (north star:
"rank-tile-size sweep"; schema after cpkern `sweep`, cli.py:343-464).

    python tools/sweep.py --shape 512 512 512 --ranks 64 --out profiles/sweep_c2.csv

Per (rank, rank_tile, block_k, engine, splits) and mode: best-of-reps CUDA-event
time, paper gflops (N R d / t / 1024^3, perfmodel.py:199-203), algorithmic
TFLOP/s (2 N R (d-1) / t) and north-star roofline fraction.  The .agg.csv
averages over modes and marks the best configuration per rank, next to the
configuration the planner picks by default ("auto").
"""

import argparse
import csv
import itertools
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, mttkrp_device, resolve_plan  # noqa: E402
from paper_2510_14891_b200.perfmodel import roofline_seconds  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs="+", default=[512, 512, 512])
    ap.add_argument("--ranks", type=int, nargs="+", default=[64])
    ap.add_argument("--rank-tiles", type=int, nargs="+", default=[0, 32, 64, 128])
    ap.add_argument("--block-ks", type=int, nargs="+", default=[0, 16, 32])
    ap.add_argument("--engines", nargs="+", default=["auto", "cpasync"])
    ap.add_argument("--splits", type=int, nargs="+", default=[0])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fp64-peak", type=float, default=0.0, help="FLOP/s; 0 = run the DFMA probe")
    ap.add_argument("--out", default="profiles/sweep.csv")
    a = ap.parse_args()

    dims = tuple(a.shape)
    d = len(dims)
    n = int(np.prod(dims))
    dev = torch.device("cuda", 0)
    t = ck.DenseTensor.uniform(dims, seed=0, device=dev)
    peak = a.fp64_peak
    if peak <= 0:
        from paper_2510_14891_b200 import _lib

        v = _lib.C.c_double(0)
        _lib.check(_lib.load().cpk_fp64_peak_probe(_lib.C.byref(v), None))
        peak = v.value
    rows, agg = [], []
    for rank in a.ranks:
        rng = np.random.Generator(np.random.Philox(1))
        fs = [torch.from_numpy(rng.random((e, rank))).to(dev) for e in dims]
        roof = roofline_seconds(dims, rank, fp64_peak=peak)
        for rt, bk, eng, sp in itertools.product(a.rank_tiles, a.block_ks, a.engines, a.splits):
            per_mode = []
            ok = True
            for k in range(d):
                plan = MttkrpPlan(Variant.B200, k, rank_tile=rt, block_k=bk, engine=eng, splits=sp)
                try:
                    info = resolve_plan(plan, dims, rank)
                    mttkrp_device(t.data, dims, fs, k, None, plan)  # warm-up
                    ts = []
                    for _ in range(a.reps):
                        _, _, timer = mttkrp_device(t.data, dims, fs, k, None, plan)
                        ts.append(timer.seconds)
                except ck.CpkernError as exc:
                    ok = False
                    print(f"skip rt={rt} bk={bk} engine={eng} splits={sp}: {exc}", file=sys.stderr)
                    break
                best = min(ts)
                per_mode.append(best)
                rows.append({
                    "variant": "b200", "mode": k + 1, "rank": rank, "rank_tile": info["rank_tile"],
                    "block_k": info["block_k"], "engine": info["engine"], "splits": info["splits"],
                    "N_T": info["tile_volume"], "time_s": best,
                    "gflops": n * rank * d / best / 1024 ** 3,
                    "tflops_alg": 2 * n * rank * (d - 1) / best / 1e12,
                    "roofline_frac": roof / best,
                    "requested": f"rt={rt} bk={bk} engine={eng} splits={sp}",
                })
            if ok:
                agg.append({"rank": rank, "requested": f"rt={rt} bk={bk} engine={eng} splits={sp}",
                            "mean_time_s": statistics.fmean(per_mode),
                            "tflops_alg": statistics.fmean(2 * n * rank * (d - 1) / x / 1e12 for x in per_mode),
                            "roofline_frac": statistics.fmean(roof / x for x in per_mode), "best": 0})
    for rank in a.ranks:
        grp = [r for r in agg if r["rank"] == rank]
        if grp:
            max(grp, key=lambda r: r["tflops_alg"])["best"] = 1
    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    with open(out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)
    agg_path = out.with_suffix(".agg.csv")
    with open(agg_path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(agg[0]))
        w.writeheader()
        w.writerows(agg)
    print(json.dumps({"rows": len(rows), "out": str(out), "agg_out": str(agg_path), "fp64_peak": peak}))


if __name__ == "__main__":
    main()
