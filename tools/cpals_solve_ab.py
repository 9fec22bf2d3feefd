"""c3 CP-ALS sweep time per normal-equation solve path (CPK_SOLVE=kernel |
sweep | cusolver set by the caller): eager and graph-replayed sweeps.

    CPK_SOLVE=sweep python tools/cpals_solve_ab.py [--rank 256] [--iters 10]
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs="+", default=[128, 128, 128, 128])
ap.add_argument("--rank", type=int, default=256)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
y = ck.DenseTensor.uniform(tuple(a.dims), seed=0, device="cuda")
cfg = ck.AlsConfig(rank=a.rank, max_iters=a.iters, tol=0.0)
ck.cp_als(y, ck.AlsConfig(rank=a.rank, max_iters=2, tol=0.0), graph=False)  # warm-up
_, te = ck.cp_als(y, cfg, graph=False)
_, tg = ck.cp_als(y, cfg, graph=True)
eager = sorted(sum(m) + o for m, o in zip(te.mttkrp_seconds, te.other_seconds))
print(json.dumps({"solve": os.environ.get("CPK_SOLVE", "default"), "rank": a.rank,
                  "eager_ms_median": 1e3 * eager[len(eager) // 2],
                  "eager_other_ms_median": 1e3 * sorted(te.other_seconds)[len(eager) // 2],
                  "graph_total_ms_per_sweep": 1e3 * tg.total_seconds / a.iters,
                  "fit_last": te.fits[-1]}))
