"""Fixed (capture) vs per-sweep cost of cp_als(graph=True): wall time of runs
of n1 and n2 sweeps; per replayed sweep = (T(n2) - T(n1)) / (n2 - n1).

    python tools/cpals_graph_cost.py [--rank 64] [--dims 128 128 128 128]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs="+", default=[128, 128, 128, 128])
ap.add_argument("--rank", type=int, default=64)
ap.add_argument("--n", type=int, nargs=2, default=[12, 36])
a = ap.parse_args()
y = ck.DenseTensor.uniform(tuple(a.dims), seed=0, device="cuda")
ck.cp_als(y, ck.AlsConfig(rank=a.rank, max_iters=2, tol=0.0), graph=False)
out = {"rank": a.rank}
for graph in (False, True):
    ts = []
    for n in a.n:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, tr = ck.cp_als(y, ck.AlsConfig(rank=a.rank, max_iters=n, tol=0.0), graph=graph)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    per = (ts[1] - ts[0]) / (a.n[1] - a.n[0])
    out["graph" if graph else "eager"] = {"per_sweep_ms": 1e3 * per, "fixed_ms": 1e3 * (ts[0] - a.n[0] * per)}
print(json.dumps(out))
