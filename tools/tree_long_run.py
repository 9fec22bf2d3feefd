"""Long CP-ALS runs, dimension tree against per-mode sweeps: c3 (128^4,
R = 256) for 100 sweeps (graph replay), c5 (4096 x 2048^2, R = 512) for 8
sweeps, and a converging run (tol 1e-6); reports the fit drift between the
two sweep structures and the sec/sweep of each.
    python tools/tree_long_run.py"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_14891_b200 as ck  # noqa: E402


def run(t, rank, iters, tree, tol=0.0, graph=None):
    _, tr = ck.cp_als(t, ck.AlsConfig(rank=rank, tol=tol, max_iters=iters, seed=0, dimtree=tree), graph=graph)
    sweeps = [sum(m) + o for m, o in zip(tr.mttkrp_seconds, tr.other_seconds)]
    return tr, statistics.median(sweeps[1:] if len(sweeps) > 1 else sweeps)


out = []
for name, dims, rank, iters, tol in (("c3", (128,) * 4, 256, 100, 0.0), ("c3-converge", (128,) * 4, 256, 200, 1e-6),
                                     ("c5", (4096, 2048, 2048), 512, 8, 0.0)):
    t = ck.DenseTensor.uniform(dims, seed=3, device="cuda")
    tr_t, s_t = run(t, rank, iters, None, tol)
    torch.cuda.empty_cache()
    tr_p, s_p = run(t, rank, iters, False, tol)
    n = min(len(tr_t.fits), len(tr_p.fits))
    drift = float(np.max(np.abs(np.asarray(tr_t.fits[:n]) - np.asarray(tr_p.fits[:n]))))
    out.append({"case": name, "dims": dims, "rank": rank, "tree_split": tr_t.tree_split,
                "iterations": [tr_t.iterations, tr_p.iterations], "converged": [tr_t.converged, tr_p.converged],
                "fit_last": [tr_t.fits[-1], tr_p.fits[-1]], "max_fit_drift": drift,
                "sec_per_sweep": {"tree": s_t, "per_mode": s_p}})
    print(json.dumps(out[-1]), flush=True)
    del t
    torch.cuda.empty_cache()
