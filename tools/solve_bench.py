"""Time the CP-ALS normal-equation solve (speculative form: factor + apply,
one launch sequence per call) for the one-CTA kernels, the multi-CTA sweep
and cuSOLVER potrf + potrs (CPK_SOLVE).

    python tools/solve_bench.py [--ranks 64 128 256 512] [--rows 128 1024 4096]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_14891_b200 import cpals  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", type=int, nargs="+", default=[256, 384, 512, 1000, 2000])
ap.add_argument("--paths", nargs="+", default=["kernel", "sweep", "cusolver"])
ap.add_argument("--rows", type=int, nargs="+", default=[128, 1024, 4096])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--lib", default=None, help="A/B: time this build of the library")
a = ap.parse_args()
if a.lib:
    from paper_2510_14891_b200 import _lib  # noqa: E402

    _lib.LIB_PATH = Path(a.lib).resolve()
dev = torch.device("cuda", 0)
for r in a.ranks:
    rng = np.random.Generator(np.random.Philox(r))
    x = rng.random((2 * r, r))
    gamma = torch.from_numpy(x.T @ x + np.eye(r)).to(dev)
    for rows in a.rows:
        g0 = torch.from_numpy(rng.random((rows, r))).to(dev)
        out = {"rank": r, "rows": rows}
        for path in a.paths:
            if path == "kernel" and r > 512:
                continue
            os.environ["CPK_SOLVE"] = path
            solver = cpals._Solver(dev, rows, r)
            info = torch.zeros(1, dtype=torch.int32, device=dev)
            g = g0.clone()
            for _ in range(3):
                g.copy_(g0)
                cpals._solve_spec(solver, gamma, g, info)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                cpals._solve_spec(solver, gamma, g, info)
            e1.record()
            torch.cuda.synchronize()
            out[path + "_us"] = round(e0.elapsed_time(e1) * 1e3 / a.reps, 1)
        print(json.dumps(out), flush=True)
