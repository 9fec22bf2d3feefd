"""Run-to-run bit reproducibility per engine / rank tile (c2 inputs, every
mode), plus a small case for compute-sanitizer.

    python tools/repro_bits.py [--reps 10] [--small]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2510_14891_b200 import harness  # noqa: E402
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, mttkrp_device, resolve_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--small", action="store_true")
a = ap.parse_args()
dims, rank = ((40, 36, 34), 130) if a.small else ((512, 512, 512), 64)
dev = torch.device("cuda", 0)
y = torch.from_numpy(np.random.Generator(np.random.Philox(0)).random(int(np.prod(dims)))).to(dev)
fs = [torch.from_numpy(np.asarray(f)).to(dev) for f in harness.bench_factors(dims, rank, 0).factors]
for engine, rt, bk in (("tma", 128, 32), ("tma", 64, 0), ("cpasync", 128, 32), ("dmma", 128, 32), ("dmma", 64, 0)):
    for k in range(3):
        plan = MttkrpPlan(Variant.B200, k, rank_tile=rt, block_k=bk, engine=engine)
        info = resolve_plan(plan, dims, rank)
        ref = mttkrp_device(y, dims, fs, k, None, plan)[0].clone()
        bad = 0
        for _ in range(a.reps):
            g = mttkrp_device(y, dims, fs, k, None, plan)[0]
            if not torch.equal(g, ref):
                bad += 1
                diff = (g - ref).abs()
                where = torch.nonzero(diff)
                first = where[0].tolist()
        msg = f"{engine:8s} rt={rt:3d} mode {k} splits={info['splits']:4d}: {bad}/{a.reps} runs differ"
        if bad:
            msg += f" (ndiff={len(where)}, first={first}, maxabs={float(diff.max()):.3e})"
        print(msg, flush=True)
