"""Run the config-4 MTTKRP of one mode a few times (for ncu captures).

    python tools/profile_one.py --mode 0 --reps 2 [--dims 1024 1024 1024 --rank 2000]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
if "--lib" in sys.argv:  # A/B: another build of the library
    from paper_2510_14891_b200 import _lib as _l  # noqa: E402

    _l.LIB_PATH = Path(sys.argv[sys.argv.index("--lib") + 1]).resolve()
import paper_2510_14891_b200 as ck  # noqa: E402
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, mttkrp_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--dims", type=int, nargs="+", default=[1024, 1024, 1024])
ap.add_argument("--rank", type=int, default=2000)
ap.add_argument("--rank-tile", type=int, default=0)
ap.add_argument("--splits", type=int, default=0)
ap.add_argument("--block-k", type=int, default=0)
ap.add_argument("--engine", default="auto")
ap.add_argument("--lib", default=None)
a = ap.parse_args()
dev = torch.device("cuda", 0)
t = ck.DenseTensor.uniform(tuple(a.dims), seed=0, device=dev)
rng = np.random.Generator(np.random.Philox(1))
fs = [torch.from_numpy(rng.random((n, a.rank))).to(dev) for n in a.dims]
modes = range(len(a.dims)) if a.mode < 0 else [a.mode]
for k in modes:
    plan = MttkrpPlan(Variant.B200, k, rank_tile=a.rank_tile, splits=a.splits, block_k=a.block_k, engine=a.engine)
    print(k, ck.resolve_plan(plan, a.dims, a.rank))
    for _ in range(a.reps):
        g, p, timer = mttkrp_device(t.data, a.dims, fs, k, None, plan)
        torch.cuda.synchronize()
        print(f"mode {k}: {timer.seconds * 1e3:.2f} ms", flush=True)
