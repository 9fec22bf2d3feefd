"""One dimension-tree CP-ALS run for profiling (ncu launch lists of the W_G
MTTKRP and the in-group contractions): python tools/dimtree_sweep.py --dims
1024,2048,2048 --rank 512 --iters 2 [--tree 0|1]."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2510_14891_b200 as ck  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="1024,2048,2048")
ap.add_argument("--rank", type=int, default=512)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--tree", type=int, default=1)
a = ap.parse_args()
dims = tuple(int(x) for x in a.dims.split(","))
t = ck.DenseTensor.uniform(dims, seed=1, device="cuda")
_, tr = ck.cp_als(t, ck.AlsConfig(rank=a.rank, tol=0.0, max_iters=a.iters, seed=0, dimtree=bool(a.tree)),
                  graph=False)
torch.cuda.synchronize()
print(json.dumps({"dims": dims, "rank": a.rank, "tree_split": tr.tree_split, "fits": tr.fits,
                  "mttkrp_seconds": tr.mttkrp_seconds, "other_seconds": tr.other_seconds}))
