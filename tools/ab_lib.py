"""A/B two builds of the library in one process pair: times the MTTKRP of
every mode at c3 / c4 / c2 with the library at --lib (default: in-tree).

    python tools/ab_lib.py --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_preog.so
"""
import argparse
import importlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
from paper_2510_14891_b200 import _lib  # noqa: E402

if a.lib:
    _lib.LIB_PATH = Path(a.lib).resolve()
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_14891_b200 as ck  # noqa: E402

mt = importlib.import_module("paper_2510_14891_b200.mttkrp")
dev = torch.device("cuda", 0)
res = {"lib": str(_lib.LIB_PATH.name)}
for name, dims, rank in (("c3", (128, 128, 128, 128), 256), ("c4", (1024, 1024, 1024), 2000), ("c2", (512, 512, 512), 64)):
    y = ck.DenseTensor.uniform(dims, seed=0, device=dev)
    rng = np.random.Generator(np.random.Philox(1))
    fs = [torch.from_numpy(rng.random((n, rank))).to(dev) for n in dims]
    per = []
    for k in range(len(dims)):
        plan = mt.MttkrpPlan(mt.Variant.B200, k)
        ts = []
        for _ in range(a.reps + 1):
            g, p, timer = mt.mttkrp_device(y.data, dims, fs, k, None, plan)
            torch.cuda.synchronize()
            ts.append(timer.seconds * 1e3)
        per.append(round(min(ts[1:]), 3))
    res[name] = per
    del y
    torch.cuda.empty_cache()
print(json.dumps(res))
