"""Per-mode MTTKRP time at the low-rank end (c2 shape 512^3 by default) for
each DMMA rank tile, plus the auto plan; reports the HBM fraction
(8 N bytes / time / peak) and the issued FP64 fraction (2 N R / time / peak).

    python tools/lowrank_sweep.py [--ranks 8 16 24 32 48 64] [--tiles 16 32 64] [--lib path]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs="+", default=[512, 512, 512])
ap.add_argument("--ranks", type=int, nargs="+", default=[8, 16, 24, 32, 48, 64])
ap.add_argument("--tiles", type=int, nargs="+", default=[16, 32, 64])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--lib", default=None)
ap.add_argument("--hbm", type=float, default=6547.2e9)
ap.add_argument("--fp64", type=float, default=37.1e12)
a = ap.parse_args()
from paper_2510_14891_b200 import _lib  # noqa: E402

if a.lib:
    _lib.LIB_PATH = Path(a.lib).resolve()
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_14891_b200 as ck  # noqa: E402
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, mttkrp_device  # noqa: E402

dev = torch.device("cuda", 0)
dims = tuple(a.dims)
n = int(np.prod(dims))
y = ck.DenseTensor.uniform(dims, seed=0, device=dev)
out = {"dims": dims, "lib": str(_lib.LIB_PATH.name), "points": []}
for r in a.ranks:
    rng = np.random.Generator(np.random.Philox(1))
    fs = [torch.from_numpy(rng.random((e, r))).to(dev) for e in dims]
    for tile in [0] + a.tiles:
        if tile and tile > 2 * max(r, 16) and tile != 64:
            continue
        per, plans = [], []
        for k in range(len(dims)):
            plan = MttkrpPlan(Variant.B200, k, rank_tile=tile, engine="dmma" if tile else "auto")
            try:
                # back to back between two events: host work overlaps the previous call
                g, p, timer = mttkrp_device(y.data, dims, fs, k, None, plan)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(4 * a.reps):
                    mttkrp_device(y.data, dims, fs, k, None, plan)
                e1.record()
                e1.synchronize()
                per.append(e0.elapsed_time(e1) * 1e-3 / (4 * a.reps))
                plans.append(p)
            except Exception as exc:  # noqa: BLE001
                per.append(None)
                plans.append(str(exc)[:80])
        ok = [t for t in per if t]
        pt = {"rank": r, "tile": tile or "auto", "ms": [round(t * 1e3, 4) if t else None for t in per]}
        if ok:
            tm = sum(ok) / len(ok)
            pt["hbm_frac"] = round(8 * n / tm / a.hbm, 3)
            pt["fp64_issued_frac"] = round(2 * n * r / tm / a.fp64, 3)
        if not tile:
            pt["plans"] = [p if isinstance(p, str) else {kk: getattr(p, kk, None) for kk in ("engine", "rank_tile", "splits")}
                           for p in plans]
        out["points"].append(pt)
        print(json.dumps(pt), flush=True)
print(json.dumps(out))
