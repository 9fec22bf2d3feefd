"""A/B the auto plan of two library builds: per case, the resolved plan and
the time of back-to-back auto-plan MTTKRPs.

    python tools/plan_ab.py --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_prechol.so
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--plans-only", action="store_true", help="resolve plans (CPU), no timing")
a = ap.parse_args()
from paper_2510_14891_b200 import _lib  # noqa: E402

if a.lib:
    _lib.LIB_PATH = Path(a.lib).resolve()
import numpy as np  # noqa: E402

CASES = [((16384, 128, 128), 0, 256), ((128, 128, 16384), 2, 256)]
CASES += [((401, 201, 12, 501), k, r) for r in (32, 64) for k in range(4)]
CASES += [((129, 129, 129, 12, 39), k, r) for r in (32, 64) for k in range(5)]
CASES += [((512, 512, 512), 0, r) for r in (16, 64, 256)]
CASES += [((1024, 1024, 1024), k, 2000) for k in range(3)]


def resolved(dims, mode, rank):
    p = _lib.CpkPlan(0, 0, 0, 0, 148)
    _lib.check(_lib.load().cpk_plan_resolve(len(dims), _lib.i64_array(dims), mode, rank, p), "plan")
    return {"engine": p.engine, "rank_tile": p.rank_tile, "block_rows": p.block_rows, "splits": p.splits,
            "merge": p.merge}


if a.plans_only:
    for dims, k, r in CASES:
        print(json.dumps({"dims": dims, "mode": k, "rank": r, **resolved(dims, k, r)}), flush=True)
    sys.exit(0)

import torch  # noqa: E402

import paper_2510_14891_b200 as ck  # noqa: E402
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, mttkrp_device  # noqa: E402

dev = torch.device("cuda", 0)
cache = {}
for dims, k, r in CASES:
    if dims not in cache:
        cache.clear()
        cache[dims] = ck.DenseTensor.uniform(dims, seed=0, device=dev).device_data(dev)
    y = cache[dims]
    rng = np.random.Generator(np.random.Philox(1))
    fs = [torch.from_numpy(rng.random((n, r))).to(dev) for n in dims]
    plan = MttkrpPlan(Variant.B200, k)
    mttkrp_device(y, dims, fs, k, None, plan)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        mttkrp_device(y, dims, fs, k, None, plan)
    e1.record()
    e1.synchronize()
    print(json.dumps({"lib": _lib.LIB_PATH.name, "dims": dims, "mode": k, "rank": r,
                      "ms": round(e0.elapsed_time(e1) / a.reps, 4), **resolved(dims, k, r)}), flush=True)
