"""A/B of the 3-way Khatri-Rao merge into the slowest mode (CPK_KR_MERGE_LAST
=1, default) against the round-2 rule (=0): per-mode times of the c2 shape
over ranks, the c3 tree's W_G view MTTKRP, the c3 tree sweep.  Run once per
setting: CPK_KR_MERGE_LAST=0 python tools/kr_last_ab.py"""
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2510_14891_b200 as ck  # noqa: E402
import importlib  # noqa: E402

from paper_2510_14891_b200 import _lib  # noqa: E402

mt = importlib.import_module("paper_2510_14891_b200.mttkrp")  # the module (the package re-exports a function)


def time_mode(y, dims, fs, k, reps=10):
    mt.mttkrp_device(y, dims, fs, k)  # warm-up, plan, workspace
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        mt.mttkrp_device(y, dims, fs, k)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def plan_of(dims, k, r):
    p = _lib.CpkPlan()
    _lib.check(_lib.load().cpk_plan_resolve(len(dims), _lib.i64_array(dims), k, r, _lib.C.byref(p)), "resolve")
    return {"merge": p.merge, "rank_tile": p.rank_tile, "splits": p.splits}


out = {"CPK_KR_MERGE_LAST": os.environ.get("CPK_KR_MERGE_LAST", "1"), "c2": [], "views": []}
dims = (512, 512, 512)
y = ck.DenseTensor.uniform(dims, seed=1, device="cuda").device_data()
g = torch.Generator(device="cuda").manual_seed(0)
for r in (16, 32, 64, 128, 512, 2000):
    fs = [torch.rand((n, r), dtype=torch.float64, device="cuda", generator=g) for n in dims]
    for k in range(3):
        out["c2"].append({"R": r, "mode": k, "ms": time_mode(y, dims, fs, k), **plan_of(dims, k, r)})
del y
for vd, k, r in (((16384, 128, 128), 0, 256), ((128, 128, 16384), 2, 256), ((1024, 2048, 2048), 0, 512)):
    y = ck.DenseTensor.uniform(vd, seed=1, device="cuda").device_data()
    fs = [torch.rand((n, r), dtype=torch.float64, device="cuda", generator=g) for n in vd]
    out["views"].append({"dims": vd, "mode": k, "R": r, "ms": time_mode(y, vd, fs, k, reps=3), **plan_of(vd, k, r)})
    del y, fs
    torch.cuda.empty_cache()
t = ck.DenseTensor.uniform((128,) * 4, seed=1, device="cuda")
ck.cp_als(t, ck.AlsConfig(rank=256, tol=0.0, max_iters=2, seed=0))
_, tr = ck.cp_als(t, ck.AlsConfig(rank=256, tol=0.0, max_iters=10, seed=0))
out["c3_tree_sweep_ms"] = 1e3 * statistics.median(sum(m) + o for m, o in zip(tr.mttkrp_seconds, tr.other_seconds))
out["c3_tree_mttkrp_ms"] = [1e3 * statistics.median(m[i] for m in tr.mttkrp_seconds) for i in range(4)]
print(json.dumps(out))
