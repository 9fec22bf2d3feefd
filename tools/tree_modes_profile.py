"""Where an all-modes dimension-tree step goes (c4 shape by default): per
piece CUDA-event times of mttkrp_modes(tree=True)'s work, and the whole call.
    python tools/tree_modes_profile.py [--dims 1024,1024,1024 --rank 2000]"""
import argparse
import importlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2510_14891_b200 as ck  # noqa: E402

mt = importlib.import_module("paper_2510_14891_b200.mttkrp")
ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="1024,1024,1024")
ap.add_argument("--rank", type=int, default=2000)
a = ap.parse_args()
dims = tuple(int(x) for x in a.dims.split(","))
r = a.rank
y = ck.DenseTensor.uniform(dims, seed=1, device="cuda").device_data()
fs = [torch.rand((n, r), dtype=torch.float64, device="cuda") for n in dims]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"dims": dims, "rank": r}
out["mttkrp_modes_tree_ms"] = timed(lambda: ck.mttkrp_modes(y, fs, tree=True))
out["mttkrp_modes_per_mode_ms"] = timed(lambda: ck.mttkrp_modes(y, fs))
out["M0_ms"] = timed(lambda: mt.mttkrp_device(y, dims, fs, 0))
vd = (dims[0], dims[1] * dims[2])
w = torch.empty((vd[1], r), dtype=torch.float64, device="cuda")
out["W_R_view_ms"] = timed(lambda: mt.mttkrp_device(y, vd, [fs[0], None], 1, out=w))
o1 = torch.empty((dims[1], r), dtype=torch.float64, device="cuda")
o2 = torch.empty((dims[2], r), dtype=torch.float64, device="cuda")
out["contract_j0_ms"] = timed(lambda: mt.dimtree_contract(w, [dims[1], dims[2]], 0, [fs[1], fs[2]], o1, r))
out["contract_j1_ms"] = timed(lambda: mt.dimtree_contract(w, [dims[1], dims[2]], 1, [fs[1], fs[2]], o2, r))
out["W_bytes"] = w.numel() * 8
out["contract_GBps"] = [w.numel() * 8 / (out[k] * 1e-3) / 1e9 for k in ("contract_j0_ms", "contract_j1_ms")]
print(json.dumps(out))
