"""Plan sweep of one MTTKRP problem through the C-ABI with explicit plans
(rank tile x block rows x splits x block_k, DMMA engine), per-call ms with
events, against the automatic plan:
    python tools/view_plan_sweep.py --dims 16384,16384 --mode 0 --rank 256"""
import argparse
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2510_14891_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="16384,16384")
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--rank", type=int, default=256)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--max-ws-gb", type=float, default=8.0, help="skip plans whose split-K workspace is larger")
a = ap.parse_args()
dims = tuple(int(x) for x in a.dims.split(","))
d, k, r = len(dims), a.mode, a.rank
lib = _lib.load()
n = 1
for x in dims:
    n *= x
y = torch.rand(n, dtype=torch.float64, device="cuda")
fs = [torch.rand((i, r), dtype=torch.float64, device="cuda") for i in dims]
out = torch.empty((dims[k], r), dtype=torch.float64, device="cuda")
dims_c = _lib.i64_array(dims)
ptrs = _lib.ptr_array([f.data_ptr() if m != k else 0 for m, f in enumerate(fs)])
lds = _lib.i64_array([r] * d)
flops = 2.0 * n * r


def run(plan, reps):
    nb = _lib.C.c_size_t(0)
    if lib.cpk_mttkrp_workspace_bytes(d, dims_c, k, r, _lib.C.byref(plan), _lib.C.byref(nb)):
        return None
    if nb.value > a.max_ws_gb * 2 ** 30:
        return None
    ws = torch.empty(max(1, (nb.value + 7) // 8), dtype=torch.float64, device="cuda")
    res = _lib.CpkPlan()
    _lib.C.memmove(_lib.C.byref(res), _lib.C.byref(plan), _lib.C.sizeof(plan))
    if lib.cpk_plan_resolve(d, dims_c, k, r, _lib.C.byref(res)):
        return None

    def call():
        return lib.cpk_mttkrp_f64(y.data_ptr(), d, dims_c, k, ptrs, lds, None, r, out.data_ptr(), r,
                                  _lib.C.byref(plan), ws.data_ptr(), nb.value, None)

    if call():
        return None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"ms": ms, "tflops": flops / ms / 1e9, **{f: getattr(res, f) for f, _ in res._fields_}}


rows = [{"plan": "auto", **(run(_lib.CpkPlan(), a.reps) or {})}]
for rt, bm, sp, bk in itertools.product((64, 128), (128, 256), (1, 2, 3, 4, 6, 8, 12, 16), (16, 32)):
    p = _lib.CpkPlan(rt, bm, 0, sp, 0, bk, 3, -1)
    res = run(p, a.reps)
    if res:
        rows.append({"plan": f"rt{rt} bm{bm} s{sp} bk{bk}", **res})
rows.sort(key=lambda x: x.get("ms", 1e9))
for x in rows[:12]:
    print(json.dumps(x))
print(json.dumps({"auto": [x for x in rows if x["plan"] == "auto"][0]}))
