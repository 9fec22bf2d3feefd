"""Optional float32 path at config 4: per-mode time of the tcgen05 3xTF32
kernel and its relative Frobenius error against the FP64 kernel on the same
(fp32-representable) inputs.

    python tools/f32_bench.py [--dims 1024 1024 1024] [--rank 2000]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402
from paper_2510_14891_b200.mttkrp import mttkrp_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs="+", default=[1024, 1024, 1024])
ap.add_argument("--rank", type=int, default=2000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dims, r = tuple(a.dims), a.rank
dev = torch.device("cuda", 0)
y64 = ck.DenseTensor.uniform(dims, seed=0, device=dev).data
y32 = y64.float()
y64 = y32.double()  # the same values in both precisions
rng = np.random.Generator(np.random.Philox(1))
f32 = [torch.from_numpy(rng.random((n, r))).to(dev).float() for n in dims]
f64 = [f.double() for f in f32]
n = int(np.prod(dims))
res = {"dims": list(dims), "rank": r, "modes": []}
for k in range(len(dims)):
    g64, _, _ = mttkrp_device(y64, dims, f64, k)
    ts = []
    for _ in range(a.reps + 1):
        g32, _, t = mttkrp_device(y32, dims, f32, k)
        ts.append(t.seconds)
    t = min(ts[1:])
    err = float(torch.linalg.norm(g32.double() - g64) / torch.linalg.norm(g64))
    res["modes"].append({"mode": k, "ms": t * 1e3, "tflops_alg": 2 * n * r * (len(dims) - 1) / t / 1e12,
                         "rel_frobenius_vs_fp64": err})
    del g64, g32
print(json.dumps(res))
