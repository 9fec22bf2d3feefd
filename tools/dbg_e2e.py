import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck
import importlib
_mt = importlib.import_module("paper_2510_14891_b200.mttkrp")
for a in sys.argv:
    if a.startswith("--slabs="):
        _mt.STREAM_SLABS = int(a.split("=")[1])
from oracle import gen
dims, R = (1024, 1024, 1024), 2000
dev = torch.device("cuda", 0)
full = ck.DenseTensor.uniform(dims, seed=0, device=dev).data
y_host = torch.empty(full.numel(), dtype=torch.float64, pin_memory=True); y_host.copy_(full); del full
fs_pinned = [torch.from_numpy(a).pin_memory() for a in gen.bench_factors(dims, R, 0)]
gp = [torch.empty((dims[k], R), dtype=torch.float64, pin_memory=True) for k in range(3)]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    yt = ck.DenseTensor(dims, y_host)
    fd = [a.to(dev, non_blocking=True) for a in fs_pinned]
    marks = []
    if "--modes" in sys.argv:
        for k, g in enumerate(ck.mttkrp_modes(yt, fd, (0, 1, 2))):
            gp[k].copy_(g, non_blocking=True)
        marks.append(("issued", None, time.perf_counter() - t0))
    else:
      for k in range(3):
        lan = yt.landing is not None if k else None
        g = ck.mttkrp(yt, fd, k)
        marks.append((k, lan, time.perf_counter() - t0))
        gp[k].copy_(g, non_blocking=True)
        marks.append(("d2h", k, time.perf_counter() - t0))
    torch.cuda.synchronize()
    print(rep, [(a, b, round(c * 1e3, 1)) for a, b, c in marks], "total %.1f ms" % ((time.perf_counter() - t0) * 1e3))
