import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import importlib
import paper_2510_14891_b200 as ck
mt = importlib.import_module("paper_2510_14891_b200.mttkrp")
from oracle import gen
dims, R = (1024, 1024, 1024), 2000
dev = torch.device("cuda", 0)
full = ck.DenseTensor.uniform(dims, seed=0, device=dev).data
y_host = torch.empty(full.numel(), dtype=torch.float64, pin_memory=True); y_host.copy_(full); del full
fs_pinned = [torch.from_numpy(a).pin_memory() for a in gen.bench_factors(dims, R, 0)]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t0.record()
    yt = ck.DenseTensor(dims, y_host)
    fd = [a.to(dev, non_blocking=True) for a in fs_pinned]
    m = ck.KruskalTensor(np.ones(R), fd, validate=False)
    fac = m.device_factors(dev)
    y_dev, bounds, events = mt._start_upload(yt, dev)
    cur = torch.cuda.current_stream(dev)
    w = []
    for (lo, hi), ev in zip(bounds, events):
        cur.wait_event(ev)
        e = torch.cuda.Event(enable_timing=True); e.record(); w.append(e)
        for k in range(3):
            mt.mttkrp_device(y_dev, dims, fac, k, None, mt.MttkrpPlan(mt.Variant.B200, k), landed=(lo, hi))
    torch.cuda.synchronize()
    print(rep, "wait resolved at", [round(t0.elapsed_time(e), 1) for e in w])
