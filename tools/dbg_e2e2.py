"""Timeline of a streamed 3-mode step: copy-slab events and per-mode piece ends."""
import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck
from paper_2510_14891_b200 import mttkrp as _m  # noqa
import importlib
mt = importlib.import_module("paper_2510_14891_b200.mttkrp")
from oracle import gen
dims, R = (1024, 1024, 1024), 2000
dev = torch.device("cuda", 0)
full = ck.DenseTensor.uniform(dims, seed=0, device=dev).data
y_host = torch.empty(full.numel(), dtype=torch.float64, pin_memory=True); y_host.copy_(full); del full
fs_pinned = [torch.from_numpy(a).pin_memory() for a in gen.bench_factors(dims, R, 0)]
fd = [a.to(dev) for a in fs_pinned]
orig = mt.mttkrp_device
marks = []
def traced(*a, **k):
    r = orig(*a, **k)
    e = torch.cuda.Event(enable_timing=True); e.record()
    marks.append((a[3], k.get("landed"), e))
    return r
for rep in range(2):
    marks.clear()
    mt.mttkrp_device = traced
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t0.record()
    yt = ck.DenseTensor(dims, y_host)
    if "--fd-inside" in sys.argv:
        fd = [a.to(dev, non_blocking=True) for a in fs_pinned]
    e_fd = torch.cuda.Event(enable_timing=True); e_fd.record()
    gs = ck.mttkrp_modes(yt, fd, (0, 1, 2)) if "--modes" in sys.argv else [ck.mttkrp(yt, fd, k) for k in range(3)]
    # copy timeline: time the copy events via a timing event recorded on the copy stream is not possible
    torch.cuda.synchronize()
    mt.mttkrp_device = orig
    out = {}
    for mode, landed, e in marks:
        out.setdefault(mode, []).append(round(t0.elapsed_time(e), 1))
    print(rep, "fd ready at %.1f" % t0.elapsed_time(e_fd), out)
# copy alone
torch.cuda.synchronize()
y_dev = torch.empty_like(y_host, device=dev)
s = torch.cuda.Stream(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    a.record(); y_dev.copy_(y_host, non_blocking=True); b.record()
torch.cuda.synchronize(); print("H2D alone %.1f ms" % a.elapsed_time(b))
