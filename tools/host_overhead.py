"""Host-side cost of issuing the per-mode calls of a CP-ALS sweep (async;
the GPU work is tiny so the host is the bottleneck): mttkrp_device, the
speculative solve halves, normalize, gram, hadamard."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402
import importlib  # noqa: E402
from paper_2510_14891_b200 import cpals  # noqa: E402
mt = importlib.import_module("paper_2510_14891_b200.mttkrp")
from paper_2510_14891_b200.kruskal import gram, hadamard  # noqa: E402

dev = torch.device("cuda", 0)
dims, r = (16, 16, 16), 8
y = ck.DenseTensor.uniform(dims, seed=0, device=dev)
fs = [torch.rand(n, r, dtype=torch.float64, device=dev) for n in dims]
grams = [gram(a) for a in fs]
gamma = torch.empty(r, r, dtype=torch.float64, device=dev)
plan = mt.MttkrpPlan(mt.Variant.B200, 0)
solver = cpals._Solver(dev, 16, r)
info = torch.zeros(1, dtype=torch.int32, device=dev)
side = torch.cuda.Stream(dev)


def bench(name, fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:24s} {1e6 * (t1 - t0) / n:8.1f} us per call (host)")


bench("mttkrp_device", lambda: mt.mttkrp_device(y.data, dims, fs, 1, None, mt.plan_for_mode(plan, dims, 1), out=fs[1]))
bench("hadamard", lambda: hadamard(grams, skip=1, out=gamma))
bench("factor_spec", lambda: cpals._factor_spec(solver, gamma, info, side))
bench("apply_spec", lambda: cpals._apply_spec(solver, fs[1], info))
bench("gram", lambda: gram(fs[1], out=grams[1]))
bench("copy_", lambda: grams[0].copy_(grams[1]))
ev = torch.cuda.Event()
bench("event record+wait", lambda: (ev.record(), side.wait_event(ev)))
