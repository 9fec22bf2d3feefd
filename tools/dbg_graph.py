import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2510_14891_b200 as ck
als = np.load(ROOT / "tests/golden/als.npz")
key = "planted_6x7x8_r3"
dims = tuple(int(x) for x in als[f"{key}/dims"])
y = ck.DenseTensor(dims, als[f"{key}/data"])
ref = als[f"{key}/fits_reference"]
for graph in (False, True):
    _, tr = ck.cp_als(y, ck.AlsConfig(rank=3, tol=0.0, max_iters=len(ref), seed=0), graph=graph)
    f = np.asarray(tr.fits)
    print("graph", graph, "maxdev", np.max(np.abs(f - ref)), "first devs", (f - ref)[:6])
