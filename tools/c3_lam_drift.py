"""How far lam drifts from the reference after 10 c3 sweeps (justifies the
test tolerance): prints rel_err(lam), max |dfit| and the per-sweep fits."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2510_14891_b200 as ck
from oracle import gen, oracle

als = dict(np.load(Path(__file__).resolve().parents[1] / "tests/golden/als.npz"))
dims = (128, 128, 128, 128)
y = ck.DenseTensor(dims, gen.philox_tensor(dims, 0))
model, tr = ck.cp_als(y, ck.AlsConfig(rank=256, tol=0.0, max_iters=10, seed=0))
print("lam rel_err", oracle.rel_err(model.weights.cpu().numpy(), als["c3/lam"]))
print("max |dfit|", float(np.max(np.abs(np.asarray(tr.fits) - als["c3/fits"]))))
for i in range(1, 11):
    _, t = ck.cp_als(y, ck.AlsConfig(rank=256, tol=0.0, max_iters=i, seed=0))
print("fits", tr.fits)
