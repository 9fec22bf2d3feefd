"""Small runs of every new device path, for compute-sanitizer (memcheck /
racecheck / synccheck): 4-way MTTKRP (Khatri-Rao merge + o-group TMEM
accumulation), 3-way with rank tails, the narrow 16/32-column DMMA tiles and
the swizzled mode-0 panels, the split chain (CPK_SPLIT_CHAIN=1), the solve
kernels (one-CTA Cholesky and the multi-CTA sweep), CP-ALS (per-mode and
dimension-tree sweeps)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant  # noqa: E402

rng = np.random.Generator(np.random.Philox(5))
for dims, r in (((32, 24, 20, 6), 70), ((40, 36, 34), 130), ((6, 5, 4, 7, 3), 9)):
    y = ck.DenseTensor(dims, rng.random(int(np.prod(dims))))
    m = ck.KruskalTensor(np.ones(r), [rng.random((n, r)) for n in dims])
    for k in range(len(dims)):
        ck.run(y, m, MttkrpPlan(Variant.B200, k))
for dims, r in (((64, 40, 34), 24), ((48, 30, 20, 4), 12)):
    y = ck.DenseTensor(dims, rng.random(int(np.prod(dims))))
    m = ck.KruskalTensor(np.ones(r), [rng.random((n, r)) for n in dims])
    for k in range(len(dims)):
        for rt in (16, 32):
            ck.run(y, m, MttkrpPlan(Variant.B200, k, rank_tile=rt, engine="dmma", splits=3))
os.environ["CPK_SPLIT_CHAIN"] = "1"
y = ck.DenseTensor((40, 36, 34), rng.random(40 * 36 * 34))
m = ck.KruskalTensor(np.ones(70), [rng.random((n, 70)) for n in (40, 36, 34)])
for k in range(3):
    for eng in ("dmma", "cpasync"):
        ck.run(y, m, MttkrpPlan(Variant.B200, k, engine=eng, rank_tile=64 if eng == "dmma" else 32, splits=4,
                                sm_count=1))
del os.environ["CPK_SPLIT_CHAIN"]
y = ck.DenseTensor((20, 18, 16, 6), rng.random(20 * 18 * 16 * 6))
ck.cp_als(y, ck.AlsConfig(rank=40, max_iters=3, tol=0.0), graph=False)
# dimension tree: W_G views and the contraction (two-mode groups, both lane
# widths: R even / odd; a three-mode group of a 5-way tensor)
for dims, r in (((20, 18, 16, 6), 40), ((21, 10, 12), 33), ((6, 5, 4, 7, 3), 9)):
    ck.cp_als(ck.DenseTensor(dims, rng.random(int(np.prod(dims)))),
              ck.AlsConfig(rank=r, max_iters=2, tol=0.0, dimtree=True), graph=False)
ck.cp_als(ck.DenseTensor((24, 20, 18), rng.random(24 * 20 * 18)), ck.AlsConfig(rank=300, max_iters=2, tol=0.0),
          graph=False)  # R > 256: the multi-CTA sweep solve
os.environ["CPK_SOLVE"] = "kernel"
ck.cp_als(ck.DenseTensor((24, 20, 18), rng.random(24 * 20 * 18)), ck.AlsConfig(rank=300, max_iters=2, tol=0.0),
          graph=False)
print("ok")
