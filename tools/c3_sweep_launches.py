"""Two eager c3 CP-ALS sweeps (for an ncu launch list of one sweep)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402

dims = tuple(int(x) for x in (sys.argv[1:] or [128, 128, 128, 128]))
rank = 256
y = ck.DenseTensor.uniform(dims, seed=0, device="cuda")
model, trace = ck.cp_als(y, ck.AlsConfig(rank=rank, max_iters=3, tol=0.0), graph=False)
print([sum(m) for m in trace.mttkrp_seconds], trace.other_seconds)
