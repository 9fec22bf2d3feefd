"""Hash of the speculative solve's output (X = G Gamma^-1 through
chol_small + chol_rows, CPK_SOLVE=kernel) per rank, for a bit-identity A/B
of two library builds (run once per --lib, compare the lines)."""
import argparse
import hashlib
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--ranks", type=int, nargs="+", default=[1, 3, 5, 31, 32, 33, 64, 100, 128, 200, 256, 300, 384, 512])
a = ap.parse_args()
from paper_2510_14891_b200 import _lib  # noqa: E402

if a.lib:
    _lib.LIB_PATH = Path(a.lib).resolve()
os.environ["CPK_SOLVE"] = "kernel"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_14891_b200 import cpals  # noqa: E402

dev = torch.device("cuda", 0)
for r in a.ranks:
    rng = np.random.Generator(np.random.Philox(r))
    x = rng.random((2 * r + 3, r))
    gamma = torch.from_numpy(x.T @ x + 1e-3 * np.eye(r)).to(dev)
    g = torch.from_numpy(rng.random((130, r))).to(dev)
    solver = cpals._Solver(dev, 130, r)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    cpals._solve_spec(solver, gamma, g, info)
    torch.cuda.synchronize()
    print(json.dumps({"rank": r, "info": int(info.item()),
                      "sha": hashlib.sha256(g.cpu().numpy().tobytes()).hexdigest()[:16]}), flush=True)
