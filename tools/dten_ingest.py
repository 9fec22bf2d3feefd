"""Time DTEN ingest into HBM (cpk_dten_load_slab_f64) on a config-4-sized file.

    python tools/dten_ingest.py [--dims 1024 1024 1024] [--dir /tmp]

Writes the file from a device-generated tensor, then times a whole-tensor
load and the mode-0 slab of one rank out of 8 (the sharded driver's ingest).
The file was just written, so reads may come from the page cache: this
measures the loader's pinned-staging/H2D pipeline, not the disk.
"""
import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402
from paper_2510_14891_b200 import sharded  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs="+", default=[1024, 1024, 1024])
ap.add_argument("--dir", default="/tmp")
a = ap.parse_args()
dims = tuple(a.dims)
path = Path(a.dir) / "ingest_probe.dten"
t = ck.DenseTensor.uniform(dims, seed=0, device="cuda")
t0 = time.perf_counter()
ck.write_dten(path, t)
tw = time.perf_counter() - t0
nbytes = 8 * int(np.prod(dims))
print(f"write {nbytes / 1e9:.2f} GB: {tw:.2f} s")
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    full = ck.read_dten(path, device="cuda")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"whole tensor -> HBM: {dt:.3f} s, {nbytes / dt / 1e9:.1f} GB/s; equal={torch.equal(full.data, t.data)}")
del full
part = sharded.partition_for(dims, 8, mode=0)
torch.cuda.synchronize()
t0 = time.perf_counter()
slab = sharded.dten_slab(path, part, 3, device="cuda")
torch.cuda.synchronize()
dt = time.perf_counter() - t0
sb = 8 * slab.size
print(f"rank 3/8 mode-0 slab ({sb / 1e9:.2f} GB, {dims[1] * int(np.prod(dims[2:]))} runs): {dt:.3f} s, "
      f"{sb / dt / 1e9:.1f} GB/s")
os.unlink(path)
