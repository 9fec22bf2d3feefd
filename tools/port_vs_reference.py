"""The bench's CPU arm times the oracle TILE port (oracle/mttkrp_ref.c, C +
OpenMP) because the reference (Python + numba) cannot travel to the GPU box.
This tool, run HERE (the container has /root/reference and numba), times the
reference's own `mttkrp_tile` against the port on the same c4 slab, plan and
thread count, and checks they agree -- the evidence that the port is a fair
stand-in.  Writes profiles/r01_port_vs_reference.json.

    python tools/port_vs_reference.py [--depth 2] [--reps 2]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from oracle import gen, oracle  # noqa: E402

DIMS, RANK, SEED, NT, F = (1024, 1024, 1024), 2000, 0, 131044, 16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import cpkern.mttkrp as rm  # the reference, imported from /root/reference
    from cpkern.dtensor import DenseTensor
    from cpkern.kruskal import KruskalTensor

    dims = (DIMS[0], DIMS[1], a.depth)
    fs = gen.bench_factors(DIMS, RANK, SEED)
    sub = [fs[0], fs[1], np.ascontiguousarray(fs[2][:a.depth])]
    y = gen.splitmix_uniform(int(np.prod(dims)), SEED)
    w = oracle.max_threads()
    flops = 3 * 2 * int(np.prod(dims)) * RANK * 2

    def port():
        return [oracle.mttkrp_tile(y, dims, k, sub, None, f_cols=F, n_t=NT, workers=w)[0] for k in range(3)]

    yt, m = DenseTensor(dims, y), KruskalTensor(np.ones(RANK), sub)

    def ref():
        out = []
        for k in range(3):
            n_s = int(np.prod(dims)) // dims[k]
            plan = rm.MttkrpPlan(rm.Variant.TILE, k, unroll=F, tile_volume=min(NT, n_s), workers=w)
            out.append(rm.run(yt, m, plan).matrix)
        return out

    res = {}
    for name, fn in (("port", port), ("reference", ref)):
        fn()  # warm-up (numba compile, page-in)
        best, out = float("inf"), None
        for _ in range(a.reps):
            t0 = time.perf_counter()
            out = fn()
            best = min(best, time.perf_counter() - t0)
        res[name] = {"seconds": best, "gflops": flops / best / 1e9, "out": out}
    err = max(oracle.rel_err(p, r) for p, r in zip(res["port"]["out"], res["reference"]["out"]))
    summary = {"slab": list(dims), "rank": RANK, "tile_volume": NT, "unroll": F, "threads": w,
               "port_seconds": res["port"]["seconds"], "port_gflops": res["port"]["gflops"],
               "reference_seconds": res["reference"]["seconds"],
               "reference_gflops": res["reference"]["gflops"],
               "port_over_reference": res["reference"]["seconds"] / res["port"]["seconds"],
               "max_rel_err": err, "host": os.uname().nodename, "cpu_count": os.cpu_count()}
    print(json.dumps(summary, indent=1))
    (ROOT / "profiles" / "r01_port_vs_reference.json").write_text(json.dumps(summary, indent=1) + "\n")


if __name__ == "__main__":
    main()
