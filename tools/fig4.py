"""MTTKRP GFLOP/s and roofline fraction vs rank R (BASELINE.json's metric),
paper Fig. 4-style: the B200 kernel (auto plan) beside the paper's two GPU
baselines on the same device -- MTTKRP-ELEM (N R FP64 atomics) and the dense
GEMM MTTKRP (partial KRPs + cuBLAS DGEMM).

    python tools/fig4.py --shape 512 512 512 --ranks 16 32 64 128 256 512 1000 2000 \
        --out profiles/r01_fig4_c2.csv

Per rank and mode: best-of-reps CUDA-event time; columns: algorithmic
TFLOP/s (2 N R (d-1) / t), paper GFLOP/s (N R d / t / 1024^3) and the
north-star roofline fraction max(8N/HBM, 2NR(d-1)/FP64) / t.  ELEM is skipped
above --elem-max-rank (N R atomics), GEMM when its scratch would not fit.
"""
import argparse
import csv
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2510_14891_b200 as ck  # noqa: E402
from paper_2510_14891_b200 import _lib  # noqa: E402
from paper_2510_14891_b200.baselines import gemm_scratch_bytes, mttkrp_elem_atomic, mttkrp_gemm_cublas  # noqa: E402
from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, mttkrp_device, resolve_plan  # noqa: E402
from paper_2510_14891_b200.perfmodel import roofline_seconds  # noqa: E402


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs="+", default=[512, 512, 512])
    ap.add_argument("--ranks", type=int, nargs="+", default=[16, 32, 64, 128, 256, 512, 1000, 2000])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--elem-max-rank", type=int, default=128)
    ap.add_argument("--out", default="profiles/fig4.csv")
    a = ap.parse_args()
    dims = tuple(a.shape)
    d, n = len(dims), int(np.prod(dims))
    dev = torch.device("cuda", 0)
    y = ck.DenseTensor.uniform(dims, seed=0, device=dev).data
    v = _lib.C.c_double(0)
    _lib.check(_lib.load().cpk_fp64_peak_probe(_lib.C.byref(v), None))
    peak = v.value
    free = torch.cuda.mem_get_info()[0]
    rows = []
    for r in a.ranks:
        rng = np.random.Generator(np.random.Philox(1))
        fs = [torch.from_numpy(rng.random((e, r))).to(dev) for e in dims]
        roof = roofline_seconds(dims, r, fp64_peak=peak)
        for k in range(d):
            impls = {"b200": lambda: mttkrp_device(y, dims, fs, k, None, MttkrpPlan(Variant.B200, k))}
            if r <= a.elem_max_rank:
                impls["elem_atomic"] = lambda: mttkrp_elem_atomic(y, dims, fs, k)
            if 2.5 * gemm_scratch_bytes(dims, r, k) < free:
                impls["gemm_cublas"] = lambda: mttkrp_gemm_cublas(y, dims, fs, k)
            for name, fn in impls.items():
                t = timed(fn, a.reps)
                row = {"impl": name, "rank": r, "mode": k + 1, "time_s": t,
                       "tflops_alg": 2 * n * r * (d - 1) / t / 1e12, "paper_gflops": n * r * d / t / 1024 ** 3,
                       "roofline_frac": roof / t}
                if name == "b200":
                    p = resolve_plan(MttkrpPlan(Variant.B200, k), dims, r)
                    row["plan"] = f"{p['engine']} rt={p['rank_tile']} splits={p['splits']}"
                rows.append(row)
                print(json.dumps(row), flush=True)
                torch.cuda.empty_cache()
    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    keys = ["impl", "rank", "mode", "time_s", "tflops_alg", "paper_gflops", "roofline_frac", "plan"]
    with open(out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=keys)
        w.writeheader()
        w.writerows(rows)
    # per (impl, rank): mean over modes
    agg = {}
    for row in rows:
        agg.setdefault((row["impl"], row["rank"]), []).append(row)
    with open(out.with_suffix(".agg.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["impl", "rank", "mean_time_s", "tflops_alg", "roofline_frac"])
        for (impl, r), grp in agg.items():
            w.writerow([impl, r, statistics.fmean(x["time_s"] for x in grp),
                        statistics.fmean(x["tflops_alg"] for x in grp),
                        statistics.fmean(x["roofline_frac"] for x in grp)])
    print(json.dumps({"out": str(out), "fp64_peak": peak}))


if __name__ == "__main__":
    main()
