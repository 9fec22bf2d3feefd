"""Rank-tile sweep measured by ncu (north star: "the rank-tile size is ...
checked by an ncu sweep reporting achieved HBM GB/s and FP64-pipe
utilisation against the B200 peaks").

    python tools/ncu_sweep.py --dims 512 512 512 --rank 64 --out profiles/r01_ncu_sweep_c2.csv

For every (engine, rank tile) and mode: one ncu capture of the MTTKRP kernel
(tools/profile_one.py under `ncu --metrics ...`), reporting its duration,
DRAM bytes -> achieved HBM GB/s and fraction of the measured copy
bandwidth, and FP64-pipe utilisation (max of the DFMA pipe and the tensor
pipe's DMMA subpipe, % of peak sustained) -- plus which plan the auto
heuristic picks.  ncu times are cold-cache and serialized: compare configs,
do not read them as bench values.
"""
import argparse
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "%": 1.0}


def capture(dims, rank, mode, engine, rank_tile):
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "--csv", "-k", "regex:mttkrp_f64",
           "-s", "1", "-c", "1", sys.executable, str(ROOT / "tools" / "profile_one.py"), "--mode", str(mode),
           "--reps", "2", "--rank", str(rank), "--engine", engine, "--rank-tile", str(rank_tile), "--dims",
           *map(str, dims)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600).stdout
    rows = [r for r in csv.reader(io.StringIO(out[out.find('"ID"'):])) if len(r) > 10]
    if len(rows) < 2:
        return None
    h = rows[0]
    iname, iunit, ival, ikern = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"), \
        h.index("Kernel Name")
    vals = {}
    kern = None
    for r in rows[1:]:
        kern = r[ikern]
        vals[r[iname]] = float(r[ival].replace(",", "")) * SCALE.get(r[iunit], 1.0)
    return kern, vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs="+", default=[512, 512, 512])
    ap.add_argument("--rank", type=int, default=64)
    ap.add_argument("--configs", nargs="+",
                    default=["dmma:64", "dmma:128", "dmma:256", "tma:64", "tma:128", "tma:256", "cpdmma:64",
                             "cpdmma:128", "cpasync:32", "cpasync:64", "cpasync:128"])
    ap.add_argument("--out", default="profiles/ncu_sweep.csv")
    a = ap.parse_args()
    dims, rank = tuple(a.dims), a.rank
    peaks = {"hbm_gbs": 6508.2}
    try:
        peaks["hbm_gbs"] = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        pass
    auto = json.loads(subprocess.run(
        [sys.executable, "-c", "import json,sys; sys.path.insert(0, %r); import paper_2510_14891_b200 as ck; "
         "from paper_2510_14891_b200.mttkrp import MttkrpPlan, Variant, resolve_plan; "
         "print(json.dumps([resolve_plan(MttkrpPlan(Variant.B200, k), %r, %d) for k in range(%d)]))"
         % (str(ROOT), dims, rank, len(dims))], capture_output=True, text=True).stdout.strip().splitlines()[-1])
    rows = []
    for cfg in a.configs:
        engine, rt = cfg.split(":")
        for k in range(len(dims)):
            res = capture(dims, rank, k, engine, int(rt))
            if res is None:
                print(f"skip {cfg} mode {k}", flush=True)
                continue
            kern, v = res
            t = v["gpu__time_duration.sum"]
            dram = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
            fp64 = max(v.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0),
                       v.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 0.0))
            n = 1
            for e in dims:
                n *= e
            row = {"engine": engine, "rank_tile": int(rt), "mode": k + 1, "ms": t * 1e3,
                   "tflops_alg": 2 * n * rank * (len(dims) - 1) / t / 1e12, "dram_gb": dram / 1e9,
                   "hbm_gbs": dram / t / 1e9, "hbm_frac": dram / t / 1e9 / peaks["hbm_gbs"],
                   "fp64_pipe_pct": fp64,
                   "auto": int(auto[k]["engine"] == engine and auto[k]["rank_tile"] == int(rt)),
                   "kernel": kern.split("(")[0][:60]}
            rows.append(row)
            print(json.dumps(row), flush=True)
    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    with open(out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)
    print(json.dumps({"out": str(out), "rows": len(rows), "auto": auto}))


if __name__ == "__main__":
    main()
