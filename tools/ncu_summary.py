"""Summarize ncu captures (run here, no GPU) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_c4_mode0_r01.ncu-rep [...] --tag r01
    python tools/ncu_summary.py --launches gpurun_out/launches_r01.csv --tag r01
    python tools/ncu_summary.py gpurun_out/prof_c3_mode1.ncu-rep --tag r01 --aux   # not the c4 kernel

Writes profiles/<tag>_<report-stem>.txt (key metrics, stall reasons, shared-
memory wavefronts per LDS, SASS opcode mix) and updates
profiles/ncu_summary.json (dram bytes per launch of the dominant kernel,
read by bench.py for the roofline `traffic` field).
"""

import argparse
import csv
import io
import json
import subprocess
from collections import Counter, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.avg.per_second",
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize_report(path: Path, tag: str) -> dict:
    rows = ncu_csv(["-i", str(path), "--page", "raw"])
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    lines = [f"# ncu --set full summary: {path.name}", f"kernel: {m.get('Kernel Name', ('?',))[0]}", ""]
    for k in KEYS:
        if k in m:
            lines.append(f"{k:70s} {m[k][0]} {m[k][1]}")
    stalls = []
    for h, (v, u) in m.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    lines += ["", "stall reasons (warps per issue-active cycle):"]
    for v, n in sorted(stalls, reverse=True)[:10]:
        lines.append(f"  {n:28s} {v:.3f}")
    # SASS opcode mix and shared wavefronts per LDS
    src = ncu_csv(["-i", str(path), "--page", "source", "--print-source", "sass"])
    sh = src[1]
    isrc, iex = sh.index("Source"), sh.index("Instructions Executed")
    iwf = sh.index("L1 Wavefronts Shared")
    ops, lds_n, lds_wf = Counter(), 0, 0
    for r in src[2:]:
        try:
            ex = int(r[iex])
        except (ValueError, IndexError):
            continue
        toks = r[isrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        ops[op] += ex
        if op.startswith("LDS") and ex:
            lds_n += ex
            lds_wf += int(r[iwf] or 0)
    total = sum(ops.values())
    lines += ["", f"SASS mix (warp instructions, total {total:.3e}):"]
    for op, n in ops.most_common(12):
        lines.append(f"  {op:28s} {n:.3e}  {100 * n / total:5.1f}%")
    if lds_n:
        lines.append(f"  shared wavefronts per LDS: {lds_wf / lds_n:.2f}")
    out = PROF / f"{tag}_{path.stem}.txt"
    out.write_text("\n".join(lines) + "\n")
    print(out)

    def num(k):
        try:
            return float(m[k][0].replace(",", ""))
        except (KeyError, ValueError):
            return None

    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = num("dram__bytes_read.sum") * scale.get(m["dram__bytes_read.sum"][1], 1)
    wr = num("dram__bytes_write.sum") * scale.get(m["dram__bytes_write.sum"][1], 1)
    return {"report": path.name, "dram_bytes_per_launch": rd + wr,
            # DFMA issues on the fp64 pipe, DMMA on the tensor pipe's dmma
            # subpipe (the same FP64 datapath, tools/microbench4.cu)
            "fp64_pipe_pct": max(num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") or 0.0,
                                 num("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")
                                 or 0.0),
            "duration_ms": num("gpu__time_duration.sum")}


def summarize_launches(path: Path, tag: str):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    t, n = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        t[r[ik]] += v
        n[r[ik]] += 1
    tot = sum(t.values())
    lines = [f"# launch list ({path.name}): gpu__time_duration.sum, --clock-control none; cold, serialized", ""]
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        lines.append(f"{v / 1e6:10.3f} ms  {100 * v / tot:6.2f}%  n={n[k]:4d}  {k}")
    out = PROF / f"{tag}_launches.txt"
    out.write_text("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--launches")
    ap.add_argument("--aux", action="store_true",
                    help="not the bench's dominant kernel: write the .txt summaries only, leave ncu_summary.json")
    ap.add_argument("--out", default=None, help="directory for the summaries (default profiles/)")
    a = ap.parse_args()
    if a.out:
        PROF = Path(a.out)
    PROF.mkdir(exist_ok=True)
    if a.launches:
        summarize_launches(Path(a.launches), a.tag)
    res = [summarize_report(Path(p), a.tag) for p in a.reports]
    if res and not a.aux:
        summ = {"tag": a.tag, "reports": res,
                "dram_bytes_per_launch": sum(r["dram_bytes_per_launch"] for r in res) / len(res)}
        (PROF / "ncu_summary.json").write_text(json.dumps(summ, indent=1) + "\n")
