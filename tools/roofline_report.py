"""One table per BASELINE config from a bench.py JSON line: measured time,
the north-star roofline max(8N / HBM, 2 N R (d-1) / FP64 peak), the issued
FP64 fraction (2 N R per mode: the Khatri-Rao scaling is folded per o-group)
and the HBM fraction, next to the CPU reference arm.

    python tools/roofline_report.py profiles/r02e_bench.json [ref.json] > profiles/r02_roofline.md
"""
import json
import sys

d = json.loads(open(sys.argv[1]).read())
ref = json.loads(open(sys.argv[2]).read()) if len(sys.argv) > 2 else None
HBM = d["rank_sweep"]["hbm_peak_gbs"] * 1e9
FP64 = d["roofline"]["peak"] * 1e12  # live probe of this run


def row(name, dims, r, ms_per_mode):
    n = 1
    for e in dims:
        n *= e
    k = len(dims)
    t = sum(ms_per_mode) / len(ms_per_mode) * 1e-3
    roof = max(8 * n / HBM, 2 * n * r * (k - 1) / FP64)
    return (f"| {name} | {'x'.join(map(str, dims))}, R = {r} | {t * 1e3:.3f} | {roof * 1e3:.3f} | {roof / t:.2f} | "
            f"{2 * n * r / t / FP64:.3f} | {8 * n / t / HBM:.3f} |")


print(f"# Roofline per config ({sys.argv[1]})\n")
print(f"FP64 peak {FP64 / 1e12:.2f} TFLOP/s (live probe), HBM {HBM / 1e9:.0f} GB/s (MEASURED_PEAKS.json); "
      "roofline = max(8 N / HBM, 2 N R (d-1) / FP64) per mode; the issued fraction counts 2 N R per mode "
      "(the (d-1) Khatri-Rao multiplies are folded once per o-group, so the north-star fraction can exceed 1).\n")
print("| config | shape | ms per mode | roofline ms | roofline / measured | FP64 issued | HBM |")
print("|---|---|---|---|---|---|---|")
print(row("c4 headline", d["config"]["dims"], d["config"]["rank"], d["per_mode_ms"]))
for p in d["rank_sweep"]["points"]:
    print(row(f"c2 shape (rank sweep)", d["rank_sweep"]["shape"], p["rank"], p["ms_per_mode"]))
cp, c5 = d["cp_als"], d["cp_als_c5"]
print("\n| CP-ALS | sec / sweep | roofline sweep | roofline / measured |")
print("|---|---|---|---|")
tree = " [dimension tree, split {}]".format(cp["tree_split"]) if cp.get("tree_split") else ""
print(f"| {cp['config']} ({cp['iters']} sweeps){tree} | {cp['sec_per_iter']:.4f} (graph replay "
      f"{cp['graph_sec_per_replayed_sweep']:.4f}) | {cp['roofline_sec_per_iter']:.4f} | {cp['roofline_frac']:.2f} |")
if cp.get("per_mode"):
    pm = cp["per_mode"]
    print(f"| same, per-mode sweep (4 MTTKRPs, the reference's structure) | {pm['sec_per_iter']:.4f} (graph replay "
          f"{pm['graph_sec_per_replayed_sweep']:.4f}) | {cp['roofline_sec_per_iter']:.4f} | "
          f"{cp['roofline_sec_per_iter'] / pm['sec_per_iter']:.2f} |")
if "sec_per_iter" in c5 and c5.get("sec_per_iter"):
    tree = " [dimension tree, split {}]".format(c5["tree_split"]) if c5.get("tree_split") else ""
    print(f"| {c5['config']} ({c5['gpus']} GPU){tree} | {c5['sec_per_iter']:.4f} | {c5['roofline_sec_per_iter']:.4f} | "
          f"{c5['roofline_frac']:.2f} |")
    if c5.get("per_mode"):
        pm = c5["per_mode"]
        print(f"| same, per-mode sweep (3 MTTKRPs) | {pm['sec_per_iter']:.4f} | {c5['roofline_sec_per_iter']:.4f} | "
              f"{c5['roofline_sec_per_iter'] / pm['sec_per_iter']:.2f} |")
    for p in c5.get("projection", {}).get("points", []):
        roof = c5["roofline_sec_per_iter"] / p["gpus"]
        extra = (f"; per-mode {p['per_mode_rank0_sec_per_iter']:.4f}"
                 if p.get("per_mode_rank0_sec_per_iter") else "")
        print(f"| c5 rank-0 sweep at P = {p['gpus']} (projection, collectives elided) | {p['rank0_sec_per_iter']:.4f}"
              f"{extra} | {roof:.4f} | {roof / p['rank0_sec_per_iter']:.2f} |")
print("\n| baseline | value |")
print("|---|---|")
print(f"| this repo, c4 device-resident | {d['value'] / 1e3:.2f} TFLOP/s |")
print(f"| this repo, c4 end to end from pinned host memory | {d['e2e']['value'] / 1e3:.2f} TFLOP/s |")
print(f"| cuBLAS DGEMM partial-KRP MTTKRP, same GPU | {d['gemm_baseline']['gflops'] / 1e3:.2f} TFLOP/s |")
print(f"| DFMA (CUDA-core FMA) engine, same GPU | {d['dfma_engine']['gflops'] / 1e3:.2f} TFLOP/s |")
print(f"| optional float32 path (3xTF32) | {d['fp32_path']['gflops'] / 1e3:.1f} TFLOP/s at {max(d['fp32_path']['rel_frobenius_vs_fp64']):.1e} |")
cb = d["cpu_baseline"]
print(f"| CPU reference arm ({cb['kind']}, {cb['cores']} threads): {cb['sample'][:80]} | {cb['value']:.1f} GFLOP/s |")
if ref:
    print(f"| `bench.py --impl reference` line | {ref['value']:.1f} GFLOP/s; reference cp_als c3 {ref['cp_als']['sec_per_iter']:.2f} s/sweep |")
