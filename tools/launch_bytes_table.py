"""Per-launch table (time, DRAM bytes, GB/s) from an ncu --csv launch list
with gpu__time_duration.sum / dram__bytes_read.sum / dram__bytes_write.sum:
    python tools/launch_bytes_table.py gpurun_out/dt_launch_c5p_dt2.csv [--min-us 20]"""
import argparse
import csv
import io

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "msecond": 1e3, "nsecond": 1e-3, "s": 1e6, "second": 1e6}

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--min-us", type=float, default=20.0)
a = ap.parse_args()
txt = open(a.csv).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
launches = {}
for r in rows:
    m = launches.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
    m[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * SCALE[r["Metric Unit"]]
print(f"| id | kernel | us | DRAM read GB | DRAM write GB | GB/s |\n|---|---|---|---|---|---|")
for i, m in sorted(launches.items()):
    t = m["gpu__time_duration.sum"]
    if t < a.min_us:
        continue
    rd, wr = m["dram__bytes_read.sum"] / 1e9, m["dram__bytes_write.sum"] / 1e9
    name = m["name"].split("(")[0].replace("void ", "")
    print(f"| {i} | `{name}` | {t:.1f} | {rd:.3f} | {wr:.3f} | {(rd + wr) * 1e9 / (t * 1e-6) / 1e9:.0f} |")
