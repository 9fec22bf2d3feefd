"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list.

    python tools/launch_table.py gpurun_out/launches.csv [--last N]
"""
import argparse
import collections
import csv

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--last", type=int, default=0, help="only the last N launches")
a = ap.parse_args()
rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
ks = [(r[ik].split("(")[0][:80], float(r[iv].replace(",", "")) * SCALE[r[iu]]) for r in rows[1:]]
if a.last:
    ks = ks[-a.last:]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, t in ks:
    agg[k][0] += 1
    agg[k][1] += t
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:12.1f} us {v[0]:5d} launches  {100 * v[1] / tot:5.1f}%  {k}")
print(f"{tot:12.1f} us total, {len(ks)} launches")
