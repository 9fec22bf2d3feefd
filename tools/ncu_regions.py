"""Instruction-count and stall-sample histogram over SASS line windows of one
kernel in an ncu report (find the loop that costs the time).

    python tools/ncu_regions.py report.ncu-rep kernel_regex [window] [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
win = int(sys.argv[3]) if len(sys.argv) > 3 else 50
top = int(sys.argv[4]) if len(sys.argv) > 4 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
isrc, ist, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) == len(h) and r[ist] != h[ist]]
tot_ex = sum(int(r[iex]) for r in body) or 1
tot_s = sum(float(r[ist]) for r in body) or 1.0
print(f"{len(body)} SASS lines, {tot_ex} warp instructions, {tot_s:.0f} samples")
ex, st = collections.Counter(), collections.Counter()
for i, r in enumerate(body):
    ex[i // win] += int(r[iex])
    st[i // win] += float(r[ist])
for k, v in sorted(st.items(), key=lambda x: -x[1])[:top]:
    first = body[k * win][isrc].strip()[:50]
    print(f"lines {k * win:5d}-{k * win + win - 1:5d}: samples {100 * v / tot_s:5.1f}%  exec {100 * ex[k] / tot_ex:5.1f}%  {first}")
