"""Top SASS lines by warp-stall samples for one kernel of an ncu report.

    python tools/ncu_hot.py report.ncu-rep kernel_regex [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
isrc, ist, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) == len(h) and r[ist] != h[ist]]
tot = sum(float(r[ist]) for r in body) or 1.0
print(f"{len(body)} SASS lines, {tot:.0f} samples")
for i, r in sorted(enumerate(body), key=lambda x: -float(x[1][ist]))[:n]:
    print(f"{i:6d} {100 * float(r[ist]) / tot:5.1f}%  exec {r[iex]:>8}  {r[isrc].strip()[:90]}")
if len(sys.argv) > 4:  # context lines around an index
    c = int(sys.argv[4])
    for i in range(max(0, c - 12), min(len(body), c + 6)):
        r = body[i]
        print(f"{i:6d} {float(r[ist]):5.0f}  exec {r[iex]:>8}  {r[isrc].strip()[:90]}")
