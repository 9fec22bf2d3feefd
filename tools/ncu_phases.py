"""Stall samples and executed instructions per barrier-delimited phase of a
kernel (one CTA-wide phase per BAR.SYNC), from an ncu report.

    python tools/ncu_phases.py report.ncu-rep kernel_regex
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
isrc, ist, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) == len(h) and r[ist] != h[ist]]
half = len(body) // 2
if half and body[0][isrc] == body[half][isrc]:
    body = body[:half]  # the page lists the function twice
tot_s = sum(float(r[ist]) for r in body) or 1.0
tot_e = sum(int(r[iex]) for r in body) or 1
start = 0
for i, r in enumerate(body + [None]):
    if r is None or "BAR.SYNC" in r[isrc]:
        seg = body[start:i + 1] if r is not None else body[start:]
        s = sum(float(x[ist]) for x in seg)
        e = sum(int(x[iex]) for x in seg)
        if s or e:
            print(f"lines {start:5d}-{i:5d}: samples {100 * s / tot_s:5.1f}%  instr {100 * e / tot_e:5.1f}%")
        start = i + 1
