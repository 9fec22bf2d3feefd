"""Shared-memory wavefronts per SASS instruction of one kernel (ncu source page).

    python tools/ncu_lds.py report.ncu-rep [kernel_regex] [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "regex:mttkrp"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
rows = rows[hi:]
iw, iid, iex, isrc = (h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"),
                      h.index("Instructions Executed"), h.index("Source"))
body = [r for r in rows[1:] if len(r) == len(h)]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(num(r[iw]) for r in body)
print(f"total shared wavefronts {tot:.3e}, ideal {sum(num(r[iid]) for r in body):.3e}")
for r in sorted(body, key=lambda r: -num(r[iw]))[:n]:
    ex = num(r[iex]) or 1
    print(f"{num(r[iw]):10.3e} ({num(r[iw]) / ex:5.2f}/inst, ideal {num(r[iid]) / ex:5.2f})  exec {ex:9.0f}  {r[isrc].strip()[:80]}")
