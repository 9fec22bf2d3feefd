"""Per-kernel stack / spill summary from `nvcc -Xptxas -v` output on stdin.

    nvcc ... -Xptxas -v -c file.cu 2>&1 | python tools/ptxas_spills.py [filter]
"""
import re
import subprocess
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
for line in sys.stdin:
    m = re.search(r"(Compiling entry function|Function properties for) '?([^' ]+)'?", line)
    if m:
        cur = m.group(2)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur and flt in cur:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        print(f"{m.group(1):>6} stack {m.group(2):>6} st {m.group(3):>6} ld  {name[:110]}")
