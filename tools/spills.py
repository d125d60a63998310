"""List kernels with register spills from build/ptxas.log (nvcc -Xptxas -v)."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "build/ptxas.log").read().splitlines()
cur = None
for ln in log:
    m = re.search(r"Function properties for (\S+)", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur and (int(m.group(1)) or int(m.group(2))):
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        print(f"{m.group(1):>5} st {m.group(2):>5} ld  {name[:150]}")
