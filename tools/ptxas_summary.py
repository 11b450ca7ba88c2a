"""Per-kernel registers / spills from the build's ptxas log:
python tools/ptxas_summary.py [paper_2601_02540_b200/_native/ptxas.log]"""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 else "paper_2601_02540_b200/_native/ptxas.log"
name = None
for line in open(log):
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = dem.replace("hsgn_dev::", "").replace("(hsgn_dev::StageArgs, hsgn_dev::KPtrs)", "")
        print(f"{m.group(1):>4} regs  spill st/ld {spill[0]:>4}/{spill[1]:<4} {dem}")
        name = None
