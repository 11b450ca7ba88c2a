"""Spill instructions inside each loop of a kernel's SASS (a loop = the span
from a backward branch's target to the branch): python tools/loop_spills.py obj [name-filter]"""
import re
import subprocess
import sys

obj = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
for fn in re.split(r"\n\s+Function : ", out)[1:]:
    name = fn.split("\n", 1)[0].strip()
    if flt not in name:
        continue
    ins = re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", fn)
    addr = [(int(a, 16), t.strip()) for a, t in ins]
    loops = []
    for a, t in addr:
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
        if m and m.group(1) and int(m.group(1), 16) < a and a - int(m.group(1), 16) > 0x400:
            lo = int(m.group(1), 16)
            sp = sum(1 for b, u in addr if lo <= b <= a and re.search(r"\b(LDL|STL)\b", u))
            loops.append(f"[{lo:#x},{a:#x}] {(a - lo) // 16 + 1} instr, {sp} LDL/STL")
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    print(dem.replace("hsgn_dev::", "")[:60], "|", "; ".join(loops))
