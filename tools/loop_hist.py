"""Opcode histogram of the longest loop of a kernel (static SASS):
python tools/loop_hist.py obj name-filter [obj2 name-filter2]"""
import collections
import re
import subprocess
import sys


def hist(obj, flt):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    for fn in re.split(r"\n\s+Function : ", out)[1:]:
        if flt not in fn.split("\n", 1)[0]:
            continue
        ins = [(int(a, 16), t.strip()) for a, t in re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", fn)]
        best = None
        for a, t in ins:
            m = re.search(r"BRA\s+0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a and (best is None or a - int(m.group(1), 16) > best[1] - best[0]):
                best = (int(m.group(1), 16), a)
                break
        lo, hi = best
        c = collections.Counter()
        for a, t in ins:
            if lo <= a <= hi:
                op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
                c[op] += 1
        return c


a = hist(sys.argv[1], sys.argv[2])
if len(sys.argv) > 3:
    b = hist(sys.argv[3], sys.argv[4])
    keys = sorted(set(a) | set(b), key=lambda k: -(a[k] + b[k]))
    print(f"{'op':10s} {sum(a.values()):6d} {sum(b.values()):6d}")
    for k in keys:
        if a[k] != b[k]:
            print(f"{k:10s} {a[k]:6d} {b[k]:6d} {b[k] - a[k]:+5d}")
else:
    print(sum(a.values()), a.most_common())
