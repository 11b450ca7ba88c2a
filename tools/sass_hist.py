"""Aggregate an `ncu --page source --csv --print-source sass` dump by opcode:
executed warp instructions and stall samples.  Usage: sass_hist.py file.csv [points]"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
    hdr.index("Warp Stall Sampling (All Samples)")
ex, st = Counter(), Counter()
tot_ex = tot_st = 0
for r in rows[2:]:
    if len(r) <= iex:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc])
    if not m:
        continue
    op = m.group(2)
    if not r[iex].isdigit():
        continue
    e = int(r[iex] or 0)
    s = int(r[ist] or 0)
    ex[op] += e
    st[op] += s
    tot_ex += e
    tot_st += s
pts = float(sys.argv[2]) if len(sys.argv) > 2 else 0
print(f"total warp instr {tot_ex:.4g}" + (f"  per point (thread instr) {tot_ex * 32 / pts:.1f}" if pts else ""))
for op, e in ex.most_common(40):
    print(f"{op:10s} {e:14d} {100 * e / tot_ex:6.2f}%  " + (f"{e * 32 / pts:7.1f}/pt  " if pts else "")
          + f"stall {100 * st[op] / max(tot_st, 1):5.1f}%")
