"""Top stall-sampled SASS instructions (with the preceding instructions for
context) from `ncu --page source --csv --print-source sass`:
python tools/top_stalls.py file.csv [n] [context]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ist, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) > iex]
tot = sum(int(r[ist] or 0) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
order = sorted(range(len(body)), key=lambda k: -int(body[k][ist] or 0))
for k in order[:n]:
    r = body[k]
    print(f"{100 * int(r[ist]) / tot:5.1f}%  {r[ia][-5:]}  {r[isrc].strip()}   (exec {r[iex]})")
    for c in range(max(0, k - ctx), k):
        print(f"        {body[c][ia][-5:]}  {body[c][isrc].strip()}")
