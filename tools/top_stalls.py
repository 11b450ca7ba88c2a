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


def reasons(path, addr_suffix):
    """Per-reason stall samples of one instruction (address suffix)."""
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    for r in rows[2:]:
        if len(r) > cols[-1] and r[0].endswith(addr_suffix):
            return {hdr[i][6:]: int(r[i] or 0) for i in cols if int(r[i] or 0)}
