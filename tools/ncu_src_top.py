"""Top SASS instructions by warp-stall samples from `ncu --page source --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iall = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[iall] or 0) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("total samples", tot)
idx = sorted(range(len(body)), key=lambda i: -int(body[i][iall] or 0))[:n]
for i in sorted(idx):
    r = body[i]
    print(f"{i:5d} {int(r[iall]):6d} {100*int(r[iall])/tot:5.1f}%  {r[isrc].strip()[:90]}")
