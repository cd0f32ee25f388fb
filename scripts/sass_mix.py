"""Opcode mix of an ncu source page (SASS, with execution counts):
    ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv
    python scripts/sass_mix.py s.csv [iterations]   # per-iteration counts if given"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
# several kernels: keep the first section (or the one named by $KERNEL)
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] or [0]
want = __import__("os").environ.get("KERNEL")
k0 = next((i for i in starts if want and want in rows[i][1]), starts[0])
k1 = next((i for i in starts if i > k0), len(rows))
rows = rows[k0:k1]
h = rows[1]
isrc, iex, istall = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
per = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cnt = collections.Counter()
stall = collections.Counter()
for r in rows[2:]:
    if len(r) <= iex:
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    if not r[iex].isdigit():
        continue
    cnt[o] += int(r[iex] or 0)
    stall[o] += int(r[istall] or 0)
tot = sum(cnt.values())
tst = sum(stall.values())
for o, c in cnt.most_common(40):
    print(f"{o:10s} {c / per:10.1f} {100 * c / tot:5.1f}%   stall samples {100 * stall[o] / max(1, tst):5.1f}%")
print(f"total {tot / per:.1f}")
