"""Join an ncu SASS source page (execution counts) with nvdisasm -g line info:
per source line, executed instructions (and top opcodes).

    nvdisasm -g X.cubin > all.sass
    ncu -i R.ncu-rep --page source --csv --print-source sass > s.csv
    python scripts/sass_lines.py all.sass KERNEL_MANGLED s.csv [per]"""
import collections
import csv
import re
import sys

sass, kern, ncsv = sys.argv[1], sys.argv[2], sys.argv[3]
per = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
lines = open(sass).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":"))
off2line = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'line (\d+)', l)
    if "//##" in l and m:
        cur = int(m.group(1))
        fm = re.search(r'File "([^"]+)"', l)
        curf = fm.group(1).split("/")[-1] if fm else "?"
        continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+(.*?);', l)
    if m and cur is not None:
        off2line[int(m.group(1), 16)] = (curf, cur)
rows = list(csv.reader(open(ncsv)))
h = rows[1]
ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
base = int(rows[2][ia], 16)
agg = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if len(r) <= iex:
        continue
    off = int(r[ia], 16) - base
    key = off2line.get(off, ("?", -1))
    n = int(r[iex] or 0)
    agg[key] += n
    tok = r[isrc].strip().split()
    o = tok[1] if tok and tok[0].startswith("@") else (tok[0] if tok else "?")
    ops[key][o] += n
tot = sum(agg.values())
for key, n in agg.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 50):
    top = ", ".join(f"{o} {c / per:.0f}" for o, c in ops[key].most_common(4))
    print(f"{n / per:8.1f} {100 * n / tot:5.1f}%  {key[0]}:{key[1]}  {top}")
