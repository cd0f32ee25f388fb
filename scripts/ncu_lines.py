"""Aggregate ncu warp-stall samples per CUDA source line from a report:
    python scripts/ncu_lines.py report.ncu-rep [top]
(uses `ncu -i ... --page source --print-source=cuda,sass --csv`)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr = None, None
agg = collections.Counter(); stall = collections.defaultdict(collections.Counter); txt = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit(): continue
    d = dict(zip(hdr[2:], r[2:]))  # sass columns (after line no + source)
    try: s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError: continue
    key = (cur_file, int(r[0]))
    agg[key] += s; txt[key] = r[1].strip()[:70]
    for k, v in d.items():
        if k.startswith("stall_") and v not in ("", "0"):
            try: stall[key][k[6:]] += int(float(v))
            except ValueError: pass
tot = sum(agg.values()) or 1
print(f"total samples {tot}")
for key, s in agg.most_common(top):
    st = ", ".join(f"{k} {v}" for k, v in stall[key].most_common(3))
    print(f"{100*s/tot:5.1f}% {key[0]}:{key[1]:<4} {txt[key]:<70} | {st}")
