"""Aggregate ncu source-page stall samples per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > f.csv; python tools/ncu_lines.py f.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None; hdr = None; items = []; tot = 0; inst_tot = 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        s = int(r[4]); ni = int(r[5]); ie = int(r[7])
    except ValueError:
        continue
    tot += s; inst_tot += ie
    items.append((s, ni, ie, f"{fname}:{r[0]}", r[1][:100]))
items.sort(reverse=True)
print("total samples", tot, "warp-instr executed", inst_tot)
for s, ni, ie, loc, src in items[:top]:
    print(f"{s:6d} {100*s/max(tot,1):5.1f}% notiss={ni:6d} inst={ie:10d} {loc:22s} {src}")

# instruction counts per line
agg = {}
fname = None; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        ie = int(r[7])
    except ValueError:
        continue
    agg[(fname, int(r[0]))] = (ie, r[1][:100])
tot = sum(v[0] for v in agg.values())
print("\nTOTAL warp instr", tot)
for (f, l), (ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ie:11d} {100*ie/tot:5.1f}% {f}:{l:<5d} {src}")
