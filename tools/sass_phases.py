"""Per-barrier-phase instruction counts and stall reasons of an ncu capture's SASS page."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) >= len(h)]
iS, iE, iSm = h.index("Source"), h.index("Instructions Executed"), h.index("# Samples")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
segs, cur = [], {}
for r in data:
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            cur[h[i]] = cur.get(h[i], 0) + v
    cur["_inst"] = cur.get("_inst", 0) + int(r[iE] or 0)
    cur["_samples"] = cur.get("_samples", 0) + int(r[iSm] or 0)
    if r[iS].strip().startswith("BAR"):
        segs.append(cur)
        cur = {}
segs.append(cur)
tot = sum(s.get("_inst", 0) for s in segs)
print("total warp instructions", tot)
for k, s in enumerate(segs):
    items = sorted(((v, c) for c, v in s.items() if not c.startswith("_")), reverse=True)[:5]
    print(k, s.get("_inst"), s.get("_samples"), items)
top = sorted(((int(r[iSm] or 0), r[iS].strip()[:70]) for r in data), reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for t in top:
    print(t)
