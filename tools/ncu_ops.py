"""Opcode histogram (executed warp instructions) from an ncu source-page csv (SASS view)."""
import csv, sys, re
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
cnt = Counter(); tot = 0
for r in rows[2:]:
    try: ie = int(r[idx['Instructions Executed']])
    except (ValueError, IndexError): continue
    src = r[1].strip()
    src = re.sub(r'^@!?U?P[T0-9]+\s+', '', src)
    op = src.split()[0] if src else '?'
    cnt[op] += ie; tot += ie
n = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
for op, c in cnt.most_common(40):
    print(f"{op:28s} {c:11d} {100*c/tot:5.1f}%  {32*c/n:6.2f}/sym")
print("total", tot, f"{32*tot/n:.2f}/sym")
