"""ALU-pipe opcodes per CUDA source line (ncu source page, --print-source cuda,sass)."""
import csv, sys, re
from collections import defaultdict
ALU = ('LOP3', 'SHF', 'SEL', 'ISETP', 'IADD3', 'PRMT', 'PLOP3', 'VIADD', 'LEA', 'FLO', 'BMSK', 'SGXT', 'IABS', 'IMNMX', 'VIMNMX', 'ICMP', 'P2R', 'R2P', 'POPC', 'BREV')
rows = list(csv.reader(open(sys.argv[1])))
n = float(sys.argv[2]); top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur = None; fname = None
alu = defaultdict(int); allc = defaultdict(int); src = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if not r or r[0] == "Line No": continue
    if r[0] != "":
        cur = (fname, r[0]); src[cur] = r[1][:90]; continue
    if len(r) < 10 or cur is None: continue
    try: ie = int(r[7])
    except ValueError: continue
    op = re.sub(r'^@!?U?P[T0-9]+\s+', '', r[3].strip()).split()
    op = op[0].split('.')[0] if op else '?'
    allc[cur] += ie
    if op in ALU: alu[cur] += ie
tot = sum(alu.values())
print(f"ALU total {32*tot/n:.2f}/sym  all {32*sum(allc.values())/n:.2f}/sym")
for k, v in sorted(alu.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{32*v/n:6.2f} alu/sym {32*allc[k]/n:6.2f} all/sym  {k[0]}:{k[1]:5s} {src.get(k,'')}")
