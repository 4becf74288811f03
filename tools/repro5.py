import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import wt_inputs
import paper_1610_05994_b200 as wt
cfg = int(sys.argv[1]); n = int(sys.argv[2])
S, sigma = wt_inputs.generate(cfg, n)
w = S.dtype.itemsize
d = torch.from_numpy(S.view(np.int32) if S.dtype == np.uint32 else S).cuda()
L = wt.sizes(n, sigma, w).levels
ws = wt.alloc_workspace(n, sigma, w, d.device)
tree = wt.alloc_tree(n, sigma, w, d.device)
try:
    wt.build(d, sigma, tree=tree, workspace=ws)
except Exception as e:
    print("build:", e)
off = wt.debug_offsets(n, sigma, w)
print(off)
W = ws.cpu().numpy()
cnt0 = W[off["cnt"]: off["cnt"] + off["cnt_stride"]].view(np.uint32)
cnt1 = W[off["cnt"] + off["cnt_stride"]: off["cnt"] + 2 * off["cnt_stride"]].view(np.uint32)
S64 = S.astype(np.int64)
for lvl, buf in [(18, cnt0), (17, cnt1)]:
    exp = np.bincount(S64 >> (L - lvl), minlength=1 << lvl)
    got = buf[: 1 << lvl].astype(np.int64)
    bad = np.nonzero(exp != got)[0]
    print(f"counts level {lvl}: {bad.size} wrong", bad[:10], exp[bad[:5]], got[bad[:5]], "sum", got.sum(), n)
# T_17 (written by pass 16 into bufA) vs S stably sorted by the top 17 bits
T = W[off["bufA"]: off["bufA"] + n * w].view(S.dtype)
exp = S[np.argsort(S64 >> (L - 17), kind="stable")]
bad = np.nonzero(T != exp)[0]
print("T_17 wrong positions:", bad.size, bad[:10])
if bad.size:
    i = bad[0]; tile = 512
    print("first bad at", i, "tile", i // tile, "offset", i % tile, "got", T[i - 2:i + 3], "exp", exp[i - 2:i + 3])
    print("bad tiles:", np.unique(bad // tile)[:20], "count", np.unique(bad // tile).size)
