import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import wt_inputs, oracle
import paper_1610_05994_b200 as wt
cfg = int(sys.argv[1]); n = int(sys.argv[2]); K = int(sys.argv[3])
S, sigma = wt_inputs.generate(cfg, n)
d = torch.from_numpy(S.view(np.int32) if S.dtype == np.uint32 else S).cuda()
try:
    t = wt.build(d, sigma)
except Exception as e:
    print("build failed", e)
B = t.bitmaps.cpu().numpy().view(np.uint32)
SB = t.superblocks.cpu().numpy().view(np.uint64)
for l in range(K):
    ob, osb, _ = oracle.build_level(S, sigma, l)
    okb = np.array_equal(B[l], ob); oks = np.array_equal(SB[l], osb)
    nb = int((B[l] != ob).sum())
    print(f"level {l}: bitmap {'ok' if okb else 'BAD %d words' % nb} superblocks {'ok' if oks else 'BAD'}")
