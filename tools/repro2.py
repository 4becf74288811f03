import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import wt_inputs, oracle
import paper_1610_05994_b200 as wt
cfg = int(sys.argv[1]); n = int(sys.argv[2])
S, sigma = wt_inputs.generate(cfg, n)
d = torch.from_numpy(S.view(np.int32) if S.dtype == np.uint32 else S).cuda()
t = wt.build(d, sigma)
torch.cuda.synchronize()
print("built", cfg, n)
ot = oracle.build(S, sigma)
B = t.bitmaps.cpu().numpy().view(np.uint32)
for l in range(ot.L):
    if not np.array_equal(B[l], ot.bitmaps[l]):
        print("level", l, "differs"); break
else:
    print("bitmaps ok", np.array_equal(t.node_offsets.cpu().numpy().view(np.uint64), ot.node_offsets))
