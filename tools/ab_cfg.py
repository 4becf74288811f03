"""A/B probe: one config's build, ms per build and per launch kind (median of runs).
usage: python tools/ab_cfg.py CFG [reps]   (WT_LIB=... selects an experiment library)"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1610_05994_b200 as wt
import wt_inputs

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
S, sigma = wt_inputs.generate(cfg)
w = S.dtype.itemsize
d = torch.from_numpy(S.view(np.int32) if w == 4 else S).cuda()
n = S.size
tree = wt.alloc_tree(n, sigma, w, d.device)
ws = wt.alloc_workspace(n, sigma, w, d.device)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    wt.build_async(d, sigma, tree=tree, workspace=ws, status=st)
torch.cuda.synchronize()
assert int(st.item()) == 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    wt.build_async(d, sigma, tree=tree, workspace=ws, status=st)
e1.record()
torch.cuda.synchronize()
plan = wt.launch_plan(n, sigma, w)
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * len(plan))] for _ in range(reps)]
for k in range(reps):
    wt.set_profile_events(evs[k])
    wt.build_async(d, sigma, tree=tree, workspace=ws, status=st)
wt.set_profile_events(None)
torch.cuda.synchronize()
per = [sum(evs[k][2 * i].elapsed_time(evs[k][2 * i + 1]) for k in range(reps)) / reps for i in range(len(plan))]
kinds = {}
for p, t in zip(plan, per):
    kinds[p] = kinds.get(p, 0.0) + t
print(f"cfg{cfg} {wt.LIB_PATH.split('/')[-1]}: {e0.elapsed_time(e1) / reps:.4f} ms/build  " +
      " ".join(f"{k}={v:.4f}" for k, v in kinds.items()))
print("   per launch:", " ".join(f"{t:.3f}" for t in per))
