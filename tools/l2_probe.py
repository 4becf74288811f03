"""Probe: cfg2-shaped builds (n = 2^N u8, sigma = 4): ms per build and per launch."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1610_05994_b200 as wt
import wt_inputs

N = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
S, sigma = wt_inputs.generate(2, 1 << N)
d = torch.from_numpy(S).cuda()
tree = wt.alloc_tree(S.size, sigma, 1, d.device)
ws = wt.alloc_workspace(S.size, sigma, 1, d.device)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(reps):
    wt.build_async(d, sigma, tree=tree, workspace=ws, status=st)
torch.cuda.synchronize()
assert int(st.item()) == 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    wt.build_async(d, sigma, tree=tree, workspace=ws, status=st)
e1.record()
torch.cuda.synchronize()
plan = wt.launch_plan(S.size, sigma, 1)
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * len(plan))] for _ in range(10)]
for k in range(10):
    wt.set_profile_events(evs[k])
    wt.build_async(d, sigma, tree=tree, workspace=ws, status=st)
wt.set_profile_events(None)
torch.cuda.synchronize()
per = [sum(evs[k][2 * i].elapsed_time(evs[k][2 * i + 1]) for k in range(10)) / 10 for i in range(len(plan))]
print(f"n=2^{N}: {e0.elapsed_time(e1) / 10:.4f} ms/build  " + " ".join(f"{p}={t:.4f}" for p, t in zip(plan, per)))
