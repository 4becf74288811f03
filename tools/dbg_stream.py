import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_05994_b200 as wt
import wt_inputs
print([l.split()[-1] for l in open('/proc/self/maps') if 'cudart' in l][:3])
S = wt_inputs.random_case(3, 200_000, 256, "zipf")
d = torch.from_numpy(S).cuda()
for name, s in [("default", None), ("side", torch.cuda.Stream())]:
    try:
        t = wt.build_async(d, 256, stream=s); torch.cuda.synchronize(); print(name, "ok")
    except Exception as e:
        print(name, "FAIL", e)
S, sig = wt_inputs.generate(3)
d = torch.from_numpy(S).cuda()
try:
    t = wt.build(d, sig); print("cfg3 ok")
except Exception as e:
    print("cfg3 FAIL", e)
