"""Debug helper: build one seeded case on cuda:0 and report the first level that differs from the oracle."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, wt_inputs
import paper_1610_05994_b200 as wt

def run(seed, n, sigma, kind, dtype=None):
    S = wt_inputs.random_case(seed, n, sigma, kind, dtype=dtype)
    d = torch.from_numpy(S.view(np.int32) if S.dtype == np.uint32 else S).cuda()
    try:
        t = wt.build(d, sigma)
    except Exception as e:
        print("build error", seed, n, sigma, kind, e); return False
    ot = oracle.build(S, sigma)
    B = t.bitmaps.cpu().numpy().view(np.uint32)
    for l in range(ot.L):
        if not np.array_equal(B[l], ot.bitmaps[l]):
            bad = np.nonzero(B[l] != ot.bitmaps[l])[0]
            print(f"seed={seed} n={n} sigma={sigma} {kind}: level {l} differs in {bad.size} words, first {bad[:8]}")
            return False
    return True

if __name__ == "__main__":
    ok = True
    for sigma in [1000, 4096, 65536, 300, 256, 27]:
        for kind in ["uniform", "zipf", "sorted", "runs"]:
            for n in [1024, 5000, 70000]:
                ok &= run(sigma + n, n, sigma, kind)
    print("ALL OK" if ok else "FAILURES")
