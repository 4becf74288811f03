"""Quick parity check of builds with interior fused groups (k_quad) against the
oracle, on assorted small cases; prints the first mismatching level."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
import wt_inputs  # noqa: E402
import paper_1610_05994_b200 as wt  # noqa: E402

cases = [(16, 5000, "uniform"), (16, 100_000, "uniform"), (256, 300_000, "zipf"), (256, 8192 * 3 + 17, "uniform"),
         (32, 77_777, "runs"), (256, 1_000_003, "sorted"), (1 << 12, 200_001, "zipf"), (1 << 16, 123_457, "zipf"),
         (1 << 16, 500_000, "uniform"), (1 << 20, 300_001, "zipf"), (200, 1, "uniform"), (200, 15, "uniform"),
         (17, 8191, "uniform"), (1000, 65536, "runs"), (256, 5, "uniform")]
bad = 0
for i, (sigma, n, kind) in enumerate(cases):
    S = wt_inputs.random_case(1000 + i, n, sigma, kind)
    d = torch.from_numpy(S.view(np.int32) if S.dtype == np.uint32 else S).cuda()
    plan = wt.launch_plan(n, sigma, S.itemsize)
    try:
        tree = wt.build(d, sigma)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(f"sigma={sigma} n={n} {kind}: ERROR {e}")
        bad += 1
        continue
    ot = oracle.build(S, sigma)
    B = tree.bitmaps.cpu().numpy().view(np.uint32)
    SB = tree.superblocks.cpu().numpy().view(np.uint64)
    C = tree.node_offsets.cpu().numpy().view(np.uint64)
    msg = []
    if not np.array_equal(C, ot.node_offsets):
        msg.append("C")
    for l in range(ot.L):
        if not np.array_equal(B[l], ot.bitmaps[l]):
            k = int(np.nonzero(B[l] != ot.bitmaps[l])[0][0])
            msg.append(f"B{l}@w{k}({np.count_nonzero(B[l] != ot.bitmaps[l])})")
        if not np.array_equal(SB[l], ot.superblocks[l]):
            k = int(np.nonzero(SB[l] != ot.superblocks[l])[0][0])
            msg.append(f"SB{l}@{k}")
    print(f"sigma={sigma} n={n} {kind} dtype={S.dtype} quads={plan.count('quad')}: {'OK' if not msg else ' '.join(msg[:8])}",
          flush=True)
    bad += bool(msg)
print("BAD", bad)
