"""Select query throughput with and without the select index (NEXT-1) on a
bench config's tree: m random (c, j) pairs over present symbols, CUDA events
around the batched query after warm-up.  usage: python tools/select_bench.py [cfg] [m]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1610_05994_b200 as wt  # noqa: E402
import wt_inputs  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
    S, sigma = wt_inputs.generate(cfg)
    w = S.dtype.itemsize
    d = torch.from_numpy(S.view(np.int32) if w == 4 else S).cuda()
    tree = wt.build(d, sigma)
    idx = wt.select_index(tree)
    C = tree.node_offsets.cpu().numpy()
    cnt = np.diff(C)
    present = np.nonzero(cnt)[0]
    rng = np.random.default_rng(7)
    c = present[rng.integers(0, present.size, m)]
    j = 1 + (rng.random(m) * cnt[c]).astype(np.int64)
    c_t = torch.from_numpy(c.astype(np.int32)).cuda()
    j_t = torch.from_numpy(j).cuda()
    res = {}
    for name, kw in (("plain", {}), ("indexed", {"index": idx})):
        for _ in range(3):
            out = wt.select(tree, c_t, j_t, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            out = wt.select(tree, c_t, j_t, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[name] = {"ms": ms, "Mqueries_per_s": m / (ms * 1e-3) / 1e6}
        res[name + "_out"] = out
    assert torch.equal(res["plain_out"], res["indexed_out"])
    # index build time
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        wt.select_index(tree)
    e1.record()
    torch.cuda.synchronize()
    line = {"config": cfg, "queries": m, "plain": res["plain"], "indexed": res["indexed"],
            "index_build_ms": e0.elapsed_time(e1) / 5, "index_bytes": idx.numel() * 4}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
