"""NEXT-3 on one GPU: the paper's domain decomposition (k segment builds, then
the merge) against the direct build, on a bench config.  Reports the merge time
alone (what a k-GPU or out-of-core build adds after its per-segment builds) and
checks the merged tree equals the direct one.  usage: python tools/dd_bench.py [cfg] [k ...]"""
import ctypes
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
    ks = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
    S, sigma = wt_inputs.generate(cfg)
    w = S.dtype.itemsize
    d = torch.from_numpy(S.view(np.int32) if w == 4 else S).cuda()
    n = d.numel()
    direct = wt.build(d, sigma)
    for k in ks:
        step = -(-(-(-n // k)) // (16 // w)) * (16 // w)
        cuts = [min(i * step, n) for i in range(k)] + [n]
        segs = [wt.build(d[cuts[i]:cuts[i + 1]], sigma) for i in range(k)]
        out = wt.alloc_tree(n, sigma, 4, d.device)
        arr = (wt.WtTree * k)(*[t._ctree() for t in segs])
        ns = (ctypes.c_uint64 * k)(*[t.n for t in segs])
        scratch = torch.empty((int(wt._lib.wt_dd_merge_scratch_bytes(n)),), dtype=torch.uint8, device=d.device)
        ct = out._ctree()
        s = torch.cuda.current_stream()

        def merge():
            st = wt._lib.wt_dd_merge(k, ctypes.cast(arr, ctypes.c_void_p), ctypes.cast(ns, ctypes.c_void_p), sigma,
                                     ctypes.byref(ct), scratch.data_ptr(), scratch.numel(), s.cuda_stream)
            assert st == wt.WT_OK
        for _ in range(2):
            merge()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            merge()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        same = (torch.equal(out.bitmaps, direct.bitmaps) and torch.equal(out.superblocks, direct.superblocks)
                and torch.equal(out.node_offsets, direct.node_offsets))
        print(json.dumps({"config": cfg, "k": k, "n": n, "merge_ms": ms, "merged_equals_direct": same}), flush=True)
        assert same
        del segs, out, scratch
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
