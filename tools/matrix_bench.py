"""Wavelet matrix (NEXT-4) build throughput on the bench configs, beside the
wavelet tree: K builds back to back on one stream, CUDA events, after warm-up.
usage: python tools/matrix_bench.py [cfg ...]"""
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


def timed(fn, k=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]
    for cfg in cfgs:
        S, sigma = wt_inputs.generate(cfg)
        w = S.dtype.itemsize
        n = S.size
        d = torch.from_numpy(S.view(np.int32) if w == 4 else S).cuda()
        ws = wt.alloc_workspace(n, sigma, w, d.device)
        mx = wt.build_matrix(d, sigma, workspace=ws)
        cm = mx._cmatrix()
        st = torch.zeros(1, dtype=torch.int32, device=d.device)
        stream = torch.cuda.current_stream()

        def build_m():
            wt._lib.wt_matrix_build_async(d.data_ptr(), n, sigma, w, ctypes.byref(cm), ws.data_ptr(), ws.numel(),
                                          st.data_ptr(), stream.cuda_stream)
        tree = wt.alloc_tree(n, sigma, w, d.device)

        def build_t():
            wt.build_async(d, sigma, tree, ws, st, stream=stream)
        mm, mt = timed(build_m), timed(build_t)
        assert int(st.item()) == wt.WT_OK
        print(json.dumps({"config": cfg, "n": n, "sigma": sigma, "matrix_ms": mm, "matrix_Gsym_s": n / mm / 1e6,
                          "tree_ms": mt, "tree_Gsym_s": n / mt / 1e6}), flush=True)
        del ws, mx, tree, d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
