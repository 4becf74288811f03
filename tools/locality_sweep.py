"""NEXT-2: the paper's locality sweep on the GPU.

cont = n/sigma copies of every symbol, sorted; rand = the same multiset at
random positions; n = 2^30 4-byte symbols, sigma = 2^y
for y in {4, 6, 8, 10, 12, 14}.  The inputs are made on the device (seeded
torch generator): they are synthetic and the bench contract's host-side
generators are not involved.  Every build is checked with oracle-independent
invariants at full size:
  * node offsets: C[c] = c * n / sigma (the multiset is the same for cont and rand);
  * per level, popcount(B_l) = n / 2 and the last superblock equals it;
  * cont: every T_l equals S (the scatter is the identity), so B_l is bit
    (L-1-l) of S[j] -- checked word by word against bits packed from S.
Times: CUDA events around K builds on the build stream after warm-up.

usage: python tools/locality_sweep.py [--n N] [--steps K] [--out FILE]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1610_05994_b200 as wt  # noqa: E402


def pack_bits(bits: torch.Tensor, words: int) -> torch.Tensor:
    """bool[n] -> int32 words (LSB-first, zero-padded to `words`), as the library stores them."""
    n = bits.numel()
    pad = torch.zeros(words * 32, dtype=torch.int64, device=bits.device)
    pad[:n] = bits.to(torch.int64)
    w = (pad.view(words, 32) << torch.arange(32, device=bits.device, dtype=torch.int64)).sum(dim=1)
    return torch.where(w >= 2 ** 31, w - 2 ** 32, w).to(torch.int32)


def popcount(words: torch.Tensor) -> int:
    x = words.to(torch.int64) & 0xFFFFFFFF
    c = torch.zeros_like(x)
    for k in range(32):
        c += (x >> k) & 1
    return int(c.sum().item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 30)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ys", default="4,6,8,10,12,14")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = args.n
    gen = torch.Generator(device=dev)
    gen.manual_seed(2016)
    stream = torch.cuda.current_stream()
    rows = []
    for y in [int(v) for v in args.ys.split(",")]:
        sigma = 1 << y
        cont = (torch.arange(n, device=dev, dtype=torch.int64) * sigma // n).to(torch.int32)
        for kind in ("cont", "rand"):
            S = cont if kind == "cont" else cont[torch.randperm(n, generator=gen, device=dev)]
            tree = wt.alloc_tree(n, sigma, 4, dev)
            ws = wt.alloc_workspace(n, sigma, 4, dev)
            st = torch.zeros(1, dtype=torch.int32, device=dev)
            for _ in range(2):
                wt.build_async(S, sigma, tree, ws, st, stream=stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                wt.build_async(S, sigma, tree, ws, st, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            assert int(st.item()) == wt.WT_OK
            # invariants
            C = tree.node_offsets
            expect_C = torch.arange(sigma + 1, device=dev, dtype=torch.int64) * (n // sigma)
            ok_c = bool(torch.equal(C, expect_C))
            L = tree.levels
            ok_pop, ok_bits = True, True
            for l in range(L):
                b = tree.bitmaps[l]
                pop = popcount(b)
                ok_pop &= pop == n // 2 and int(tree.superblocks[l, -1].item()) == pop
                if kind == "cont":
                    ref = pack_bits(((S >> (L - 1 - l)) & 1).bool(), b.numel())
                    ok_bits &= bool(torch.equal(ref, b))
            row = {"y": y, "sigma": sigma, "kind": kind, "n": n, "ms_per_build": ms,
                   "Gsym_per_s": n / (ms * 1e-3) / 1e9, "C_closed_form": ok_c, "popcounts": ok_pop,
                   "cont_identity_bits": ok_bits if kind == "cont" else None}
            print(json.dumps(row), flush=True)
            rows.append(row)
            assert ok_c and ok_pop and ok_bits, row
            del tree, ws, S
            torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
