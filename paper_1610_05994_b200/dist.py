"""Multi-GPU domain decomposition: the paper's dd
 with one segment per GPU.

Each rank holds a contiguous segment of S (rank order = segment order) and:

1. builds its segment's tree with the single-GPU path (createPartialBA,
   P:691-732) -- no communication;
2. all-gathers the segments' lengths and node offsets (NCCL); the merged node
   offsets C are their sum (``wt_dd_offsets``), and the per-(level, node,
   segment) destinations follow from them alone (the per-level prefix over
   segments, Alg. 2 lines 7-8): ``wt_dd_plan_async`` gives, for every
   level l, part p and segment g, the contiguous range of g's level-l bits
   that lands in part p (part p = the merged tree's 512-bit blocks rank p owns,
   ``wt_dd_part_blocks``);
3. exchanges bit words point to point (NCCL send/recv in one group; ``dd_exchange``):
   rank g sends rank p the words of its level-l bitmap covering that range
   -- about L*n/8 bytes over the whole job, each rank receiving ~1/G of it;
4. merges its own part of every level from the received words (mergeBA,
   P:734-765: ``wt_dd_merge_level``, every merged word written once, the
   boundary words of the paper's concat assembled from both neighbours' bits);
5. rescans its part's superblocks (``wt_superblocks``) from a base = the ones
   of the level before the part: sum over segments of rank1 at the plan's lo,
   one all-reduce of L x G counts.

The result is a tree SHARDED by position: rank p holds bitmap words
[16 b, 16 e) and superblock entries [b, e] of every level (b, e its block
range) and the whole C.  This module is orchestration (collectives and
argument marshalling); every step of the build and the merge runs in the
library's kernels.  The exchange and the plan arithmetic are device-agnostic,
so they run under gloo on CPU tensors in the tests (tests/test_multirank.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import (WaveletTree, build, dd_merge_level, dd_offsets, dd_part_blocks, dd_plan_device, rank1,
               superblocks, _sync)


@dataclass
class ShardedTree:
    """Rank `part`'s share of a tree of n symbols split into `parts` parts."""
    n: int
    sigma: int
    levels: int
    parts: int
    part: int
    block_begin: int
    block_end: int
    bitmaps: torch.Tensor       # (L, 16 * (block_end - block_begin)) int32: merged words [16 b, 16 e)
    superblocks: torch.Tensor   # (L, block_end - block_begin + 1) int64: merged entries [b, e]
    node_offsets: torch.Tensor  # (2^L + 1,) int64: the merged C


def word_range(lo: int, hi: int) -> tuple[int, int]:
    """Words of a segment's level bitmap that hold its bits [lo, hi)."""
    if hi <= lo:
        return 0, 0
    return lo // 32, (hi + 31) // 32


def dd_exchange(local_bits: torch.Tensor, plan: np.ndarray, rank: int, group=None) -> list:
    """Point-to-point exchange of bit words: for every level l and part p, this
    rank (segment `rank`) sends the words of local_bits[l] covering
    plan[l, p, rank] to rank p, and receives from every segment g the words
    covering plan[l, rank, g].  Returns recv[l][g] (1-D int32 tensors; the own
    segment's words are a slice, no copy).  Works for NCCL (CUDA tensors) and
    gloo (CPU tensors)."""
    L, parts, k, _ = plan.shape
    ops, recv = [], [[None] * k for _ in range(L)]
    dev = local_bits.device
    for l in range(L):
        for g in range(k):
            a, b = word_range(int(plan[l, rank, g, 0]), int(plan[l, rank, g, 1]))
            if g == rank:
                recv[l][g] = local_bits[l, a:b] if b > a else local_bits.new_empty(0)
            elif b > a:
                buf = torch.empty(b - a, dtype=local_bits.dtype, device=dev)
                recv[l][g] = buf
                ops.append(dist.P2POp(dist.irecv, buf, g, group))
            else:
                recv[l][g] = local_bits.new_empty(0)
        for p in range(parts):
            if p == rank:
                continue
            a, b = word_range(int(plan[l, p, rank, 0]), int(plan[l, p, rank, 1]))
            if b > a:
                ops.append(dist.P2POp(dist.isend, local_bits[l, a:b].contiguous(), p, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return recv


def merge_part(seg_offsets: list, offsets: torch.Tensor, sigma: int, n: int, parts: int, part: int, plan: np.ndarray,
               recv: list, bases, stream=None) -> ShardedTree:
    """Steps 4-5 on one device: part `part` of every level merged from recv[l][g]
    (the words of segment g covering plan[l, part, g]) and its superblocks from
    bases[l] (ones of level l before the part)."""
    L = plan.shape[0]
    k = len(seg_offsets)
    dev = offsets.device
    b_lo, b_hi = dd_part_blocks(n, parts, part)
    nw = 16 * (b_hi - b_lo)
    bits = torch.empty((L, nw), dtype=torch.int32, device=dev)
    sbs = torch.empty((L, b_hi - b_lo + 1), dtype=torch.int64, device=dev)
    for l in range(L):
        base = [32 * word_range(int(plan[l, part, g, 0]), int(plan[l, part, g, 1]))[0] for g in range(k)]
        dd_merge_level(seg_offsets, offsets, sigma, n, l, [recv[l][g] for g in range(k)], base, 16 * b_lo,
                       16 * b_hi, bits[l], stream)
        superblocks(bits[l], b_hi - b_lo, int(bases[l]), sbs[l], stream)
    return ShardedTree(n=n, sigma=sigma, levels=L, parts=parts, part=part, block_begin=b_lo, block_end=b_hi,
                       bitmaps=bits, superblocks=sbs, node_offsets=offsets)


def ones_before_parts(tree: WaveletTree, plan: np.ndarray, seg: int) -> torch.Tensor:
    """This segment's share of every part's superblock base: ones of its level-l
    bits before plan[l, p, seg, 0], for all (l, p) -> (L, parts) int64 tensor
    (summed over the segments by one all-reduce)."""
    L, parts = plan.shape[0], plan.shape[1]
    dev = tree.node_offsets.device
    if L == 0 or tree.n == 0:
        return torch.zeros((L, parts), dtype=torch.int64, device=dev)
    lv = torch.arange(L, dtype=torch.int32, device=dev).repeat_interleave(parts)
    pos = torch.from_numpy(np.ascontiguousarray(plan[:, :, seg, 0]).reshape(-1)).to(dev)
    return rank1(tree, lv, pos).view(L, parts)


def build_distributed(seq_local: torch.Tensor, sigma: int, group=None, stream=None) -> ShardedTree:
    """The multi-GPU build: this rank's contiguous segment of S in `seq_local`
    (a CUDA tensor; segments in rank order), every rank calls it.  Returns this
    rank's part of the merged tree."""
    G = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev = seq_local.device
    local = build(seq_local, sigma, stream=stream)   # step 1 (one sync: the range flag)
    L = local.levels
    # step 2: segment lengths and node offsets of every rank
    ns = torch.tensor([local.n], dtype=torch.int64, device=dev)
    all_n = [torch.empty_like(ns) for _ in range(G)]
    dist.all_gather(all_n, ns, group=group)
    n = int(sum(int(x.item()) for x in all_n))
    Cs = torch.empty((G, local.node_offsets.numel()), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(Cs, local.node_offsets, group=group)
    seg_offsets = [Cs[g] for g in range(G)]
    C = torch.empty_like(local.node_offsets)
    dd_offsets(seg_offsets, sigma, C, stream)
    plan_d = dd_plan_device(seg_offsets, sigma, n, G, stream)
    _sync(stream)
    plan = plan_d.cpu().numpy()
    # step 5's bases: sum over segments of rank1 at the plan's lo
    bases = ones_before_parts(local, plan, r)
    if L:
        dist.all_reduce(bases, group=group)
    # step 3: point-to-point exchange of the bit words
    recv = dd_exchange(local.bitmaps, plan, r, group)
    # steps 4-5: this rank's part
    out = merge_part(seg_offsets, C, sigma, n, G, r, plan, recv, bases[:, r].tolist() if L else [], stream)
    _sync(stream)
    return out
