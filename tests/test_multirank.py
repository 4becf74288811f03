"""The N > 1 path of bench.py ("replicas only" -- every rank builds
its own tree, no data-path collective): the job's step time is the slowest rank's
(all_reduce MAX) and the reported value is the whole-job throughput.  Runs on CPU
with the gloo backend, world size 2, rendezvous on 127.0.0.1."""
import os
import socket
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local_ms = [3.0, 5.5][rank]                      # rank 1 is the straggler
    ms = bench.max_over_ranks(local_ms, world, torch.device("cpu"))
    value = bench.job_throughput(1 << 28, world, ms)
    out[rank] = (ms, value)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_max_and_throughput():
    world, port = 2, _free_port()
    out = mp.Manager().dict()
    mp.spawn(_rank_main, args=(world, port, out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == 5.5             # both ranks report the slowest rank
    expect = 2 * (1 << 28) / (5.5e-3) / 1e9          # both replicas' symbols over that time
    assert abs(out[0][1] - expect) < 1e-9 and out[0][1] == out[1][1]


def test_single_rank_is_identity():
    import bench
    assert bench.max_over_ranks(4.25, 1, torch.device("cpu")) == 4.25
    assert abs(bench.job_throughput(1 << 20, 1, 1.0) - (1 << 20) / 1e6) < 1e-12


# ------------------------------------------------------------------ multi-GPU dd
# The N-rank build's host logic on CPU tensors under gloo: every rank builds its
# segment's tree (here the oracle stands in for the GPU build), the ranks
# all-gather node offsets, compute the library's plan (wt_dd_plan), exchange bit
# words with the library's dd_exchange, and every rank's part -- assembled from
# what it received by the test-side reference walk (tests/dd_ref.py) -- must be
# the oracle's whole-sequence tree on that part; the superblock bases summed by
# all-reduce must be the oracle's superblocks at the part starts.

def _dd_rank_main(rank, world, port, out, sigma, n, seed):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import dd_ref
    import oracle
    import wt_inputs
    import paper_1610_05994_b200 as wt
    from paper_1610_05994_b200.dist import dd_exchange, word_range
    S = wt_inputs.random_case(seed, n, sigma, "zipf")
    cuts = [rank_ * n // world for rank_ in range(world)] + [n]
    mine = oracle.build(S[cuts[rank]:cuts[rank + 1]], sigma)
    L = mine.L
    Cloc = torch.from_numpy(mine.node_offsets.view(np.int64).copy())
    Cs = [torch.empty_like(Cloc) for _ in range(world)]
    dist.all_gather(Cs, Cloc)
    seg_C = [c.numpy().view(np.uint64) for c in Cs]
    plan = wt.dd_plan_host(seg_C, sigma, world)
    recv = dd_exchange(torch.from_numpy(mine.bitmaps.view(np.int32).copy()), plan, rank)
    full = oracle.build(S, sigma)
    b, e = wt.dd_part_blocks(n, world, rank)
    q_lo, q_hi = min(n, 512 * b), min(n, 512 * e)
    ok = True
    for l in range(L):
        part = np.zeros(q_hi - q_lo, np.uint8)
        dest = dd_ref.merged_dest(seg_C, L, l)
        for g in range(world):
            lo, hi = int(plan[l, rank, g, 0]), int(plan[l, rank, g, 1])
            a, _ = word_range(lo, hi)
            got = dd_ref.unpack(recv[l][g].numpy().view(np.uint32), 32 * recv[l][g].numel())
            part[dest[g][lo:hi] - q_lo] = got[lo - 32 * a: hi - 32 * a]
        want = dd_ref.unpack(full.bitmaps[l], n)[q_lo:q_hi]
        ok &= bool(np.array_equal(part, want))
    # superblock bases: this segment's ones before the plan's lo, summed over ranks
    bases = torch.zeros((L, world), dtype=torch.int64)
    for l in range(L):
        bits = dd_ref.unpack(mine.bitmaps[l], mine.n).astype(np.int64)
        csum = np.concatenate([[0], np.cumsum(bits)])
        for p in range(world):
            bases[l, p] = int(csum[int(plan[l, p, rank, 0])])
    dist.all_reduce(bases)
    for l in range(L):
        for p in range(world):
            bp, _ = wt.dd_part_blocks(n, world, p)
            ok &= int(bases[l, p]) == int(full.superblocks[l][bp])
    out[rank] = ok
    dist.barrier()
    dist.destroy_process_group()


import pytest  # noqa: E402


@pytest.mark.parametrize("world,sigma,n,seed", [(2, 256, 20011, 1), (3, 1 << 12, 30000, 2), (2, 4, 1537, 3),
                                                (4, 27, 2049, 4)])
def test_dd_exchange_gloo(world, sigma, n, seed):
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_dd_rank_main, args=(world, port, out, sigma, n, seed), nprocs=world, join=True)
    assert all(out[r] for r in range(world)), dict(out)
