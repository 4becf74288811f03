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
