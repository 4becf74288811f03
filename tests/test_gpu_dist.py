"""The multi-GPU build's code path (paper_1610_05994_b200.dist.build_distributed)
on real CUDA tensors with NCCL, world size 1 (this environment has one GPU):
the all-gathers, the plan kernel, the send/recv group (empty at one rank), the
part merge and the superblock rescan run as they do on N GPUs, and the one part
is the whole tree -- compared with the oracle.  The N-rank exchange itself is
covered under gloo (tests/test_multirank.py) and the N-part merge on one device
(tests/test_gpu_dd.py)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import wt_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    from conftest import build_native
    build_native()
    import torch.distributed as dist
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("sigma,n,dtype", [(4, 1_000_003, np.uint8), (256, 300_001, np.uint8),
                                           (1 << 16, 200_000, np.uint16), (1 << 20, 100_003, np.uint32),
                                           (1, 5000, np.uint8)])
def test_build_distributed_one_rank(pg, sigma, n, dtype):
    from paper_1610_05994_b200.dist import build_distributed
    S = wt_inputs.random_case(n + 1, n, sigma, "zipf" if sigma > 2 else "uniform", dtype=dtype)
    d = torch.from_numpy(S.view(np.int32) if dtype == np.uint32 else S).cuda()
    part = build_distributed(d, sigma)
    ot = oracle.build(S, sigma)
    assert part.parts == 1 and part.block_begin == 0 and part.block_end == (n + 511) // 512
    assert np.array_equal(part.node_offsets.cpu().numpy().view(np.uint64), ot.node_offsets)
    for l in range(ot.L):
        assert np.array_equal(part.bitmaps[l].cpu().numpy().view(np.uint32), ot.bitmaps[l]), f"level {l}"
        assert np.array_equal(part.superblocks[l].cpu().numpy().view(np.uint64), ot.superblocks[l]), f"sb {l}"
