"""Per-kernel device times of one distributed build step (world size 1) --
where the dd step's time beyond the local build goes."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import wt_inputs  # noqa: E402
from paper_1610_05994_b200.dist import build_distributed  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
S, sigma = wt_inputs.generate(cfg)
d = torch.from_numpy(S.view(np.int32) if S.itemsize == 4 else S).to(dev)
for _ in range(3):
    build_distributed(d, sigma)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as p:
    for _ in range(5):
        build_distributed(d, sigma)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=25))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    build_distributed(d, sigma)
e1.record()
torch.cuda.synchronize()
print("dd step ms", e0.elapsed_time(e1) / 10)
dist.destroy_process_group()
