#!/usr/bin/env python
"""Benchmark: levelwise wavelet-tree build on B200 (BASELINE.json metric
"wavelet tree build Gsymbols/s and achieved HBM GB/s vs roofline on 1 B200").

A step = one whole build (pass over S, scans, node tables, every level pass) of
one config's sequence, through the C ABI (wt_build_async), inputs resident in
HBM.  Default workload = BASELINE configs[1] (cfg2, DNA-like, n=2^30 uint8,
sigma=4).  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): every rank builds its own copy of
the config (independent problems, no data-path collective) -> "scaling":
"weak"; value = symbols of all ranks / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import wt_inputs  # noqa: E402

METRIC = "wavelet tree build Gsymbols/s (HBM GB/s vs roofline in 'roofline')"
UNIT = "Gsymbols/s"
DTYPE = {1: "u8", 2: "u16", 4: "u32"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=9)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay timing")
    ap.add_argument("--out", default=None, help="also write the JSON line (plus per-kernel detail) here")
    return ap.parse_args()


def algorithmic_bytes(kind: str, n: int, w: int, L: int) -> int:
    """Bytes the levelwise method itself must move per launch."""
    nsb = (n + 511) // 512 + 1
    bitmap = 4 * 16 * ((n + 511) // 512)
    if kind == "level":      # read T_l, write T_{l+1}, bitmap words, superblocks
        return 2 * n * w + bitmap + 8 * nsb
    if kind == "last_level":  # read T_{L-1}, bitmap words, superblocks (L = 1 only)
        return n * w + bitmap + 8 * nsb
    if kind == "pair":        # level L-2 fused with L-1: read T_{L-2}, both bitmaps, superblocks of L-2
        return n * w + 2 * bitmap + 8 * nsb
    if kind == "sb_scan":     # superblocks of level L-1 from the block counts
        return 4 * (nsb - 1) + 8 * nsb
    if kind == "prologue":    # read S once (range check, level-0 tile ones)
        return n * w
    if kind == "scan":        # node_offsets: read 2^L uint32 leaf counts, write 2^L + 1 uint64
        return 4 * (1 << L) + 8 * ((1 << L) + 1)
    if kind in ("prep", "tile_scan"):  # tile prefixes (read agg, write pre), node tables, zeroed counts; avg per launch
        tile = {1: 2048, 2: 1024, 4: 512}[w]
        tiles = (n + tile - 1) // tile
        levels = max(L - 1, 1)
        tables = sum(4 * (2 << l) + 8 * (1 << l) for l in range(max(L - 1, 0)))
        zero = sum(16 * (1 << l) for l in range(max(L - 1, 0))) + (bitmap if L >= 2 else 0)
        return 8 * tiles + (tables + zero) // levels
    if kind == "final_scan":  # last-level superblocks from its bitmap, C from the leaf counts
        return bitmap + 8 * nsb + 4 * (1 << L) + 8 * ((1 << L) + 1)
    return 0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                rows.append((float(f[0]), float(f[1]), f[3:7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, x in enumerate(r) if x.lower() == "active"})
        load = [r[0] for r in rows]
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_time(cfg: int, n_sample: int, reps: int):
    """Time the CPU oracle (as it stands, one thread) on a prefix sample of the config."""
    import oracle
    S, sigma = wt_inputs.generate(cfg, n_sample)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.build(S, sigma)
        ts.append(time.perf_counter() - t0)
    return S.size, ts


ORACLE_SAMPLE = {1: 1 << 20, 2: 1 << 28, 3: 1 << 26, 4: 1 << 24, 5: 1 << 23}


def run_reference(args, rank):
    """--impl reference: the CPU oracle is this tier's reference arm."""
    if rank != 0:
        return
    cfg = wt_inputs.CONFIGS[args.config]
    n_s = ORACLE_SAMPLE[args.config] // 4
    steps = args.steps or 3
    for _ in range(args.warmup if args.warmup < 2 else 1):
        oracle_time(args.config, n_s, 1)
    n, ts = oracle_time(args.config, n_s, steps)
    t = statistics.median(ts)
    val = n / t / 1e9
    w = np.dtype(cfg["dtype"]).itemsize
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE[w], "data": "synthetic",
        "config": {"workload": f"{cfg['name']} (BASELINE configs[{args.config - 1}])", "n": cfg["n"],
                   "sigma": cfg["sigma"], "width": w},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {n} symbols of the config's sequence, oracle (Alg. 1 sequential, "
                                   f"gcc -O2, 1 thread), median of {steps}",
                         "host": cpu_model(), "host_cores": os.cpu_count()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def max_over_ranks(ms: float, world: int, device) -> float:
    """The step time of an N-rank job: the slowest rank's device time (all_reduce MAX).
    device: the collective's tensor device (cuda for NCCL, cpu for gloo)."""
    if world <= 1:
        return ms
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(n_per_rank: int, world: int, ms_per_step: float) -> float:
    """Whole-job Gsymbols/s: every rank builds its own replica of n symbols (weak scaling)."""
    return world * n_per_rank / (ms_per_step * 1e-3) / 1e9


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_1610_05994_b200 as wt

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = wt_inputs.CONFIGS[args.config]
    S, sigma = wt_inputs.generate(args.config)
    n = S.size
    w = S.dtype.itemsize
    L = wt.sizes(n, sigma, w).levels
    h_seq = torch.from_numpy(S.view(np.int32) if w == 4 else S)
    d_seq = h_seq.to(dev)
    stream = torch.cuda.Stream(device=dev)
    tree = wt.alloc_tree(n, sigma, w, dev)
    ws = wt.alloc_workspace(n, sigma, w, dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    plan = wt.launch_plan(n, sigma, w)
    steps = args.steps or {1: 2000, 2: 200, 3: 200, 4: 60, 5: 25}[args.config]
    warmup = max(3, args.warmup)

    def step():
        wt.build_async(d_seq, sigma, tree=tree, workspace=ws, status=status, stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            step()
    stream.synchronize()
    assert int(status.item()) == wt.WT_OK

    # timed region 1 (the reported value): K builds back to back, no instrumentation
    nl = len(plan)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_start.record(stream)
        for k in range(steps):
            step()
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    elapsed_ms = max_over_ranks(t_start.elapsed_time(t_end), world, dev)
    ms_per_step = elapsed_ms / steps
    value = job_throughput(n, world, ms_per_step)

    # timed region 2 (the per-kernel breakdown and roofline): the same K builds
    # with a CUDA event pair recorded by the library around every launch, on
    # the build stream (event records add small gaps, so the value above is
    # taken without them)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nl)] for _ in range(steps)]
    p_start = torch.cuda.Event(enable_timing=True)
    p_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    p_start.record(stream)
    for k in range(steps):
        wt.set_profile_events(evs[k])
        step()
    p_end.record(stream)
    wt.set_profile_events(None)
    torch.cuda.synchronize()
    profiled_ms_per_step = p_start.elapsed_time(p_end) / steps

    # the same build captured once in a CUDA graph and replayed (launch gaps
    # removed); reported beside the direct-launch value, not instead of it
    graph = None
    if not args.no_graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step()
            g.replay()
            torch.cuda.synchronize()
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(steps):
                    g.replay()
            g1.record(stream)
            torch.cuda.synchronize()
            gms = g0.elapsed_time(g1) / steps
            graph = {"ms_per_step": gms, "value": job_throughput(n, world, gms), "unit": UNIT}
            assert int(status.item()) == wt.WT_OK
        except Exception as e:  # report, do not fail the bench line
            graph = {"error": str(e)[:200]}

    # per-kernel durations (same stream as the launches)
    per_kind: dict[str, list[float]] = {}
    per_launch = [0.0] * nl
    for k in range(steps):
        for i in range(nl):
            d = evs[k][2 * i].elapsed_time(evs[k][2 * i + 1])
            per_launch[i] += d / steps
            per_kind.setdefault(plan[i], []).append(d)
    kind_total = {kd: sum(v) / steps for kd, v in per_kind.items()}
    dom = max(kind_total, key=kind_total.get)
    launches_of = {kd: plan.count(kd) for kd in kind_total}
    avg_launch_ms = kind_total[dom] / launches_of[dom]
    ab = algorithmic_bytes(dom, n, w, L)
    achieved = ab / (avg_launch_ms * 1e-3) / 1e9
    peak, peak_src = measured_peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(dom)
    kernels = {kd: {"launches_per_step": launches_of[kd], "ms_per_step": kind_total[kd],
                    "share": kind_total[kd] / ms_per_step,
                    "algorithmic_GBps": algorithmic_bytes(kd, n, w, L) * launches_of[kd] /
                    (kind_total[kd] * 1e-3) / 1e9}
               for kd in kind_total}

    # end-to-end through the public host API: every step is H2D of S from pinned
    # memory, the build, and D2H of the whole tree (wt_build_from_host_async).
    # INFLIGHT builds are in flight on as many streams with their own workspaces,
    # so one build's copies overlap the others' compute (H2D and D2H use separate
    # copy engines); a build's H2D -> build -> D2H chain is ~2-3x one copy.
    e2e = None
    if args.e2e_steps > 0:
        h_pinned = h_seq.pin_memory()
        del ws
        torch.cuda.empty_cache()
        INFLIGHT = 3
        streams = [torch.cuda.Stream(device=dev) for _ in range(INFLIGHT)]
        h_trees = [wt.alloc_host_tree(n, sigma, w) for _ in range(INFLIGHT)]
        wss = [wt.alloc_workspace(n, sigma, w, dev, host=True) for _ in range(INFLIGHT)]
        stats = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(INFLIGHT)]
        for i in range(INFLIGHT):  # warm-up, every slot
            wt.build_from_host_async(h_pinned, sigma, h_trees[i], wss[i], stats[i], stream=streams[i])
        sz = wt.sizes(n, sigma, w)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        for s_ in streams[1:]:
            s_.wait_event(e0)
        for k in range(args.e2e_steps):
            i = k % INFLIGHT
            wt.build_from_host_async(h_pinned, sigma, h_trees[i], wss[i], stats[i], stream=streams[i])
        for s_ in streams[1:]:
            done = torch.cuda.Event()
            done.record(s_)
            streams[0].wait_event(done)
        e1.record(streams[0])
        torch.cuda.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, world, dev)
        e2e = {"value": job_throughput(n, world, e_ms), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": n * w,
               "d2h_bytes_per_step": int(sz.bitmap_bytes + sz.superblock_bytes + sz.node_offset_bytes + 4),
               "api": f"wt_build_from_host_async (pinned host buffers; {INFLIGHT} builds in flight on "
                      f"{INFLIGHT} streams)"}
        # correctness guard on the e2e results: status words and C[2^L] = n
        assert all(int(x.item()) == wt.WT_OK for x in stats)
        assert all(int(t.node_offsets[-1].item()) == n for t in h_trees)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_s = min(ORACLE_SAMPLE[args.config], n)
        ns, ts = oracle_time(args.config, n_s, 3)
        cpu = {"value": ns / statistics.median(ts) / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {ns} symbols of {cfg['name']}, oracle (Alg. 1 sequential, gcc -O2, 1 thread), "
                         f"median of 3 ({statistics.median(ts):.2f} s each)",
               "host": cpu_model(), "host_cores": os.cpu_count()}

    clocks = sampler.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DTYPE[w], "data": "synthetic",
        "config": {"workload": f"{cfg['name']} (BASELINE configs[{args.config - 1}])", "n": n, "sigma": sigma,
                   "width": w, "levels": L, "per_rank": "independent replica of the config",
                   "l2": "inputs exceed L2 (n*w >= 256 MiB > 126 MB), no flush" if n * w > (200 << 20)
                   else "inputs fit in L2 (latency config), no flush",
                   "parallelism": f"replicas x{world}"},
        "profiled_ms_per_step": profiled_ms_per_step,
        "graph": graph,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": ab, "avg_launch_ms": avg_launch_ms},
        "e2e": e2e,
        "gpu_launches": steps * nl,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "kernels": kernels,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump(dict(line, per_launch_ms=per_launch, plan=plan), f, indent=1)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
