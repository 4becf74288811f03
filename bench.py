#!/usr/bin/env python
"""Benchmark: levelwise wavelet-tree build on B200 (BASELINE.json metric
"wavelet tree build Gsymbols/s and achieved HBM GB/s vs roofline on 1 B200").

A step = one whole build (pass over S, scans, node tables, every level pass) of
one config's sequence, through the C ABI (wt_build_async), inputs resident in
HBM.  Default workload = BASELINE configs[1] (cfg2, DNA-like, n=2^30 uint8,
sigma=4).  Prints ONE JSON line on rank 0.  The same run also times the three
north-star configs (cfg3-5, n = 2^28) device-side and reports them under
"north_star_configs" (build Gsym/s and per-kernel-kind fractions of the HBM
roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

Multi-GPU (one process per GPU; `--gpus N` without torchrun re-launches itself
under torch.distributed.run): see DESIGN.md §8 for the N > 1 step.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
# kernel kinds whose per-launch HBM fraction is a roofline statement (the scans
# move a few MB and are latency-bound)
STREAMING_KINDS = ("prologue", "level", "pair", "last_level", "final_scan")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=9)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay timing")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg3-5 device-timed lines")
    ap.add_argument("--extra-steps", type=int, default=10)
    ap.add_argument("--dd", action="store_true",
                    help="run the multi-GPU (domain decomposition) step even at N = 1 (its merge overhead)")
    ap.add_argument("--out", default=None, help="also write the JSON line (plus per-kernel detail) here")
    return ap.parse_args(argv)


def algorithmic_bytes(kind: str, n: int, w: int, L: int, c_in_final: bool = True) -> int:
    """Bytes the levelwise method itself must move per launch (DESIGN.md §6 table)."""
    nsb = (n + 511) // 512 + 1
    bitmap = 4 * 16 * ((n + 511) // 512)
    if kind == "level":      # read T_l, write T_{l+1}, bitmap words, superblocks
        return 2 * n * w + bitmap + 8 * nsb
    if kind == "last_level":  # read T_{L-1}, bitmap words, superblocks (L = 1 only)
        return n * w + bitmap + 8 * nsb
    if kind == "pair":        # level L-2 fused with L-1: read T_{L-2}, both bitmaps, superblocks of L-2
        return n * w + 2 * bitmap + 8 * nsb
    if kind == "prologue":    # read S once (range check, level-0 tile ones)
        return n * w
    if kind == "scan":        # node_offsets: read 2^L uint32 leaf counts, write 2^L + 1 uint64
        return 4 * (1 << L) + 8 * ((1 << L) + 1)
    if kind == "prep":        # tile prefixes (read agg, write pre), node tables, zeroed counts; avg per launch
        tile = {1: 2048, 2: 1024, 4: 512}[w]
        tiles = (n + tile - 1) // tile
        levels = max(L - 1, 1)
        tables = sum(4 * (2 << l) + 8 * (1 << l) for l in range(max(L - 1, 0)))
        zero = sum(16 * (1 << l) for l in range(max(L - 1, 0))) + (bitmap if L >= 2 else 0)
        return 8 * tiles + (tables + zero) // levels
    if kind == "final_scan":  # last-level superblocks from its bitmap (and C from the leaf counts)
        return bitmap + 8 * nsb + ((4 * (1 << L) + 8 * ((1 << L) + 1)) if c_in_final else 0)
    if kind == "class_count":  # (opt-in triple) read T_{L-3}, per-tile class counts (agg01, agg11)
        tile = {1: 2048, 2: 1024, 4: 512}[w]
        return n * w + 8 * ((n + tile - 1) // tile)
    if kind == "triple":       # (opt-in) read T_{L-3}, three bitmaps, superblocks of level L-3
        return n * w + 3 * bitmap + 8 * nsb
    if kind == "leaf_offsets":  # C from the level-(L-2) node table and B_{L-1}'s ranks at the node starts
        return 8 * ((1 << L) + 1) + 8 * (1 << max(L - 2, 0))
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


def config_of(cfg: int, world: int = 1) -> dict:
    """The `config` object of the JSON line -- identical for both arms."""
    c = wt_inputs.CONFIGS[cfg]
    w = np.dtype(c["dtype"]).itemsize
    L = max(0, (c["sigma"] - 1).bit_length())
    return {"workload": f"{c['name']} (BASELINE configs[{cfg - 1}])", "n": c["n"], "sigma": c["sigma"],
            "width": w, "levels": L,
            "l2": "inputs exceed L2 (n*w >= 256 MiB > 126 MB), no flush" if c["n"] * w > (200 << 20)
            else "inputs fit in L2 (latency config), no flush",
            "parallelism": f"dd x{world}" if world > 1 else "1 GPU"}


def oracle_time(cfg: int, n_sample: int, reps: int):
    """Time the CPU oracle (as it stands: single-threaded C, Alg. 1) on the first
    n_sample symbols of the config, pinned to ONE host core (os.sched_setaffinity),
    `reps` repetitions.  Returns (n, seconds per repetition, core)."""
    import oracle
    S, sigma = wt_inputs.generate(cfg, n_sample)
    oracle.lib()
    old = os.sched_getaffinity(0)
    core = max(old)                      # one core of those this process may use
    os.sched_setaffinity(0, {core})
    try:
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            oracle.build(S, sigma)
            ts.append(time.perf_counter() - t0)
    finally:
        os.sched_setaffinity(0, old)
    return S.size, ts, core


# bounded samples (~3 s of single-core oracle work per repetition)
ORACLE_SAMPLE = {1: 1 << 20, 2: 1 << 28, 3: 1 << 26, 4: 1 << 24, 5: 1 << 23}


def cpu_baseline_of(cfg: int, n: int, ts, core, reps_note: str) -> dict:
    c = wt_inputs.CONFIGS[cfg]
    t = statistics.median(ts)
    return {"value": n / t / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {n} of the {c['n']} symbols of {c['name']} (a bounded prefix; throughput = "
                      f"prefix symbols / time), oracle (Alg. 1 sequential, gcc -O2, 1 thread pinned to host "
                      f"core {core} by sched_setaffinity), {reps_note} ({t:.2f} s each)",
            "sample_n": n, "host": cpu_model(), "host_cores": os.cpu_count()}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    n_s = ORACLE_SAMPLE[args.config] // 4
    steps = args.steps or 5
    for _ in range(min(args.warmup, 1)):
        oracle_time(args.config, n_s, 1)
    n, ts, core = oracle_time(args.config, n_s, steps)
    t = statistics.median(ts)
    val = n / t / 1e9
    w = np.dtype(wt_inputs.CONFIGS[args.config]["dtype"]).itemsize
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE[w], "data": "synthetic",
        "config": config_of(args.config, world),
        "cpu_baseline": cpu_baseline_of(args.config, n, ts, core, f"median of {steps}"),
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
    """Whole-job Gsymbols/s: every rank processes n symbols per step (weak scaling)."""
    return world * n_per_rank / (ms_per_step * 1e-3) / 1e9


def time_builds(wt, d_seq, sigma, stream, steps, warmup, profile=True):
    """Device-time `steps` builds back to back (CUDA events on the build stream),
    then the same builds with a library-recorded event pair around every launch
    (per-kernel durations on the launching stream).  Returns a dict."""
    import torch
    n = d_seq.numel()
    w = wt.width_of(d_seq)
    dev = d_seq.device
    tree = wt.alloc_tree(n, sigma, w, dev)
    ws = wt.alloc_workspace(n, sigma, w, dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    plan = wt.launch_plan(n, sigma, w)

    def step():
        wt.build_async(d_seq, sigma, tree=tree, workspace=ws, status=status, stream=stream)

    for _ in range(warmup):
        step()
    stream.synchronize()
    assert int(status.item()) == wt.WT_OK
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    res = {"ms_per_step": t0.elapsed_time(t1) / steps, "plan": plan, "tree": tree, "ws": ws, "status": status,
           "step": step}
    if not profile:
        return res
    nl = len(plan)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * nl)] for _ in range(steps)]
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    p0.record(stream)
    for k in range(steps):
        wt.set_profile_events(evs[k])
        step()
    p1.record(stream)
    wt.set_profile_events(None)
    torch.cuda.synchronize()
    per_launch = [[evs[k][2 * i].elapsed_time(evs[k][2 * i + 1]) for k in range(steps)] for i in range(nl)]
    res["profiled_ms_per_step"] = p0.elapsed_time(p1) / steps
    res["per_launch_ms"] = [sum(x) / steps for x in per_launch]
    return res


def kernel_table(res, n, w, L, peak):
    """Per kernel kind: launches, time share of the step, algorithmic GB/s and the
    min / mean / max per-launch fraction of the HBM roofline."""
    plan, pl, ms = res["plan"], res["per_launch_ms"], res["ms_per_step"]
    kinds = {}
    for kd, t in zip(plan, pl):
        kinds.setdefault(kd, []).append(t)
    out = {}
    for kd, ts in kinds.items():
        ab = algorithmic_bytes(kd, n, w, L, c_in_final="leaf_offsets" not in plan)
        fr = [ab / (t * 1e-3) / 1e9 / peak for t in ts if t > 0]
        e = {"launches_per_step": len(ts), "ms_per_step": sum(ts), "share": sum(ts) / ms,
             "per_launch_ms": {"min": min(ts), "mean": sum(ts) / len(ts), "max": max(ts)},
             "algorithmic_GBps": ab * len(ts) / (sum(ts) * 1e-3) / 1e9}
        if kd in STREAMING_KINDS and fr:
            e["roofline_frac"] = {"min": min(fr), "mean": sum(fr) / len(fr), "max": max(fr)}
        out[kd] = e
    return out


def north_star_line(wt, cfg, stream, dev, steps, warmup, peak):
    """Device-timed build of one north-star config (cfg3-5): Gsym/s plus the
    per-kind roofline fractions (the level-partition kernels' target is >= 0.6)."""
    import torch
    S, sigma = wt_inputs.generate(cfg)
    n, w = S.size, S.dtype.itemsize
    d_seq = torch.from_numpy(S.view(np.int32) if w == 4 else S).to(dev)
    del S
    L = wt.sizes(n, sigma, w).levels
    res = time_builds(wt, d_seq, sigma, stream, steps, warmup)
    kt = kernel_table(res, n, w, L, peak)
    lvl = [k for k in ("level", "pair", "last_level") if k in kt]
    line = {"workload": config_of(cfg)["workload"], "n": n, "sigma": sigma, "width": w, "levels": L,
            "steps": steps, "ms_per_step": res["ms_per_step"], "value": n / (res["ms_per_step"] * 1e-3) / 1e9,
            "unit": UNIT, "level_partition_frac_min": min(kt[k]["roofline_frac"]["min"] for k in lvl),
            "kernels": kt}
    del d_seq, res
    torch.cuda.empty_cache()
    return line


def e2e_throughput(wt, h_seq, sigma, dev, steps, world):
    """End to end through the public host API: every step is the H2D of S from
    pinned memory, the build, and the D2H of the whole tree and its status word
    (wt_build_from_host_async).  Three builds are in flight on three streams with
    their own workspaces, so one build's copies overlap the others' compute: the
    value is the pipelined whole-job throughput of back-to-back host-to-host
    builds (PCIe-bound), not one call's latency, which is reported beside it."""
    import torch
    n, w = h_seq.numel(), wt.width_of(h_seq)
    h_pinned = h_seq.pin_memory()
    INFLIGHT = 3
    streams = [torch.cuda.Stream(device=dev) for _ in range(INFLIGHT)]
    h_trees = [wt.alloc_host_tree(n, sigma, w) for _ in range(INFLIGHT)]
    wss = [wt.alloc_workspace(n, sigma, w, dev, host=True) for _ in range(INFLIGHT)]
    stats = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(INFLIGHT)]
    for i in range(INFLIGHT):  # warm-up, every slot
        wt.build_from_host_async(h_pinned, sigma, h_trees[i], wss[i], stats[i], stream=streams[i])
    torch.cuda.synchronize()
    # one call alone: H2D -> build -> D2H latency
    l0 = torch.cuda.Event(enable_timing=True)
    l1 = torch.cuda.Event(enable_timing=True)
    l0.record(streams[0])
    wt.build_from_host_async(h_pinned, sigma, h_trees[0], wss[0], stats[0], stream=streams[0])
    l1.record(streams[0])
    torch.cuda.synchronize()
    single_ms = l0.elapsed_time(l1)
    sz = wt.sizes(n, sigma, w)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for s_ in streams[1:]:
        s_.wait_event(e0)
    for k in range(steps):
        i = k % INFLIGHT
        wt.build_from_host_async(h_pinned, sigma, h_trees[i], wss[i], stats[i], stream=streams[i])
    for s_ in streams[1:]:
        done = torch.cuda.Event()
        done.record(s_)
        streams[0].wait_event(done)
    e1.record(streams[0])
    torch.cuda.synchronize()
    e_ms = max_over_ranks(e0.elapsed_time(e1) / steps, world, dev)
    # correctness guard on the e2e results: status words and C[2^L] = n
    assert all(int(x.item()) == wt.WT_OK for x in stats)
    assert all(int(t.node_offsets[-1].item()) == n for t in h_trees)
    return {"value": job_throughput(n, world, e_ms), "unit": UNIT, "ms_per_step": e_ms,
            "h2d_bytes_per_step": n * w,
            "d2h_bytes_per_step": int(sz.bitmap_bytes + sz.superblock_bytes + sz.node_offset_bytes + 4),
            "pipelined": True, "single_build_ms": single_ms,
            "single_build_value": n / (single_ms * 1e-3) / 1e9,
            "api": f"wt_build_from_host_async (pinned host buffers; {INFLIGHT} builds in flight on "
                   f"{INFLIGHT} streams; single_build_* = one call alone)"}


def run_dd(args, wt, rank, world, local, dev):
    """N > 1: the multi-GPU domain decomposition.
    Every rank holds one contiguous segment of the job's sequence -- the config's
    n symbols (its seeded sequence; the job's sequence is the G segments in rank
    order, G*n symbols) -- and a step is one whole distributed build
    (paper_1610_05994_b200.dist.build_distributed): the rank's segment build,
    all-gather of node offsets, plan, NCCL send/recv of the bit words, merge of
    the rank's part of every level, superblock rescan.  Weak scaling: value =
    G*n / the slowest rank's device time."""
    import torch
    import torch.distributed as dist
    from paper_1610_05994_b200.dist import build_distributed
    cfg = args.config
    S, sigma = wt_inputs.generate(cfg)
    n, w = S.size, S.dtype.itemsize
    h_seq = torch.from_numpy(S.view(np.int32) if w == 4 else S)
    d_seq = h_seq.to(dev)
    steps = args.steps or {1: 200, 2: 50, 3: 50, 4: 20, 5: 10}[cfg]
    warmup = max(3, args.warmup)
    peak, peak_src = measured_peaks()
    for _ in range(warmup):
        part = build_distributed(d_seq, sigma)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            part = build_distributed(d_seq, sigma)
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, world, dev)
    # the rank's local segment build alone (its kernels and roofline)
    stream = torch.cuda.Stream(device=dev)
    L = wt.sizes(n, sigma, w).levels
    prof = time_builds(wt, d_seq, sigma, stream, min(steps, 20), 1, profile=True)
    kt = kernel_table(prof, n, w, L, peak)
    dom = max(kt, key=lambda k: kt[k]["ms_per_step"])
    avg_launch_ms = kt[dom]["ms_per_step"] / kt[dom]["launches_per_step"]
    ab = algorithmic_bytes(dom, n, w, L)
    local_ms = max_over_ranks(prof["ms_per_step"], world, dev)
    # end to end: H2D of the rank's segment from pinned memory, the distributed
    # build, D2H of the rank's part of the tree
    h_pinned = h_seq.pin_memory()
    h_bits = torch.empty(part.bitmaps.shape, dtype=part.bitmaps.dtype, pin_memory=True)
    h_sb = torch.empty(part.superblocks.shape, dtype=part.superblocks.dtype, pin_memory=True)
    e_steps = max(1, min(args.e2e_steps, 5))
    dist.barrier()
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(e_steps):
        d_in = h_pinned.to(dev, non_blocking=True)
        part = build_distributed(d_in, sigma)
        h_bits.copy_(part.bitmaps, non_blocking=True)
        h_sb.copy_(part.superblocks, non_blocking=True)
    f1.record()
    torch.cuda.synchronize()
    e_ms = max_over_ranks(f0.elapsed_time(f1) / e_steps, world, dev)
    line = {
        "metric": METRIC, "value": job_throughput(n, world, ms), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DTYPE[w], "data": "synthetic",
        "config": dict(config_of(cfg, world), parallelism=f"dd x{world} (one segment of n per rank, merged tree "
                                                            f"of {world}*n symbols sharded by position)"),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": ab / (avg_launch_ms * 1e-3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": ab / (avg_launch_ms * 1e-3) / 1e9 / peak, "traffic": None,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": ab, "avg_launch_ms": avg_launch_ms,
                     "scope": "the rank's local segment build"},
        "dd": {"local_build_ms": local_ms, "exchange_merge_ms": ms - local_ms},
        "e2e": {"value": job_throughput(n, world, e_ms), "unit": UNIT, "ms_per_step": e_ms,
                "h2d_bytes_per_step": n * w,
                "d2h_bytes_per_step": int(h_bits.numel() * 4 + h_sb.numel() * 8),
                "api": "per rank: H2D of its segment, dist.build_distributed, D2H of its part"},
        "gpu_launches": None,
        "clocks": sampler.summary(),
        "cpu_baseline": None,
        "kernels": kt,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump(line, f, indent=1)


def relaunch_under_torchrun(args):
    """`--gpus N` (N > 1) without torchrun: start N ranks ourselves."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1610_05994_b200 as wt

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.dd:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if "MASTER_PORT" not in os.environ:
                with socket.socket() as s:
                    s.bind(("127.0.0.1", 0))
                    os.environ["MASTER_PORT"] = str(s.getsockname()[1])
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    cfg = args.config
    if world > 1 or args.dd:
        run_dd(args, wt, rank, world, local, dev)
        dist.destroy_process_group()
        return
    S, sigma = wt_inputs.generate(cfg)
    n = S.size
    w = S.dtype.itemsize
    L = wt.sizes(n, sigma, w).levels
    h_seq = torch.from_numpy(S.view(np.int32) if w == 4 else S)
    d_seq = h_seq.to(dev)
    stream = torch.cuda.Stream(device=dev)
    steps = args.steps or {1: 2000, 2: 200, 3: 200, 4: 60, 5: 25}[cfg]
    warmup = max(3, args.warmup)
    peak, peak_src = measured_peaks()

    # timed region 1 (the reported value): K builds back to back, no instrumentation
    sampler = ClockSampler(local)
    with sampler:
        if world > 1:
            dist.barrier()
        res = time_builds(wt, d_seq, sigma, stream, steps, warmup, profile=False)
        if world > 1:
            dist.barrier()
    ms_per_step = max_over_ranks(res["ms_per_step"], world, dev)
    value = job_throughput(n, world, ms_per_step)
    # timed region 2 (per-kernel breakdown and roofline): the same builds with an
    # event pair recorded by the library around every launch, on the build stream
    prof = time_builds(wt, d_seq, sigma, stream, steps, 1, profile=True)
    plan = prof["plan"]
    kt = kernel_table(prof, n, w, L, peak)
    dom = max(kt, key=lambda k: kt[k]["ms_per_step"])
    avg_launch_ms = kt[dom]["ms_per_step"] / kt[dom]["launches_per_step"]
    ab = algorithmic_bytes(dom, n, w, L)
    achieved = ab / (avg_launch_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{cfg}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(dom)

    # the same build captured once in a CUDA graph and replayed (launch gaps
    # removed); reported beside the direct-launch value, not instead of it
    graph = None
    if not args.no_graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                prof["step"]()
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
            assert int(prof["status"].item()) == wt.WT_OK
            del g
        except Exception as e:  # report, do not fail the bench line
            graph = {"error": str(e)[:200]}
    del res, prof
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    e2e = None
    if args.e2e_steps > 0:
        e2e = e2e_throughput(wt, h_seq, sigma, dev, args.e2e_steps, world)
    del d_seq
    torch.cuda.empty_cache()

    # the north-star configs (n = 2^28), device-timed, on rank 0 of a 1-GPU run
    extra = None
    if rank == 0 and world == 1 and not args.no_extra and cfg == 2:
        extra = {}
        for c in (3, 4, 5):
            extra[f"cfg{c}"] = north_star_line(wt, c, stream, dev, args.extra_steps, 3, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ns, ts, core = oracle_time(cfg, min(ORACLE_SAMPLE[cfg], n), 5)
        cpu = cpu_baseline_of(cfg, ns, ts, core, "median of 5")

    clocks = sampler.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DTYPE[w], "data": "synthetic",
        "config": config_of(cfg, world),
        "graph": graph,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": ab, "avg_launch_ms": avg_launch_ms},
        "e2e": e2e,
        "gpu_launches": steps * len(plan),
        "clocks": clocks,
        "cpu_baseline": cpu,
        "kernels": kt,
        "north_star_configs": extra,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump(dict(line, plan=plan), f, indent=1)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
