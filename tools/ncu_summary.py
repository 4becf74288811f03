"""Summarise an ncu launch list (gpu__time_duration per launch) and a full
capture of the level pass into a text summary under profiles/, plus the
per-launch DRAM traffic of the level pass for bench.py's roofline.traffic.

usage: python tools/ncu_summary.py <cfg> <round_tag>
reads gpurun_out/launches_cfg<cfg>.csv and gpurun_out/prof_cfg<cfg>.ncu-rep
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kind_of(name: str) -> str:
    if "k_leaf_offsets" in name:
        return "leaf_offsets"
    if "k_triple" in name:
        return "triple"
    if "k_cls3" in name:
        return "class_count"
    if "k_pair2" in name or "k_pairn" in name:
        return "pair"
    if "k_prep" in name:
        return "final_scan" if ("OpBitsPop" in name or "OpBlockPop" in name) else "prep"
    if "k_prologue" in name:
        return "prologue"
    if "k_level" in name:
        return {", 1>(": "level", ", 2>(": "pair"}.get(next((k for k in (", 1>(", ", 2>(") if k in name), ""),
                                                          "last_level")
    if "OpTilePrefix" in name:
        return "tile_scan"
    if "OpLevelTab" in name:
        return "tables"
    if "OpLeafC" in name:
        return "scan"
    if "OpBitsPop" in name or "OpBlockPop" in name:
        return "sb_scan"
    if "k_block_pop" in name:
        return "block_pop"
    return "other(" + re.sub(r"\(.*", "", name)[:40] + ")"


def launches(cfg: int):
    path = os.path.join(ROOT, "gpurun_out", f"launches_cfg{cfg}.csv")
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    out = []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        out.append((kind_of(r["Kernel Name"]), float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)))
    return out


def full_capture(cfg: int):
    rep = os.path.join(ROOT, "gpurun_out", f"prof_cfg{cfg}.ncu-rep")
    if not os.path.exists(rep):
        return None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))

        def val(k, to_bytes=False):
            x = d.get(k)
            if x in (None, ""):
                return None
            x = float(x.replace(",", ""))
            if to_bytes:
                x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(k), 1)
            return x
        dur_us = val("gpu__time_duration.sum") * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u.get("gpu__time_duration.sum"), 1.0)
        rd, wr = val("dram__bytes_read.sum", True), val("dram__bytes_write.sum", True)
        res.append(OrderedDict(kernel=re.sub(r"\(.*", "", d["Kernel Name"]), duration_us=dur_us, dram_read=rd,
                               dram_write=wr, dram_GBps=(rd + wr) / dur_us / 1e3,
                               issue_active_pct=val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                               alu_pipe_pct=val("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                               fma_pipe_pct=val("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                               smem_wavefront_pct=val(
                                   "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                               warps_active_pct=val("sm__warps_active.avg.pct_of_peak_sustained_active"),
                               registers=val("launch__registers_per_thread"),
                               inst_executed=val("smsp__inst_executed.sum")))
    return res


def main():
    cfg, tag = int(sys.argv[1]), sys.argv[2]
    outdir = os.path.join(ROOT, "profiles", tag)
    os.makedirs(outdir, exist_ok=True)
    L = launches(cfg)
    # drop the warm-up builds: keep the launches of the last build (from its last prologue)
    starts = [i for i, (k, _) in enumerate(L) if k == "prologue"]
    last = L[starts[-1]:] if starts else L
    tot = sum(t for _, t in last)
    per = OrderedDict()
    for k, t in last:
        a = per.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    lines = [f"ncu launch list, cfg{cfg}: one build = {len(last)} launches, {tot:.1f} us serialized "
             "(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache per launch: compare shares)"]
    for k, (c, t) in per.items():
        lines.append(f"  {k:12s} launches={c:3d} total={t:9.1f} us share={100 * t / tot:5.1f}%")
    fc = full_capture(cfg)
    if fc:
        lines.append(f"ncu --set full capture (level pass), cfg{cfg}:")
        for r in fc:
            lines.append("  " + json.dumps(r))
        lvl = [r for r in fc if "k_level" in r["kernel"] or "k_pair2" in r["kernel"] or "k_pairn" in r["kernel"]]
        if lvl:
            traffic = {}
            for r in lvl:
                kd = ("pair" if (", 2>" in r["kernel"] or "k_pair2" in r["kernel"] or "k_pairn" in r["kernel"]) else
                      "level" if ", 1>" in r["kernel"] else "last_level")
                traffic.setdefault(kd, r["dram_read"] + r["dram_write"])
            traffic["_source"] = f"profiles/{tag}/ncu_summary_cfg{cfg}.txt"
            with open(os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{cfg}.json"), "w") as f:
                json.dump(traffic, f)
    with open(os.path.join(outdir, f"ncu_summary_cfg{cfg}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
