"""Host-side checks of the C ABI (no GPU): the library loads, exports every
symbol include/wt.h declares, and its pure-host entry points (sizes, launch
plan, argument validation) behave as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def wt():
    from conftest import build_native
    build_native()
    import paper_1610_05994_b200 as wt
    return wt


def declared_symbols():
    with open(os.path.join(ROOT, "include", "wt.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(wt_\w+)\s*\(", src, re.M)))


def test_exports_every_declared_symbol(wt):
    syms = declared_symbols()
    assert len(syms) >= 10
    lib = ctypes.CDLL(wt.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(wt.EXPORTS)


def test_library_is_sm100a_only(wt):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", wt.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_sizes(wt):
    s = wt.sizes(30, 16, 1)
    assert (s.levels, s.words_per_level, s.sb_per_level, s.c_len) == (4, 16, 2, 17)
    s = wt.sizes(0, 16, 1)
    assert (s.levels, s.words_per_level, s.sb_per_level, s.c_len) == (4, 0, 1, 17)
    s = wt.sizes(1 << 28, 1 << 24, 4)
    assert s.levels == 24 and s.words_per_level == (1 << 28) // 32 and s.sb_per_level == (1 << 19) + 1
    assert s.bitmap_bytes == 24 * (1 << 23) * 4 and s.superblock_bytes == 24 * ((1 << 19) + 1) * 8
    # two ping-pong permuted copies of the sequence at most (T_1..T_{L-2}), plus
    # node tables, two 2^L uint32 node-count buffers, per-tile and per-block counts
    assert 2 * (1 << 30) <= s.workspace_bytes < 2 * (1 << 30) + 450 * (1 << 20)
    assert wt.sizes(1 << 20, 4, 1).workspace_bytes < 1 << 20   # L=2: the fused pass writes no permuted copy
    assert wt.sizes(1 << 20, 8, 1).workspace_bytes > 1 << 20   # L=3: T_1
    assert s.host_workspace_bytes > s.workspace_bytes + (1 << 30)
    assert wt.sizes(5, 1, 1).levels == 0
    assert wt.sizes(5, 2, 1).workspace_bytes < 1 << 20   # L=1: no permuted copy
    for n, sigma, w, L in [(10, 3, 1, 2), (10, 256, 1, 8), (10, 257, 2, 9), (10, 1 << 16, 2, 16)]:
        assert wt.sizes(n, sigma, w).levels == L


@pytest.mark.parametrize("n,sigma,width", [(10, 4, 3), (10, 0, 1), (10, 257, 1), (10, 1 << 17, 2),
                                           (10, (1 << 31), 4), ((1 << 36) + 1, 256, 1)])
def test_sizes_rejects_bad_args(wt, n, sigma, width):
    with pytest.raises(wt.WtError) as e:
        wt.sizes(n, sigma, width)
    assert e.value.status == wt.WT_ERR_ARG


def test_build_validates_before_touching_the_device(wt):
    lib = wt._lib
    tree = wt.WtTree(None, None, None)
    assert lib.wt_build_async(None, 10, 4, 1, ctypes.byref(tree), None, 0, None, None) == wt.WT_ERR_ARG
    tree = wt.WtTree(16, 16, 16)
    assert lib.wt_build_async(None, 10, 4, 1, ctypes.byref(tree), None, 0, None, None) == wt.WT_ERR_ARG
    assert lib.wt_build_async(32, 10, 4, 1, ctypes.byref(tree), None, 0, None, None) == wt.WT_ERR_WORKSPACE
    assert lib.wt_build_async(33, 10, 4, 1, ctypes.byref(tree), 256, 1 << 20, None, None) == wt.WT_ERR_ARG
    assert lib.wt_build_async(32, 10, 4, 1, ctypes.byref(tree), 257, 1 << 20, None, None) == wt.WT_ERR_ARG
    assert lib.wt_build_async(32, 10, 4, 3, ctypes.byref(tree), 256, 1 << 20, None, None) == wt.WT_ERR_ARG
    # misaligned outputs (the pair passes store 16-byte bitmap words)
    for bad in (wt.WtTree(20, 16, 16), wt.WtTree(16, 20, 16), wt.WtTree(16, 16, 12)):
        assert lib.wt_build_async(32, 10, 4, 1, ctypes.byref(bad), 256, 1 << 20, None, None) == wt.WT_ERR_ARG
        assert b"aligned" in lib.wt_last_error()
    assert lib.wt_access(None, 10, 4, None, 1, None, None, None) == wt.WT_ERR_ARG
    # the host-buffer build: NULL status word / host pointers, then the workspace size
    htree = wt.WtTree(16, 16, 16)
    assert lib.wt_build_from_host_async(32, 10, 4, 1, ctypes.byref(htree), 256, 1 << 20, None, None) == wt.WT_ERR_ARG
    assert lib.wt_build_from_host_async(None, 10, 4, 1, ctypes.byref(htree), 256, 1 << 20, 64, None) == wt.WT_ERR_ARG
    assert lib.wt_build_from_host_async(32, 10, 4, 1, ctypes.byref(htree), 256, 16, 64, None) == wt.WT_ERR_WORKSPACE
    assert b"workspace" in lib.wt_last_error() or lib.wt_last_error() == b"tree is NULL"
    assert lib.wt_status_string(2) == b"WT_ERR_SYMBOL_RANGE"


def test_launch_plan(wt):
    # per level one prep launch (tile prefixes, node tables, zeroing) and the
    # pass; pass L-2 is fused with level L-1 (writes B_{L-1}), then the last
    # level's superblocks (from its bitmap) and C in one launch
    lv = ["prep", "level"]
    # (the fused final pair counts no leaves: C from B_{L-1}'s ranks at the node starts)
    pair = ["prep", "pair", "final_scan", "leaf_offsets"]
    # interior fused groups (a5, k = 2) at l = 0, 2, .. <= 6 while l + 2 <= L - 2:
    # tile prefixes + zeroing, the quad pass, the superblocks of its level l+1
    # (opt-in, WT_QUAD=1: slower than the level passes on B200)
    assert wt.launch_plan(1 << 20, 256, 1) == ["prologue"] + lv * 6 + pair
    assert wt.launch_plan(1 << 20, 8, 1) == ["prologue"] + lv + pair
    # the fused final three levels (opt-in, WT_TRIPLE=1: slower than a level pass
    # + the pair on B200): the level's prep, the class counts,
    # their prep, the pass, the superblocks of its two OR-ed levels, C
    trip = ["prep", "class_count", "prep", "triple", "final_scan", "leaf_offsets"]
    os.environ["WT_TRIPLE"] = "1"
    try:
        assert wt.launch_plan(1 << 20, 256, 1) == ["prologue"] + lv * 5 + trip
        assert wt.launch_plan(1 << 20, 8, 1) == ["prologue"] + trip
        assert wt.launch_plan(1 << 20, 1 << 16, 2) == ["prologue"] + lv * 13 + trip
        assert wt.launch_plan(1 << 20, 4, 1) == ["prologue"] + pair   # (L = 2)
    finally:
        del os.environ["WT_TRIPLE"]
    quad = ["prep", "quad", "sb_scan"]
    os.environ["WT_QUAD"] = "1"
    try:
        assert wt.launch_plan(1 << 20, 256, 1) == ["prologue"] + quad * 3 + pair
        assert wt.launch_plan(1 << 20, 1 << 16, 2) == ["prologue"] + quad * 4 + lv * 6 + pair
        assert wt.launch_plan(1 << 20, 32, 1) == ["prologue"] + quad + lv + pair
        assert wt.launch_plan(1 << 20, 16, 4) == ["prologue"] + quad + pair
        assert wt.launch_plan(1 << 20, 8, 1) == ["prologue"] + lv + pair   # L = 3: no quad
        os.environ["WT_TRIPLE"] = "1"
        assert wt.launch_plan(1 << 20, 32, 1) == ["prologue"] + quad + trip   # (T_2 from the quad)
        assert wt.launch_plan(1 << 20, 16, 4) == ["prologue"] + quad + pair   # (the quad reaches T_2 > T_{L-3})
        del os.environ["WT_TRIPLE"]
    finally:
        del os.environ["WT_QUAD"]
    # two levels of 1-byte symbols: the specialised pair pass (k_pair2)
    assert wt.launch_plan(1 << 20, 4, 1) == ["prologue"] + pair
    assert wt.launch_plan(1 << 20, 4, 2) == ["prologue"] + pair
    # fewer than 128 bytes of symbols (no TMA tensor rows) or WT_NO_PAIRN=1: the
    # general fused pair, which counts the leaves (C from the final scan)
    gpair = ["prep", "pair", "final_scan"]
    assert wt.launch_plan(127, 256, 1) == ["prologue"] + lv * 6 + gpair
    assert wt.launch_plan(31, 1 << 20, 4) == ["prologue"] + lv * 18 + gpair
    os.environ["WT_NO_PAIRN"] = "1"
    try:
        assert wt.launch_plan(1 << 20, 256, 1) == ["prologue"] + lv * 6 + gpair
        assert wt.launch_plan(1 << 20, 4, 1) == ["prologue"] + pair      # (k_pair2 is separate)
        assert wt.launch_plan(1 << 20, 4, 2) == ["prologue"] + gpair
    finally:
        del os.environ["WT_NO_PAIRN"]
    assert wt.launch_plan(1 << 20, 8, 1) == ["prologue"] + lv + pair
    assert wt.launch_plan(100, 2, 1) == ["prologue", "prep", "last_level"]
    assert wt.launch_plan(100, 1, 1) == ["prologue", "scan"]
    assert wt.launch_plan(0, 16, 1) == []
