"""GPU parity of the interior fused groups (a5, k = 2: k_quad, wt_quad.cuh)
against the oracle.  The quad pass is opt-in (WT_QUAD=1; slower than the two
level passes on B200), so these tests switch it on: every level
of the tree -- the ones the quads write (B_l, SB_l, B_{l+1} and its scanned
superblocks) and the ones the passes after them write from the T_{l+2},
per-tile counts and node sizes the quads hand over -- compared word for word
(Alg. 1 lines 5-14)."""
import os

import numpy as np
import pytest
import torch

import oracle
import wt_inputs

pytestmark = pytest.mark.gpu

QTILE = {1: 8192, 2: 4096, 4: 2048}   # quad tile (symbols) per width


@pytest.fixture(scope="module")
def wt():
    from conftest import build_native
    build_native()
    import paper_1610_05994_b200 as wt
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return wt


@pytest.fixture
def quad_on():
    old = os.environ.get("WT_QUAD")
    os.environ["WT_QUAD"] = "1"
    yield
    if old is None:
        del os.environ["WT_QUAD"]
    else:
        os.environ["WT_QUAD"] = old


def to_dev(S):
    return torch.from_numpy(S.view(np.int32) if S.dtype == np.uint32 else S).cuda()


def check(wt, S, sigma, ctx=""):
    plan = wt.launch_plan(S.size, sigma, S.itemsize)
    tree = wt.build(to_dev(S), sigma)
    ot = oracle.build(S, sigma)
    B = tree.bitmaps.cpu().numpy().view(np.uint32)
    SB = tree.superblocks.cpu().numpy().view(np.uint64)
    C = tree.node_offsets.cpu().numpy().view(np.uint64)
    assert np.array_equal(C, ot.node_offsets), f"C {ctx}"
    for l in range(ot.L):
        if not np.array_equal(B[l], ot.bitmaps[l]):
            bad = np.nonzero(B[l] != ot.bitmaps[l])[0]
            raise AssertionError(f"level {l} bitmap differs at {bad.size} words, first {bad[:5]} {ctx}")
        assert np.array_equal(SB[l], ot.superblocks[l]), f"level {l} superblocks {ctx}"
    return plan


@pytest.mark.parametrize("sigma,n,kind", [
    (16, 100_000, "uniform"), (256, 300_000, "zipf"), (32, 77_777, "runs"), (256, 1_000_003, "sorted"),
    (1 << 12, 200_001, "zipf"), (1 << 16, 123_457, "zipf"), (1 << 16, 500_000, "uniform"),
    (1 << 20, 300_001, "zipf"), (1000, 65_536, "runs"), (17, 8191, "uniform"), (1 << 10, 400_000, "zipf"),
    (3000, 250_000, "sorted"), (1 << 24, 100_000, "uniform"),
])
def test_quad_random(wt, quad_on, sigma, n, kind):
    S = wt_inputs.random_case(4242 + n % 1000, n, sigma, kind)
    plan = check(wt, S, sigma, f"sigma={sigma} n={n} {kind}")
    assert "quad" in plan


@pytest.mark.parametrize("width", [1, 2, 4])
def test_quad_edge_sizes(wt, quad_on, width):
    # empty, tiny, one tile +- 1, a partial 16-byte chunk at the tail, many tiles
    sigma = {1: 200, 2: 3000, 4: 70_000}[width]
    dt = {1: np.uint8, 2: np.uint16, 4: np.uint32}[width]
    T = QTILE[width]
    for n in (0, 1, 5, 15, 16, 17, 511, 512, 513, T - 1, T, T + 1, 3 * T + 7, 17 * T - 3):
        S = wt_inputs.random_case(n + 7, n, sigma, "uniform", dtype=dt)
        check(wt, S, sigma, f"width={width} n={n}")


def test_quad_many_small_nodes(wt, quad_on):
    # the deepest quad (l = 6: 64 nodes, up to 64 segments per tile) over many
    # tiny and empty nodes: a sparse alphabet with a few heavy symbols
    rng = np.random.default_rng(7)
    sigma = 1 << 12
    n = 200_000
    S = rng.choice(np.arange(0, sigma, 37, dtype=np.uint16), size=n)
    S[rng.integers(0, n, n // 3)] = 5
    check(wt, S.astype(np.uint16), sigma, "sparse alphabet")
    # every node of level 6 is tiny: one tile spans dozens of them
    S = (np.arange(n, dtype=np.uint32) % sigma).astype(np.uint16)
    check(wt, np.sort(S), sigma, "sorted cycles")


def test_quad_symbol_range_error(wt, quad_on):
    S = wt_inputs.random_case(3, 50_000, 200, "uniform")
    S[31_337] = 201
    with pytest.raises(wt.WtError) as e:
        wt.build(to_dev(S), 200)
    assert e.value.status == wt.WT_ERR_SYMBOL_RANGE


def test_quad_full_size_cfg3(wt, quad_on):
    # the u8 n = 2^28, sigma = 256 configuration (BASELINE configs[2]) with
    # three quads: every level word for word
    from test_gpu_parity import oracle_levels_parallel
    S, sigma = wt_inputs.generate(3)
    assert wt.launch_plan(S.size, sigma, 1).count("quad") == 3
    tree = wt.build(to_dev(S), sigma)
    torch.cuda.synchronize()
    B = tree.bitmaps.cpu().numpy().view(np.uint32)
    SB = tree.superblocks.cpu().numpy().view(np.uint64)
    C = tree.node_offsets.cpu().numpy().view(np.uint64)
    assert np.array_equal(C, oracle.node_offsets(S, sigma))
    for l, (ob, osb, _) in oracle_levels_parallel(S, sigma, tree.levels):
        assert np.array_equal(B[l], ob), f"level {l} bitmap"
        assert np.array_equal(SB[l], osb), f"level {l} superblocks"


def test_quad_inside_segmented_build(wt, quad_on):
    # a segmented build (n > seg_max, here lowered) runs the direct sequence --
    # with its quads -- on every segment, then merges
    old = os.environ.get("WT_SEG_MAX")
    os.environ["WT_SEG_MAX"] = str(4 * 4096)
    try:
        for sigma, n, kind in [(256, 100_003, "zipf"), (1 << 16, 70_001, "uniform")]:
            S = wt_inputs.random_case(n, n, sigma, kind)
            plan = check(wt, S, sigma, f"segmented sigma={sigma} n={n}")
            assert "dd_merge" in plan and "quad" in plan
    finally:
        if old is None:
            del os.environ["WT_SEG_MAX"]
        else:
            os.environ["WT_SEG_MAX"] = old
