"""GPU parity of the domain-decomposition paths (NEXT-3, the paper's dd,
P:633-687, 773-822) against the oracle:

* segmented builds (n > seg_max: segments built, then merged with 64-bit
  positions) -- at small n with WT_SEG_MAX lowered, and at n = 2^32 + 12345;
* the multi-GPU merge's device steps for G parts on one device: the plan
  kernel (== the host plan), every part merged from exactly the words the
  exchange would deliver, superblocks from the rank1 bases, the assembled
  parts == the oracle's tree of the concatenation.  (The transport itself,
  NCCL send/recv, is covered under gloo in tests/test_multirank.py.)
"""
import os

import numpy as np
import pytest
import torch

import oracle
import wt_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wt():
    from conftest import build_native
    build_native()
    import paper_1610_05994_b200 as wt
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return wt


def to_dev(S):
    return torch.from_numpy(S.view(np.int32) if S.dtype == np.uint32 else S).cuda()


def assert_tree(tree, ot, ctx=""):
    B = tree.bitmaps.cpu().numpy().view(np.uint32)
    SB = tree.superblocks.cpu().numpy().view(np.uint64)
    C = tree.node_offsets.cpu().numpy().view(np.uint64)
    assert np.array_equal(C, ot.node_offsets), f"node offsets {ctx}"
    for l in range(ot.L):
        assert np.array_equal(B[l], ot.bitmaps[l]), f"level {l} bitmap {ctx}"
        assert np.array_equal(SB[l], ot.superblocks[l]), f"level {l} superblocks {ctx}"


@pytest.fixture
def small_segments():
    old = os.environ.get("WT_SEG_MAX")
    os.environ["WT_SEG_MAX"] = str(3 * 4096)
    yield 3 * 4096
    if old is None:
        del os.environ["WT_SEG_MAX"]
    else:
        os.environ["WT_SEG_MAX"] = old


@pytest.mark.parametrize("sigma,n,dtype,kind", [(4, 100_003, None, "uniform"), (256, 50_000, None, "zipf"),
                                                (1 << 16, 40_961, np.uint16, "runs"),
                                                (1 << 20, 30_011, np.uint32, "zipf"), (2, 24_577, None, "uniform"),
                                                (1, 20_000, None, "uniform"), (230, 12_289, None, "sorted")])
def test_segmented_build_small(wt, small_segments, sigma, n, dtype, kind):
    S = wt_inputs.random_case(n + sigma, n, sigma, kind, dtype=dtype)
    assert n > small_segments
    plan = wt.launch_plan(n, sigma, S.itemsize)
    assert "dd_merge" in plan or sigma == 1
    tree = wt.build(to_dev(S), sigma)
    assert_tree(tree, oracle.build(S, sigma), f"segmented sigma={sigma} n={n}")
    # the range flag of a later segment reaches the status
    bad = S.copy()
    bad[-1] = sigma if sigma < (1 << (8 * S.itemsize)) else bad[-1]
    if sigma < (1 << (8 * S.itemsize)):
        with pytest.raises(wt.WtError) as e:
            wt.build(to_dev(bad), sigma)
        assert e.value.status == wt.WT_ERR_SYMBOL_RANGE


def test_segmented_build_beyond_2_32(wt):
    # n = 2^32 + 12345 (the paper's datasets reach n = 1.46e10; the
    # limit at n < 2^32 of other systems): three segments of <= 2^31,
    # merged with 64-bit positions; every level compared with the oracle word for
    # word, and access(i) == S[i] for all i
    from test_gpu_parity import device_access_all, oracle_levels_parallel
    n = (1 << 32) + 12345
    S, sigma = wt_inputs.generate(2, n)      # the cfg2 (DNA-like) recipe, extended
    d = torch.from_numpy(S).cuda()
    tree = wt.build(d, sigma)
    torch.cuda.synchronize()
    L = tree.levels
    B = tree.bitmaps.cpu().numpy().view(np.uint32)
    SB = tree.superblocks.cpu().numpy().view(np.uint64)
    C = tree.node_offsets.cpu().numpy().view(np.uint64)
    assert np.array_equal(C, oracle.node_offsets(S, sigma))
    for l, (ob, osb, onl) in oracle_levels_parallel(S, sigma, L):
        assert np.array_equal(B[l], ob), f"level {l} bitmap"
        assert np.array_equal(SB[l], osb), f"level {l} superblocks"
        assert np.array_equal(C[:: 1 << (L - l)], onl)
    del B, SB
    device_access_all(tree, S)


def simulate_parts(wt, S, sigma, cuts, parts):
    """The multi-GPU build's device steps with every 'rank' on this device."""
    from paper_1610_05994_b200.dist import merge_part, ones_before_parts, word_range
    k = len(cuts) - 1
    segs = [wt.build(to_dev(S[cuts[g]:cuts[g + 1]]), sigma) for g in range(k)]
    n = S.size
    offs = [t.node_offsets for t in segs]
    C = torch.empty_like(offs[0])
    wt.dd_offsets(offs, sigma, C)
    plan_d = wt.dd_plan_device(offs, sigma, n, parts)
    torch.cuda.synchronize()
    plan = plan_d.cpu().numpy()
    host = wt.dd_plan_host([o.cpu().numpy() for o in offs], sigma, parts)
    assert np.array_equal(plan, host), "device plan != host plan"
    L = plan.shape[0]
    bases = sum(ones_before_parts(segs[g], plan, g) for g in range(k)) if L else None
    out = []
    for p in range(parts):
        recv = [[None] * k for _ in range(L)]
        for l in range(L):
            for g in range(k):
                a, b = word_range(int(plan[l, p, g, 0]), int(plan[l, p, g, 1]))
                recv[l][g] = segs[g].bitmaps[l, a:b].clone()   # what the exchange delivers
        out.append(merge_part(offs, C, sigma, n, parts, p, plan, recv,
                              bases[:, p].tolist() if L else []))
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("sigma,n,k,dtype,kind", [(16, 30, 3, None, "uniform"), (4, 1_000_003, 2, None, "uniform"),
                                                  (256, 300_001, 5, None, "zipf"),
                                                  (1 << 16, 200_000, 8, np.uint16, "runs"),
                                                  (1 << 20, 150_001, 4, np.uint32, "zipf"),
                                                  (3, 5000, 7, None, "uniform"), (256, 100, 8, None, "zipf")])
def test_multi_part_merge(wt, sigma, n, k, dtype, kind):
    S = wt_inputs.random_case(n * k + 7, n, sigma, kind, dtype=dtype)
    step = -(-n // k)
    step = -(-step // 16) * 16
    cuts = [min(g * step, n) for g in range(k)] + [n]   # (16-byte aligned cuts; trailing ones may be empty)
    ot = oracle.build(S, sigma)
    for parts in sorted({1, k, 3}):
        shards = simulate_parts(wt, S, sigma, cuts, parts)
        L = ot.L
        for sh in shards:
            assert np.array_equal(sh.node_offsets.cpu().numpy().view(np.uint64), ot.node_offsets)
            b, e = sh.block_begin, sh.block_end
            for l in range(L):
                got = sh.bitmaps[l].cpu().numpy().view(np.uint32)
                assert np.array_equal(got, ot.bitmaps[l][16 * b:16 * e]), f"part {sh.part}/{parts} level {l}"
                sb = sh.superblocks[l].cpu().numpy().view(np.uint64)
                assert np.array_equal(sb, ot.superblocks[l][b:e + 1]), f"part {sh.part}/{parts} sb level {l}"
