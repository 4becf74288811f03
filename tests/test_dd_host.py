"""Host arithmetic of the domain-decomposition merge (NEXT-3, the paper's dd,
P:633-687, 799-822), no GPU: the library's plan (wt_dd_plan, the same
__host__ __device__ code its plan kernel runs) against a brute-force walk of
the merged node order over oracle segment trees, and the part split."""
import numpy as np
import pytest

import dd_ref
import oracle
import wt_inputs


@pytest.fixture(scope="module")
def wt():
    from conftest import build_native
    build_native()
    import paper_1610_05994_b200 as wt
    return wt


def segment_trees(S, sigma, cuts):
    return [oracle.build(S[cuts[i]:cuts[i + 1]], sigma) for i in range(len(cuts) - 1)]


@pytest.mark.parametrize("sigma,n,k,parts,kind", [
    (16, 30, 3, 2, "uniform"), (4, 5000, 2, 3, "uniform"), (256, 20000, 5, 4, "zipf"),
    (1 << 12, 9000, 8, 8, "runs"), (3, 1000, 4, 7, "uniform"), (1 << 16, 3000, 3, 2, "zipf"),
    (2, 700, 1, 1, "uniform"), (1000, 4096 + 13, 6, 5, "sorted"), (1, 500, 3, 2, "uniform"),
])
def test_plan_matches_brute_force(wt, sigma, n, k, parts, kind):
    S = wt_inputs.random_case(n * k + parts, n, sigma, kind)
    rng = np.random.default_rng(n)
    cuts = np.sort(np.concatenate([[0, n], rng.integers(0, n + 1, k - 1)]))   # (empty segments allowed)
    trees = segment_trees(S, sigma, cuts)
    L = oracle.levels(sigma)
    ranges = []
    for p in range(parts):
        b, e = wt.dd_part_blocks(n, parts, p)
        ranges.append((min(n, 512 * b), min(n, 512 * e)))
    got = wt.dd_plan_host([t.node_offsets for t in trees], sigma, parts)
    want = dd_ref.plan_brute([t.node_offsets for t in trees], L, n, ranges)
    assert got.shape == (L, parts, k, 2)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,parts", [(0, 3), (1, 1), (511, 2), (512, 2), (513, 2), (5000, 3), (1 << 20, 7),
                                     ((1 << 33) + 5, 8)])
def test_part_blocks_tile_the_tree(wt, n, parts):
    nblk = (n + 511) // 512
    prev = 0
    for p in range(parts):
        b, e = wt.dd_part_blocks(n, parts, p)
        assert b == prev and b <= e <= nblk
        assert e - b <= -(-nblk // parts)
        prev = e
    assert prev == nblk
    assert wt.dd_part_blocks(n, parts, parts) == (0, 0)    # out of range: empty


def test_segmented_sizes_and_plan(wt):
    # n beyond seg_max (2^31): the build is segmented; its workspace holds the segment
    # trees and one segment's build workspace; the launch plan lists each segment's
    # build, then the merge (offsets, per level merge + superblock scan, flag OR)
    n = (1 << 32) + 12345
    s = wt.sizes(n, 4, 1)
    assert s.levels == 2 and s.words_per_level == 16 * ((n + 511) // 512)
    assert s.workspace_bytes > 2 * n // 8   # three segment trees of two levels
    plan = wt.launch_plan(n, 4, 1)
    seg = ["prologue", "prep", "pair", "final_scan", "leaf_offsets"]
    assert plan == (seg + ["flags"]) * 3 + ["dd_offsets"] + ["dd_merge", "dd_superblocks"] * 2
    assert wt.launch_plan(1 << 20, 4, 1) == seg
