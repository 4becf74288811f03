"""Pins for the CPU oracle (no GPU).  The oracle is checked against things other
than itself: the paper's printed worked example, the brute-force and recursive
definitions in tests/brute.py, closed forms and invariants.  A plausible slip in
oracle/wt_oracle.c (dropped stability, wrong bit/level order, exclusive vs
inclusive rank, wrong superblock base, wrong node offsets) fails one of these.
"""
import itertools
import json
import os

import numpy as np
import pytest

import brute
import oracle
import wt_inputs

HERE = os.path.dirname(os.path.abspath(__file__))
SIGMAS = [1, 2, 3, 4, 5, 7, 16, 27, 230, 256, 1000, 1 << 10, 1 << 14, 1 << 16]


def fig2():
    with open(os.path.join(HERE, "golden", "fig2_once_upon.json")) as f:
        g = json.load(f)
    alpha = g["alphabet_first_appearance"]
    S = np.array([alpha.index(ch) for ch in g["text"]], np.uint8)
    return g, alpha, S


# ----------------------------------------------------------------- golden


def test_fig2_printed_access_path():
    g, alpha, S = fig2()
    t = oracle.build(S, g["sigma"])
    p = g["printed"]
    sym, path = t.access(24, with_path=True)
    assert alpha[sym] == p["access_24_symbol"] and sym == p["access_24_code"]
    assert path[: t.L] == p["access_24_in_node_indices"]          # 24 -> 7 -> 4 -> 2
    # bits read at each level = the code's bits MSB first (0 = left, 1 = right)
    assert [(sym >> (t.L - 1 - l)) & 1 for l in range(t.L)] == p["access_24_bits_read"]
    # the bit actually stored at the visited position of each level
    lo = 0
    v = 0
    for l in range(t.L):
        q = lo + path[l]
        bit = int((t.bitmaps[l][q >> 5] >> (q & 31)) & 1)
        assert bit == p["access_24_bits_read"][l]
        v = 2 * v + bit
        lo = int(t.node_offsets[v << (t.L - 1 - l)])
    # alphabet ranges halve as printed
    for l, (a, b) in enumerate(p["access_24_ranges"]):
        w = 1 << (t.L - l)
        assert (sym // w * w, sym // w * w + w - 1) == (a, b)


def test_fig3_caption_positions_zero_based():
    g, alpha, S = fig2()
    for pos, ch in g["printed"]["fig3_positions"].items():
        assert alpha[S[int(pos)]] == ch


def test_fig2_rank_select_and_reconstruction():
    g, alpha, S = fig2()
    t = oracle.build(S, g["sigma"])
    assert t.rank(alpha.index("t"), 29) == g["derived"]["rank_t_29"]
    assert t.select(alpha.index("a"), 2) == g["derived"]["select_a_2"]
    assert "".join(alpha[t.access(i)] for i in range(S.size)) == g["text"]


def test_fig2_matches_both_definitions():
    g, alpha, S = fig2()
    t = oracle.build(S, g["sigma"])
    rec = brute.levels_by_recursion(S, 16)
    srt = brute.levels_by_stable_sort(S, 16)
    for l in range(t.L):
        W = brute.words_per_level(S.size)
        assert np.array_equal(t.bitmaps[l], brute.pack_bits(np.array(rec[l]), W))
        assert np.array_equal(t.bitmaps[l], brute.pack_bits(srt[l], W))


# ------------------------------------------------------ definition checks


def check_against_stable_sort(S, sigma):
    t = oracle.build(S, sigma)
    n = S.size
    W = brute.words_per_level(n)
    assert t.L == brute.n_levels(sigma)
    assert np.array_equal(t.node_offsets, brute.node_offsets(S, sigma))
    for l, bits in enumerate(brute.levels_by_stable_sort(S, sigma)):
        assert np.array_equal(t.bitmaps[l], brute.pack_bits(bits, W)), f"level {l}"
        assert np.array_equal(t.superblocks[l], brute.superblocks_from_bits(bits, n)), f"SB {l}"
    return t


@pytest.mark.parametrize("sigma", SIGMAS)
def test_random_cases_vs_stable_sort(sigma):
    rng = np.random.default_rng(sigma)
    for k in range(12):
        n = int(rng.choice([0, 1, 31, 32, 33, 511, 512, 513, 1000, 4096 + 17, 20000]))
        kind = ["uniform", "zipf", "runs", "sorted", "reverse", "constant"][k % 6]
        S = wt_inputs.random_case(1000 * sigma + k, n, sigma, kind)
        check_against_stable_sort(S, sigma)


def test_two_hundred_random_cases():
    # SPEC acceptance-style: 200 seeded cases over mixed sigma and n
    rng = np.random.default_rng(2024)
    for k in range(200):
        sigma = int(rng.choice([1, 2, 3, 4, 16, 27, 230, 1 << 10, 1 << 14]))
        n = int(rng.integers(0, 3000))
        S = wt_inputs.random_case(k, n, sigma, "uniform")
        check_against_stable_sort(S, sigma)


@pytest.mark.parametrize("sigma", [1, 2, 3, 4])
def test_recursive_definition_exhaustive(sigma):
    # every sequence with n <= 5 over [0, sigma)
    W = None
    for n in range(0, 6):
        W = brute.words_per_level(n)
        for seq in itertools.product(range(sigma), repeat=n):
            S = np.array(seq, np.uint8)
            t = oracle.build(S, sigma)
            rec = brute.levels_by_recursion(S, sigma)
            for l in range(t.L):
                assert np.array_equal(t.bitmaps[l], brute.pack_bits(np.array(rec[l], np.uint8), W)), (seq, l)


def test_cfg1_full_brute_force():
    S, sigma = wt_inputs.generate(1)
    check_against_stable_sort(S, sigma)


# ------------------------------------------------ closed forms, invariants


def test_closed_forms():
    rng = np.random.default_rng(7)
    for sigma in [2, 4, 16, 256, 1 << 12]:
        L = brute.n_levels(sigma)
        S = wt_inputs.random_case(int(rng.integers(1 << 30)), 5000, sigma)
        t = oracle.build(S, sigma)
        n = S.size
        W = brute.words_per_level(n)
        # B_0 is the MSB of S in S order (no permutation at the root)
        assert np.array_equal(t.bitmaps[0], brute.pack_bits((S.astype(np.int64) >> (L - 1)) & 1, W))
        # popcount(B_l) = #{j : bit (L-1-l) of S[j]} and the last SB entry is it
        for l in range(L):
            ones = int((((S.astype(np.int64) >> (L - 1 - l)) & 1)).sum())
            assert int(t.superblocks[l][-1]) == ones
            assert sum(bin(int(w)).count("1") for w in t.bitmaps[l]) == ones
        # per-node ones = size of the right child, from C
        C = t.node_offsets.astype(np.int64)
        for l in range(L):
            s = L - l
            bits = brute.unpack_level(t.bitmaps[l], n)
            for v in range(min(1 << l, 64)):
                a, b = C[v << s], C[(v + 1) << s]
                assert int(bits[a:b].sum()) == C[(v + 1) << s] - C[(2 * v + 1) << (s - 1)]
        # node starts from level counts equal C strides (checked inside oracle_build too)
        for l in range(L):
            _, _, Nl = oracle.build_level(S, sigma, l)
            assert np.array_equal(Nl, t.node_offsets[:: 1 << (L - l)])
        # sigma == 2: B_0 = S
        if sigma == 2:
            assert np.array_equal(t.bitmaps[0], brute.pack_bits(S, W))


def test_sorted_input_is_never_permuted():
    # 'cont': every T_l = S, so B_l[j] = bit (L-1-l) of S[j]
    for sigma in [4, 16, 256, 1 << 14]:
        S = wt_inputs.random_case(0, 10000, sigma, "cont")
        t = oracle.build(S, sigma)
        L = t.L
        W = brute.words_per_level(S.size)
        for l in range(L):
            assert np.array_equal(t.bitmaps[l], brute.pack_bits((S.astype(np.int64) >> (L - 1 - l)) & 1, W))


def test_constant_sequence():
    for sigma, c in [(4, 0), (4, 3), (256, 0xA5), (1 << 16, 12345)]:
        S = np.full(3001, c, wt_inputs.dtype_for_sigma(sigma))
        t = oracle.build(S, sigma)
        for l in range(t.L):
            bit = (c >> (t.L - 1 - l)) & 1
            bits = brute.unpack_level(t.bitmaps[l], S.size)
            assert (bits == bit).all()
            assert int(t.superblocks[l][-1]) == bit * S.size


# ----------------------------------------------------------------- queries


@pytest.mark.parametrize("sigma", [1, 2, 3, 16, 230, 1 << 12])
def test_queries_vs_brute_force(sigma):
    S = wt_inputs.random_case(sigma, 1500, sigma, "zipf" if sigma > 2 else "uniform")
    t = oracle.build(S, sigma)
    assert [t.access(i) for i in range(S.size)] == [int(x) for x in S]
    rng = np.random.default_rng(1)
    for _ in range(300):
        c = int(rng.integers(sigma))
        i = int(rng.integers(S.size))
        assert t.rank(c, i) == int((S[: i + 1] == c).sum())
    total = sum(t.rank(c, S.size - 1) for c in range(min(sigma, 300)))
    if sigma <= 300:
        assert total == S.size
    for c in range(min(sigma, 40)):
        occ = np.nonzero(S == c)[0]
        for k in range(0, occ.size, max(1, occ.size // 7)):
            assert t.select(c, k + 1) == int(occ[k])


def test_select_samples_vs_brute_force():
    # the select index (NEXT-1) pinned to the brute-force bitmaps (stable-sort
    # definition) and to occurrence counting: sample k of (level l, bit b) is the
    # position of the (k * 2^s)-th b-bit; a small shift exercises many samples
    for sigma, n, kind in [(16, 5000, "zipf"), (256, 20000, "uniform"), (3, 9001, "runs"), (1 << 10, 777, "sorted")]:
        S = wt_inputs.random_case(n + sigma, n, sigma, kind)
        ot = oracle.build(S, sigma)
        shift = 5
        smp = ot.select_samples(shift)
        for l, bits in enumerate(brute.levels_by_stable_sort(S, sigma)):
            bits = np.asarray(bits, np.uint8)
            for b in (0, 1):
                cnt = 0
                for q in range(n):       # walk the level: every 2^shift-th b-bit is sampled
                    if bits[q] == b:
                        if cnt % (1 << shift) == 0:
                            assert smp[l, b, cnt >> shift] == q
                        cnt += 1
                assert np.all(smp[l, b, (cnt + (1 << shift) - 1) >> shift:] == n)   # the rest: sentinel n


def test_sigma_one_and_empty():
    t = oracle.build(np.zeros(5, np.uint8), 1)
    assert t.L == 0 and list(t.node_offsets) == [0, 5]
    assert t.access(3) == 0 and t.rank(0, 3) == 4 and t.select(0, 2) == 1
    t = oracle.build(np.zeros(0, np.uint8), 16)
    assert t.bitmaps.shape == (4, 0) and t.superblocks.shape == (4, 1)
    assert not t.superblocks.any() and not t.node_offsets.any()


def test_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(np.array([0, 1, 4], np.uint8), 4)
    assert e.value.status == oracle.ERR_SYMBOL_RANGE
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(np.array([0, 1, 2], np.uint8), 3 * 0 or 2)  # 2 >= sigma=2
    assert e.value.status == oracle.ERR_SYMBOL_RANGE
    with pytest.raises(oracle.OracleError):
        oracle.build(np.array([0], np.uint8), 0)
    with pytest.raises(oracle.OracleError):
        oracle.build(np.array([0], np.uint8), 257)  # sigma beyond the 1-byte width
    t = oracle.build(np.array([0, 1, 2], np.uint8), 3)
    with pytest.raises(oracle.OracleError):
        t.access(3)
    with pytest.raises(oracle.OracleError):
        t.rank(3, 0)
    with pytest.raises(oracle.OracleError):
        t.select(0, 2)


@pytest.mark.parametrize("sigma", [2, 3, 16, 230, 1 << 12])
def test_matrix_oracle_vs_reversed_prefix_sort(sigma):
    # the wavelet matrix (NEXT-4) pinned to an independent characterisation:
    # T_l = S stably sorted by its top l bits READ IN REVERSE (the global stable
    # partitions by bit 0, then bit 1, ... compose to that order); B_l = bit
    # (L-1-l) of T_l; zeros[l] = #{s : bit (L-1-l) of s = 0} in any order
    for kind in ("uniform", "zipf", "runs", "sorted"):
        S = wt_inputs.random_case(sigma + 7, 3001, sigma, kind)
        om = oracle.build_matrix(S, sigma)
        L = om.L
        s64 = S.astype(np.int64)
        for l in range(L):
            top = s64 >> (L - l) if l else np.zeros_like(s64)
            rev = np.zeros_like(top)
            for k in range(l):                    # reverse the l-bit prefix
                rev |= ((top >> k) & 1) << (l - 1 - k)
            T = s64[np.argsort(rev, kind="stable")]
            bits = ((T >> (L - 1 - l)) & 1).astype(np.uint8)
            assert np.array_equal(om.bitmaps[l], brute.pack_bits(bits, om.bitmaps.shape[1]))
            assert int(om.zeros[l]) == int(((s64 >> (L - 1 - l)) & 1 == 0).sum())
            assert int(om.superblocks[l, -1]) == int(bits.sum())
