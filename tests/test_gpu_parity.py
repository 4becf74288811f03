"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element, on seeded inputs.  All wavelet-tree outputs are integers, so the
bar is bit-exact equality of every bitmap word, superblock and node offset."""
import os

import numpy as np
import pytest
import torch

import brute
import oracle
import wt_inputs

pytestmark = pytest.mark.gpu

TILE = {1: 2048, 2: 1024, 4: 512}   # level-pass tile (positions) per symbol width


@pytest.fixture(scope="module")
def wt():
    from conftest import build_native
    build_native()
    import paper_1610_05994_b200 as wt
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return wt


def to_dev(S: np.ndarray) -> torch.Tensor:
    t = torch.from_numpy(S.view(np.int32) if S.dtype == np.uint32 else S)
    return t.cuda()


def np_tree(tree):
    return (tree.bitmaps.cpu().numpy().view(np.uint32), tree.superblocks.cpu().numpy().view(np.uint64),
            tree.node_offsets.cpu().numpy().view(np.uint64))


def assert_same(tree, ot, ctx=""):
    B, SB, C = np_tree(tree)
    assert tree.levels == ot.L, ctx
    assert np.array_equal(C, ot.node_offsets), f"node offsets {ctx}"
    for l in range(ot.L):
        if not np.array_equal(B[l], ot.bitmaps[l]):
            bad = np.nonzero(B[l] != ot.bitmaps[l])[0]
            raise AssertionError(f"level {l} bitmap differs at {bad.size} words, first {bad[:5]} {ctx}")
        assert np.array_equal(SB[l], ot.superblocks[l]), f"level {l} superblocks {ctx}"


def check_case(wt, S, sigma, ctx=""):
    tree = wt.build(to_dev(S), sigma)
    assert_same(tree, oracle.build(S, sigma), ctx)
    return tree


# ---------------------------------------------------------------- small cases


@pytest.mark.parametrize("sigma", [1, 2, 3, 4, 5, 16, 27, 230, 256, 1000, 1 << 12, 1 << 16, 70000, 1 << 24])
def test_random_small(wt, sigma):
    rng = np.random.default_rng(sigma)
    for k, kind in enumerate(["uniform", "zipf", "runs", "sorted", "reverse", "constant"]):
        n = int(rng.integers(1, 70000))
        S = wt_inputs.random_case(100 * sigma + k, n, sigma, kind)
        check_case(wt, S, sigma, f"sigma={sigma} n={n} kind={kind}")


@pytest.mark.parametrize("width", [1, 2, 4])
def test_edge_sizes(wt, width):
    t = TILE[width]
    sigma = {1: 256, 2: 1 << 16, 4: 1 << 20}[width]
    dtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[width]
    for n in [0, 1, 2, 31, 32, 33, 511, 512, 513, 1023, t - 1, t, t + 1, 2 * t - 1, 2 * t, 2 * t + 1,
              3 * t + 512, 7 * t + 33]:
        for sg in (sigma, 3):
            S = wt_inputs.random_case(n, n, sg, "uniform", dtype=dtype)
            check_case(wt, S, sg, f"n={n} sigma={sg} w={width}")


def test_two_hundred_random_cases(wt):
    rng = np.random.default_rng(99)
    for k in range(200):
        sigma = int(rng.choice([1, 2, 3, 4, 16, 27, 230, 1 << 10, 1 << 14, 1 << 18]))
        n = int(rng.integers(0, 40000))
        kind = ["uniform", "zipf", "runs", "sorted"][k % 4]
        dtype = [None, np.uint16, np.uint32][k % 3] if sigma <= 65536 else np.uint32
        S = wt_inputs.random_case(k, n, sigma, kind, dtype=dtype)
        check_case(wt, S, sigma, f"k={k}")


@pytest.mark.parametrize("y", [4, 8, 12, 14])
def test_cont_rand_locality(wt, y):
    # the paper's locality workloads: n/sigma copies of each symbol,
    # sorted (cont) or shuffled (rand), 4-byte symbols; cont makes every T_l = S
    sigma = 1 << y
    for kind in ("cont", "rand"):
        S = wt_inputs.random_case(y, 150_001, sigma, kind, dtype=np.uint32)
        tree = check_case(wt, S, sigma, f"{kind} sigma=2^{y}")
        if kind == "cont":
            B, _, _ = np_tree(tree)
            L = tree.levels
            bits = ((S[None, :] >> (L - 1 - np.arange(L))[:, None]) & 1).astype(np.uint8)
            packed = np.packbits(bits, axis=1, bitorder="little")
            for l in range(L):
                assert np.array_equal(B[l].view(np.uint8)[:packed.shape[1]], packed[l])


def test_many_tiles(wt):
    # thousands of level tiles: the per-level tile-prefix scans (k_prep's decoupled
    # look-back) span many 32-tile windows
    for sigma, dtype in [(4, np.uint8), (256, np.uint8), (1 << 16, np.uint16), (1 << 20, np.uint32)]:
        S = wt_inputs.random_case(7, 3_000_017, sigma, "zipf", dtype=dtype)
        check_case(wt, S, sigma, f"sigma={sigma}")


def test_symbol_range_error(wt):
    for S, sigma in [(np.array([0, 1, 4, 2], np.uint8), 4), (np.array([0, 2, 1], np.uint8), 2),
                     (np.full(100000, 300, np.uint16), 256), (np.array([5], np.uint32), 3)]:
        with pytest.raises(wt.WtError) as e:
            wt.build(to_dev(S), sigma)
        assert e.value.status == wt.WT_ERR_SYMBOL_RANGE
    # L = 2, u8 (the pass that reads S itself checks the range): a bad symbol
    # in a full tile and in the ragged last tile, sigma = 3 and 4
    for pos, val, sigma in [(3000, 3, 3), (100, 7, 4), (4500, 255, 4), (4999, 3, 3), (0, 4, 3)]:
        S = np.random.default_rng(pos).integers(0, sigma, 5000).astype(np.uint8)
        S[pos] = val
        with pytest.raises(wt.WtError) as e:
            wt.build(to_dev(S), sigma)
        assert e.value.status == wt.WT_ERR_SYMBOL_RANGE
    # a valid build afterwards on the same device still works
    check_case(wt, np.array([0, 1, 2, 3], np.uint8), 4)


def test_async_status_and_determinism(wt):
    S = wt_inputs.random_case(5, 500_000, 1 << 14, "zipf", dtype=np.uint16)
    d = to_dev(S)
    status = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    t1 = wt.build_async(d, 1 << 14, status=status)
    t2 = wt.build_async(d, 1 << 14)
    torch.cuda.synchronize()
    assert int(status.item()) == wt.WT_OK
    for a, b in zip(np_tree(t1), np_tree(t2)):
        assert np.array_equal(a, b)
    bad = d.clone()
    bad[1234] = 20000
    wt.build_async(bad, 1 << 14, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == wt.WT_ERR_SYMBOL_RANGE


def test_side_stream_and_events(wt):
    # launches on a torch-created (non-default) stream, profiled with torch events
    S = wt_inputs.random_case(3, 200_000, 256, "zipf")
    d = to_dev(S)
    s = torch.cuda.Stream()
    plan = wt.launch_plan(S.size, 256, 1)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * len(plan))]
    wt.set_profile_events(evs)
    with torch.cuda.stream(s):
        tree = wt.build_async(d, 256, stream=s)
    wt.set_profile_events(None)
    s.synchronize()
    assert all(evs[2 * i].elapsed_time(evs[2 * i + 1]) >= 0 for i in range(len(plan)))
    assert_same(tree, oracle.build(S, 256))


def test_build_from_host_matches(wt):
    S = wt_inputs.random_case(11, 1_000_003, 230, "zipf")
    h = wt.build_from_host(torch.from_numpy(S), 230)
    ot = oracle.build(S, 230)
    assert np.array_equal(h.bitmaps.numpy().view(np.uint32), ot.bitmaps)
    assert np.array_equal(h.superblocks.numpy().view(np.uint64), ot.superblocks)
    assert np.array_equal(h.node_offsets.numpy().view(np.uint64), ot.node_offsets)


def test_build_from_host_async_two_streams(wt):
    # two builds in flight on two streams (different inputs, workspaces, host trees),
    # each compared with the oracle; then the range error through the status word
    cases = [(wt_inputs.random_case(12, 700_001, 256, "zipf"), 256),
             (wt_inputs.random_case(13, 300_007, 1 << 16, "uniform", dtype=np.uint16), 1 << 16)]
    dev = torch.device("cuda", 0)
    streams = [torch.cuda.Stream(device=dev) for _ in cases]
    outs = []
    for (S, sigma), st in zip(cases, streams):
        h = torch.from_numpy(S).pin_memory()
        ht = wt.alloc_host_tree(S.size, sigma, S.itemsize)
        ws = wt.alloc_workspace(S.size, sigma, S.itemsize, dev, host=True)
        status = torch.full((1,), -1, dtype=torch.int32).pin_memory()
        wt.build_from_host_async(h, sigma, ht, ws, status, stream=st)
        outs.append((S, sigma, ht, status, h, ws))
    torch.cuda.synchronize()
    for S, sigma, ht, status, _, _ in outs:
        assert int(status.item()) == wt.WT_OK
        ot = oracle.build(S, sigma)
        assert np.array_equal(ht.bitmaps.numpy().view(np.uint32), ot.bitmaps)
        assert np.array_equal(ht.superblocks.numpy().view(np.uint64), ot.superblocks)
        assert np.array_equal(ht.node_offsets.numpy().view(np.uint64), ot.node_offsets)
    bad = np.array([0, 1, 5, 2] * 1000, np.uint8)
    ht = wt.alloc_host_tree(bad.size, 4, 1)
    ws = wt.alloc_workspace(bad.size, 4, 1, dev, host=True)
    status = torch.zeros(1, dtype=torch.int32).pin_memory()
    wt.build_from_host_async(torch.from_numpy(bad).pin_memory(), 4, ht, ws, status, stream=streams[0])
    streams[0].synchronize()
    assert int(status.item()) == wt.WT_ERR_SYMBOL_RANGE
    with pytest.raises(ValueError):
        wt.build_from_host_async(torch.from_numpy(bad), 4, ht, ws, status.cuda())


# ------------------------------------------------------------------- queries


@pytest.mark.parametrize("sigma,n", [(1, 1000), (2, 5000), (16, 70001), (230, 100000), (1 << 16, 200000),
                                     (1 << 20, 100000)])
def test_queries(wt, sigma, n):
    S = wt_inputs.random_case(sigma, n, sigma, "zipf" if sigma > 2 else "uniform",
                              dtype=np.uint32 if sigma > 65536 else None)
    tree = check_case(wt, S, sigma)
    pos = torch.arange(n, device="cuda")
    got = tree.access(pos).cpu().numpy()
    assert np.array_equal(got, S.astype(np.int64))
    rng = np.random.default_rng(3)
    m = 5000
    c = rng.integers(0, sigma, m)
    c[: m // 2] = S[rng.integers(0, n, m // 2)]          # half the queries on present symbols
    i = rng.integers(0, n, m)
    cnt = tree.rank(torch.from_numpy(c.astype(np.int32)).cuda(), torch.from_numpy(i).cuda()).cpu().numpy()
    order = np.argsort(S, kind="stable")
    ot = oracle.build(S, sigma)
    for k in range(0, m, 50):
        assert cnt[k] == ot.rank(int(c[k]), int(i[k]))
    # brute-force count for all m via sorted occurrence lists
    Ssorted = S[order]
    for k in range(m):
        lo = np.searchsorted(Ssorted, c[k], "left")
        hi = np.searchsorted(Ssorted, c[k], "right")
        assert cnt[k] == np.searchsorted(order[lo:hi], i[k], "right")
    # select: j-th occurrence
    cs, js, want = [], [], []
    for sym in np.unique(S)[:200]:
        occ = np.nonzero(S == sym)[0]
        for j in (1, occ.size, (occ.size + 1) // 2):
            cs.append(sym)
            js.append(j)
            want.append(occ[j - 1])
    got = tree.select(torch.tensor(np.array(cs, np.int32)).cuda(), torch.tensor(js).cuda()).cpu().numpy()
    assert np.array_equal(got, np.array(want))
    # the select index (NEXT-1): the samples equal the oracle's by definition, and
    # the indexed select returns the same positions
    idx = wt.select_index(tree)
    if ot.L:
        assert np.array_equal(idx.cpu().numpy().view(np.uint32), ot.select_samples(12))
        got2 = wt.select(tree, torch.tensor(np.array(cs, np.int32)).cuda(), torch.tensor(js).cuda(),
                         index=idx).cpu().numpy()
        assert np.array_equal(got2, np.array(want))


@pytest.mark.parametrize("sigma,n", [(2, 1), (4, 511), (4, 512), (256, 4097), (256, 300_001), (1 << 16, 1_000_003)])
def test_select_index_edges(wt, sigma, n):
    # sample boundaries: n around 512 / 4096, a single symbol, many samples per level
    S = wt_inputs.random_case(n, n, sigma, "uniform", dtype=np.uint16 if sigma > 256 else None)
    tree = check_case(wt, S, sigma)
    ot = oracle.build(S, sigma)
    idx = wt.select_index(tree)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ot.select_samples(12))
    rng = np.random.default_rng(n)
    cs, js, want = [], [], []
    for sym in rng.choice(np.unique(S), size=min(50, np.unique(S).size), replace=False):
        occ = np.nonzero(S == sym)[0]
        for j in np.unique(rng.integers(1, occ.size + 1, 5)):
            cs.append(sym)
            js.append(int(j))
            want.append(occ[j - 1])
    c_t = torch.tensor(np.array(cs, np.int32)).cuda()
    j_t = torch.tensor(js).cuda()
    assert np.array_equal(wt.select(tree, c_t, j_t, index=idx).cpu().numpy(), np.array(want))


def test_query_index_errors(wt):
    S = np.array([0, 1, 2, 3, 2, 1], np.uint8)
    tree = wt.build(to_dev(S), 4)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = wt.access(tree, torch.tensor([0, 6, 5], device="cuda"), status=st)
    assert out.tolist() == [0, 0xFFFFFFFF, 1] and st.item() == wt.WT_ERR_INDEX
    st.zero_()
    out = wt.rank(tree, torch.tensor([1, 4], device="cuda"), torch.tensor([5, 0], device="cuda"), status=st)
    assert out.tolist()[0] == 2 and out.tolist()[1] == -1 and st.item() == wt.WT_ERR_INDEX
    st.zero_()
    out = wt.select(tree, torch.tensor([2, 2, 0], device="cuda"), torch.tensor([2, 3, 0], device="cuda"), status=st)
    assert out.tolist() == [4, -1, -1] and st.item() == wt.WT_ERR_INDEX


def test_fig2_worked_example_on_gpu(wt):
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "fig2_once_upon.json")) as f:
        g = json.load(f)
    alpha = g["alphabet_first_appearance"]
    S = np.array([alpha.index(ch) for ch in g["text"]], np.uint8)
    tree = check_case(wt, S, 16)
    assert tree.access(torch.tensor([24], device="cuda")).item() == g["printed"]["access_24_code"]
    assert tree.rank(torch.tensor([8], device="cuda"), torch.tensor([29], device="cuda")).item() == 3


# ------------------------------------------------------- full-size configs


def gpu_invariants(tree, S, sigma):
    """Order-independent properties that hold at any size (checked on the GPU)."""
    L = tree.levels
    d = to_dev(S).to(torch.int64) & 0xFFFFFFFF
    C = tree.node_offsets
    H = torch.bincount(d, minlength=1 << L)
    assert torch.equal(C[1:], torch.cumsum(H, 0)) and C[0].item() == 0
    for l in range(L):
        ones = int(((d >> (L - 1 - l)) & 1).sum().item())
        assert int(tree.superblocks[l, -1].item()) == ones, f"level {l} total ones"
        lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int32, device="cuda")
        pc = int(lut[tree.bitmaps[l].view(torch.uint8).to(torch.int64)].sum().item())
        assert pc == ones, f"level {l} bitmap popcount"


def oracle_levels_parallel(S, sigma, L):
    """oracle.build_level for every level, the levels on a thread pool: each call is
    the single-threaded C oracle (Alg. 1, one level); ctypes releases the GIL, so
    the host's cores take different levels (the oracle itself is unchanged)."""
    from concurrent.futures import ThreadPoolExecutor
    workers = max(1, min(L, (os.cpu_count() or 2) - 1, 12))
    with ThreadPoolExecutor(workers) as ex:
        futs = {l: ex.submit(oracle.build_level, S, sigma, l) for l in range(L)}
        for l in range(L):
            yield l, futs[l].result()


def device_access_all(tree, S, chunk=1 << 26):
    """access(i) for EVERY i in [0, n), compared with S on the device, in chunks."""
    n = S.size
    d = to_dev(S).to(torch.int64) & 0xFFFFFFFF
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        got = tree.access(torch.arange(a, b, device="cuda"))
        if not torch.equal(got, d[a:b]):
            bad = torch.nonzero(got != d[a:b])[:5].flatten().tolist()
            raise AssertionError(f"access differs from S at {[a + i for i in bad]}")


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_parity(wt, cfg):
    # every level of every config, element by element: bitmap words, superblocks
    # and the level's node starts (Alg. 1 lines 5-14)
    S, sigma = wt_inputs.generate(cfg)
    tree = wt.build(to_dev(S), sigma)
    torch.cuda.synchronize()
    L = tree.levels
    B, SB, C = np_tree(tree)
    assert np.array_equal(C, oracle.node_offsets(S, sigma))
    checked = 0
    for l, (ob, osb, onl) in oracle_levels_parallel(S, sigma, L):
        assert np.array_equal(B[l], ob), f"cfg{cfg} level {l} bitmap"
        assert np.array_equal(SB[l], osb), f"cfg{cfg} level {l} superblocks"
        assert np.array_equal(C[:: 1 << (L - l)], onl), f"cfg{cfg} level {l} node starts"
        checked += 1
    assert checked == L
    gpu_invariants(tree, S, sigma)
    device_access_all(tree, S)


@pytest.mark.parametrize("cfg", [3, 4])
def test_config_parity_opt_in_bottom_groups(wt, cfg):
    # the opt-in fused final three levels (WT_TRIPLE=1) at full size: every
    # level word for word against the direct build (itself checked against the
    # oracle above), and C
    S, sigma = wt_inputs.generate(cfg)
    d = to_dev(S)
    ref = wt.build(d, sigma)
    os.environ["WT_TRIPLE"] = "1"
    try:
        assert "triple" in wt.launch_plan(S.size, sigma, S.dtype.itemsize)
        tr = wt.build(d, sigma)
    finally:
        del os.environ["WT_TRIPLE"]
    torch.cuda.synchronize()
    assert torch.equal(tr.bitmaps, ref.bitmaps)
    assert torch.equal(tr.superblocks, ref.superblocks)
    assert torch.equal(tr.node_offsets, ref.node_offsets)


# ------------------------------------------------------------ wavelet matrix (NEXT-4)


@pytest.mark.parametrize("width", [1, 2, 4])
def test_matrix_general_pair(wt, width):
    # WT_NO_PAIRN=1: the matrix's final pair through k_level<T, 2> (LV_MATRIX)
    sigma = {1: 256, 2: 1 << 16, 4: 1 << 20}[width]
    dtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[width]
    os.environ["WT_NO_PAIRN"] = "1"
    try:
        for k, (kind, s) in enumerate([("uniform", sigma), ("zipf", sigma), ("runs", 4)]):
            S = wt_inputs.random_case(1300 + k, 50_000 + 11 * k, s, kind, dtype=dtype)
            mx = wt.build_matrix(to_dev(S), s)
            om = oracle.build_matrix(S, s)
            assert np.array_equal(mx.bitmaps.cpu().numpy().view(np.uint32), om.bitmaps), kind
            assert np.array_equal(mx.superblocks.cpu().numpy().view(np.uint64), om.superblocks), kind
            assert np.array_equal(mx.zeros.cpu().numpy().view(np.uint64), om.zeros), kind
    finally:
        del os.environ["WT_NO_PAIRN"]


def test_degenerate_host_and_matrix_builds(wt):
    # n = 0 through the asynchronous host path; sigma = 1 (no levels) for the matrix
    # and the select index
    dev = torch.device("cuda", 0)
    st = torch.full((1,), -1, dtype=torch.int32).pin_memory()
    ht = wt.alloc_host_tree(0, 16, 1)
    ws = wt.alloc_workspace(0, 16, 1, dev, host=True)
    wt.build_from_host_async(torch.zeros(0, dtype=torch.uint8), 16, ht, ws, st)
    torch.cuda.synchronize()
    assert int(st.item()) == wt.WT_OK and int(ht.node_offsets.abs().sum()) == 0
    S = np.zeros(100, np.uint8)
    mx = wt.build_matrix(to_dev(S), 1)
    assert mx.levels == 0 and mx.zeros.numel() == 0
    assert np.array_equal(wt.matrix_access(mx, torch.arange(100, device="cuda")).cpu().numpy(), np.zeros(100))
    tree = check_case(wt, S, 1)
    assert wt.select_index(tree).numel() == 0


@pytest.mark.parametrize("sigma,n,dtype", [(2, 1, None), (4, 70001, None), (256, 4097, None), (256, 300_001, None),
                                           (230, 100_000, None), (1 << 16, 200_003, np.uint16),
                                           (1 << 20, 99_991, np.uint32), (5, 0, None)])
def test_matrix_parity_and_queries(wt, sigma, n, dtype):
    for kind in ("uniform", "zipf", "runs"):
        S = wt_inputs.random_case(n + sigma, n, sigma, kind, dtype=dtype)
        mx = wt.build_matrix(to_dev(S), sigma)
        om = oracle.build_matrix(S, sigma)
        B = mx.bitmaps.cpu().numpy().view(np.uint32)
        assert np.array_equal(B, om.bitmaps), f"matrix bitmaps {kind}"
        assert np.array_equal(mx.superblocks.cpu().numpy().view(np.uint64), om.superblocks), f"matrix sb {kind}"
        assert np.array_equal(mx.zeros.cpu().numpy().view(np.uint64), om.zeros), f"matrix zeros {kind}"
        if n == 0:
            continue
        got = wt.matrix_access(mx, torch.arange(n, device="cuda")).cpu().numpy()
        assert np.array_equal(got, S.astype(np.int64))
        rng = np.random.default_rng(n)
        m = 2000
        c = S[rng.integers(0, n, m)].astype(np.int64)
        i = rng.integers(0, n, m)
        cnt = wt.matrix_rank(mx, torch.from_numpy(c.astype(np.int32)).cuda(), torch.from_numpy(i).cuda()).cpu().numpy()
        for k in range(0, m, 97):
            assert cnt[k] == int((S[: i[k] + 1] == c[k]).sum())


@pytest.mark.parametrize("sigma,n,dtype,kind", [(1 << 20, 200_003, np.uint32, "zipf"), (1 << 16, 50_000, np.uint16, "runs"),
                                                (256, 4097, None, "uniform"), (1 << 32, 100_000, np.uint32, "sparse"),
                                                (7, 1, None, "uniform"), (1000, 0, np.uint16, "uniform")])
def test_alphabet_remap(wt, sigma, n, dtype, kind):
    # NEXT-4's alphabet remap against its definition (np.unique); then the tree of the
    # remapped sequence has ceil(lg sigma') levels and matches the oracle
    if kind == "sparse":   # a few thousand distinct values spread over [0, 2^32)
        rng = np.random.default_rng(5)
        vals = np.unique(rng.integers(0, 1 << 32, 3000, dtype=np.uint64)).astype(np.uint32)
        S = vals[rng.integers(0, vals.size, n)]
    else:
        S = wt_inputs.random_case(n + 3, n, min(sigma, 1 << 24), kind, dtype=dtype)
    d = to_dev(S)
    out, alphabet, s2 = wt.remap_alphabet(d, sigma)
    uniq, inv = np.unique(S, return_inverse=True)
    assert s2 == uniq.size
    assert np.array_equal(alphabet.cpu().numpy().view(np.uint32), uniq.astype(np.uint32))
    got = out.cpu().numpy()
    got = got.view(np.uint32) if got.dtype == np.int32 else got
    assert np.array_equal(got.astype(np.int64), inv.astype(np.int64))
    if n and s2 > 0:
        R = got.astype(S.dtype)
        check_case(wt, R, max(s2, 1), f"remapped sigma'={s2}")


# ------------------------------------------------------------ domain decomposition (NEXT-3)


@pytest.mark.parametrize("sigma,n,k,dtype", [(16, 30, 3, None), (4, 1_000_003, 2, None), (256, 300_001, 5, None),
                                             (1 << 16, 200_000, 8, np.uint16), (1 << 20, 150_001, 4, np.uint32),
                                             (3, 5000, 7, None), (256, 100, 8, None),
                                             # 4096 superblocks exactly: the superblock scan's grid has a
                                             # surplus CTA whose tile lies past the blocks
                                             (256, 1 << 21, 2, None)])
def test_dd_merge_equals_direct_build(wt, sigma, n, k, dtype):
    # the merged tree of k segment trees is the tree of the whole sequence
    for kind in ("uniform", "zipf", "runs"):
        S = wt_inputs.random_case(n * k + sigma, n, sigma, kind, dtype=dtype)
        merged = wt.build_dd(to_dev(S), sigma, k)
        assert_same(merged, oracle.build(S, sigma), f"dd k={k} {kind}")


def test_dd_fig2_segments(wt):
    # SURVEY Appendix A's dd split of the worked example: 3 segments of 10
    S = np.array([0, 1, 2, 3, 4, 5, 6, 0, 1, 4, 7, 4, 8, 9, 10, 3, 4, 7, 4, 11, 12, 13, 4, 14, 8, 5, 15, 3, 1, 8],
                 np.uint8)
    merged = wt.dd_merge([wt.build(to_dev(S[i:i + 10]), 16) for i in (0, 10, 20)], 16)
    assert_same(merged, oracle.build(S, 16), "fig2 dd")



# ------------------------------------------------------------ L = 2 edges


L2_EDGE = {1: 32768, 2: 16384, 4: 8192}   # 32 KiB of symbols: several level tiles


@pytest.mark.parametrize("width", [1, 2, 4])
def test_l2_edges(wt, width):
    # two-level trees (sigma 3 / 4: the fused final pair reads S itself) across
    # many level tiles, runs of one value (a level-0 half empty: Z = 0 or O = 0),
    # and the range check in full and ragged tiles
    dtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[width]
    ts = L2_EDGE[width]
    for n in [1, 31, 33, 511, 513, ts - 1, ts, ts + 1, 2 * ts + 511, 3 * ts + 777, 5 * ts]:
        for sigma in (3, 4):
            S = wt_inputs.random_case(n + sigma, n, sigma, "uniform", dtype=dtype)
            check_case(wt, S, sigma, f"l2 n={n} sigma={sigma} w={width}")
    n = 2 * ts + 100
    for fill in ([0], [3], [2], [1], [0, 3], [3, 0, 0], [1, 2]):
        S = np.resize(np.array(fill, dtype), n)
        check_case(wt, S, 4, f"l2 pattern {fill}")
    rng = np.random.default_rng(width)
    S = rng.integers(0, 4, 3 * ts + 5).astype(dtype)
    S[rng.integers(0, S.size, 3000)] = 0          # zeros-heavy region
    S[ts: 2 * ts] = 3
    check_case(wt, S, 4, "l2 mixed runs")
    for pos in (0, ts - 1, ts, S.size - 1):
        bad = S.copy()
        bad[pos] = 4 if width > 1 else 200
        with pytest.raises(wt.WtError) as e:
            wt.build(to_dev(bad), 4)
        assert e.value.status == wt.WT_ERR_SYMBOL_RANGE


@pytest.fixture
def no_pair2():
    # (and no k_pairn, which would otherwise take over the two-level trees)
    os.environ["WT_NO_PAIR2"] = "1"
    os.environ["WT_NO_PAIRN"] = "1"
    yield
    del os.environ["WT_NO_PAIR2"]
    del os.environ["WT_NO_PAIRN"]


@pytest.fixture
def no_pairn():
    os.environ["WT_NO_PAIRN"] = "1"
    yield
    del os.environ["WT_NO_PAIRN"]


@pytest.fixture
def triple_forced():
    os.environ["WT_TRIPLE"] = "1"
    yield
    del os.environ["WT_TRIPLE"]




@pytest.mark.parametrize("width", [1, 2, 4])
def test_triple(wt, triple_forced, width):
    # k_triple (the fused final three levels) on every tree with L >= 3 (forced,
    # whatever the node sizes): lanes inside one node, lanes spanning many nodes
    # (uniform over a large alphabet, sorted runs), constant and Zipf inputs,
    # tails around the 128-byte rows, the lane, the 2 KiB level tile and the
    # 4 KiB warp tile, L = 3 (the pass reads S)
    dtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[width]
    t = TILE[width]
    cases = []
    for sigma in {1: (5, 8, 27, 256), 2: (8, 300, 1 << 16), 4: (8, 1 << 12, 1 << 24)}[width]:
        for kind in ("uniform", "sorted", "runs", "constant", "zipf"):
            cases.append((sigma, kind, 3 * t + 77))
    for n in (128 // width, 128 // width + 1, t - 1, t + 5, 2 * t - 1, 2 * t + 1, 3 * t + 128 // width + 3,
              5 * t + 64 // width - 1, 9 * t):
        cases.append(({1: 256, 2: 1 << 16, 4: 1 << 24}[width], "uniform", n))
        cases.append((16, "sorted", n))
        cases.append((8, "zipf", n))
    for i, (sigma, kind, n) in enumerate(cases):
        S = wt_inputs.random_case(1100 + i, n, sigma, kind, dtype=dtype)
        if n * width >= 128 and sigma > 4:
            assert "triple" in wt.launch_plan(n, sigma, width)
        check_case(wt, S, sigma, f"triple w={width} sigma={sigma} {kind} n={n}")


def test_triple_random(wt, triple_forced):
    # forced k_triple over the small random suite's alphabets and shapes
    for sigma in (5, 8, 16, 27, 230, 256, 1000, 1 << 12, 1 << 16, 70000, 1 << 24):
        rng = np.random.default_rng(sigma + 5)
        for k, kind in enumerate(["uniform", "zipf", "runs", "sorted", "reverse", "constant"]):
            n = int(rng.integers(1, 70000))
            S = wt_inputs.random_case(300 * sigma + k, n, sigma, kind)
            check_case(wt, S, sigma, f"triple sigma={sigma} n={n} kind={kind}")


@pytest.mark.parametrize("width", [1, 2, 4])
def test_general_fused_pair(wt, no_pairn, width):
    # WT_NO_PAIRN=1: the final pair through the general k_level<T, 2> (it counts
    # the leaves itself; C from the final scan)
    sigma = {1: 256, 2: 1 << 16, 4: 1 << 20}[width]
    dtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[width]
    assert "leaf_offsets" not in wt.launch_plan(100_000, sigma, width)
    for k, kind in enumerate(["uniform", "zipf", "runs"]):
        S = wt_inputs.random_case(700 + k, 100_000 + 37 * k, sigma, kind, dtype=dtype)
        check_case(wt, S, sigma, f"general pair w={width} {kind}")


@pytest.mark.parametrize("width", [1, 2, 4])
def test_pairn_node_changes(wt, width):
    # k_pairn: a lane's symbols span many level-(L-2) nodes (sorted / uniform
    # over a large alphabet: a new node at almost every symbol), one node
    # (constant), node runs crossing lanes and tiles, every tail geometry
    # around the 128-byte tensor rows, the 2 KiB tile and the 64-byte lane
    dtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[width]
    t = TILE[width]
    rows = 128 // width
    cases = []
    for sigma in ({1: (5, 8, 256), 2: (8, 300, 1 << 16), 4: (8, 1 << 12, 1 << 24)}[width]):
        for kind in ("uniform", "sorted", "runs", "constant", "zipf"):
            cases.append((sigma, kind, 3 * t + 77))
    for n in (rows, rows + 1, 2 * rows - 1, t - 1, t + rows, 2 * t - 1, 2 * t + 1, 3 * t + 128 // width + 3,
              5 * t + 64 // width - 1, 5 * t + 64 // width + 1):
        cases.append(({1: 256, 2: 1 << 16, 4: 1 << 24}[width], "uniform", n))
        cases.append((8, "sorted", n))
    for i, (sigma, kind, n) in enumerate(cases):
        S = wt_inputs.random_case(900 + i, n, sigma, kind, dtype=dtype)
        if n * width >= 128 and sigma > 4:
            assert "leaf_offsets" in wt.launch_plan(n, sigma, width)
        check_case(wt, S, sigma, f"pairn w={width} sigma={sigma} {kind} n={n}")


@pytest.mark.parametrize("sigma,n", [(4, 300_001), (3, 100_000), (4, 2048 * 7 + 5)])
def test_l2_general_pair(wt, no_pair2, sigma, n):
    # WT_NO_PAIR2=1: two levels of 1-byte symbols through the general fused pair
    assert "pair2_offsets" not in wt.launch_plan(n, sigma, 1)
    S = wt_inputs.random_case(n, n, sigma, "zipf", dtype=np.uint8)
    check_case(wt, S, sigma, f"general pair n={n}")
