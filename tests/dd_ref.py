"""Test-side reference for the domain-decomposition merge (NEXT-3): where every
bit of every segment lands in the merged tree, by walking the nodes in order
(the definition: node v of level l holds segment 0's run of v, then segment
1's, ... -- P:633-687, 799-822).  Plain numpy over oracle segment trees; it
shares nothing with the library's plan or merge kernels."""
import numpy as np


def merged_dest(seg_C: list, L: int, l: int) -> list:
    """dest[g][q] = merged position of segment g's level-l bit q."""
    k = len(seg_C)
    sh = L - l
    nodes = 1 << l
    C = [np.asarray(c, dtype=np.int64) for c in seg_C]
    dest = [np.empty(int(c[-1]), np.int64) for c in C]
    pos = 0
    for v in range(nodes):
        for g in range(k):
            a, b = int(C[g][v << sh]), int(C[g][(v + 1) << sh])
            dest[g][a:b] = np.arange(pos, pos + (b - a))
            pos += b - a
    return dest


def unpack(words: np.ndarray, nbits: int) -> np.ndarray:
    return np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")[:nbits]


def plan_brute(seg_C: list, L: int, n: int, part_ranges: list) -> np.ndarray:
    """(L, parts, k, 2): [lo, hi) of segment g's level-l bits with merged
    position in part p's range [q_lo, q_hi)."""
    k = len(seg_C)
    out = np.zeros((L, len(part_ranges), k, 2), np.int64)
    for l in range(L):
        dest = merged_dest(seg_C, L, l)
        for p, (q_lo, q_hi) in enumerate(part_ranges):
            for g in range(k):
                out[l, p, g, 0] = int(np.count_nonzero(dest[g] < q_lo))
                out[l, p, g, 1] = int(np.count_nonzero(dest[g] < q_hi))
    return out
