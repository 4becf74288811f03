"""Independent definitions used to PIN the oracle (and, on the GPU box, to check
the CUDA path at properties that hold at any size).  Plain numpy; nothing here
is shared with oracle/ or paper_1610_05994_b200/.

Each function restates a definition from the paper, not Alg. 1:
  * levels_by_stable_sort -- the levelwise tree as "S stably sorted by its top
    l bits, then bit l" (BASELINE north_star; Prop. 1 P:485-490 + the
    per-node subsequence definition P:288-296 with stable order).
  * levels_by_recursion   -- the recursive per-node definition:
    a node over alphabet range R keeps the subsequence of S with symbols in R;
    its bitmap marks the second half; children recurse on the halves; the
    one-pointer-per-level bitmap concatenates the nodes of a level left to
    right (Fig. 1b).
"""
from __future__ import annotations

import numpy as np


def n_levels(sigma: int) -> int:
    return 0 if sigma <= 1 else int(sigma - 1).bit_length()


def pack_bits(bits: np.ndarray, n_words: int) -> np.ndarray:
    """LSB-first packing into uint32 words (R5), zero padded to n_words."""
    by = np.packbits(np.asarray(bits, np.uint8), bitorder="little")
    buf = np.zeros(n_words * 4, np.uint8)
    buf[: by.size] = by
    return buf.view("<u4")


def words_per_level(n: int) -> int:
    return 16 * ((n + 511) // 512)


def levels_by_stable_sort(S: np.ndarray, sigma: int) -> list[np.ndarray]:
    """bit lists, one per level: T_l = S stably sorted by s >> (L-l); B_l[q] = bit (L-1-l) of T_l[q]."""
    L = n_levels(sigma)
    S64 = S.astype(np.int64)
    out = []
    for l in range(L):
        order = np.argsort(S64 >> (L - l), kind="stable")
        T = S64[order]
        out.append(((T >> (L - 1 - l)) & 1).astype(np.uint8))
    return out


def levels_by_recursion(S, sigma: int) -> list[list[int]]:
    """Recursive per-node construction with the power-of-two split of
    Proposition 1 (reading R3 in DESIGN.md)."""
    L = n_levels(sigma)
    levels = [[] for _ in range(L)]

    def node(seq, lo, width, depth):
        if depth == L:
            return
        half = width // 2
        mid = lo + half
        levels[depth].extend(1 if s >= mid else 0 for s in seq)
        node([s for s in seq if s < mid], lo, half, depth + 1)
        node([s for s in seq if s >= mid], mid, half, depth + 1)

    node([int(s) for s in S], 0, 1 << L, 0)
    return levels


def superblocks_from_bits(bits: np.ndarray, n: int) -> np.ndarray:
    """SB[t] = ones in bits[0, min(512 t, n)), t = 0..ceil(n/512) (R6)."""
    c = np.concatenate([[0], np.cumsum(bits.astype(np.int64))])
    t = np.arange((n + 511) // 512 + 1, dtype=np.int64)
    return c[np.minimum(512 * t, n)].astype(np.uint64)


def node_offsets(S: np.ndarray, sigma: int) -> np.ndarray:
    """C[c] = #{j : S[j] < c}, c in [0, 2^L]."""
    L = n_levels(sigma)
    H = np.bincount(S.astype(np.int64), minlength=1 << L)
    return np.concatenate([[0], np.cumsum(H)]).astype(np.uint64)


def unpack_level(words: np.ndarray, n: int) -> np.ndarray:
    return np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")[:n]
