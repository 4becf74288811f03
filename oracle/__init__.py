"""CPU oracle for the levelwise wavelet tree (arXiv 1610.05994, Alg. 1 sequential).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1610_05994_b200`` never imports it, and
the two share no code ("Oracle").

Thin ctypes marshalling over ``wt_oracle.c`` (plain single-threaded C, built
with ``gcc -O2`` as the paper's code was).  All arithmetic lives
in the C file; this module only allocates numpy arrays and passes pointers.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ERR_ARG, ERR_SYMBOL_RANGE, ERR_INDEX, ERR_NOMEM, ERR_INTERNAL = 0, 1, 2, 3, 6, 7


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def build_lib(force: bool = False) -> str:
    """Compile wt_oracle.c into liboracle.so (gcc -O2, single-threaded)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_LIB)
        u64, u32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
        L.oracle_levels.restype = u32
        L.oracle_levels.argtypes = [u64]
        L.oracle_words_per_level.restype = u64
        L.oracle_words_per_level.argtypes = [u64]
        L.oracle_sb_per_level.restype = u64
        L.oracle_sb_per_level.argtypes = [u64]
        L.oracle_validate.argtypes = [vp, u64, u64, u32]
        L.oracle_node_offsets.argtypes = [vp, u64, u64, u32, vp]
        L.oracle_build_level.argtypes = [vp, u64, u64, u32, u32, vp, vp, vp]
        L.oracle_build.argtypes = [vp, u64, u64, u32, vp, vp, vp]
        L.oracle_rank1.restype = u64
        L.oracle_rank1.argtypes = [vp, vp, u64]
        for f in (L.oracle_access,):
            f.argtypes = [vp, vp, vp, u64, u64, u64, vp, vp]
        for f in (L.oracle_rank, L.oracle_select):
            f.argtypes = [vp, vp, vp, u64, u64, u64, u64, vp]
        for f in (L.oracle_validate, L.oracle_node_offsets, L.oracle_build_level, L.oracle_build,
                  L.oracle_access, L.oracle_rank, L.oracle_select):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _seq(S: np.ndarray) -> tuple[np.ndarray, int]:
    S = np.ascontiguousarray(S)
    if S.dtype not in (np.uint8, np.uint16, np.uint32):
        raise TypeError(f"sequence dtype must be uint8/uint16/uint32, got {S.dtype}")
    return S, S.dtype.itemsize


def levels(sigma: int) -> int:
    return int(lib().oracle_levels(sigma))


def words_per_level(n: int) -> int:
    return int(lib().oracle_words_per_level(n))


def sb_per_level(n: int) -> int:
    return int(lib().oracle_sb_per_level(n))


@dataclass
class OracleTree:
    n: int
    sigma: int
    L: int
    bitmaps: np.ndarray        # (L, words_per_level) uint32, LSB-first
    superblocks: np.ndarray    # (L, sb_per_level) uint64
    node_offsets: np.ndarray   # (2^L + 1,) uint64

    def access(self, i: int, with_path: bool = False):
        sym = np.zeros(1, np.uint64)
        path = np.zeros(self.L + 1, np.uint64)
        st = lib().oracle_access(_ptr(self.bitmaps), _ptr(self.superblocks), _ptr(self.node_offsets),
                                 self.n, self.sigma, i, _ptr(sym), _ptr(path))
        if st != OK:
            raise OracleError(st, "access")
        return (int(sym[0]), [int(x) for x in path]) if with_path else int(sym[0])

    def rank(self, c: int, i: int) -> int:
        out = np.zeros(1, np.uint64)
        st = lib().oracle_rank(_ptr(self.bitmaps), _ptr(self.superblocks), _ptr(self.node_offsets),
                               self.n, self.sigma, c, i, _ptr(out))
        if st != OK:
            raise OracleError(st, "rank")
        return int(out[0])

    def select(self, c: int, j: int) -> int:
        out = np.zeros(1, np.uint64)
        st = lib().oracle_select(_ptr(self.bitmaps), _ptr(self.superblocks), _ptr(self.node_offsets),
                                 self.n, self.sigma, c, j, _ptr(out))
        if st != OK:
            raise OracleError(st, "select")
        return int(out[0])

    def rank1(self, level: int, q: int) -> int:
        return int(lib().oracle_rank1(_ptr(self.bitmaps[level]), _ptr(self.superblocks[level]), q))

    def select_samples(self, shift: int = 12) -> np.ndarray:
        """The select index by its definition (createRankSelect's select half,
        P:556, 599-600): out[l, b, k] = position of the (k * 2^shift)-th (0-based)
        bit equal to b in B_l, n where the level has fewer; shape (L, 2, n >> shift + 2).
        Plain numpy over this oracle's bitmaps."""
        q = (self.n >> shift) + 2
        out = np.full((self.L, 2, q), self.n, np.uint32)
        for l in range(self.L):
            bits = np.unpackbits(self.bitmaps[l].view(np.uint8), bitorder="little")[: self.n]
            for b in (0, 1):
                pos = np.flatnonzero(bits == b)[:: 1 << shift]
                out[l, b, : pos.size] = pos
        return out


def validate(S: np.ndarray, sigma: int) -> int:
    S, w = _seq(S)
    return int(lib().oracle_validate(_ptr(S), S.size, sigma, w))


def node_offsets(S: np.ndarray, sigma: int) -> np.ndarray:
    S, w = _seq(S)
    C = np.zeros((1 << levels(sigma)) + 1, np.uint64)
    st = lib().oracle_node_offsets(_ptr(S), S.size, sigma, w, _ptr(C))
    if st != OK:
        raise OracleError(st, "node_offsets")
    return C


def build_level(S: np.ndarray, sigma: int, level: int):
    """One level of Alg. 1: (bitmap words, superblocks, node starts Nl)."""
    S, w = _seq(S)
    n = S.size
    B = np.zeros(words_per_level(n), np.uint32)
    SB = np.zeros(sb_per_level(n), np.uint64)
    Nl = np.zeros((1 << level) + 1, np.uint64)
    st = lib().oracle_build_level(_ptr(S), n, sigma, w, level, _ptr(B), _ptr(SB), _ptr(Nl))
    if st != OK:
        raise OracleError(st, "build_level")
    return B, SB, Nl


def build(S: np.ndarray, sigma: int) -> OracleTree:
    """Alg. 1, sequential form, all levels + leaf node offsets."""
    S, w = _seq(S)
    n = S.size
    L = levels(sigma)
    B = np.zeros((L, words_per_level(n)), np.uint32)
    SB = np.zeros((L, sb_per_level(n)), np.uint64)
    C = np.zeros((1 << L) + 1, np.uint64)
    st = lib().oracle_build(_ptr(S), n, sigma, w, _ptr(B), _ptr(SB), _ptr(C))
    if st != OK:
        raise OracleError(st, "build")
    return OracleTree(n=n, sigma=sigma, L=L, bitmaps=B, superblocks=SB, node_offsets=C)


@dataclass
class OracleMatrix:
    n: int
    sigma: int
    L: int
    bitmaps: np.ndarray        # (L, words_per_level) uint32, LSB-first
    superblocks: np.ndarray    # (L, sb_per_level) uint64
    zeros: np.ndarray          # (L,) uint64


def build_matrix(S: np.ndarray, sigma: int) -> OracleMatrix:
    """The wavelet matrix (NEXT-4) by its definition, plain numpy:
    T_0 = S; B_l[j] = bit (L-1-l) of T_l[j]; T_{l+1} = the zeros of T_l then its
    ones, each in order (a global stable partition, no nodes); zeros[l] = the
    number of zeros of level l; superblocks as the tree's (one cumulative count
    per 512 bits plus the total)."""
    seq = np.asarray(S).astype(np.int64)
    n = seq.size
    L = levels(sigma)
    if n and int(seq.max(initial=0)) >= sigma:
        raise OracleError(2, "symbol >= sigma")
    W, NSB = words_per_level(n), sb_per_level(n)
    bm = np.zeros((L, W), np.uint32)
    sb = np.zeros((L, NSB), np.uint64)
    zeros = np.zeros(L, np.uint64)
    T = seq
    for l in range(L):
        bits = ((T >> (L - 1 - l)) & 1).astype(np.uint8)
        buf = np.zeros(W * 4, np.uint8)
        packed = np.packbits(bits, bitorder="little")
        buf[: packed.size] = packed
        bm[l] = buf.view("<u4")
        ones_before = np.concatenate([[0], np.cumsum(bits, dtype=np.uint64)])
        sb[l] = ones_before[np.minimum(np.arange(NSB) * 512, n)]
        zeros[l] = n - int(bits.sum())
        T = np.concatenate([T[bits == 0], T[bits == 1]])
    return OracleMatrix(n, sigma, L, bm, sb, zeros)

