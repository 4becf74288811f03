"""paper_1610_05994_b200 -- B200-native levelwise wavelet-tree construction
(arXiv 1610.05994, "Parallel Construction of Wavelet Trees on Multicore
Architectures"), as hand-written sm_100a CUDA behind the C ABI of
``include/wt.h`` (``libwt.so``).

This module is argument marshalling only: it allocates device memory with
torch, passes raw pointers and the current CUDA stream to the C ABI, and wraps
the results.  Every step of the build runs in the library's kernels; there is
no CPU fallback -- importing fails loudly if ``libwt.so`` is missing.

Names follow the C ABI: ``sizes``, ``build`` / ``build_async``,
``build_from_host``, ``access``, ``rank``, ``select``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WT_LIB") or os.path.join(_HERE, "libwt.so")  # WT_LIB: experiment builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is deliberately no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

WT_OK, WT_ERR_ARG, WT_ERR_SYMBOL_RANGE, WT_ERR_INDEX, WT_ERR_CUDA, WT_ERR_WORKSPACE = range(6)
KIND_NAMES = {1: "prologue", 2: "scan", 3: "tables", 4: "level", 5: "last_level", 6: "tile_scan", 7: "memset",
              8: "pair", 9: "sb_scan", 10: "block_pop", 11: "prep", 12: "final_scan", 13: "dd_offsets",
              14: "dd_merge", 15: "dd_superblocks", 16: "flags", 17: "leaf_offsets", 18: "quad",
              21: "class_count", 22: "triple"}


class WtSizes(ctypes.Structure):
    _fields_ = [
        ("levels", ctypes.c_uint32),
        ("width", ctypes.c_uint32),
        ("words_per_level", ctypes.c_uint64),
        ("sb_per_level", ctypes.c_uint64),
        ("c_len", ctypes.c_uint64),
        ("bitmap_bytes", ctypes.c_uint64),
        ("superblock_bytes", ctypes.c_uint64),
        ("node_offset_bytes", ctypes.c_uint64),
        ("workspace_bytes", ctypes.c_size_t),
        ("host_workspace_bytes", ctypes.c_size_t),
    ]


class WtTree(ctypes.Structure):
    _fields_ = [("bitmaps", ctypes.c_void_p), ("superblocks", ctypes.c_void_p),
                ("node_offsets", ctypes.c_void_p)]


_u64, _u32, _vp, _sz = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t
_lib.wt_sizes.argtypes = [_u64, _u64, _u32, ctypes.POINTER(WtSizes)]
_lib.wt_build_async.argtypes = [_vp, _u64, _u64, _u32, ctypes.POINTER(WtTree), _vp, _sz, _vp, _vp]
_lib.wt_build.argtypes = [_vp, _u64, _u64, _u32, ctypes.POINTER(WtTree), _vp, _sz, _vp]
_lib.wt_build_from_host.argtypes = [_vp, _u64, _u64, _u32, ctypes.POINTER(WtTree), _vp, _sz, _vp]
_lib.wt_build_from_host_async.argtypes = [_vp, _u64, _u64, _u32, ctypes.POINTER(WtTree), _vp, _sz, _vp, _vp]
_lib.wt_access.argtypes = [ctypes.POINTER(WtTree), _u64, _u64, _vp, _u64, _vp, _vp, _vp]
_lib.wt_rank.argtypes = [ctypes.POINTER(WtTree), _u64, _u64, _vp, _vp, _u64, _vp, _vp, _vp]
_lib.wt_select.argtypes = [ctypes.POINTER(WtTree), _u64, _u64, _vp, _vp, _u64, _vp, _vp, _vp]
class WtMatrix(ctypes.Structure):
    _fields_ = [("bitmaps", _vp), ("superblocks", _vp), ("zeros", _vp)]


_lib.wt_matrix_build_async.argtypes = [_vp, _u64, _u64, _u32, ctypes.POINTER(WtMatrix), _vp, _sz, _vp, _vp]
_lib.wt_matrix_access.argtypes = [ctypes.POINTER(WtMatrix), _u64, _u64, _vp, _u64, _vp, _vp, _vp]
_lib.wt_matrix_rank.argtypes = [ctypes.POINTER(WtMatrix), _u64, _u64, _vp, _vp, _u64, _vp, _vp, _vp]
_lib.wt_dd_merge_scratch_bytes.argtypes = [_u64]
_lib.wt_dd_merge_scratch_bytes.restype = _sz
_lib.wt_dd_merge.argtypes = [_u32, _vp, _vp, _u64, ctypes.POINTER(WtTree), _vp, _sz, _vp]
_lib.wt_dd_part_blocks.argtypes = [_u64, _u64, _u64, _vp, _vp]
_lib.wt_dd_part_blocks.restype = None
_lib.wt_dd_offsets.argtypes = [_u32, _vp, _u64, _vp, _vp]
_lib.wt_dd_plan.argtypes = [_u32, _vp, _u64, _u64, _vp]
_lib.wt_dd_plan_async.argtypes = [_u32, _vp, _u64, _u64, _u64, _vp, _vp]
_lib.wt_dd_merge_level.argtypes = [_u32, _vp, _vp, _u64, _u64, _u32, _vp, _vp, _u64, _u64, _vp, _vp]
_lib.wt_superblocks_scratch_bytes.argtypes = [_u64]
_lib.wt_superblocks_scratch_bytes.restype = _sz
_lib.wt_superblocks.argtypes = [_vp, _u64, _u64, _vp, _vp, _sz, _vp]
_lib.wt_rank1.argtypes = [ctypes.POINTER(WtTree), _u64, _u64, _vp, _vp, _u64, _vp, _vp]
_lib.wt_remap_workspace_bytes.argtypes = [_u64]
_lib.wt_remap_workspace_bytes.restype = _sz
_lib.wt_remap_alphabet.argtypes = [_vp, _u64, _u64, _u32, _vp, _vp, _vp, _vp, _sz, _vp, _vp]
_lib.wt_select_index_entries.argtypes = [_u64, _u64]
_lib.wt_select_index_entries.restype = _u64
_lib.wt_select_index.argtypes = [ctypes.POINTER(WtTree), _u64, _u64, _vp, _vp]
_lib.wt_select_indexed.argtypes = [ctypes.POINTER(WtTree), _u64, _u64, _vp, _vp, _vp, _u64, _vp, _vp, _vp]
_lib.wt_launch_plan.argtypes = [_u64, _u64, _u32, _vp, _u32]
_lib.wt_launch_plan.restype = _u32
_lib.wt_debug_offsets.argtypes = [_u64, _u64, _u32, _vp, _u32]
_lib.wt_debug_offsets.restype = _u32
_lib.wt_set_profile_events.argtypes = [_vp, _u32]
_lib.wt_set_profile_events.restype = None
_lib.wt_status_string.argtypes = [ctypes.c_int]
_lib.wt_status_string.restype = ctypes.c_char_p
_lib.wt_last_error.argtypes = []
_lib.wt_last_error.restype = ctypes.c_char_p
for _f in (_lib.wt_sizes, _lib.wt_build_async, _lib.wt_build, _lib.wt_build_from_host,
           _lib.wt_build_from_host_async, _lib.wt_access, _lib.wt_rank, _lib.wt_select, _lib.wt_select_index,
           _lib.wt_select_indexed, _lib.wt_matrix_build_async, _lib.wt_matrix_access, _lib.wt_matrix_rank,
           _lib.wt_remap_alphabet, _lib.wt_dd_merge, _lib.wt_dd_offsets, _lib.wt_dd_plan, _lib.wt_dd_plan_async,
           _lib.wt_dd_merge_level, _lib.wt_superblocks, _lib.wt_rank1):
    _f.restype = ctypes.c_int

EXPORTS = ["wt_sizes", "wt_build_async", "wt_build", "wt_build_from_host", "wt_build_from_host_async",
           "wt_access", "wt_rank", "wt_select_index_entries", "wt_select_index", "wt_select_indexed",
           "wt_matrix_build_async", "wt_matrix_access", "wt_matrix_rank", "wt_remap_workspace_bytes",
           "wt_remap_alphabet", "wt_dd_merge_scratch_bytes", "wt_dd_merge", "wt_dd_part_blocks", "wt_dd_offsets",
           "wt_dd_plan", "wt_dd_plan_async", "wt_dd_merge_level", "wt_superblocks_scratch_bytes", "wt_superblocks",
           "wt_rank1",
           "wt_select", "wt_launch_plan", "wt_debug_offsets", "wt_set_profile_events", "wt_status_string",
           "wt_last_error"]


class WtError(RuntimeError):
    def __init__(self, status: int, what: str):
        detail = _lib.wt_last_error().decode()
        super().__init__(f"{what}: {_lib.wt_status_string(status).decode()} {detail}".strip())
        self.status = status


def _check(st: int, what: str):
    if st != WT_OK:
        raise WtError(st, what)


_WIDTH = {torch.uint8: 1, torch.int8: 1, torch.uint16: 2, torch.int16: 2, torch.int32: 4, torch.uint32: 4}


def width_of(t: torch.Tensor) -> int:
    if t.dtype not in _WIDTH:
        raise TypeError(f"sequence dtype must be 1/2/4-byte integer, got {t.dtype}")
    return _WIDTH[t.dtype]


def _stream_ptr(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _keep_for(stream, *tensors):
    """Tensors allocated here on torch's current stream but used by kernels enqueued
    on another `stream`: tell the caching allocator, so their memory is not handed out
    again before that stream's work completes (torch Tensor.record_stream)."""
    if stream is None:
        return
    for t in tensors:
        if t is not None and t.is_cuda and t.numel():
            t.record_stream(stream)


def _sync(stream):
    (stream if stream is not None else torch.cuda.current_stream()).synchronize()


def _status_tensor(device):
    return torch.zeros(1, dtype=torch.int32, device=device)


def sizes(n: int, sigma: int, width: int) -> WtSizes:
    out = WtSizes()
    _check(_lib.wt_sizes(n, sigma, width, ctypes.byref(out)), "wt_sizes")
    return out


def launch_plan(n: int, sigma: int, width: int) -> list[str]:
    cnt = _lib.wt_launch_plan(n, sigma, width, None, 0)
    buf = (ctypes.c_uint32 * max(cnt, 1))()
    _lib.wt_launch_plan(n, sigma, width, ctypes.cast(buf, _vp), cnt)
    return [KIND_NAMES.get(buf[i], str(buf[i])) for i in range(cnt)]


def debug_offsets(n: int, sigma: int, width: int) -> dict:
    """Workspace layout of a build (debug aid)."""
    buf = (ctypes.c_uint64 * 16)()
    k = _lib.wt_debug_offsets(n, sigma, width, ctypes.cast(buf, _vp), 16)
    names = ["flag", "ones0", "agg", "pre", "tab", "cnt", "cnt_stride", "bufA", "bufB", "ntiles"]
    return dict(zip(names, [int(buf[i]) for i in range(k)]))


def set_profile_events(events: list | None):
    """events: list of torch.cuda.Event (enable_timing=True) or None."""
    global _prof_keep
    if not events:
        _lib.wt_set_profile_events(None, 0)
        _prof_keep = None
        return
    for e in events:            # torch creates the CUDA event lazily, on first record
        if not e.cuda_event:
            e.record()
    arr = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
    _prof_keep = arr
    _lib.wt_set_profile_events(ctypes.cast(arr, _vp), len(events))


_prof_keep = None


@dataclass
class WaveletTree:
    """Device-resident tree (all torch tensors on the build's device)."""
    n: int
    sigma: int
    levels: int
    bitmaps: torch.Tensor       # (L, words_per_level) int32 storage of uint32 words
    superblocks: torch.Tensor   # (L, sb_per_level) int64 storage of uint64 counts
    node_offsets: torch.Tensor  # (2^L + 1,) int64 storage of uint64 offsets

    def _ctree(self) -> WtTree:
        return WtTree(self.bitmaps.data_ptr() if self.bitmaps.numel() else None,
                      self.superblocks.data_ptr() if self.superblocks.numel() else None,
                      self.node_offsets.data_ptr())

    def access(self, pos: torch.Tensor, stream=None) -> torch.Tensor:
        return access(self, pos, stream)

    def rank(self, c: torch.Tensor, pos: torch.Tensor, stream=None) -> torch.Tensor:
        return rank(self, c, pos, stream)

    def select(self, c: torch.Tensor, j: torch.Tensor, stream=None) -> torch.Tensor:
        return select(self, c, j, stream)


def alloc_tree(n: int, sigma: int, width: int, device) -> WaveletTree:
    sz = sizes(n, sigma, width)
    L = sz.levels
    return WaveletTree(
        n=n, sigma=sigma, levels=L,
        bitmaps=torch.empty((L, sz.words_per_level), dtype=torch.int32, device=device),
        superblocks=torch.empty((L, sz.sb_per_level), dtype=torch.int64, device=device),
        node_offsets=torch.empty((sz.c_len,), dtype=torch.int64, device=device))


def alloc_workspace(n: int, sigma: int, width: int, device, host: bool = False) -> torch.Tensor:
    sz = sizes(n, sigma, width)
    nbytes = sz.host_workspace_bytes if host else sz.workspace_bytes
    return torch.empty((max(nbytes, 256),), dtype=torch.uint8, device=device)


def build_async(seq: torch.Tensor, sigma: int, tree: WaveletTree | None = None,
                workspace: torch.Tensor | None = None, status: torch.Tensor | None = None,
                stream=None) -> WaveletTree:
    """Enqueue wt_build_async on `stream` (default: torch's current stream).
    `status` (int32 device tensor, optional) receives WT_OK / WT_ERR_SYMBOL_RANGE."""
    if not seq.is_cuda:
        raise ValueError("seq must be a CUDA tensor (use build_from_host for host data)")
    seq_in = seq
    seq = seq.contiguous()
    w = width_of(seq)
    n = seq.numel()
    own_tree, own_ws = tree is None, workspace is None
    if tree is None:
        tree = alloc_tree(n, sigma, w, seq.device)
    if workspace is None:
        workspace = alloc_workspace(n, sigma, w, seq.device)
    _keep_for(stream, seq if seq is not seq_in else None, workspace if own_ws else None,
              *((tree.bitmaps, tree.superblocks, tree.node_offsets) if own_tree else ()))
    ct = tree._ctree()
    st = _lib.wt_build_async(seq.data_ptr() if n else None, n, sigma, w, ctypes.byref(ct),
                             workspace.data_ptr(), workspace.numel(),
                             status.data_ptr() if status is not None else None, _stream_ptr(stream))
    _check(st, "wt_build_async")
    return tree


def build(seq: torch.Tensor, sigma: int, tree: WaveletTree | None = None,
          workspace: torch.Tensor | None = None, stream=None) -> WaveletTree:
    """wt_build: enqueue the build and synchronise once to read the range flag."""
    if not seq.is_cuda:
        raise ValueError("seq must be a CUDA tensor (use build_from_host for host data)")
    seq = seq.contiguous()
    w = width_of(seq)
    n = seq.numel()
    if tree is None:
        tree = alloc_tree(n, sigma, w, seq.device)
    if workspace is None:
        workspace = alloc_workspace(n, sigma, w, seq.device)
    ct = tree._ctree()
    st = _lib.wt_build(seq.data_ptr() if n else None, n, sigma, w, ctypes.byref(ct),
                       workspace.data_ptr(), workspace.numel(), _stream_ptr(stream))
    _check(st, "wt_build")
    return tree


@dataclass
class HostTree:
    n: int
    sigma: int
    levels: int
    bitmaps: torch.Tensor       # host (pinned) tensors
    superblocks: torch.Tensor
    node_offsets: torch.Tensor


def alloc_host_tree(n: int, sigma: int, width: int, pin: bool = True) -> HostTree:
    sz = sizes(n, sigma, width)
    L = sz.levels
    return HostTree(n=n, sigma=sigma, levels=L,
                    bitmaps=torch.empty((L, sz.words_per_level), dtype=torch.int32, pin_memory=pin),
                    superblocks=torch.empty((L, sz.sb_per_level), dtype=torch.int64, pin_memory=pin),
                    node_offsets=torch.empty((sz.c_len,), dtype=torch.int64, pin_memory=pin))


def build_from_host(h_seq: torch.Tensor, sigma: int, h_tree: HostTree | None = None,
                    workspace: torch.Tensor | None = None, device=None, stream=None) -> HostTree:
    """wt_build_from_host: H2D of the sequence, build, D2H of the whole tree, one sync."""
    if h_seq.is_cuda:
        raise ValueError("h_seq must be a host tensor")
    h_seq = h_seq.contiguous()
    w = width_of(h_seq)
    n = h_seq.numel()
    device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    if h_tree is None:
        h_tree = alloc_host_tree(n, sigma, w)
    if workspace is None:
        workspace = alloc_workspace(n, sigma, w, device, host=True)
    ct = WtTree(h_tree.bitmaps.data_ptr() if h_tree.bitmaps.numel() else None,
                h_tree.superblocks.data_ptr() if h_tree.superblocks.numel() else None,
                h_tree.node_offsets.data_ptr())
    st = _lib.wt_build_from_host(h_seq.data_ptr() if n else None, n, sigma, w, ctypes.byref(ct),
                                 workspace.data_ptr(), workspace.numel(), _stream_ptr(stream))
    _check(st, "wt_build_from_host")
    return h_tree


def build_from_host_async(h_seq: torch.Tensor, sigma: int, h_tree: HostTree, workspace: torch.Tensor,
                          h_status: torch.Tensor, stream=None) -> HostTree:
    """wt_build_from_host_async: H2D, build and D2H of the tree enqueued on `stream`, no
    synchronisation; after the stream is synchronised, h_status (a pinned int32 host
    tensor of one element) holds WT_OK or WT_ERR_SYMBOL_RANGE.  Two builds on two
    streams with two workspaces overlap each other's copies and compute."""
    if h_seq.is_cuda or h_status.is_cuda:
        raise ValueError("h_seq and h_status must be host tensors")
    if h_status.dtype != torch.int32 or h_status.numel() < 1:
        raise ValueError("h_status must be an int32 host tensor")
    h_seq = h_seq.contiguous()
    w = width_of(h_seq)
    n = h_seq.numel()
    ct = WtTree(h_tree.bitmaps.data_ptr() if h_tree.bitmaps.numel() else None,
                h_tree.superblocks.data_ptr() if h_tree.superblocks.numel() else None,
                h_tree.node_offsets.data_ptr())
    st = _lib.wt_build_from_host_async(h_seq.data_ptr() if n else None, n, sigma, w, ctypes.byref(ct),
                                       workspace.data_ptr(), workspace.numel(), h_status.data_ptr(),
                                       _stream_ptr(stream))
    _check(st, "wt_build_from_host_async")
    return h_tree




def access(tree: WaveletTree, pos: torch.Tensor, stream=None, status: torch.Tensor | None = None) -> torch.Tensor:
    """S[pos] for a batch of positions (int64 device tensor) -> int64 tensor (uint32 values)."""
    pos = pos.to(torch.int64).contiguous()
    m = pos.numel()
    out = torch.empty(m, dtype=torch.int32, device=pos.device)
    ct = tree._ctree()
    st = _lib.wt_access(ctypes.byref(ct), tree.n, tree.sigma, pos.data_ptr() if m else None, m,
                        out.data_ptr() if m else None, status.data_ptr() if status is not None else None,
                        _stream_ptr(stream))
    _check(st, "wt_access")
    return out.to(torch.int64) & 0xFFFFFFFF


def rank(tree: WaveletTree, c: torch.Tensor, pos: torch.Tensor, stream=None,
         status: torch.Tensor | None = None) -> torch.Tensor:
    """inclusive rank_c(S, pos) for paired batches (c: int32/uint32, pos: int64)."""
    c = c.to(torch.int32).contiguous()
    pos = pos.to(torch.int64).contiguous()
    m = pos.numel()
    out = torch.empty(m, dtype=torch.int64, device=pos.device)
    ct = tree._ctree()
    st = _lib.wt_rank(ctypes.byref(ct), tree.n, tree.sigma, c.data_ptr() if m else None,
                      pos.data_ptr() if m else None, m, out.data_ptr() if m else None,
                      status.data_ptr() if status is not None else None, _stream_ptr(stream))
    _check(st, "wt_rank")
    return out


SELECT_SAMPLE_SHIFT = 12  # the select index samples every 2^12-th bit of each value


def select_index(tree: WaveletTree, stream=None) -> torch.Tensor:
    """wt_select_index: per level l and bit b, the positions of every 4096-th bit equal to
    b, as an int32 tensor of shape (L, 2, n // 4096 + 2) (entries past the count hold n)."""
    e = int(_lib.wt_select_index_entries(tree.n, tree.sigma))
    L = tree.levels
    q = tree.n // 4096 + 2
    out = torch.empty((L, 2, q) if L else (0,), dtype=torch.int32, device=tree.bitmaps.device)
    assert out.numel() == e
    ct = tree._ctree()
    st = _lib.wt_select_index(ctypes.byref(ct), tree.n, tree.sigma, out.data_ptr() if e else None,
                              _stream_ptr(stream))
    _check(st, "wt_select_index")
    return out


def select(tree: WaveletTree, c: torch.Tensor, j: torch.Tensor, stream=None,
           status: torch.Tensor | None = None, index: torch.Tensor | None = None) -> torch.Tensor:
    """position of the j-th (1-based) occurrence of c, for paired batches; with the tree's
    select index (select_index) each level's search is narrowed to one sample stretch."""
    c = c.to(torch.int32).contiguous()
    j = j.to(torch.int64).contiguous()
    m = j.numel()
    out = torch.empty(m, dtype=torch.int64, device=j.device)
    ct = tree._ctree()
    if index is None:
        st = _lib.wt_select(ctypes.byref(ct), tree.n, tree.sigma, c.data_ptr() if m else None,
                            j.data_ptr() if m else None, m, out.data_ptr() if m else None,
                            status.data_ptr() if status is not None else None, _stream_ptr(stream))
        _check(st, "wt_select")
    else:
        st = _lib.wt_select_indexed(ctypes.byref(ct), tree.n, tree.sigma,
                                    index.data_ptr() if index.numel() else None,
                                    c.data_ptr() if m else None, j.data_ptr() if m else None, m,
                                    out.data_ptr() if m else None,
                                    status.data_ptr() if status is not None else None, _stream_ptr(stream))
        _check(st, "wt_select_indexed")
    return out


# ---------------------------------------------------------------- wavelet matrix (NEXT-4)


@dataclass
class WaveletMatrix:
    n: int
    sigma: int
    levels: int
    bitmaps: torch.Tensor       # (L, words_per_level) int32 (uint32 bit pattern)
    superblocks: torch.Tensor   # (L, sb_per_level) int64
    zeros: torch.Tensor         # (L,) int64: zeros of each level

    def _cmatrix(self) -> WtMatrix:
        return WtMatrix(self.bitmaps.data_ptr() if self.bitmaps.numel() else None,
                        self.superblocks.data_ptr() if self.superblocks.numel() else None,
                        self.zeros.data_ptr() if self.zeros.numel() else None)


def build_matrix(seq: torch.Tensor, sigma: int, workspace: torch.Tensor | None = None,
                 stream=None) -> WaveletMatrix:
    """wt_matrix_build_async + one synchronisation to read the range flag."""
    if not seq.is_cuda:
        raise ValueError("seq must be a CUDA tensor")
    seq = seq.contiguous()
    w = width_of(seq)
    n = seq.numel()
    sz = sizes(n, sigma, w)
    L = sz.levels
    dev = seq.device
    mx = WaveletMatrix(n=n, sigma=sigma, levels=L,
                       bitmaps=torch.empty((L, sz.words_per_level), dtype=torch.int32, device=dev),
                       superblocks=torch.empty((L, sz.sb_per_level), dtype=torch.int64, device=dev),
                       zeros=torch.empty((L,), dtype=torch.int64, device=dev))
    if workspace is None:
        workspace = alloc_workspace(n, sigma, w, dev)
    status = _status_tensor(dev)
    cm = mx._cmatrix()
    st = _lib.wt_matrix_build_async(seq.data_ptr() if n else None, n, sigma, w, ctypes.byref(cm),
                                    workspace.data_ptr(), workspace.numel(), status.data_ptr(), _stream_ptr(stream))
    _check(st, "wt_matrix_build_async")
    _sync(stream)  # the status word is written on `stream`, which need not be torch's current one
    if int(status.item()) != WT_OK:
        raise WtError(int(status.item()), "wt_matrix_build_async: a symbol is >= sigma")
    return mx


def matrix_access(mx: WaveletMatrix, pos: torch.Tensor, stream=None) -> torch.Tensor:
    pos = pos.to(torch.int64).contiguous()
    m = pos.numel()
    out = torch.empty(m, dtype=torch.int32, device=pos.device)
    cm = mx._cmatrix()
    st = _lib.wt_matrix_access(ctypes.byref(cm), mx.n, mx.sigma, pos.data_ptr() if m else None, m,
                               out.data_ptr() if m else None, None, _stream_ptr(stream))
    _check(st, "wt_matrix_access")
    return out.to(torch.int64) & 0xFFFFFFFF


def matrix_rank(mx: WaveletMatrix, c: torch.Tensor, pos: torch.Tensor, stream=None) -> torch.Tensor:
    c = c.to(torch.int32).contiguous()
    pos = pos.to(torch.int64).contiguous()
    m = pos.numel()
    out = torch.empty(m, dtype=torch.int64, device=pos.device)
    cm = mx._cmatrix()
    st = _lib.wt_matrix_rank(ctypes.byref(cm), mx.n, mx.sigma, c.data_ptr() if m else None,
                             pos.data_ptr() if m else None, m, out.data_ptr() if m else None, None,
                             _stream_ptr(stream))
    _check(st, "wt_matrix_rank")
    return out


def remap_alphabet(seq: torch.Tensor, sigma: int, stream=None):
    """wt_remap_alphabet: (remapped sequence, sorted alphabet, sigma') for a CUDA tensor
    of symbols < sigma; every symbol becomes its rank among the distinct values present."""
    if not seq.is_cuda:
        raise ValueError("seq must be a CUDA tensor")
    seq = seq.contiguous()
    w = width_of(seq)
    n = seq.numel()
    dev = seq.device
    out = torch.empty_like(seq)
    # at most min(sigma, n) distinct values can occur (sigma may be 2^32)
    alphabet = torch.empty((max(min(sigma, n), 1),), dtype=torch.int32, device=dev)
    sig = torch.zeros(1, dtype=torch.int64, device=dev)
    status = _status_tensor(dev)
    ws = torch.empty((max(int(_lib.wt_remap_workspace_bytes(sigma)), 256),), dtype=torch.uint8, device=dev)
    st = _lib.wt_remap_alphabet(seq.data_ptr() if n else None, n, sigma, w, out.data_ptr() if n else None,
                                alphabet.data_ptr(), sig.data_ptr(), ws.data_ptr(), ws.numel(), status.data_ptr(),
                                _stream_ptr(stream))
    _check(st, "wt_remap_alphabet")
    _sync(stream)
    if int(status.item()) != WT_OK:
        raise WtError(int(status.item()), "wt_remap_alphabet: a symbol is >= sigma")
    s2 = int(sig.item())
    return out, alphabet[:s2], s2


# ---------------------------------------------------------------- domain decomposition (NEXT-3)


DD_MAX_SEGMENTS = 32


def _ptr_array(ptrs):
    return (ctypes.c_void_p * len(ptrs))(*ptrs)


def dd_merge(segments: list, sigma: int, stream=None) -> WaveletTree:
    """wt_dd_merge: the tree of the concatenation of k <= 32 segment trees (each a
    WaveletTree over the same sigma, on the same device)."""
    k = len(segments)
    if not 1 <= k <= DD_MAX_SEGMENTS:
        raise ValueError(f"1..{DD_MAX_SEGMENTS} segments")
    n = sum(t.n for t in segments)
    dev = segments[0].node_offsets.device
    w = 4  # (the tree layout does not depend on the symbol width; 4 admits every sigma)
    out = alloc_tree(n, sigma, w, dev)
    arr = (WtTree * k)(*[t._ctree() for t in segments])
    ns = (ctypes.c_uint64 * k)(*[t.n for t in segments])
    scratch = torch.empty((max(int(_lib.wt_dd_merge_scratch_bytes(n)), 256),), dtype=torch.uint8, device=dev)
    ct = out._ctree()
    st = _lib.wt_dd_merge(k, ctypes.cast(arr, _vp), ctypes.cast(ns, _vp), sigma, ctypes.byref(ct),
                          scratch.data_ptr(), scratch.numel(), _stream_ptr(stream))
    _check(st, "wt_dd_merge")
    _sync(stream)
    return out


def build_dd(seq: torch.Tensor, sigma: int, k: int) -> WaveletTree:
    """The paper's domain decomposition on one GPU: k contiguous segments built
    separately (16-byte-aligned cut points), then merged."""
    seq = seq.contiguous()
    n = seq.numel()
    w = width_of(seq)
    step = -(-n // k) if n else 0
    align = 16 // w
    step = -(-step // align) * align if step else 0
    cuts = [min(i * step, n) for i in range(k)] + [n]
    segs = [build(seq[cuts[i]:cuts[i + 1]], sigma) for i in range(k)]
    return dd_merge(segs, sigma)


# ---------------------------------------------------------------- dd building blocks (multi-GPU merge)


def dd_part_blocks(n: int, parts: int, part: int) -> tuple[int, int]:
    """wt_dd_part_blocks: the 512-bit blocks [b, e) part `part` of `parts` owns."""
    b, e = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _lib.wt_dd_part_blocks(n, parts, part, ctypes.byref(b), ctypes.byref(e))
    return int(b.value), int(e.value)


def dd_plan_host(seg_offsets: list, sigma: int, parts: int):
    """wt_dd_plan on host arrays: seg_offsets[g] = segment g's node offsets (numpy
    uint64 or int64, 2^L + 1 entries).  Returns an int64 numpy array of shape
    (L, parts, k, 2): the source range [lo, hi) of segment g's level-l bits that
    land in part p."""
    import numpy as np
    k = len(seg_offsets)
    L = sizes(1, sigma, 4).levels
    arrs = [np.ascontiguousarray(np.asarray(c).view(np.uint64)) for c in seg_offsets]
    ptrs = _ptr_array([a.ctypes.data for a in arrs])
    plan = np.zeros((L, parts, k, 2), np.uint64)
    _check(_lib.wt_dd_plan(k, ctypes.cast(ptrs, _vp), sigma, parts, plan.ctypes.data if plan.size else None),
           "wt_dd_plan")
    return plan.astype(np.int64)


def dd_plan_device(seg_offsets: list, sigma: int, n: int, parts: int, stream=None) -> torch.Tensor:
    """wt_dd_plan_async: the same plan from device node offsets (a device int64
    tensor of shape (L, parts, k, 2))."""
    k = len(seg_offsets)
    L = sizes(1, sigma, 4).levels
    dev = seg_offsets[0].device
    plan = torch.empty((L, parts, k, 2), dtype=torch.int64, device=dev)
    ptrs = _ptr_array([c.data_ptr() for c in seg_offsets])
    _check(_lib.wt_dd_plan_async(k, ctypes.cast(ptrs, _vp), sigma, n, parts,
                                 plan.data_ptr() if plan.numel() else None, _stream_ptr(stream)),
           "wt_dd_plan_async")
    return plan


def dd_offsets(seg_offsets: list, sigma: int, out: torch.Tensor, stream=None) -> torch.Tensor:
    """wt_dd_offsets: out = sum of the segments' node offsets (device tensors)."""
    ptrs = _ptr_array([c.data_ptr() for c in seg_offsets])
    _check(_lib.wt_dd_offsets(len(seg_offsets), ctypes.cast(ptrs, _vp), sigma, out.data_ptr(), _stream_ptr(stream)),
           "wt_dd_offsets")
    return out


def dd_merge_level(seg_offsets: list, offsets: torch.Tensor, sigma: int, n: int, level: int, src_bits: list,
                   src_base: list, word_begin: int, word_end: int, out: torch.Tensor, stream=None):
    """wt_dd_merge_level: merged words [word_begin, word_end) of `level` into `out`
    from the segments' source words (src_bits[g]: device tensor whose word j holds
    segment g's level bits [src_base[g] + 32 j, +32))."""
    k = len(seg_offsets)
    offs = _ptr_array([c.data_ptr() for c in seg_offsets])
    bits = _ptr_array([b.data_ptr() if b.numel() else 0 for b in src_bits])
    base = (ctypes.c_uint64 * k)(*[int(x) for x in src_base])
    _check(_lib.wt_dd_merge_level(k, ctypes.cast(offs, _vp), offsets.data_ptr(), sigma, n, level,
                                  ctypes.cast(bits, _vp), ctypes.cast(base, _vp), word_begin, word_end,
                                  out.data_ptr() if out.numel() else None, _stream_ptr(stream)),
           "wt_dd_merge_level")


def superblocks(bits: torch.Tensor, nblocks: int, base: int, out: torch.Tensor, stream=None):
    """wt_superblocks: out[t] = base + ones in the first t 512-bit blocks of `bits`, t <= nblocks."""
    dev = out.device
    scratch = torch.empty((max(int(_lib.wt_superblocks_scratch_bytes(nblocks)), 256),), dtype=torch.uint8,
                          device=dev)
    _keep_for(stream, scratch)
    _check(_lib.wt_superblocks(bits.data_ptr() if nblocks else None, nblocks, base, out.data_ptr(),
                               scratch.data_ptr(), scratch.numel(), _stream_ptr(stream)), "wt_superblocks")


def rank1(tree: WaveletTree, level: torch.Tensor, pos: torch.Tensor, stream=None) -> torch.Tensor:
    """wt_rank1: ones of level[j] before pos[j] in a finished tree."""
    level = level.to(torch.int32).contiguous()
    pos = pos.to(torch.int64).contiguous()
    m = pos.numel()
    out = torch.empty(m, dtype=torch.int64, device=pos.device)
    ct = tree._ctree()
    _check(_lib.wt_rank1(ctypes.byref(ct), tree.n, tree.sigma, level.data_ptr() if m else None,
                         pos.data_ptr() if m else None, m, out.data_ptr() if m else None, _stream_ptr(stream)),
           "wt_rank1")
    return out
