/*
 * wt.h -- C ABI of the B200-native levelwise wavelet-tree builder
 * (libwt.so, package paper_1610_05994_b200).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   the one-pointer-per-level wavelet tree (Fig. 1b) of a sequence
 *   S[0..n) over the contiguous alphabet [0, sigma), i.e. for each
 *   of the L = ceil(lg sigma) levels (L = 0 when sigma == 1):
 *     - the level bitmap B_l: bit (L-1-l) of every symbol, taken in the order
 *       of S stably sorted by the symbol's top l bits (Prop. 1, P:485-490;
 *       node of s at level l is s >> (L-l); Alg. 1 lines 8-13);
 *     - the rank directory of B_l (createRankSelect, Alg. 1 line 14):
 *       one 64-bit cumulative popcount per 512-bit block;
 *   and the node offsets C (the prefix-summed counters of Alg. 1 lines 5-7,
 *   P:539-543, at the leaf granularity): C[c] = #{j : S[j] < c}, c in [0, 2^L].
 *
 * Output layout (the parity contract; the oracle emits the identical bytes):
 *   bitmaps      uint32[L * words_per_level], level-major.  Bit q of level l is
 *                (bitmaps[l*words_per_level + q/32] >> (q%32)) & 1 (LSB-first).
 *                words_per_level = 16*ceil(n/512); bits >= n are zero.
 *   superblocks  uint64[L * sb_per_level], sb_per_level = ceil(n/512) + 1.
 *                superblocks[l*sb_per_level + t] = popcount of level-l bits in
 *                [0, min(512 t, n)); the last entry is the level's total ones.
 *   node_offsets uint64[2^L + 1].  Level-l node v spans positions
 *                [node_offsets[v << (L-l)], node_offsets[(v+1) << (L-l)]).
 *
 * Conventions: 0-based positions; bit 0 = left child, 1 = right child
 * (P:293-296); access/rank are the paper's traversals with
 * INCLUSIVE rank ("i = rank1(B,24) - 1 = 7").
 *
 * Ownership: every d_ pointer is DEVICE memory owned by the caller (e.g. torch
 * tensors); every h_ pointer is host memory owned by the caller.  The library
 * allocates nothing, keeps no global state (only a thread-local last-error
 * string and thread-local profiling events), never retains a pointer after a
 * call's work has completed on the stream, and is stream-ordered: all device
 * work is enqueued on `stream`.  Concurrent builds on different streams need
 * different workspaces.  A finished tree is immutable; queries on it may run
 * concurrently.
 *
 * Errors: status codes only -- no exceptions, aborts or printing.
 */
#ifndef WT_H_
#define WT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Layout-compatible with cudaStream_t (a CUstream_st*); NULL = legacy default stream. */
typedef struct CUstream_st* wt_stream_t;
/* Layout-compatible with cudaEvent_t. */
typedef struct CUevent_st* wt_event_t;

typedef enum {
  WT_OK = 0,
  WT_ERR_ARG = 1,           /* bad width / sigma / n / pointer / alignment */
  WT_ERR_SYMBOL_RANGE = 2,  /* some S[j] >= sigma; outputs unspecified */
  WT_ERR_INDEX = 3,         /* query position >= n, or symbol >= sigma, or ordinal out of range */
  WT_ERR_CUDA = 4,          /* a CUDA runtime call or launch failed (see wt_last_error) */
  WT_ERR_WORKSPACE = 5      /* workspace NULL or smaller than wt_sizes().workspace_bytes */
} wt_status;

typedef struct {
  uint32_t levels;           /* L = ceil(lg sigma); 0 when sigma == 1 */
  uint32_t width;            /* bytes per input symbol (1, 2 or 4) */
  uint64_t words_per_level;  /* uint32 words per level bitmap = 16*ceil(n/512) */
  uint64_t sb_per_level;     /* uint64 superblock entries per level = ceil(n/512) + 1 */
  uint64_t c_len;            /* uint64 node offsets = 2^L + 1 */
  uint64_t bitmap_bytes;     /* 4 * L * words_per_level */
  uint64_t superblock_bytes; /* 8 * L * sb_per_level */
  uint64_t node_offset_bytes;/* 8 * c_len */
  size_t workspace_bytes;    /* device scratch wt_build needs (ping-pong permuted
                                sequences T_l, node tables, scan state, flag) */
  size_t host_workspace_bytes; /* device scratch wt_build_from_host needs: the
                                workspace plus a device copy of S and of the tree */
} wt_sizes_t;

/* A tree in memory the caller owns (device pointers for the device API, host
 * pointers for the *_from_host output). */
typedef struct {
  uint32_t* bitmaps;
  uint64_t* superblocks;
  uint64_t* node_offsets;
} wt_tree_t;

/*
 * wt_sizes: sizes of every output and of the workspace for a build of n
 * symbols of `width` bytes over [0, sigma).  Pure host arithmetic.
 * n may exceed 2^32: a build of more than seg_max = 2^31 symbols is
 * SEGMENTED -- S is cut into k = ceil(n / 2^31) contiguous segments, each built
 * by the direct launch sequence (all of its in-kernel positions 32-bit), and
 * the k segment trees are merged into the output with 64-bit positions (the
 * paper's domain decomposition; its datasets reach
 * n = 1.46e10).  workspace_bytes then includes the k segment trees
 * and one segment's build workspace.  (WT_SEG_MAX, read per call, lowers the
 * segment length for tests: a multiple of 4096 in [4096, 2^31].)
 * Errors: WT_ERR_ARG if width not in {1,2,4}, sigma == 0,
 * sigma > 2^(8*width), L > 30, n > 32 * seg_max, or out == NULL.
 */
wt_status wt_sizes(uint64_t n, uint64_t sigma, uint32_t width, wt_sizes_t* out);

/*
 * wt_build_async: enqueue the whole construction on `stream`:
 *   a1 one pass over S (symbol-range check, level-0 tile ones), a3 one
 *   stable bit-partition pass per level l < L-2 (bitmap words, superblocks,
 *   T_{l+1}, and -- progressive counting -- the sizes of the level-(l+2)
 *   nodes), each preceded by a2 scans building that level's node tables;
 *   a5 the pass of level L-2 fused with level L-1 (both bitmaps from T_{L-2}
 *   with no symbol moved), then the last level's superblocks and
 *   node_offsets from its ranks at the node starts; a4 the single level when
 *   L = 1.  No host synchronisation; CUDA-graph capturable.
 * d_seq       n symbols, little-endian, `width` bytes each; 16-byte aligned
 *             (any torch/cudaMalloc allocation is).  Read only.
 * out         device pointers sized per wt_sizes (bitmaps, superblocks,
 *             node_offsets); fully overwritten.  bitmaps 16-byte aligned
 *             (the pair passes store 16-byte words), superblocks and
 *             node_offsets 8-byte aligned (any torch/cudaMalloc allocation is).
 * d_workspace >= wt_sizes().workspace_bytes of device memory, 256-byte aligned;
 *             contents on entry are irrelevant.
 * d_status    optional (may be NULL): receives WT_OK or WT_ERR_SYMBOL_RANGE
 *             (int32) when the stream reaches the end of the build.
 * Returns WT_ERR_ARG / WT_ERR_WORKSPACE on bad arguments (nothing enqueued;
 * WT_ERR_ARG also for a misaligned d_seq, d_workspace or output pointer),
 * WT_ERR_CUDA if a launch failed, else WT_OK.
 */
wt_status wt_build_async(const void* d_seq, uint64_t n, uint64_t sigma, uint32_t width,
                         const wt_tree_t* out, void* d_workspace, size_t workspace_bytes,
                         int32_t* d_status, wt_stream_t stream);

/*
 * wt_build: wt_build_async, then one stream synchronisation to read the
 * range-check flag.  Returns WT_ERR_SYMBOL_RANGE if any S[j] >= sigma.
 */
wt_status wt_build(const void* d_seq, uint64_t n, uint64_t sigma, uint32_t width,
                   const wt_tree_t* out, void* d_workspace, size_t workspace_bytes,
                   wt_stream_t stream);

/*
 * wt_build_from_host: end-to-end build from HOST memory.  Copies h_seq
 * (n*width bytes, ideally pinned) to the device, builds, and copies the tree
 * back into the host buffers of h_out (sizes per wt_sizes), all on `stream`,
 * then synchronises.  d_workspace >= wt_sizes().host_workspace_bytes.
 * Errors as wt_build.
 */
wt_status wt_build_from_host(const void* h_seq, uint64_t n, uint64_t sigma, uint32_t width,
                             const wt_tree_t* h_out, void* d_workspace, size_t workspace_bytes,
                             wt_stream_t stream);

/*
 * wt_build_from_host_async: the same, enqueued on `stream` WITHOUT the final
 * synchronisation: H2D of h_seq, the build, D2H of the tree into h_out, and
 * the build's status word into *h_status (host memory, pinned for the copy
 * to stay asynchronous).  After synchronising the stream, *h_status is WT_OK
 * or WT_ERR_SYMBOL_RANGE (h_out is then unspecified).  Builds on different
 * streams with different workspaces run concurrently (their copies overlap
 * each other's compute: H2D and D2H use separate copy engines).  The host
 * buffers must stay valid until the stream reaches the end of the build.
 * Errors (returned at once): as wt_build_from_host, WT_ERR_ARG if h_status
 * is NULL.
 */
wt_status wt_build_from_host_async(const void* h_seq, uint64_t n, uint64_t sigma, uint32_t width,
                                   const wt_tree_t* h_out, void* d_workspace, size_t workspace_bytes,
                                   int32_t* h_status, wt_stream_t stream);

/*
 * wt_access: d_sym[k] = S[d_pos[k]] for k < m, by the top-down traversal of
 * P:353-380 simulated with rank on the level bitmaps.
 * tree: device pointers of a finished build of (n, sigma).
 * Positions >= n get d_sym[k] = UINT32_MAX and set *d_status = WT_ERR_INDEX
 * (d_status optional; initialise it to WT_OK yourself).  Asynchronous.
 */
wt_status wt_access(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint64_t* d_pos,
                    uint64_t m, uint32_t* d_sym, int32_t* d_status, wt_stream_t stream);

/*
 * wt_rank: d_cnt[k] = #{ j <= d_pos[k] : S[j] == d_c[k] } (inclusive rank,
 * P:279-281).  Pairs with pos >= n or c >= sigma get UINT64_MAX and set
 * *d_status = WT_ERR_INDEX.  Asynchronous.
 */
wt_status wt_rank(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint32_t* d_c,
                  const uint64_t* d_pos, uint64_t m, uint64_t* d_cnt, int32_t* d_status,
                  wt_stream_t stream);

/*
 * wt_select: d_out[k] = position of the d_j[k]-th (1-based) occurrence of
 * d_c[k] in S, by the bottom-up traversal.  Invalid pairs
 * (c >= sigma, j == 0, j > occurrences of c) get UINT64_MAX and set
 * *d_status = WT_ERR_INDEX.  Asynchronous.
 */
wt_status wt_select(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint32_t* d_c,
                    const uint64_t* d_j, uint64_t m, uint64_t* d_out, int32_t* d_status,
                    wt_stream_t stream);

/*
 * Select index (createRankSelect's select half):
 * per level l and bit value b, the position of every 4096-th bit equal to b:
 *   d_samples[(2 l + b) * Q + k] = position of the (4096 k)-th (0-based) bit
 *   equal to b in B_l, or n when the level has fewer such bits,
 * with Q = wt_select_index_entries(n) / (2 L) = n / 4096 + 2 uint32 entries.
 * Built from a finished tree (device pointers) in one pass over the bitmaps
 * (L * n / 8 bytes); like the paper's rank/select structures it is not part
 * of the tree construction.  d_samples: caller-owned device memory of
 * wt_select_index_entries(n, sigma) uint32.  Asynchronous.
 * Errors: WT_ERR_ARG (NULL pointers, bad sigma, n >= 2^32: the samples are
 * 32-bit positions), WT_ERR_CUDA.
 */
uint64_t wt_select_index_entries(uint64_t n, uint64_t sigma);
wt_status wt_select_index(const wt_tree_t* tree, uint64_t n, uint64_t sigma, uint32_t* d_samples,
                          wt_stream_t stream);

/*
 * wt_select_indexed: wt_select with the select index of the same tree: each
 * level's superblock search is narrowed to the stretch between two samples
 * (at most 4096 bits of that value).  Same results and errors as wt_select.
 */
wt_status wt_select_indexed(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint32_t* d_samples,
                            const uint32_t* d_c, const uint64_t* d_j, uint64_t m, uint64_t* d_out,
                            int32_t* d_status, wt_stream_t stream);

/*
 * Wavelet matrix (NEXT-4; the variant P:1409-1413 names): level l is the
 * sequence T_l stably partitioned, over the WHOLE sequence (no nodes), by bit
 * (L-1-l): T_0 = S, T_{l+1} = zeros of T_l then ones; B_l[j] = bit (L-1-l) of
 * T_l[j]; zeros[l] = number of zeros of level l.  Same bitmap and superblock
 * layout as the tree (bitmaps L x words_per_level, superblocks L x
 * sb_per_level); zeros: L uint64.  Built by the same level kernels with one
 * global node per level; workspace as wt_sizes().workspace_bytes.
 * d_status as wt_build_async.  Errors as wt_build_async.
 */
typedef struct {
  uint32_t* bitmaps;
  uint64_t* superblocks;
  uint64_t* zeros;
} wt_matrix_t;

wt_status wt_matrix_build_async(const void* d_seq, uint64_t n, uint64_t sigma, uint32_t width,
                                const wt_matrix_t* out, void* d_workspace, size_t workspace_bytes,
                                int32_t* d_status, wt_stream_t stream);
/* d_sym[k] = S[d_pos[k]] (positions >= n: UINT32_MAX and *d_status = WT_ERR_INDEX). */
wt_status wt_matrix_access(const wt_matrix_t* mx, uint64_t n, uint64_t sigma, const uint64_t* d_pos,
                           uint64_t m, uint32_t* d_sym, int32_t* d_status, wt_stream_t stream);
/* d_cnt[k] = #{j <= d_pos[k] : S[j] = d_c[k]} (inclusive; invalid: UINT64_MAX, WT_ERR_INDEX). */
wt_status wt_matrix_rank(const wt_matrix_t* mx, uint64_t n, uint64_t sigma, const uint32_t* d_c,
                         const uint64_t* d_pos, uint64_t m, uint64_t* d_cnt, int32_t* d_status,
                         wt_stream_t stream);

/*
 * Alphabet remap (NEXT-4, the effective alphabet of P:467-470): replaces every
 * symbol of d_seq (n symbols of `width` bytes, all < sigma) by its rank among
 * the distinct values present, so a sequence over a sparse alphabet builds a
 * tree of ceil(lg sigma') levels, sigma' = number of distinct values.
 *   d_out[j] = #{distinct values < d_seq[j]}   (same width; may alias d_seq)
 *   d_alphabet[r] = the r-th smallest distinct value, r < sigma' (capacity sigma)
 *   *d_sigma_out = sigma' (uint64, device)
 * sigma <= 2^(8 width) (<= 2^32).  Device scratch: wt_remap_workspace_bytes(sigma)
 * (a presence bitmap of sigma bits plus per-word ranks).  Asynchronous; *d_status
 * (device, optional) becomes WT_ERR_SYMBOL_RANGE if a symbol is >= sigma.
 * Errors: WT_ERR_ARG, WT_ERR_WORKSPACE, WT_ERR_CUDA.
 */
size_t wt_remap_workspace_bytes(uint64_t sigma);
wt_status wt_remap_alphabet(const void* d_seq, uint64_t n, uint64_t sigma, uint32_t width, void* d_out,
                            uint32_t* d_alphabet, uint64_t* d_sigma_out, void* d_workspace,
                            size_t workspace_bytes, int32_t* d_status, wt_stream_t stream);

/*
 * Domain decomposition (NEXT-3; the paper's dd).  S is cut
 * into k <= 32 contiguous segments, each built on its own (the partial trees of
 * createPartialBA) -- on one GPU, or one segment per GPU -- and the
 * tree of the whole sequence is their merge (mergeBA): C is the sum
 * of the segments' node offsets, and node v of every level holds segment 0's
 * run of v, then segment 1's, ... (the per-level prefix over segments of
 * Alg. 2 lines 7-8).  All positions are 64-bit (n may be >= 2^32).
 *
 * wt_dd_merge: the whole merge on one device.  segs[g]: device trees of
 * seg_n[g] symbols over the same sigma; out: a tree of n = sum seg_n symbols.
 * d_scratch: wt_dd_merge_scratch_bytes(n).  Asynchronous.
 * Errors: WT_ERR_ARG (k = 0 or > 32, NULL pointers), WT_ERR_WORKSPACE.
 */
size_t wt_dd_merge_scratch_bytes(uint64_t n);
wt_status wt_dd_merge(uint32_t k, const wt_tree_t* segs, const uint64_t* seg_n, uint64_t sigma,
                      const wt_tree_t* out, void* d_scratch, size_t scratch_bytes, wt_stream_t stream);

/*
 * The merge's building blocks, for a merge whose output is split into `parts`
 * (one per GPU: each rank merges and owns one part):
 *
 * wt_dd_part_blocks: part p of a merged tree of n symbols owns the 512-bit
 *   blocks [*block_begin, *block_end) -- bitmap words [16 b, 16 e), merged
 *   positions [min(n, 512 b), min(n, 512 e)), superblock entries [b, e]
 *   (e - b + 1 entries; the last equals the next part's first).  Parts get
 *   ceil(ceil(n/512) / parts) blocks each, the trailing ones fewer (or none).
 * wt_dd_offsets: d_offsets[i] = sum_g d_seg_offsets[g][i], i <= 2^L (the
 *   merged node offsets C).  d_seg_offsets: HOST array of k device pointers.
 * wt_dd_plan (host arithmetic on HOST arrays h_seg_offsets[g][0..2^L]) and
 * wt_dd_plan_async (the same arithmetic in a kernel, DEVICE arrays; n = the
 *   merged length): for level l < L, part p < parts, segment g < k,
 *     plan[((l * parts + p) * k + g) * 2 + 0] = lo, [... + 1] = hi
 *   where [lo, hi) are the positions of segment g's level-l bitmap whose
 *   merged positions fall in part p (a contiguous range: inside a segment the
 *   nodes are in order, and so are they in the merge).  lo counts the
 *   segment-g bits whose merged position is before the part: by node offsets
 *   alone (binary search for the node holding the part's first position).
 *   The plan has L * parts * k entries; with L = 0 (sigma = 1) it may be NULL.
 * wt_dd_merge_level: level `level` of the merge over merged words
 *   [word_begin, word_end) into d_out[0 .. word_end - word_begin).  Segment g's
 *   local bit q of that level is bit (q - src_base[g]) of the words at
 *   d_src_bits[g] (HOST arrays of k entries; src_base multiples of 32, NULL =
 *   all 0); the merge reads exactly the bits the plan assigns to the range,
 *   i.e. words [lo/32, ceil(hi/32)) relative to src_base.  d_seg_offsets,
 *   d_offsets as above.  Words past n are written as zeros.
 * wt_superblocks: superblocks of nblocks 512-bit blocks of d_bits plus the
 *   final total: d_sb[t] = base + ones in blocks [0, t), t <= nblocks.  One
 *   decoupled-look-back scan; d_scratch: wt_superblocks_scratch_bytes(nblocks).
 * wt_rank1: d_out[j] = ones of level d_level[j] before position d_pos[j]
 *   (d_pos[j] <= n) of a finished tree (the base of a part's superblocks is the
 *   sum over segments of rank1 at the plan's lo).
 * All asynchronous on `stream` except wt_dd_plan and wt_dd_part_blocks.
 * Errors: WT_ERR_ARG (k = 0 or > 32, NULL pointers, bad ranges), WT_ERR_WORKSPACE.
 */
void wt_dd_part_blocks(uint64_t n, uint64_t parts, uint64_t part, uint64_t* block_begin, uint64_t* block_end);
wt_status wt_dd_offsets(uint32_t k, const uint64_t* const* d_seg_offsets, uint64_t sigma, uint64_t* d_offsets,
                        wt_stream_t stream);
wt_status wt_dd_plan(uint32_t k, const uint64_t* const* h_seg_offsets, uint64_t sigma, uint64_t parts,
                     uint64_t* h_plan);
wt_status wt_dd_plan_async(uint32_t k, const uint64_t* const* d_seg_offsets, uint64_t sigma, uint64_t n,
                           uint64_t parts, uint64_t* d_plan, wt_stream_t stream);
wt_status wt_dd_merge_level(uint32_t k, const uint64_t* const* d_seg_offsets, const uint64_t* d_offsets,
                            uint64_t sigma, uint64_t n, uint32_t level, const uint32_t* const* d_src_bits,
                            const uint64_t* src_base, uint64_t word_begin, uint64_t word_end, uint32_t* d_out,
                            wt_stream_t stream);
size_t wt_superblocks_scratch_bytes(uint64_t nblocks);
wt_status wt_superblocks(const uint32_t* d_bits, uint64_t nblocks, uint64_t base, uint64_t* d_sb, void* d_scratch,
                         size_t scratch_bytes, wt_stream_t stream);
wt_status wt_rank1(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint32_t* d_level, const uint64_t* d_pos,
                   uint64_t m, uint64_t* d_out, wt_stream_t stream);

/* Kernel launches one wt_build_async(n, sigma, width) enqueues, and their kinds
 * (kinds may be NULL): 1 pass over S (prologue), 2 scan of node_offsets
 * (sigma = 1 only), 4 level pass with scatter (a3), 5 last level (a4, only
 * when L = 1), 8 level pass L-2 fused with level L-1 (a5 with k = 2: writes
 * B_{L-2} and B_{L-1}, no T_{L-1}),
 * 11 per-level preparation (the level's tile-prefix scan, its node-table scan
 * and the zeroing of the node counts the pass fills -- and of B_{L-1} before
 * pass 8), 12 final scans (superblocks of level L-1 straight from its bitmap,
 * and node_offsets from the leaf counts when kind 8 is the general pass),
 * 17 node_offsets from B_{L-1}'s ranks at the level-(L-1) node starts (after
 * the no-move fused pair, which counts no leaves: the default for L >= 2),
 * 18 interior fused pair of levels (opt-in).
 * A segmented build (n > seg_max) lists each segment's launches followed by
 * 16 (its range flag OR-ed into the build's), then 13 the merged node
 * offsets and, per level, 14 the level merge and 15 its superblock scan
 * (the merge kernels do nothing once a range flag is set).
 * Kinds 3, 6, 7, 9, 10 are retired (folded into 11 and 12). */
uint32_t wt_launch_plan(uint64_t n, uint64_t sigma, uint32_t width, uint32_t* kinds, uint32_t cap);

/* Debug aid: byte offsets inside the workspace of wt_build_async(n, sigma,
 * width): {flag, ones0, agg, pre, node tables, node counts, node-count buffer
 * stride, T_odd, T_even, tiles per level}.  Returns the number of entries. */
uint32_t wt_debug_offsets(uint64_t n, uint64_t sigma, uint32_t width, uint64_t* offsets, uint32_t cap);

/* Profiling hook (thread-local): when events != NULL, the next wt_build_async
 * calls on this thread record events[2k] before and events[2k+1] after launch
 * k (k < count/2) on the build stream.  Pass NULL to disable. */
void wt_set_profile_events(wt_event_t* events, uint32_t count);

const char* wt_status_string(wt_status status);
/* Detail of the last error on this thread ("" if none). */
const char* wt_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* WT_H_ */
