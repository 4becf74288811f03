// wt_kernels.cuh -- the build's scan kernels and the query / merge / remap
// kernels (sm_100a).  The launch sequence of a build (PAPER.md = P:n):
//   a1 k_prologue     (wt_prologue.cuh) one pass over S: symbol-range flag and the
//                     level-0 ones of every level tile.  No histogram of S is
//                     taken: Alg. 1's per-level counters (lines 5-6)
//                     are node sizes (Prop. 1), counted two levels
//                     ahead by the level passes ("progressive counting").
//   a2 k_prep         per level: decoupled-look-back scans (this file) of the
//                     per-tile ones (tile prefixes) and of the node sizes (node
//                     tables); the final one writes the last level's
//                     superblocks (and C, line 7, exclusive, after
//                     the general fused pair).
//   a3 k_level        (wt_level.cuh) the per-level stable segmented bit-partition
//                     of T_l, levels 0 .. L-3.
//   a5 k_pairn        (wt_pairn.cuh) pass L-2 fused with level L-1, no symbol
//                     moves; k_pair2 (wt_pair2.cuh) for two-level byte trees;
//                     k_leaf_offsets (this file) then C from B_{L-1}'s ranks.
//                     Opt-in: k_quad (interior pairs of levels), k_triple (the
//                     final three levels, wt_triple.cuh).
#pragma once
#include "wt_device.cuh"
#include "wt_prologue.cuh"
#include "wt_pair2.cuh"
#include "wt_pairn.cuh"
#include "wt_triple.cuh"
#include "wt_quad.cuh"

namespace wt {

// ================================================================ a2 scans

// CTA sizes: 512 threads for the scans that read a bitmap's 512-bit blocks
// themselves (SCAN_ITEMS_BITS = 8 blocks per thread: their loads want bytes in
// flight), 1024 for the scans of per-tile / per-node values (4 per thread:
// latency-bound -- fewer tiles shorten the look-back; 512 threads: cfg5 preps
// 0.54 ms per build, 1024: 0.45).  A k_prep launch hosts two scans in CTAs of
// one size, that of its first scan.
constexpr int SCAN_THREADS_BITS = 512;
constexpr int SCAN_THREADS_VALS = 1024;
constexpr int SCAN_ITEMS_BITS = 8;
#ifndef WT_SCAN_ITEMS_V
#define WT_SCAN_ITEMS_V 4
#endif
constexpr int SCAN_ITEMS_VALS = WT_SCAN_ITEMS_V;
// the smallest scan tile (sizes the look-back state: an upper bound on the tiles of any scan)
constexpr int SCAN_TILE_MIN = SCAN_THREADS_BITS * (SCAN_ITEMS_VALS < SCAN_ITEMS_BITS ? SCAN_ITEMS_VALS : SCAN_ITEMS_BITS);

// Scan ops whose values are the popcounts of consecutive 512-bit blocks of a
// bitmap (`bits`): scan_tile loads the tile's blocks itself, coalesced.
template <class Op>
struct ScanOfBits {
  static constexpr bool value = false;
};

// Exclusive scan of uint64 values over [0, count) with a decoupled look-back.
// Op supplies load(i) and store(i, exclusive, value).  One CTA of NT threads
// scans one tile of NT * items values; tile ids come from an atomic ticket
// (forward progress).
template <class Op>
constexpr int scan_items_of() { return ScanOfBits<Op>::value ? SCAN_ITEMS_BITS : SCAN_ITEMS_VALS; }
template <class Op>
constexpr int scan_threads_of() { return ScanOfBits<Op>::value ? SCAN_THREADS_BITS : SCAN_THREADS_VALS; }
template <class Op, int NT = scan_threads_of<Op>()>
constexpr uint64_t scan_tile_of() { return (uint64_t)NT * scan_items_of<Op>(); }

template <class Op, int NT>
__device__ __forceinline__ void scan_tile(const Op& op, uint64_t count, const LookbackState& status,
                                          uint32_t* tile_counter, uint32_t epoch) {
  constexpr int SCAN_ITEMS = scan_items_of<Op>();
  constexpr uint64_t SCAN_TILE = scan_tile_of<Op, NT>();
  __shared__ uint64_t s_warp[NT / 32];
  __shared__ uint64_t s_P;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
  uint64_t v[SCAN_ITEMS];
  uint64_t tsum = 0;
  if constexpr (ScanOfBits<Op>::value) {
    // the tile's blocks as 16-byte chunks, chunk c read by thread c % NT
    // (a warp reads 512 consecutive bytes per load); 4 consecutive lanes
    // hold one block: two shuffles sum it, its first lane stores the count
    __shared__ __align__(16) uint32_t s_cnt[SCAN_TILE];
    static_assert(SCAN_ITEMS % 4 == 0, "16-byte item loads");
    constexpr uint32_t CH = 4 * SCAN_TILE / NT;  // chunks per thread
    const uint4* src = reinterpret_cast<const uint4*>(op.bits) + 4 * tile * SCAN_TILE;
    const uint64_t t0 = tile * SCAN_TILE;  // (a surplus CTA's tile lies past count: no chunks)
    const uint64_t nch = t0 < count ? 4 * min((uint64_t)SCAN_TILE, count - t0) : 0;
#pragma unroll
    for (uint32_t j0 = 0; j0 < CH; j0 += 8) {
      uint32_t c[8];
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t ch = threadIdx.x + NT * (j0 + k);
        const uint4 q = ch < nch ? ldg_nc_v4(src + ch) : make_uint4(0, 0, 0, 0);
        c[k] = (uint32_t)(__popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w));
      }
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        c[k] += __shfl_xor_sync(FULL, c[k], 1);
        c[k] += __shfl_xor_sync(FULL, c[k], 2);
        if ((threadIdx.x & 3) == 0) s_cnt[(threadIdx.x + NT * (j0 + k)) >> 2] = c[k];
      }
    }
    __syncthreads();
    uint32_t cv[SCAN_ITEMS];  // the thread's items as 16-byte shared loads
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k += 4) {
      const uint4 q = *reinterpret_cast<const uint4*>(&s_cnt[threadIdx.x * SCAN_ITEMS + k]);
      cv[k] = q.x, cv[k + 1] = q.y, cv[k + 2] = q.z, cv[k + 3] = q.w;
    }
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      v[k] = (base + k < count) ? cv[k] : 0;
      tsum += v[k];
    }
  } else {
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      v[k] = (base + k < count) ? op.load(base + k) : 0;
      tsum += v[k];
    }
  }
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t incl = warp_incl_scan_u64(tsum);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint64_t run;
  if constexpr (ScanOfBits<Op>::value) {
    // (the bitmap scans fill a wave of CTAs that still stream their blocks: a
    // whole CTA polling its predecessors slowed cfg2's final scan 0.049 -> 0.052 ms)
    if (warp == 0) {
      const uint64_t w = (lane < NT / 32) ? s_warp[lane] : 0;
      const uint64_t wi = warp_incl_scan_u64(w);
      const uint64_t total = __shfl_sync(FULL, wi, 31);
      if (lane < NT / 32) s_warp[lane] = wi - w;
      const uint64_t P = lookback(status, tile, total, epoch);
      if (lane == 0) s_P = P;
    }
    __syncthreads();
    run = s_P + s_warp[warp] + incl - tsum;
  } else {
    // the look-back by the whole CTA: one round trip covers NT predecessors
    __shared__ uint64_t s_sum[NT / 32];
    __shared__ uint32_t s_has[NT / 32];
    if (warp == 0) {
      const uint64_t w = (lane < NT / 32) ? s_warp[lane] : 0;
      const uint64_t wi = warp_incl_scan_u64(w);
      if (lane < NT / 32) s_warp[lane] = wi - w;
      if (lane == 31) s_P = wi;  // the tile's total
    }
    __syncthreads();
    run = block_lookback<NT>(status, tile, s_P, epoch, s_sum, s_has) + s_warp[warp] + incl - tsum;
  }
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < count) op.store(base + k, run, v[k]);
    run += v[k];
  }
}

template <class Op>
__global__ void __launch_bounds__(scan_threads_of<Op>()) k_scan(Op op, uint64_t count, LookbackState status,
                                                                uint32_t* tile_counter, uint32_t epoch,
                                                                const int32_t* __restrict__ flag) {
  if (*flag) return;
  scan_tile<Op, scan_threads_of<Op>()>(op, count, status, tile_counter, epoch);
}

// Two independent scans (each with its own look-back state and ticket) and a
// zero fill of up to two buffers in ONE launch: CTAs [0, ga) scan A, the next
// gb scan B, the rest zero-fill.  Per level: the tile prefixes of the level,
// its node tables, and the node-count buffer the pass fills (plus, before the
// fused pass, the last level's bitmap); at the end: the last level's
// superblocks and C.
struct ZeroFill {
  uint4* p0;
  uint64_t n0;  // 16-byte units
  uint4* p1;
  uint64_t n1;
};
template <class OpA, class OpB>
__global__ void __launch_bounds__(scan_threads_of<OpA>())
    k_prep(OpA a, uint64_t na, LookbackState sta, uint32_t* ca, uint32_t ea, OpB b, uint64_t nb, LookbackState stb,
           uint32_t* cb, uint32_t eb, ZeroFill z, const int32_t* __restrict__ flag) {
  constexpr int NT = scan_threads_of<OpA>();  // (both scans in CTAs of the first one's size)
  pdl_wait();
  if (*flag) return;
  const uint32_t ga = (uint32_t)((na + scan_tile_of<OpA, NT>() - 1) / scan_tile_of<OpA, NT>()),
                 gb = (uint32_t)((nb + scan_tile_of<OpB, NT>() - 1) / scan_tile_of<OpB, NT>());
  if (blockIdx.x < ga) {
    scan_tile<OpA, NT>(a, na, sta, ca, ea);
  } else if (blockIdx.x < ga + gb) {
    scan_tile<OpB, NT>(b, nb, stb, cb, eb);
  } else {
    const uint64_t nt = (uint64_t)(gridDim.x - ga - gb) * NT;
    const uint64_t t0 = (uint64_t)(blockIdx.x - ga - gb) * NT + threadIdx.x;
    for (uint64_t i = t0; i < z.n0; i += nt) z.p0[i] = make_uint4(0, 0, 0, 0);
    for (uint64_t i = t0; i < z.n1; i += nt) z.p1[i] = make_uint4(0, 0, 0, 0);
  }
  pdl_trigger();  // at the tail: the next pass's CTAs launch as this grid drains
}

// Wavelet matrix (NEXT-4): a level is one global node.  The level's zeros
// Z_l = n - (ones of the level) come out of a scan of its per-tile ones: the
// last element writes tab[0] = {0 ones before the node, Z_l} and zeros[0] = Z_l.
struct OpMatrixTab {
  const uint32_t* agg;
  uint2* tab;
  unsigned long long* zeros;
  uint64_t n, count;
  __device__ uint64_t load(uint64_t i) const { return agg[i]; }
  __device__ void store(uint64_t i, uint64_t excl, uint64_t val) const {
    if (i + 1 == count) {
      const uint64_t z = n - (excl + val);
      tab[0] = make_uint2(0u, (uint32_t)z);
      zeros[0] = z;
    }
  }
};
// Superblocks of a level from its finished bitmap (the last level, whose bits
// the fused pass L-2 wrote in place; every level after a dd merge):
// SB[t] = ones in the 512-bit blocks before t, SB[nblocks] = the level's total
// (reading R7 of DESIGN.md).  One scan launch: scan_tile takes the
// block popcounts itself (ScanOfBits), coalesced.
struct OpBitsPop {
  const uint32_t* bits;
  unsigned long long* sb;
  uint64_t nblocks;
  uint64_t base;  // ones before block 0 (a part of a merged level: the ones of the earlier parts)
  __device__ uint64_t load(uint64_t) const { return 0; }  // (unused: ScanOfBits)
  __device__ void store(uint64_t i, uint64_t excl, uint64_t val) const {
    sb[i] = base + excl;
    if (i + 1 == nblocks) sb[nblocks] = base + excl + val;
  }
};
template <>
struct ScanOfBits<OpBitsPop> {
  static constexpr bool value = true;
};
struct OpBitsPopZ {  // (wavelet matrix: also the level's zeros)
  const uint32_t* bits;
  unsigned long long* sb;
  uint64_t nblocks;
  unsigned long long* zeros;
  uint64_t n;
  __device__ uint64_t load(uint64_t) const { return 0; }  // (unused: ScanOfBits)
  __device__ void store(uint64_t i, uint64_t excl, uint64_t val) const {
    sb[i] = excl;
    if (i + 1 == nblocks) {
      sb[nblocks] = excl + val;
      zeros[0] = n - (excl + val);
    }
  }
};
template <>
struct ScanOfBits<OpBitsPopZ> {
  static constexpr bool value = true;
};

// ---------------------------------------------------------------- alphabet remap (NEXT-4)
// The symbols that occur, ranked: map(s) = #{present values < s} (P:467-470's
// effective alphabet; the tree over the remapped sequence has ceil(lg sigma')
// levels for sigma' distinct values).  A presence bitmap over [0, sigma), a
// scan of its word popcounts, then every symbol is replaced by its rank.
template <typename T>
__global__ void k_remap_mark(const T* __restrict__ seq, uint64_t n, uint64_t sigma, uint32_t* present,
                             int32_t* __restrict__ flag) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = (uint64_t)seq[j];
    if (s >= sigma) {
      *flag = 2;  // WT_ERR_SYMBOL_RANGE
      continue;
    }
    const uint32_t bit = 1u << (s & 31);
    uint32_t* w = present + (s >> 5);
    // (a coherent relaxed read -- other threads OR into `present` during this
    // kernel, so no read-only-cache load -- skips the atomic for repeats)
    if (!(ld_relaxed_u32(w) & bit)) atomicOr(w, bit);
  }
}
struct OpPopPrefix {  // rank of the first value of word w = set bits of the words before w
  const uint32_t* present;
  uint32_t* rank;
  uint64_t words;
  unsigned long long* total;
  __device__ uint64_t load(uint64_t w) const { return (uint64_t)__popc(present[w]); }
  __device__ void store(uint64_t w, uint64_t excl, uint64_t val) const {
    rank[w] = (uint32_t)excl;
    if (w + 1 == words) *total = excl + val;
  }
};
template <typename T>
__global__ void k_remap_apply(const T* __restrict__ seq, uint64_t n, const uint32_t* __restrict__ present,
                              const uint32_t* __restrict__ rank, T* __restrict__ out, const int32_t* __restrict__ flag) {
  if (*flag) return;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = (uint64_t)seq[j];
    const uint64_t w = s >> 5;
    out[j] = (T)(rank[w] + (uint32_t)__popc(present[w] & ((1u << (s & 31)) - 1u)));
  }
}
// alphabet[rank] = value: one thread per presence word
__global__ void k_remap_alphabet(const uint32_t* __restrict__ present, const uint32_t* __restrict__ rank,
                                 uint64_t words, uint32_t* __restrict__ alphabet) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= words) return;
  uint32_t x = present[w], r = rank[w];
  while (x) {
    const uint32_t b = (uint32_t)(__ffs(x) - 1);
    x &= x - 1;
    alphabet[r++] = (uint32_t)(32 * w + b);
  }
}

// a scan job that does nothing (count 0)
struct OpNone {
  __device__ uint64_t load(uint64_t) const { return 0; }
  __device__ void store(uint64_t, uint64_t, uint64_t) const {}
};

// Per-tile prefixes: pre[t] = sum_{t' < t} agg[t'] (ones of the level before
// tile t), from the per-tile ones counted by the previous pass.
struct OpTilePrefix {  // (n < 2^32: the prefixes fit 32 bits)
  const uint32_t* agg;
  uint32_t* pre;
  __device__ uint64_t load(uint64_t i) const { return agg[i]; }
  __device__ void store(uint64_t i, uint64_t excl, uint64_t) const { pre[i] = (uint32_t)excl; }
};

// The class-count tile prefixes of a quad pass (wt_quad.cuh): classes 01 and
// 11 of the bit pair (l, l+1) packed in one 64-bit value (each prefix <= n <
// 2^32, so the low half never carries into the high half).
struct OpTilePrefix2 {
  const uint32_t* a01;
  const uint32_t* a11;
  uint32_t* p01;
  uint32_t* p11;
  __device__ uint64_t load(uint64_t i) const { return a01[i] | ((uint64_t)a11[i] << 32); }
  __device__ void store(uint64_t i, uint64_t excl, uint64_t) const {
    p01[i] = (uint32_t)excl;
    p11[i] = (uint32_t)(excl >> 32);
  }
};

// k_triple's node table: per level-(L-3) node the class-01 and class-11
// symbols before it (exclusive scan of the packed class sizes cls[v] = {01,
// 11}; each prefix < 2^32, no carry between the halves).
struct OpNodeCls {
  const uint2* cls;
  uint2* tab3;
  __device__ uint64_t load(uint64_t v) const {
    const uint2 c = cls[v];
    return c.x | ((uint64_t)c.y << 32);
  }
  __device__ void store(uint64_t v, uint64_t excl, uint64_t) const {
    tab3[v] = make_uint2((uint32_t)excl, (uint32_t)(excl >> 32));
  }
};

// Node tables of level l from the sizes of the level-(l+1) nodes
// (cnt[u], u < 2^(l+1); counted by pass l-1, or by the prologue for l = 0:
// cnt1 = ones0, cnt0 = n - ones0).  For level-l node v:
//   left(v) = cnt[2v]                         (its left child)
//   N(v)    = sum_{u < 2v} cnt[u]             (its first position)
//   Zn[v]   = sum_{v' <= v} left(v')          (zeros of level l before node v+1)
//   ob[v]   = N(v) - (Zn[v] - left(v))        (ones of level l before node v)
// One scan over v of the packed pair (left | total << 32); n < 2^32.
struct OpLevelTab {
  const uint32_t* cnt;
  uint2* tab;  // the level's slice: {ob, Zn} (n < 2^32)
  uint64_t n;
  const unsigned long long* ones0;  // non-null for level 0
  __device__ uint64_t load(uint64_t v) const {
    uint64_t l, r;
    if (ones0) {
      r = *ones0;
      l = n - r;
    } else {
      l = cnt[2 * v];
      r = cnt[2 * v + 1];
    }
    return l | ((l + r) << 32);
  }
  __device__ void store(uint64_t v, uint64_t excl, uint64_t val) const {
    const uint64_t left = val & 0xffffffffull;
    const uint64_t zn = (excl & 0xffffffffull) + left, N = excl >> 32;
    tab[v] = make_uint2((uint32_t)(N - (zn - left)), (uint32_t)zn);
  }
};

// Leaf node offsets C[c] = sum_{c' < c} H[c'] (the output), C[2^L] = n, from
// the leaf counts H = sizes of the level-L nodes (counted by pass L-2, or by
// the prologue when L = 1).
struct OpLeafC {
  const uint32_t* cnt;
  unsigned long long* C;
  uint64_t count, n;
  const unsigned long long* ones0;  // non-null when L = 1 (cnt and ones0 null when L = 0)
  __device__ uint64_t load(uint64_t i) const {
    if (ones0) return i ? *ones0 : n - *ones0;  // L = 1
    if (!cnt) return n;                         // L = 0: one leaf
    return cnt[i];
  }
  __device__ void store(uint64_t i, uint64_t excl, uint64_t val) const {
    C[i] = excl;
    if (i + 1 == count) C[count] = excl + val;
  }
};

}  // namespace wt


namespace wt {

// ================================================================ queries

// ones in positions [0, q) of one level (superblock + word popcounts)
__device__ __forceinline__ uint64_t rank1(const uint32_t* __restrict__ B,
                                          const unsigned long long* __restrict__ SB, uint64_t q) {
  const uint64_t t = q >> 9;
  uint64_t r = SB[t];
  const uint32_t wi = (uint32_t)(q >> 5) & 15u, bi = (uint32_t)q & 31u;
  if (wi == 0 && bi == 0) return r;
  const uint32_t* blk = B + 16 * t;
  for (uint32_t w = 0; w < wi; ++w) r += (uint32_t)__popc(blk[w]);
  if (bi) r += (uint32_t)__popc(blk[wi] & ((1u << bi) - 1u));
  return r;
}

// Node offsets C (the output, line 7's exclusive prefix of the leaf counts,
// P:541-543) of a tree whose last pass was the fused pair (k_pairn, k_pair2),
// which counts no leaves.  Level-(L-1) node q = leaf pair (2q, 2q+1) spans
// [s_q, s_{q+1}); its start from the level-(L-2) node table {ob, Zn} of its
// parent v = q >> 1 (the zeros of level L-2 before v's end, Zn[v], plus the
// ones before v, ob[v], for the right child; Zn[v-1] + ob[v] for the left);
// leaf 2q+1's size is the ones of B_{L-1} inside node q (Prop. 1: bit 0).  So
//   C[2q] = s_q,   C[2q+1] = s_{q+1} - (rank1(s_{q+1}) - rank1(s_q)),   C[2^L] = n.
// B_{L-1}'s superblocks must be final.

// ones of one level in [s0, s1): short ranges (the deep trees' small nodes)
// by popcounts of their words, long ones as a rank difference
__device__ __forceinline__ uint64_t ones_between(const uint32_t* __restrict__ B,
                                                 const unsigned long long* __restrict__ SB, uint64_t s0, uint64_t s1) {
  if (s1 <= s0) return 0;
  if (s1 - s0 > 512) return rank1(B, SB, s1) - rank1(B, SB, s0);
  const uint64_t w0 = s0 >> 5, w1 = (s1 - 1) >> 5;  // words holding the first and the last bit
  const uint32_t head = 0xffffffffu << (s0 & 31), tail = 0xffffffffu >> (31 - ((s1 - 1) & 31));
  if (w0 == w1) return (uint32_t)__popc(B[w0] & head & tail);
  uint64_t c = (uint32_t)__popc(B[w0] & head) + (uint32_t)__popc(B[w1] & tail);
  for (uint64_t w = w0 + 1; w < w1; ++w) c += (uint32_t)__popc(B[w]);
  return c;
}

// One thread per level-(L-2) node v: its two children q = 2v, 2v+1 (starts
// s_{2v} = Zn[v-1] + ob[v], s_{2v+1} = Zn[v] + ob[v], s_{2v+2} = Zn[v] + ob[v+1]),
// C[4v .. 4v+3] as two 16-byte stores when C is 16-byte aligned.
__global__ void k_leaf_offsets(const uint2* __restrict__ tab, uint32_t L, const uint32_t* __restrict__ B,
                               const unsigned long long* __restrict__ SB, uint64_t n,
                               unsigned long long* __restrict__ C, const int32_t* __restrict__ flag) {
  pdl_wait();
  if (*flag) return;
  const uint64_t nv = 1ull << (L - 2);
  const bool al16 = (reinterpret_cast<uintptr_t>(C) & 15u) == 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 t = tab[v];
    const uint64_t s0 = (v ? (uint64_t)tab[v - 1].y : 0ull) + t.x;
    const uint64_t s1 = (uint64_t)t.y + t.x;
    const uint64_t s2 = v + 1 < nv ? (uint64_t)t.y + tab[v + 1].x : n;
    const uint64_t c1 = s1 - ones_between(B, SB, s0, s1), c3 = s2 - ones_between(B, SB, s1, s2);
    if (al16) {
      reinterpret_cast<ulonglong2*>(C)[2 * v] = make_ulonglong2(s0, c1);
      reinterpret_cast<ulonglong2*>(C)[2 * v + 1] = make_ulonglong2(s1, c3);
    } else {
      C[4 * v] = s0, C[4 * v + 1] = c1, C[4 * v + 2] = s1, C[4 * v + 3] = c3;
    }
    if (v + 1 == nv) C[4 * nv] = n;
  }
  pdl_trigger();
}

// Node offsets C after k_triple (which counts no leaves): per level-(L-3) node
// v its level-(L-1) nodes q = 4v + c start at N(4v) = s_v, N(4v+1) = s_v +
// size00, N(4v+2) = s_v + zeros_v, N(4v+3) = N(4v+2) + size10, N(4v+4) = the
// next node's start; C[2q] = N(q), C[2q+1] = N(q+1) - (ones of B_{L-1} in
// [N(q), N(q+1))).  B_{L-1}'s superblocks must be final.  One thread per v.
__global__ void k_leaf3(const uint2* __restrict__ tab, const uint2* __restrict__ tab3, const uint2* __restrict__ cls,
                        uint32_t L, const uint32_t* __restrict__ B, const unsigned long long* __restrict__ SB,
                        uint64_t n, unsigned long long* __restrict__ C, const int32_t* __restrict__ flag) {
  pdl_wait();
  if (*flag) return;
  const uint32_t nv = 1u << (L - 3);
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
    const TrNode d = tr_node(tab, tab3, cls, (uint32_t)v, nv, (uint32_t)n);
    const uint64_t sv = (uint64_t)d.zb + d.ob, zv = (uint64_t)d.Zn - d.zb, ov = (uint64_t)d.ob1 - d.ob;
    const uint64_t N[5] = {sv, sv + zv - d.s01, sv + zv, sv + zv + ov - d.s11, sv + zv + ov};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      C[8 * v + 2 * c] = N[c];
      C[8 * v + 2 * c + 1] = N[c + 1] - ones_between(B, SB, N[c], N[c + 1]);
    }
    if (v + 1 == nv) C[8ull * nv] = n;
  }
  pdl_trigger();
}

// out[k] = ones of level lv[k] before position pos[k] (pos <= n): bit-level
// rank of a finished tree (superblock + word popcounts).
__global__ void k_rank1(const uint32_t* __restrict__ bitmaps, const unsigned long long* __restrict__ sb, uint64_t W,
                        uint64_t NSB, const uint32_t* __restrict__ lv, const unsigned long long* __restrict__ pos,
                        uint64_t m, unsigned long long* __restrict__ out) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t l = lv[k];
  out[k] = rank1(bitmaps + l * W, sb + l * NSB, pos[k]);
}

struct TreeView {
  const uint32_t* bitmaps;
  const unsigned long long* sb;
  const unsigned long long* C;
  uint64_t n, W, NSB;
  uint32_t L;
};

__global__ void k_access(TreeView t, const uint64_t* __restrict__ pos, uint64_t m,
                         uint32_t* __restrict__ sym, int32_t* status) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t i = pos[k];
  if (i >= t.n) {
    sym[k] = 0xffffffffu;
    if (status) *status = 3;
    return;
  }
  uint64_t lo = 0, p = i, v = 0;
  for (uint32_t l = 0; l < t.L; ++l) {
    const uint32_t* B = t.bitmaps + l * t.W;
    const unsigned long long* SB = t.sb + l * t.NSB;
    const uint64_t q = lo + p;
    const uint32_t b = (B[q >> 5] >> (q & 31)) & 1u;
    const uint64_t ones_before = rank1(B, SB, q) - rank1(B, SB, lo);
    p = b ? ones_before : p - ones_before;
    v = 2 * v + b;
    lo = t.C[v << (t.L - 1 - l)];
  }
  sym[k] = (uint32_t)v;
}

__global__ void k_rank(TreeView t, uint64_t sigma, const uint32_t* __restrict__ cs,
                       const uint64_t* __restrict__ pos, uint64_t m, unsigned long long* __restrict__ cnt,
                       int32_t* status) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t i = pos[k];
  const uint64_t c = cs[k];
  if (i >= t.n || c >= sigma) {
    cnt[k] = ~0ull;
    if (status) *status = 3;
    return;
  }
  uint64_t lo = 0, r = i + 1;
  for (uint32_t l = 0; l < t.L; ++l) {
    const uint32_t* B = t.bitmaps + l * t.W;
    const unsigned long long* SB = t.sb + l * t.NSB;
    const uint32_t b = (uint32_t)(c >> (t.L - 1 - l)) & 1u;
    const uint64_t ones = rank1(B, SB, lo + r) - rank1(B, SB, lo);
    r = b ? ones : r - ones;
    lo = t.C[(c >> (t.L - 1 - l)) << (t.L - 1 - l)];
  }
  cnt[k] = r;
}

// Wavelet matrix queries (NEXT-4).  Level l partitions the whole sequence by
// bit (L-1-l), zeros first, stably (no nodes); zeros[l] = Z_l.
//   access(i): b = B_l[i]; i = b ? Z_l + rank1_l(i) : i - rank1_l(i)
//   rank(c, i) (inclusive): the prefix [0, i] of S maps to [s, e) per level
__global__ void k_matrix_access(TreeView t, const unsigned long long* __restrict__ zeros,
                                const uint64_t* __restrict__ pos, uint64_t m, uint32_t* __restrict__ sym,
                                int32_t* status) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  uint64_t i = pos[k];
  if (i >= t.n) {
    sym[k] = 0xffffffffu;
    if (status) *status = 3;
    return;
  }
  uint32_t v = 0;
  for (uint32_t l = 0; l < t.L; ++l) {
    const uint32_t* B = t.bitmaps + l * t.W;
    const unsigned long long* SB = t.sb + l * t.NSB;
    const uint32_t b = (B[i >> 5] >> (i & 31)) & 1u;
    const uint64_t r1 = rank1(B, SB, i);
    i = b ? zeros[l] + r1 : i - r1;
    v = 2 * v + b;
  }
  sym[k] = v;
}

__global__ void k_matrix_rank(TreeView t, const unsigned long long* __restrict__ zeros, uint64_t sigma,
                              const uint32_t* __restrict__ cs, const uint64_t* __restrict__ pos, uint64_t m,
                              unsigned long long* __restrict__ cnt, int32_t* status) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t i = pos[k], c = cs[k];
  if (i >= t.n || c >= sigma) {
    cnt[k] = ~0ull;
    if (status) *status = 3;
    return;
  }
  uint64_t s = 0, e = i + 1;  // the symbols equal to c's top bits so far lie in [s, e) of T_l
  for (uint32_t l = 0; l < t.L; ++l) {
    const uint32_t* B = t.bitmaps + l * t.W;
    const unsigned long long* SB = t.sb + l * t.NSB;
    const uint32_t b = (uint32_t)(c >> (t.L - 1 - l)) & 1u;
    const uint64_t rs = rank1(B, SB, s), re = rank1(B, SB, e);
    if (b) s = zeros[l] + rs, e = zeros[l] + re;
    else s = s - rs, e = e - re;
  }
  cnt[k] = e - s;
}

// ---------------------------------------------------------------- domain decomposition merge (NEXT-3)
// The paper's dd: S is split into k contiguous segments,
// each built on its own (the partial trees), then every level's node runs are
// concatenated: node v of level l in the merged tree holds segment 0's run of
// node v, then segment 1's, ... (stability across segments).  With Cg the
// segments' node offsets and C = sum_g Cg, segment g's run of node v goes to
//   C[v << (L-l)] + sum_{g' < g} (Cg'[(v+1) << (L-l)] - Cg'[v << (L-l)])
// (the paper's per-level prefix over segments, Alg. 2 lines 7-8).
// All positions are 64-bit: the merged tree may hold n >= 2^32 symbols.
constexpr int DD_MAX_SEGMENTS = 32;
struct DdOffsets {  // the segments' node offsets (device, 2^L + 1 each)
  const unsigned long long* C[DD_MAX_SEGMENTS];
  uint32_t k, L;
};
// One level's source bits: segment g's local bit p (of that level) is bit
// (p - base[g]) of the words at bits[g]; base[g] is a multiple of 32.  (The
// whole level bitmap of a segment tree: base 0.  A multi-GPU merge: the word
// range of the segment's bitmap received from its rank.)
struct DdLevelSrc {
  const uint32_t* bits[DD_MAX_SEGMENTS];
  unsigned long long base[DD_MAX_SEGMENTS];
};

// Number of segment-g bits of level l whose merged position is < p, for
// p in [0, n]: the node v holding p (the last v with node start <= p), the
// bits of g in nodes < v, plus g's part of node v before p.  `cg(h, i)` reads
// segment h's node offset i.  Shared by the host plan (wt_dd_plan) and the
// device plan kernel -- the same arithmetic on both sides.
template <class CG>
__host__ __device__ inline uint64_t dd_src_before(const CG& cg, uint32_t k, uint32_t L, uint32_t l, uint32_t g,
                                                  uint64_t p) {
  const uint32_t sh = L - l;
  auto cum = [&](uint64_t i) {
    uint64_t s = 0;
    for (uint32_t h = 0; h < k; ++h) s += cg(h, i);
    return s;
  };
  if (p >= cum(1ull << L)) return cg(g, 1ull << L);
  uint64_t lo = 0, hi = 1ull << l;  // cum(lo << sh) <= p < cum(hi << sh)
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (cum(mid << sh) <= p) lo = mid;
    else hi = mid;
  }
  uint64_t off = p - cum(lo << sh), before = 0;
  for (uint32_t h = 0; h < g; ++h) before += cg(h, (lo + 1) << sh) - cg(h, lo << sh);
  const uint64_t a = cg(g, lo << sh), sz = cg(g, (lo + 1) << sh) - a;
  const uint64_t in = off > before ? off - before : 0;
  return a + (in < sz ? in : sz);
}

// The merged tree's blocks are split into `parts` contiguous ranges of whole
// 512-bit blocks (one per rank in a multi-GPU merge): part p owns blocks
// [b_lo, b_hi), i.e. bitmap words [16 b_lo, 16 b_hi) and merged positions
// [min(n, 512 b_lo), min(n, 512 b_hi)).
__host__ __device__ inline void dd_part_blocks(uint64_t n, uint64_t parts, uint64_t p, uint64_t* b_lo,
                                               uint64_t* b_hi) {
  const uint64_t nblk = (n + 511) / 512, per = (nblk + parts - 1) / parts;
  *b_lo = p * per < nblk ? p * per : nblk;
  *b_hi = (p + 1) * per < nblk ? (p + 1) * per : nblk;
}

struct DevCg {  // device accessor of the segments' node offsets
  const DdOffsets* sg;
  __device__ uint64_t operator()(uint32_t h, uint64_t i) const { return sg->C[h][i]; }
};
// plan[((l * parts + p) * k + g) * 2 + {0, 1}] = the source range [lo, hi) of
// segment g's level-l bits that land in part p: one thread per (l, p, g).
__global__ void k_dd_plan(DdOffsets sg, uint64_t n, uint64_t parts, unsigned long long* __restrict__ plan) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t k = sg.k;
  if (t >= (uint64_t)sg.L * parts * k) return;
  const uint32_t g = (uint32_t)(t % k);
  const uint64_t p = (t / k) % parts;
  const uint32_t l = (uint32_t)(t / (k * parts));
  uint64_t b_lo, b_hi;
  dd_part_blocks(n, parts, p, &b_lo, &b_hi);
  const uint64_t q_lo = min(n, 512 * b_lo), q_hi = min(n, 512 * b_hi);
  const DevCg cg{&sg};
  plan[2 * t] = dd_src_before(cg, sg.k, sg.L, l, g, q_lo);
  plan[2 * t + 1] = dd_src_before(cg, sg.k, sg.L, l, g, q_hi);
}

// Destination-driven merge of one level: one thread per DD_WPT consecutive
// words of the merged bitmap, within the word range [w_begin, w_end) (a part;
// out[w - w_begin] receives merged word w).  The thread finds the node v
// holding its first position (binary search over C's level-l node starts) and
// the segment run inside v, then walks the runs (v, 0), (v, 1), ..., (v + 1, 0),
// ... in merged order, funnel-shifting up to 32 source bits at a time into the
// word it assembles; every word is written once with a plain store (no zero
// fill, no atomics: the paper's concat of bit runs, done from the
// destination side), words past n as zeros.  When one run covers the thread's
// whole range (long runs: shallow levels, few segments) the words are a
// funnel-shifted copy with all source loads issued first.  The thread's words
// leave as two 16-byte stores (one L2 request per 4 words: per-word stores of
// 8-word-strided threads made the merge L2-request-bound, 140 -> 49 us per
// cfg2 level).
constexpr uint32_t DD_WPT = 8;     // merged words per thread (two 16-byte stores)
constexpr uint32_t DD_THREADS = 256;
// (flag, optional: a segmented build's range flag; set = the segment trees are
// unspecified, nothing is merged)
__global__ void __launch_bounds__(DD_THREADS) k_dd_merge_level(DdOffsets sg, DdLevelSrc src, uint32_t l,
                                                               const unsigned long long* __restrict__ C, uint64_t n,
                                                               uint64_t w_begin, uint64_t w_end,
                                                               uint32_t* __restrict__ out,
                                                               const int32_t* __restrict__ flag) {
  __shared__ uint32_t sbuf[DD_THREADS * DD_WPT];  // the run walk's words (dynamic index) before the vector stores
  if (flag && *flag) return;
  const uint64_t w0 = w_begin + ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * DD_WPT;
  if (w0 >= w_end) return;
  const uint64_t w1 = min(w0 + DD_WPT, w_end);
  const uint64_t qend = min(32 * w1, n);
  const uint32_t sh = sg.L - l;  // node v of level l spans leaves [v << sh, (v + 1) << sh)
  const uint64_t nodes = 1ull << l;
  uint32_t v8[DD_WPT];  // the thread's words (zero past n)
#pragma unroll
  for (uint32_t i = 0; i < DD_WPT; ++i) v8[i] = 0;
  uint64_t q = 32 * w0;
  if (q < qend) {
    uint64_t v = 0, sp = 0, rem = 0;  // current run: segment h, source positions [sp, sp + rem)
    uint32_t h = 0;
    // (v, h, sp, rem) for merged position q, v searched in [lo, nodes)
    auto enter = [&](uint64_t lo) {
      uint64_t z = nodes;
      while (z - lo > 1) {
        const uint64_t mid = (lo + z) >> 1;
        if (C[mid << sh] <= q) lo = mid;
        else z = mid;
      }
      v = lo;
      uint64_t off = q - C[v << sh];
      for (h = 0;; ++h) {  // q < C[(v + 1) << sh]: some segment holds it
        const uint64_t a = sg.C[h][v << sh], sz = sg.C[h][(v + 1) << sh] - a;
        if (off < sz) {
          sp = a + off;
          rem = sz - off;
          return;
        }
        off -= sz;
      }
    };
    enter(0);
    if (rem >= qend - q) {  // one run: a funnel-shifted copy
      const uint32_t len = (uint32_t)(qend - q);
      const uint32_t* sbits = src.bits[h];
      const uint64_t sw = (sp - src.base[h]) >> 5;
      const uint32_t o = (uint32_t)(sp & 31);
      const uint32_t last = (o + len - 1) >> 5;  // the last source word holding a needed bit
      uint32_t x[DD_WPT + 1];
#pragma unroll
      for (uint32_t i = 0; i <= DD_WPT; ++i) x[i] = i <= last ? sbits[sw + i] : 0u;
#pragma unroll
      for (uint32_t i = 0; i < DD_WPT; ++i) {
        const uint32_t y = __funnelshift_r(x[i], x[i + 1], o);
        v8[i] = 32 * (i + 1) <= len ? y : (32 * i < len ? y & ((1u << (len - 32 * i)) - 1u) : 0u);
      }
    } else {  // the run walk, words into this thread's shared slot
      uint32_t* mine = sbuf + threadIdx.x * DD_WPT;
#pragma unroll
      for (uint32_t i = 0; i < DD_WPT; ++i) mine[i] = 0;
      uint32_t acc = 0;
      for (;;) {
        const uint32_t d = (uint32_t)(q & 31);
        const uint32_t len = (uint32_t)min(min(rem, qend - q), (uint64_t)(32 - d));
        const uint32_t* s = src.bits[h];
        const uint64_t sw = (sp - src.base[h]) >> 5;
        const uint32_t o = (uint32_t)(sp & 31);
        const uint32_t lo_w = s[sw];
        const uint32_t hi_w = (o + len > 32) ? s[sw + 1] : 0u;
        uint32_t x = __funnelshift_r(lo_w, hi_w, o);
        if (len < 32) x &= (1u << len) - 1u;
        acc |= x << d;
        q += len;
        sp += len;
        rem -= len;
        if ((q & 31) == 0) {
          mine[(q >> 5) - 1 - w0] = acc;
          acc = 0;
        }
        if (q >= qend) break;
        if (rem == 0) {  // next non-empty run: later segment of v, else a later node
          uint32_t g = h + 1;
          for (; g < sg.k; ++g) {
            const uint64_t a = sg.C[g][v << sh], sz = sg.C[g][(v + 1) << sh] - a;
            if (sz) {
              h = g;
              sp = a;
              rem = sz;
              break;
            }
          }
          if (g == sg.k) enter(v + 1);
        }
      }
      if (q & 31) mine[(q >> 5) - w0] = acc;  // q == n: the last, partial word
#pragma unroll
      for (uint32_t i = 0; i < DD_WPT; ++i) v8[i] = mine[i];
    }
  }
  uint32_t* dst = out + (w0 - w_begin);
  if (w1 - w0 == DD_WPT && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
    reinterpret_cast<uint4*>(dst)[0] = make_uint4(v8[0], v8[1], v8[2], v8[3]);
    reinterpret_cast<uint4*>(dst)[1] = make_uint4(v8[4], v8[5], v8[6], v8[7]);
  } else {
#pragma unroll
    for (uint32_t i = 0; i < DD_WPT; ++i)
      if (w0 + i < w1) dst[i] = v8[i];
  }
}

// C = sum over the segments' node offsets
__global__ void k_dd_sum_offsets(DdOffsets sg, uint64_t count, unsigned long long* __restrict__ C,
                                 const int32_t* __restrict__ flag) {
  if (flag && *flag) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long s = 0;
    for (uint32_t g = 0; g < sg.k; ++g) s += sg.C[g][i];
    C[i] = s;
  }
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *p = v;
}

// *flag |= *seg_flag (a segmented build accumulates its segments' range flags)
__global__ void k_or_flag(const int32_t* __restrict__ seg_flag, int32_t* __restrict__ flag) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *flag |= *seg_flag;
}

// Select index (NEXT-1; createRankSelect's select half):
// per level and bit value b, the position of every 2^SEL_SHIFT-th bit equal to
// b: samples[l][b][k] = position of the (k * 2^SEL_SHIFT)-th (0-based) such bit;
// entries past the level's count hold n.  One thread per 512-bit block finds
// the multiples of 2^SEL_SHIFT that fall inside its block from SB.
constexpr uint32_t SEL_SHIFT = 12;
__host__ __device__ constexpr uint64_t select_samples_per_level(uint64_t n) { return (n >> SEL_SHIFT) + 2; }

__global__ void k_fill_u32(uint32_t* __restrict__ p, uint64_t count, uint32_t value) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = value;
}

__global__ void k_select_samples_fill(TreeView t, uint32_t* __restrict__ samples) {
  const uint64_t nblk = t.NSB - 1, Q = select_samples_per_level(t.n);
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (uint64_t)t.L * nblk) return;
  const uint32_t l = (uint32_t)(gid / nblk);
  const uint64_t blk = gid % nblk;
  const uint32_t* B = t.bitmaps + (uint64_t)l * t.W + 16 * blk;
  const unsigned long long* SB = t.sb + (uint64_t)l * t.NSB;
  const uint64_t pos0 = blk * 512, len = min((uint64_t)512, t.n - pos0);
  const uint64_t r1 = SB[blk], r0 = pos0 - r1;
  const uint64_t c1 = SB[blk + 1] - r1, c0 = len - c1;
#pragma unroll
  for (uint32_t b = 0; b < 2; ++b) {
    const uint64_t r = b ? r1 : r0, c = b ? c1 : c0;
    const uint64_t S = 1ull << SEL_SHIFT;
    uint64_t k = (r + S - 1) >> SEL_SHIFT;  // first multiple of S at or after rank r
    for (; (k << SEL_SHIFT) < r + c; ++k) {  // (at most one per block: 512 < S)
      uint64_t need = (k << SEL_SHIFT) - r + 1;  // 1-based rank inside the block
      for (uint32_t w = 0; w < 16; ++w) {
        uint32_t word = b ? B[w] : ~B[w];
        if (32 * w + 32 > len) word &= (len > 32 * w) ? ((len - 32 * w >= 32) ? ~0u : ((1u << (len - 32 * w)) - 1u)) : 0u;
        const uint32_t pc = (uint32_t)__popc(word);
        if (need <= pc) {
          for (uint64_t d = 1; d < need; ++d) word &= word - 1;
          samples[((uint64_t)l * 2 + b) * Q + k] = (uint32_t)(pos0 + 32 * w + (uint32_t)(__ffs(word) - 1));
          break;
        }
        need -= pc;
      }
    }
  }
}

// position of the `target`-th (1-based, global) bit equal to b in one level;
// [tlo, thi] brackets the answer's superblock (the whole level without an index)
__device__ uint64_t select_bit(const uint32_t* __restrict__ B, const unsigned long long* __restrict__ SB,
                               uint64_t n, uint64_t nsb, uint32_t b, uint64_t target, uint64_t tlo = 0,
                               uint64_t thi = ~0ull) {
  // rank_b at superblock t
  auto rb = [&](uint64_t t) -> uint64_t {
    const uint64_t ones = SB[t];
    const uint64_t pos = min(t * 512, n);
    return b ? ones : pos - ones;
  };
  // largest t with rb(t) < target
  uint64_t lo = tlo, hi = min(thi, nsb - 1);  // rb(lo) < target <= rb(hi)
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (rb(mid) < target) lo = mid;
    else hi = mid;
  }
  uint64_t need = target - rb(lo);
  const uint32_t* blk = B + 16 * lo;
  for (uint32_t w = 0; w < 16; ++w) {
    uint32_t word = b ? blk[w] : ~blk[w];
    const uint32_t c = (uint32_t)__popc(word);
    if (need <= c) {
      for (uint64_t d = 1; d < need; ++d) word &= word - 1;  // drop need-1 lowest set bits
      return lo * 512 + 32 * w + (uint32_t)(__ffs(word) - 1);
    }
    need -= c;
  }
  return ~0ull;  // unreachable for valid input
}

__global__ void k_select(TreeView t, uint64_t sigma, const uint32_t* __restrict__ cs,
                         const uint64_t* __restrict__ js, uint64_t m, unsigned long long* __restrict__ out,
                         int32_t* status, const uint32_t* __restrict__ samples) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t c = cs[k], j = js[k];
  if (c >= sigma || j == 0 || t.C[c + 1] - t.C[c] < j) {
    out[k] = ~0ull;
    if (status) *status = 3;
    return;
  }
  uint64_t p = j - 1;  // index inside the leaf
  for (uint32_t l = t.L; l-- > 0;) {
    const uint32_t* B = t.bitmaps + l * t.W;
    const unsigned long long* SB = t.sb + l * t.NSB;
    const uint64_t v = c >> (t.L - l);
    const uint64_t lo = t.C[v << (t.L - l)];
    const uint32_t b = (uint32_t)(c >> (t.L - 1 - l)) & 1u;
    const uint64_t before = b ? rank1(B, SB, lo) : lo - rank1(B, SB, lo);
    const uint64_t target = before + p + 1;
    uint64_t tlo = 0, thi = ~0ull;
    if (samples) {  // the sampled positions bracket the target's superblock
      const uint64_t Q = select_samples_per_level(t.n);
      const uint32_t* sm = samples + ((uint64_t)l * 2 + b) * Q;
      const uint64_t kk = (target - 1) >> SEL_SHIFT;
      tlo = sm[kk] / 512;                 // the (kk * 2^s)-th bit is at or before the target
      const uint32_t nx = sm[kk + 1];     // the next sample (or n) is at or after it
      thi = (uint64_t)nx / 512 + 1;
    }
    const uint64_t q = select_bit(B, SB, t.n, t.NSB, b, target, tlo, thi);
    p = q - lo;
  }
  out[k] = p;
}

}  // namespace wt
