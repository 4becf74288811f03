// wt_level.cuh -- a3/a4: the per-level stable segmented bit-partition (sm_100a).
//
// One pass over T_l produces B_l (bitmap words), SB_l (superblocks) and, for
// l < L-1, T_{l+1} = T_l stably partitioned inside every level-l node by bit
// sh = L-1-l (Alg. 1 lines 8-13, with the "C[node]++" cursors
// replaced by closed-form ranks; node of s at level l is s >> (sh+1),
// Proposition 1).  Global destinations, with r(j) the ones of
// level l before position j, ob[v] the ones before node v and Zn[v] the zeros
// before the end of node v (node tables, built from C):
//   b = 0: dest = j - r(j) + ob[v]            b = 1: dest = r(j) + Zn[v]
//
// Execution model (B200-first, not the paper's thread-per-level): barrier-free
// WARP TILES.  Every CTA is one warp, a persistent worker; 20 of them per SM
// run independently (no block barriers to wait on, only __syncwarp).  A warp
// tile is 2 KiB of symbols (2048 / 1024 / 512 for 1 / 2 / 4-byte symbols, a
// multiple of 512 positions: every bitmap word and superblock belongs to one
// tile); every warp takes a contiguous chunk of tiles.  Per warp a ring of 4 buffers:
// tile `it` is TMA-bulk-loaded (cp.async.bulk + mbarrier) into buf[it % 4]
// and its partitioned output is staged in buf[(it-1) % 4], the previous
// tile's input buffer.
//   * NO look-back: the ones of level l in every tile (agg_l[t]) were counted
//     by the pass that wrote T_l (the prologue for l = 0) and a tiny scan
//     (k_prep) turned them into pre_l[t], so the tiles of a pass are independent;
//   * phase A (lane owns 64 consecutive bytes, read in a lane-rotated chunk
//     order against bank conflicts): SWAR bit extraction, bitmap words, warp
//     scan of popcounts -> tile-local rank R(q), superblocks;
//   * ONE-SEGMENT tiles (the whole tile in one node: the common case) take a
//     dedicated path: the zeros go to one run, the ones to another, each
//     staged congruent mod 16 bytes to its HBM destination; the split of each
//     run at its destination tile boundary (for agg_{l+1}) is counted from the
//     staged symbols around the boundary;
//   * MULTI-SEGMENT tiles: a first segment (node vF, may start before the
//     tile), interior nodes (wholly inside the tile: by node locality their
//     destinations are their own positions, an identity region), a last
//     segment (node vL); the first and last segments' runs go to four side
//     regions; a per-tile segment table in shared memory gives each word its
//     stage addresses (global node tables beyond MAXSEG segments);
//   * phase D (word w = lane + 32 k: lanes touch consecutive 32-bit words, so
//     the byte stores are bank-conflict free) writes every symbol to its stage
//     position: u8 words are partitioned by a PRMT from a 16-entry selector
//     table, u16 words store each symbol straight to its slot;
//   * phase E: TMA bulk stores (cp.async.bulk shared->global) of each region's
//     16-byte-aligned body, lane-parallel stores of the edge symbols, and the
//     next level's ones per destination tile as a few global atomics;
//   * MODE 2 (pass L-2 fused with level L-1) writes B_{L-1} instead of T_{L-1}:
//     one-segment tiles compact the last-level bits per lane (no symbol moves)
//     and store the two runs' words from a bit stage (or, with LV_RED, OR
//     each lane's strings straight into B_{L-1}: the L = 2 pass);
//     multi-segment tiles take them from the byte stage;
//   * LV_MATRIX (wavelet matrix): one global node per level, every tile is a
//     one-segment tile.
#pragma once
#include "wt_ptx.cuh"

namespace wt {

// ------------------------------------------------------------ configuration
constexpr int LV_NREG = 5;  // regions: identity, first zeros/ones, last zeros/ones
constexpr int LV_NKEY = 2 * LV_NREG;
constexpr int LV_THREADS = 32;  // one warp per CTA
constexpr uint32_t LV_MATRIX = 0x100;  // k_level `shf` flag: wavelet-matrix level (global partition)
constexpr uint32_t LV_RED = 0x200;     // k_level `shf` flag (MODE 2): B_{L-1} runs as global OR-reductions

template <typename T>
struct LvTile {
  static constexpr int W = (int)sizeof(T);
  static constexpr int E = 64 / W;               // symbols per lane in phase A (64 bytes)
  static constexpr int TILE = 32 * E;            // symbols per warp tile: 2048 / 1024 / 512
  static constexpr int NH = (E + 31) / 32;       // 32-bit mask halves per lane (2 / 1 / 1)
  static constexpr int A = 16 / W;               // symbols per 16-byte chunk
  static constexpr int SPW = 4 / W;              // symbols per 32-bit word
  static constexpr int XW = 16;                  // 32-bit words per lane (phase A and phase D)
  static constexpr int MARGIN = 4 * A;           // side-region slack before/after the tile
  static constexpr int BUF = TILE + 2 * MARGIN;  // ring buffer (symbols)
  static constexpr int NB = 4;                   // ring buffers per warp
  static constexpr int MINB = 20;                // warps (CTAs) per SM the register budget is sized for
  static constexpr int MAXSEG = W == 1 ? 32 : 64;  // segment table capacity (else global node tables)
  static_assert(TILE % 512 == 0, "tiles hold whole superblocks");
  static_assert(NH == 1 || NH == 2, "mask halves");
};

template <typename T>
struct LevelSmem {
  using C = LvTile<T>;
  alignas(128) T buf[C::NB][C::BUF];  // ring: input tiles land at buf[b][MARGIN], outputs are staged
  uint4 own[32 * C::NH];              // lane l, mask half h at [NH l + h] (the NH entries of a lane adjacent:
                                      // phase D's loads of a word round then hit distinct banks):
                                      // {bits, ones before, head bits, heads before}
  uint16_t seg_a[C::MAXSEG + 1];      // segment g starts at tile position seg_a[g] (g >= 1)
  uint16_t seg_R[C::MAXSEG + 1];      // tile-local ones before seg_a[g]
  uint2 kt[C::MAXSEG];                // segment g: shared-memory byte addresses {Z0, O0}: a zero at q with
                                      // R ones before it goes to Z0 + (q - R) W, a one to O0 + R W
  uint2 lut[16];                      // in-word stable partition: {selector | nz << 16 (nz zeros first),
                                      // 2^nz - 1 (the zero slots)}
  uint2 lutp[16];                     // MODE 2 bit compaction: {2^nz, 2^(SPW-nz)} (string position multipliers)
  int32_t s1, am, Rs1, Ram;           // first-segment end, last-segment start, ranks there
  alignas(8) unsigned long long bar[C::NB];
};

template <typename T>
constexpr size_t level_smem_bytes() {
  return sizeof(LevelSmem<T>);
}

// ------------------------------------------------------------ the kernel
// blockDim.x == 32 (one warp per CTA).
// MODE 0: level L-1 (bitmap and superblocks only); MODE 1: level l < L-2,
// also T_{l+1} to `out`; MODE 2: level L-2 fused with level L-1: instead of
// T_{L-1} it writes B_{L-1} (the last level's bits of T_{L-1}, in T_{L-1}
// order) to `out` reinterpreted as uint32 words, which must be zero on entry
// (words shared with other tiles are OR-ed); no next-level tile counts.
template <typename T, int MODE>
__global__ void __launch_bounds__(32, LvTile<T>::MINB)
    k_level(const T* __restrict__ in, T* __restrict__ out, uint32_t n32, uint32_t ntiles, uint32_t shf,
            const uint2* __restrict__ tab, uint32_t* __restrict__ bits, uint32_t words_per_level,
            unsigned long long* __restrict__ sb, uint32_t nsb, const uint32_t* __restrict__ pre,
            uint32_t* __restrict__ agg_next, uint32_t* __restrict__ cnt_next, const int32_t* __restrict__ flag) {
  constexpr bool SCATTER = MODE != 0, BITS = MODE == 2;
  using Cfg = LvTile<T>;
  constexpr int TILE = Cfg::TILE, A = Cfg::A, E = Cfg::E, SPW = Cfg::SPW, XW = Cfg::XW, NH = Cfg::NH;
  constexpr int MARGIN = Cfg::MARGIN, NB = Cfg::NB;
  constexpr uint32_t EM = (E >= 32) ? 0xffffffffu : ((1u << E) - 1u);  // bits of a half that are symbols
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LevelSmem<T>& S = *reinterpret_cast<LevelSmem<T>*>(smem_raw);

  // n < 2^32 (wt_sizes rejects larger n): every position, rank and node
  // offset of the pass fits 32 bits; only pointers are 64-bit.
  const uint32_t lane = threadIdx.x;
  // shf = the level's bit sh, | LV_MATRIX for the wavelet matrix (NEXT-4,
  // P:1409-1413): one global node per level (symbols < 2^30, so s >> 31 = 0)
  // and tab[0] = {0, zeros of the level}; every tile is then a one-segment tile
  const uint32_t sh = shf & 0xffu;
  const uint32_t nsh = (shf & LV_MATRIX) ? 31u : sh + 1;  // node id = symbol >> nsh
  const uint32_t i0 = lane * E;  // first tile position of this lane (phase A)

#ifndef WT_LV_ROUND_ROBIN
  // every warp takes a contiguous chunk of tiles: its tiles mostly stay in one
  // node, so the progressive counts (cc_flush) leave rarely and warps do not
  // meet on the same counters (round-robin tiles put all warps in the same one
  // or two nodes at once: cfg5 levels 7-9 0.51 / 0.49 / 0.45 -> 0.41 ms)
  const uint32_t chunk = (ntiles + gridDim.x - 1) / gridDim.x;
  auto tile_of = [&](uint32_t it) -> uint32_t { return it < chunk ? blockIdx.x * chunk + it : 0xffffffffu; };
#else
  auto tile_of = [&](uint32_t it) -> uint32_t { return blockIdx.x + it * gridDim.x; };
#endif
  auto issue = [&](uint32_t it) {  // lane 0: bulk-copy the warp's it-th tile into buf[it % NB]
    const uint32_t t = tile_of(it);
    if (t >= ntiles) return;
    const int b = (int)(it % NB);
    const uint32_t T0 = t * (uint32_t)TILE;
    const uint32_t len = min((uint32_t)TILE, n32 - T0);
    const uint32_t bytes = (uint32_t)(len * sizeof(T)) & ~15u;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&S.bar[b], bytes);
    if (bytes) bulk_g2s(S.buf[b] + MARGIN, in + T0, bytes, &S.bar[b]);
  };

  if (lane == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&S.bar[b], 1);
    fence_mbar_init();
  }
  // everything above overlaps the predecessor (k_prep): from here on its
  // outputs (tile prefixes, node tables, zeroed counts) and T_l are read
  pdl_wait();
  if (*flag) return;
  if (lane == 0)
    for (int b = 0; b < (SCATTER ? NB - 1 : NB); ++b) issue((uint32_t)b);
  if (SCATTER && lane < 16) {
    const uint32_t e = partition_lut_entry<T>(lane), nz = e >> 16;
    S.lut[lane] = make_uint2(e, (1u << nz) - 1u);
    S.lutp[lane] = make_uint2(1u << nz, 1u << (4 / sizeof(T) - nz));
  }
  __syncwarp();

  // sizes of the level-(l+2) nodes below the node this warp's tiles were in
  // (lane k < 4: node 4 v + k), flushed when the node changes
  uint32_t cc_node = 0xffffffffu, cc_acc = 0;
  auto cc_flush = [&]() {  // lanes 0 and 2 add (k, k+1) pairs with one 64-bit atomic
    const uint32_t hi = __shfl_down_sync(FULL, cc_acc, 1);
    const unsigned long long pair = (unsigned long long)cc_acc | ((unsigned long long)hi << 32);
    if ((lane == 0 || lane == 2) && pair)
      atomicAdd(reinterpret_cast<unsigned long long*>(cnt_next + 4ull * cc_node + lane), pair);
    cc_acc = 0;
  };

  for (uint32_t it = 0;; ++it) {
    const uint32_t tile = tile_of(it);
    if (tile >= ntiles) break;
    const int ib = (int)(it % NB), ob = (int)((it + NB - 1) % NB);
    const uint32_t T0 = tile * (uint32_t)TILE;
    const uint32_t len = min((uint32_t)TILE, n32 - T0);
    const uint32_t P = __ldg(&pre[tile]);  // ones of this level before the tile
    T* const B = S.buf[ib] + MARGIN;                 // tile position q lives at B[q]
    mbar_wait(&S.bar[ib], (it / NB) & 1u);
    if (len < TILE) {  // tail bytes the 16-byte bulk copy did not cover
      const uint32_t done = ((len * (uint32_t)sizeof(T)) & ~15u) / (uint32_t)sizeof(T);
      for (uint32_t i = done + lane; i < len; i += 32) B[i] = in[T0 + i];
      __syncwarp();
    }

    // ---------------- phase A: the lane's 64 bytes -> E bits, bitmap word(s)
    // The lane's four 16-byte chunks are read in a lane-rotated order (slot
    // v holds chunk (v + rot) & 3): lanes 64 bytes apart would otherwise hit
    // the same banks 4-way.  Masks are built in slot order and rotated back.
    constexpr int CS = E / 4;  // symbols per chunk
    // (not for the last level, which is not smem-bound, nor for MODE 2, whose
    // one-segment tiles compact the bits from xw[] in position order)
    const uint32_t rot = (MODE == 1) ? (lane >> 1) & 3u : 0u;
    uint32_t xw[XW];
    {
      const uint4* src = reinterpret_cast<const uint4*>(B + i0);
#pragma unroll
      for (int v = 0; v < XW / 4; ++v) {
        const uint4 q = src[(v + rot) & 3u];
        xw[4 * v] = q.x, xw[4 * v + 1] = q.y, xw[4 * v + 2] = q.z, xw[4 * v + 3] = q.w;
      }
    }
    // slot-order bits (bit CS v + j = symbol j of slot v) -> position order
    auto unrot = [&](uint32_t (&x)[NH]) {
      if constexpr (NH == 2) {  // 64 bits: rotate left by 16 rot
        uint32_t lo = (rot & 2u) ? x[1] : x[0], hi = (rot & 2u) ? x[0] : x[1];
        const uint32_t s16 = (rot & 1u) * 16u;
        x[0] = __funnelshift_l(hi, lo, s16);
        x[1] = __funnelshift_l(lo, hi, s16);
      } else if constexpr (E == 32) {
        x[0] = __funnelshift_l(x[0], x[0], 8u * rot);
      } else {  // E == 16: a 16-bit field
        x[0] = ((x[0] * 0x10001u) >> (16u - 4u * rot)) & 0xffffu;
      }
    };
    const uint32_t nvalid = (i0 >= len) ? 0u : min((uint32_t)E, len - i0);
    uint32_t m[NH], nbm[NH], vm[NH];
    vm[0] = lowmask(min(nvalid, 32u)) & EM;
    if constexpr (NH == 2) vm[NH - 1] = lowmask(nvalid > 32 ? nvalid - 32 : 0u);
    if constexpr (sizeof(T) == 4) {
      // one funnel rotation per symbol serves both masks: rotr(x, sh - k)
      // puts bit sh at k and bit sh-1 at k-1 (mod 32); nbm is accumulated
      // rotated by one and fixed at the end
      uint32_t mm = 0, nn = 0;
#pragma unroll
      for (int k = 0; k < XW; ++k) {
        const uint32_t r = __funnelshift_r(xw[k], xw[k], sh - (uint32_t)k);
        mm |= r & (1u << k);
        if (SCATTER) nn |= r & (1u << ((k + 31) & 31));
      }
      m[0] = mm;
      nbm[0] = SCATTER ? __funnelshift_l(nn, nn, 1) & 0xffffu : 0u;  // next level's bits
    } else {
      // (MODE 2: the next level's bits only on multi-segment tiles, below)
      m[0] = swar_bits<T, XW / NH, 0>(xw, sh);
      nbm[0] = MODE == 1 ? swar_bits<T, XW / NH, 0>(xw, sh - 1) : 0u;  // next level's bits
      if constexpr (NH == 2) {
        m[NH - 1] = swar_bits<T, XW / 2, XW / 2>(xw, sh);
        nbm[NH - 1] = MODE == 1 ? swar_bits<T, XW / 2, XW / 2>(xw, sh - 1) : 0u;
      }
    }
    unrot(m);
    if (SCATTER) unrot(nbm);
#pragma unroll
    for (int h = 0; h < NH; ++h) m[h] &= vm[h], nbm[h] &= vm[h];
    {  // bitmap words (LSB-first)
      const uint32_t gw = (T0 + i0) / 32;
      if constexpr (E == 64) {
        if (gw < words_per_level) *reinterpret_cast<uint2*>(bits + gw) = make_uint2(m[0], m[NH - 1]);
      } else if constexpr (E == 32) {
        if (gw < words_per_level) bits[gw] = m[0];
      } else {  // E == 16: two lanes per word
        const uint32_t w = m[0] | (__shfl_down_sync(FULL, m[0], 1) << 16);
        if ((lane & 1) == 0 && gw < words_per_level) bits[gw] = w;
      }
    }
    uint32_t vF = 0, vL = 0;
    uint2 tabF = make_uint2(0, 0), tabL = make_uint2(0, 0);
    uint32_t hm[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) hm[h] = 0;
    if (SCATTER) {
      vF = (uint32_t)B[0] >> nsh;
      vL = (uint32_t)B[len - 1] >> nsh;
      tabF = __ldg(&tab[vF]);  // issued early: at deep levels these miss L1
      tabL = __ldg(&tab[vL]);
      if (vF != vL) {  // warp-uniform: segment heads (positions q > 0 whose node differs from q-1's)
        // in slot order: the first symbol of slot v follows the last symbol of
        // slot v - 1, or the previous lane's last symbol when it is chunk 0
        const uint32_t pl = lane ? ((uint32_t)B[i0 - 1] >> nsh) : vF;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint32_t prev = (v == (int)((4u - rot) & 3u)) ? pl : (sym_of<T>(xw, ((v + 3) & 3) * CS + CS - 1) >> nsh);
#pragma unroll
          for (int j = 0; j < CS; ++j) {
            const int q = v * CS + j;
            const uint32_t nd = sym_of<T>(xw, q) >> nsh;
            hm[q / 32] |= (nd != prev ? 1u : 0u) << (q % 32);
            prev = nd;
          }
        }
        unrot(hm);
#pragma unroll
        for (int h = 0; h < NH; ++h) hm[h] &= vm[h];
      }
    }
    uint32_t c = 0;  // packed heads << 16 | ones of the lane
#pragma unroll
    for (int h = 0; h < NH; ++h) c += ((uint32_t)__popc(hm[h]) << 16) | (uint32_t)__popc(m[h]);
    const uint32_t incl = warp_incl_scan_u32(c);
    const uint32_t totp = __shfl_sync(FULL, incl, 31);
    const uint32_t prep = incl - c;
    const uint32_t mypre = prep & 0xffffu, hpre = prep >> 16;
    const uint32_t tot = totp & 0xffffu, nseg = (totp >> 16) + 1;
    if ((i0 & 511u) == 0 && T0 + i0 < n32) sb[(T0 + i0) >> 9] = P + mypre;
    // (the last tile by index: T0 + TILE can wrap to 0 when n is within a tile of 2^32)
    if (lane == 0 && tile + 1 == ntiles) sb[nsb - 1] = P + tot;
    if (!SCATTER) {
      __syncwarp();  // every read of this buffer is done
      if (lane == 0) issue(it + NB);
      continue;
    }

    // stage offsets (symbols, relative to the output buffer) -> shared-memory byte addresses
    const int32_t sbuf = (int32_t)(smem_u32(S.buf[ob]) / (uint32_t)sizeof(T));
    auto sa = [&](int32_t K) { return (uint32_t)(sbuf + K) * (uint32_t)sizeof(T); };
    // symbols of a side region with rank < ksplit land in destination tile
    // floor(D / TILE), the rest in the next tile
    auto ksplit = [&](uint32_t D, int32_t l) { return min(l, (int32_t)(TILE - D % TILE)); };
    // ---------------- phase D helpers
    const uint32_t* Win = reinterpret_cast<const uint32_t*>(B);
    // word w = lane + 32 k is owned by phase-A lane w / XW, at symbol offset
    // (w % XW) * SPW = (lane % XW) * SPW of that lane: mask half hh, bit sub
    const uint32_t soff = (lane % (uint32_t)XW) * SPW;
    const uint32_t hh = soff / 32, sub = soff % 32;
    const uint32_t submask = lowmask(sub), subhead = lowmask(sub + 1);
    const uint32_t lutrot = (sub - 3u) & 31u;  // rotr by this puts bits [sub, sub + 4) at [3, 7)
    const uint32_t rot2 = (sub - 1u) & 31u;    // rotr by this puts bits [sub, sub + 2) at [1, 3)
    const uint4* own = S.own + (NH == 1 ? 0 : hh);  // own[NH * owner]
    // (4-byte entries: the 16 entries span 16 banks, one wavefront per word round)
    auto lut_of = [&](uint32_t m4) -> uint2 {
      if constexpr (SPW <= 2) return make_uint2(0, 0);  // (u16 stores without the table)
      else if constexpr (SPW == 4) return make_uint2(S.lut[m4 & 15u].x, 0u);  // (u8: .y unused, 4-byte loads)
      else return S.lut[m4 & ((1u << SPW) - 1u)];
    };
    // stores the SPW symbols of word x (tile position q0, R ones before it,
    // bits m4, in-word partition e) into the segment with byte addresses
    // (Z0, O0) (kt[]).  Slot k of the partitioned word y is a zero iff
    // k < nz: it goes to Az + k, else to Ao + k; the symbol extraction is a
    // multiply-high (FMA pipe).
    auto word_one_segment = [&](uint32_t x, uint32_t q0, uint32_t R, uint32_t m4, uint32_t Z0, uint32_t O0,
                                uint2 e2) {
      if constexpr (SPW == 1) {
        st_shared<T>((m4 & 1u) ? O0 + R * (uint32_t)sizeof(T) : Z0 + (q0 - R) * (uint32_t)sizeof(T), x);
      } else if constexpr (SPW == 2) {  // u16: each symbol straight to its slot (no partition table)
        const uint32_t t = 2u * (m4 & 1u);              // 2 if symbol 0 is a one
        const uint32_t Az = Z0 + (q0 - R) * 2u, Ao = O0 + R * 2u;
        st_shared<T, 0>(t ? Ao : Az, x);
        st_shared<T, 0>((m4 & 2u) ? Ao + t : Az + 2u - t, x >> 16);
      } else {
        const uint32_t e = e2.x;
        uint32_t y;
        asm("prmt.b32 %0, %1, 0, %2;" : "=r"(y) : "r"(x), "r"(e));  // selector = e[15:0]
        const uint32_t nz = e >> 16;
        const uint32_t Az = Z0 + (q0 - R) * (uint32_t)sizeof(T);
        const uint32_t Ao = O0 + (R - nz) * (uint32_t)sizeof(T);
        st_shared<T, 0>(e >= (1u << 16) ? Az : Ao, y);
        st_shared<T, sizeof(T)>(e >= (2u << 16) ? Az : Ao, __umulhi(y, 1u << (32 - 8 * sizeof(T))));
        if constexpr (SPW > 2) {
          st_shared<T, 2>(e >= (3u << 16) ? Az : Ao, __umulhi(y, 1u << 16));
          st_shared<T, 3>(e >= (4u << 16) ? Az : Ao, __umulhi(y, 1u << 8));
        }
      }
    };
    // the symbols of a word that spans segments (or the tile end), one by one
    auto word_split = [&](uint32_t x, uint32_t q0, uint32_t R, uint32_t m4, uint32_t h4, uint32_t nv, auto zo) {
#pragma unroll
      for (int j = 0; j < SPW; ++j) {
        if ((uint32_t)j < nv) {
          const uint32_t sym = sym_in_word<T>(x, j);
          const uint2 k = zo(j, sym, h4);
          const uint32_t Rj = R + (uint32_t)__popc(m4 & lowmask(j));
          st_shared<T>(((m4 >> j) & 1u) ? k.y + Rj * (uint32_t)sizeof(T) : k.x + (q0 + j - Rj) * (uint32_t)sizeof(T),
                       sym);
        }
      }
    };

    // MODE 2: the staged symbols of region [b, b + l) (congruent to HBM
    // position D mod 16 bytes) -> their last-level bits (bit 0) at bit
    // positions [D, D + l) of B_{L-1}.  Global word gw covers stage
    // positions [32 gw - D + b, +32), a 16-byte-aligned window; whole words
    // are stored, words shared with other regions or tiles are OR-ed.
    auto emit_bits = [&](int nreg, const int32_t* rb_, const int32_t* rl_, const uint32_t* rD_) {
      uint32_t* const nbits = reinterpret_cast<uint32_t*>(out);
      uint32_t wb[LV_NREG], cum[LV_NREG + 1];
      cum[0] = 0;
#pragma unroll
      for (int r = 0; r < LV_NREG; ++r) {
        const bool live = r < nreg && rl_[r] > 0;
        wb[r] = rD_[r] / 32u;
        cum[r + 1] = cum[r] + (live ? (rD_[r] + (uint32_t)rl_[r] - 1u) / 32u - wb[r] + 1u : 0u);
      }
      for (uint32_t s0 = 0; s0 < cum[LV_NREG]; s0 += 32) {  // warp-uniform trip count
        const uint32_t s = s0 + lane;
        int r = 0;
#pragma unroll
        for (int k = 1; k < LV_NREG; ++k) r += s >= cum[k] ? 1 : 0;
        int32_t b = rb_[0], l = rl_[0];
        uint32_t D = rD_[0], w0 = wb[0], c0 = cum[0];
#pragma unroll
        for (int k = 1; k < LV_NREG; ++k)
          if (r == k) b = rb_[k], l = rl_[k], D = rD_[k], w0 = wb[k], c0 = cum[k];
        const uint32_t gw = w0 + (s - c0);
        const int32_t p = (int32_t)(32u * gw - D) + b;  // stage position of bit 0 of word gw
        uint32_t word = 0;
        if (s < cum[LV_NREG]) {
          constexpr int CH = 32 * (int)sizeof(T) / 16;  // 16-byte chunks per 32 symbols
          constexpr int PC = 16 / (int)sizeof(T);       // symbols per chunk
          uint32_t xv[4 * CH];
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const int32_t pc = p + PC * c;
            uint4 q = make_uint4(0, 0, 0, 0);
            if (pc + PC > b && pc < b + l) q = *reinterpret_cast<const uint4*>(S.buf[ob] + pc);  // (pc >= 0)
            xv[4 * c] = q.x, xv[4 * c + 1] = q.y, xv[4 * c + 2] = q.z, xv[4 * c + 3] = q.w;
          }
          word = swar_bits<T, 4 * CH, 0>(xv, 0u);
          const int32_t lo = max(b - p, 0), hi = min(b + l - p, 32);  // valid bits [lo, hi)
          const uint32_t msk = lowmask((uint32_t)hi) & ~lowmask((uint32_t)lo);
          word &= msk;
          if (msk == 0xffffffffu) nbits[gw] = word;
          else if (word) atomicOr(&nbits[gw], word);
        }
      }
    };
    if (BITS && nseg == 1) {
      // ================= MODE 2, one segment (node vF): no symbol moves at
      // all.  The last-level bits (bit 0) of the tile's zeros, in order, form
      // the bit run [D0z, D0z + z0) of B_{L-1}, those of its ones the run
      // [D0o, D0o + o0).  Each lane compacts the bits of its E symbols (the
      // in-word partition PRMT of phase D, then a multiply gathers bit 0 of
      // the partitioned symbols), ORs its two strings into a bit stage in the
      // free output buffer, and the warp stores the runs' words (whole words
      // plain, the two boundary words of each run OR-ed: other tiles share them).
      const uint32_t z0 = len - tot, o0 = tot;
      const uint32_t D0z = T0 - P + tabF.x, D0o = P + tabF.y;
      uint32_t nol = 0;
#pragma unroll
      for (int h = 0; h < NH; ++h) nol += (uint32_t)__popc(m[h]);
      const uint32_t nzl = nvalid - nol, rz = i0 - mypre, ro = mypre;
      // compaction: strings of the zeros' / ones' bits, 32 symbols per half
      constexpr int HW = (XW + NH - 1) / NH;  // words per half
      uint32_t Zh[NH], Oh[NH], nzh[NH];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        uint32_t Zs = 0, Os = 0;
        if constexpr (SPW == 1) {
          uint32_t zp = 0, op = 0;
#pragma unroll
          for (int kk = 0; kk < HW; ++kk) {
            const int k = h * HW + kk;
            const uint32_t b = (m[h] >> kk) & 1u, g = xw[k] & 1u;
            Zs |= (b ? 0u : g) << zp;
            Os |= (b ? g : 0u) << op;
            zp += 1u - b;
            op += b;
          }
        } else {
          // the string positions as multipliers (pz = 2^zp, po = 2^op): the
          // appends and position updates are multiply-adds (FMA pipe), the
          // ALU pipe keeps only the table index, PRMT, gather and mask
          uint32_t pz = 1, po = 1;
#pragma unroll
          for (int kk = 0; kk < HW; ++kk) {
            const int k = h * HW + kk;
            const uint32_t m4 = (m[h] >> (SPW * kk)) & ((1u << SPW) - 1u);
            const uint2 ee = S.lut[m4], pp = S.lutp[m4];
            uint32_t y;
            asm("prmt.b32 %0, %1, 0, %2;" : "=r"(y) : "r"(xw[k]), "r"(ee.x));
            uint32_t g;  // bit 0 of the partitioned symbols, slot j at bit j
            if constexpr (SPW == 4) g = ((y & 0x01010101u) * 0x10204080u) >> 28;
            else g = (y & 1u) | ((y >> 15) & 2u);
            Zs += (g & ee.y) * pz;          // disjoint bits: + is |
            Os += (g >> (ee.x >> 16)) * po;
            pz *= pp.x;
            po *= pp.y;
          }
        }
        Zh[h] = Zs, Oh[h] = Os;
        nzh[h] = (uint32_t)(HW * SPW) - (uint32_t)__popc(m[h]);  // (positions past the tile end count as zeros)
      }
      // 64-bit strings (low, high).  Positions past the tile end (m = 0)
      // count as zeros after every valid zero: the zero string is cut to nzl
      uint32_t Z[2], O[2];
      if constexpr (NH == 2) {
        Z[0] = Zh[0] | __funnelshift_lc(0u, Zh[1], nzh[0]);
        Z[1] = __funnelshift_lc(Zh[1], 0u, nzh[0]);
        const uint32_t noh0 = (uint32_t)__popc(m[0]);
        O[0] = Oh[0] | __funnelshift_lc(0u, Oh[1], noh0);
        O[1] = __funnelshift_lc(Oh[1], 0u, noh0);
      } else {
        Z[0] = Zh[0], Z[1] = 0, O[0] = Oh[0], O[1] = 0;
      }
      Z[0] &= lowmask(nzl);
      Z[1] &= lowmask(nzl > 32u ? nzl - 32u : 0u);
      // progressive counting: (b, nb) pair counts of node vF from the strings
      const uint32_t red = __reduce_add_sync(
          FULL, (uint32_t)(__popc(Z[0]) + __popc(Z[1])) | ((uint32_t)(__popc(O[0]) + __popc(O[1])) << 16));
      const uint32_t c01 = red & 0xffffu, c11 = red >> 16;
#ifndef WT_EXP_SKIP_PCOUNT
      if (vF != cc_node) {
        cc_flush();
        cc_node = vF;
      }
      {
        const uint32_t cx = (lane & 2u) ? c11 : c01;
        cc_acc += (lane & 1u) ? cx : ((lane & 2u) ? o0 : z0) - cx;
      }
#endif
      // LV_RED: each lane ORs its two strings (at most three words each) into
      // B_{L-1} with global reductions -- fewer instructions than the stage
      // below, but every touched line of B_{L-1} is read back from HBM for the
      // read-modify-write: the host sets it where the pass is ALU-bound (L = 2)
      if (shf & LV_RED) {
        uint32_t* const nbits = reinterpret_cast<uint32_t*>(out);
        auto red = [&](uint32_t pos, const uint32_t (&v)[2], uint32_t nb) {  // nb bits of v at global bit pos
          if (nb == 0) return;
          const uint32_t j = pos >> 5, off = pos & 31u;
          const uint32_t w0 = v[0] << off;
          const uint32_t w1 = __funnelshift_lc(v[0], v[1], off);
          const uint32_t w2 = __funnelshift_lc(v[1], 0u, off);
          if (w0) atomicOr(&nbits[j], w0);
          if (w1) atomicOr(&nbits[j + 1], w1);
          if (w2) atomicOr(&nbits[j + 2], w2);
        };
        red(D0z + rz, Z, nzl);
        red(D0o + ro, O, nol);
      } else {
        // bit stage in the output buffer: zero-run words [0, WZ), one-run words [WZ, 2 WZ)
        constexpr uint32_t WZ = (TILE / 32 + 2 + 3) & ~3u;  // (a multiple of 4 words: 16-byte zeroing)
        uint32_t* const st = reinterpret_cast<uint32_t*>(S.buf[ob]);
        for (uint32_t j = lane; j < 2 * WZ / 4; j += 32) reinterpret_cast<uint4*>(st)[j] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        auto put = [&](uint32_t base, uint32_t pos, const uint32_t (&v)[2], uint32_t nb) {  // nb bits of v at bit pos
          if (nb == 0) return;
          const uint32_t j = pos >> 5, off = pos & 31u;
          const uint32_t w0 = v[0] << off;
          const uint32_t w1 = __funnelshift_lc(v[0], v[1], off);
          const uint32_t w2 = __funnelshift_lc(v[1], 0u, off);
          if (w0) atomicOr(&st[base + j], w0);
          if (w1) atomicOr(&st[base + j + 1], w1);
          if (w2) atomicOr(&st[base + j + 2], w2);
        };
        put(0, (D0z & 31u) + rz, Z, nzl);
        put(WZ, (D0o & 31u) + ro, O, nol);
        __syncwarp();
        uint32_t* const nbits = reinterpret_cast<uint32_t*>(out);
        // the two runs' words as one lane-parallel list: zero-run words [0, nwz), then one-run words
        const uint32_t nwz = z0 ? ((D0z & 31u) + z0 + 31u) / 32u : 0u;
        const uint32_t nwo = o0 ? ((D0o & 31u) + o0 + 31u) / 32u : 0u;
        for (uint32_t s = lane; s < nwz + nwo; s += 32) {
          const bool one_run = s >= nwz;
          const uint32_t j = one_run ? s - nwz : s, nw = one_run ? nwo : nwz;
          const uint32_t D = one_run ? D0o : D0z, l = one_run ? o0 : z0;
          const uint32_t wv = st[(one_run ? WZ : 0u) + j];
          const bool full = (j > 0 || (D & 31u) == 0) && (j + 1 < nw || ((D + l) & 31u) == 0);
          if (full) nbits[D / 32u + j] = wv;
          else if (wv) atomicOr(&nbits[D / 32u + j], wv);
        }
      }
    } else if (nseg == 1) {
      // ================= one segment: the whole tile lies in node vF.  Zeros
      // go to D0z.., ones to D0o..; staged at b1 / b2 (congruent mod 16 B)
      {
        uint32_t po = mypre;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          *reinterpret_cast<uint2*>(&S.own[NH * lane + h]) = make_uint2(m[h], po);
          po += (uint32_t)__popc(m[h]);
        }
      }
      const uint32_t z0 = len - tot, o0 = tot;
      const uint32_t D0z = T0 - P + tabF.x, D0o = P + tabF.y;  // (mod 2^32; positions < n)
      const uint32_t b1 = D0z & (A - 1);
      const uint32_t b2 = ((b1 + z0 + A - 1) & ~(uint32_t)(A - 1)) + (D0o & (A - 1));
      const uint32_t Z0 = sa((int32_t)b1), O0 = sa((int32_t)b2);
      // next level's ones among the zeros / the ones, and the part of each
      // run below its destination tile boundary (ranks < kz / ko): lanes
      // wholly below count here, the one lane straddling the boundary counts
      // its part in the stage after phase D (window below)
      const uint32_t kz = (uint32_t)ksplit(D0z, (int32_t)z0), ko = (uint32_t)ksplit(D0o, (int32_t)o0);
      uint32_t nol = 0, tbz = 0, tbo = 0;
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        nol += (uint32_t)__popc(m[h]);
        tbz += (uint32_t)__popc(nbm[h] & ~m[h]);
        tbo += (uint32_t)__popc(nbm[h] & m[h]);
      }
      const uint32_t nzl = nvalid - nol, rz = i0 - mypre, ro = mypre;
      const uint32_t redz = __reduce_add_sync(FULL, ((rz + nzl <= kz) ? tbz : 0u) | (tbz << 16));
      const uint32_t redo = __reduce_add_sync(FULL, ((ro + nol <= ko) ? tbo : 0u) | (tbo << 16));
      const uint32_t c01 = redz >> 16, c11 = redo >> 16;
      uint32_t Lz = redz & 0xffffu, Lo = redo & 0xffffu;
      const uint32_t splz = __ballot_sync(FULL, rz < kz && rz + nzl > kz);
      const uint32_t splo = __ballot_sync(FULL, ro < ko && ro + nol > ko);
      const uint32_t sz0 = __shfl_sync(FULL, rz, (__ffs(splz) - 1) & 31);
      const uint32_t so0 = __shfl_sync(FULL, ro, (__ffs(splo) - 1) & 31);
#ifndef WT_EXP_SKIP_PCOUNT
      // progressive counting: the (b, nb) pair counts of node vF are the run
      // sizes and their next-level ones
      if (vF != cc_node) {
        cc_flush();
        cc_node = vF;
      }
      {  // lane k < 4 adds count k = {00, 01, 10, 11}; lanes >= 4 hold don't-cares (cc_flush reads lanes 0..3)
        const uint32_t cx = (lane & 2u) ? c11 : c01;
        cc_acc += (lane & 1u) ? cx : ((lane & 2u) ? o0 : z0) - cx;
      }
#endif
      __syncwarp();  // own[]
#ifndef WT_EXP_SKIP_D
      if (len == (uint32_t)TILE) {  // warp-uniform: full tile
        // batches of BK words: the batch's shared loads first (independent), then its stores
        constexpr int BK = sizeof(T) == 2 ? 4 : 8;  // (measured: u8, u32 8; u16 4)
#pragma unroll
        for (int k0 = 0; k0 < XW; k0 += BK) {
          uint32_t xs[BK], Rs[BK], ms[BK];
          uint2 es[BK];
#pragma unroll
          for (int k = 0; k < BK; ++k) {
            const uint32_t w = lane + 32 * (k0 + k);
            const uint2 ow = *reinterpret_cast<const uint2*>(&own[NH * (w / XW)]);
            xs[k] = Win[w];
            Rs[k] = ow.y + (uint32_t)__popc(ow.x & submask);
            ms[k] = SPW == 1 ? ow.x >> sub : ow.x;  // (u8, u16: rotated at use)
          }
#pragma unroll
          for (int k = 0; k < BK; ++k) {
            if constexpr (SPW == 4) {  // (u8) entry byte offset m4 * 8 by one funnel rotation of the bits
              const uint32_t o8 = __funnelshift_r(ms[k], ms[k], lutrot) & 0x78u;
              es[k] = make_uint2(*reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(S.lut) + o8), 0u);
            } else {
              es[k] = lut_of(ms[k]);
            }
          }
#pragma unroll
          for (int k = 0; k < BK; ++k) {
            if constexpr (SPW == 2) {
              // u16: one rotation brings both symbols' bits to bits 1 and 2
              // (bit 1 = 2 if symbol 0 is a one); Az / Ao are symbol 0's zero /
              // one slots, symbol 1 goes 2 bytes after the slot of its kind
              // minus what symbol 0 took
              const uint32_t r = __funnelshift_r(ms[k], ms[k], rot2), t = r & 2u;
              const uint32_t q0 = (lane + 32 * (k0 + k)) * 2u;
              const uint32_t Az = Z0 + 2u * q0 - 2u * Rs[k], Ao = O0 + 2u * Rs[k];
              st_shared<T, 0>(t ? Ao : Az, xs[k]);
              st_shared<T, 0>((r & 4u) ? Ao + t : Az + 2u - t, xs[k] >> 16);
            } else {
              word_one_segment(xs[k], (lane + 32 * (k0 + k)) * SPW, Rs[k], ms[k], Z0, O0, es[k]);
            }
          }
        }
      } else {  // the last, partial tile
        const uint2 kF = make_uint2(Z0, O0);
#pragma unroll
        for (int k = 0; k < XW; ++k) {
          const uint32_t w = lane + 32 * k;
          const uint32_t q0 = w * SPW;
          if (q0 >= len) break;
          const uint2 ow = *reinterpret_cast<const uint2*>(&own[NH * (w / XW)]);
          const uint32_t R = ow.y + (uint32_t)__popc(ow.x & submask);
          const uint32_t m4 = ow.x >> sub;
          const uint32_t x = Win[w];
          const uint32_t nv = min((uint32_t)SPW, len - q0);
          if (nv == (uint32_t)SPW) word_one_segment(x, q0, R, m4, Z0, O0, lut_of(m4));
          else word_split(x, q0, R, m4, 0u, nv, [&](int, uint32_t, uint32_t) { return kF; });
        }
      }
#endif
      fence_proxy_async_smem();
      __syncwarp();  // stage written (and the input buffer fully read)
      // the straddling lane's symbols below the boundary: stage positions
      // [bst + r0, bst + k), fewer than E, their next-level bits counted here
      auto window = [&](uint32_t bst, uint32_t r0, uint32_t k) {
        const int32_t lo = (int32_t)(bst + r0), hi = (int32_t)(bst + k);
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < (E + 31) / 32; ++j) {
          const int32_t q = hi - E + 32 * j + (int32_t)lane;
          const bool in = q >= lo && q < hi;
          const uint32_t sym = in ? (uint32_t)S.buf[ob][q] : 0u;
          c += (uint32_t)__popc(__ballot_sync(FULL, (sym >> (sh - 1)) & 1u));
        }
        return c;
      };
      if constexpr (BITS) {  // the two runs' last-level bits
        const int32_t rb2[2] = {(int32_t)b1, (int32_t)b2}, rl2[2] = {(int32_t)z0, (int32_t)o0};
        const uint32_t rD2[2] = {D0z, D0o};
        emit_bits(2, rb2, rl2, rD2);
      } else {
      if (splz) Lz += window(b1, sz0, kz);
      if (splo) Lo += window(b2, so0, ko);
      // ---------------- phase E: lanes 0 / 1 bulk-store the two runs' aligned
      // bodies, the warp stores their edge symbols
      {
        const bool r2 = lane == 1;
        const uint32_t b = r2 ? b2 : b1, l = r2 ? o0 : z0, D = r2 ? D0o : D0z;
        const uint32_t fs = (b + A - 1) & ~(uint32_t)(A - 1), fe = (b + l) & ~(uint32_t)(A - 1);
        if (lane < 2 && fe > fs) bulk_s2g(out + (D - b + fs), S.buf[ob] + fs, (fe - fs) * (uint32_t)sizeof(T));
        bulk_commit();  // every lane (empty groups too): no divergence
#pragma unroll
        for (uint32_t base = 0; base < (uint32_t)(4 * A); base += 32) {
          const uint32_t slot = base + lane, e = slot % (2 * A);
          const bool s2 = slot >= (uint32_t)(2 * A);
          const uint32_t bb = s2 ? b2 : b1, end = bb + (s2 ? o0 : z0), DD = s2 ? D0o : D0z;
          const uint32_t hend = min((bb + A - 1) & ~(uint32_t)(A - 1), end);
          const uint32_t tst = max(end & ~(uint32_t)(A - 1), hend);
          const uint32_t q = e < (uint32_t)A ? bb + e : tst + e - A;
          if (slot < (uint32_t)(4 * A) && (e < (uint32_t)A ? q < hend : q < end)) out[DD - bb + q] = S.buf[ob][q];
        }
      }
      {  // next-level ones per destination tile: lanes 0..3, one predicated reduction (no branch)
        const uint32_t cx = (lane & 2u) ? c11 : c01, lx = (lane & 2u) ? Lo : Lz;
        const uint32_t v = lane < 4 ? ((lane & 1u) ? cx - lx : lx) : 0u;
        const uint32_t dt = ((lane & 2u) ? D0o : D0z) / TILE + (lane & 1u);
        if (v) atomicAdd(&agg_next[dt], v);
      }
      }  // !BITS
    } else {
      // ================= several segments
      if constexpr (MODE == 2 && sizeof(T) != 4) {  // the next level's bits (phase A skipped them)
        nbm[0] = swar_bits<T, XW / NH, 0>(xw, sh - 1) & vm[0];
        if constexpr (NH == 2) nbm[NH - 1] = swar_bits<T, XW / 2, XW / 2>(xw, sh - 1) & vm[NH - 1];
      }

      {
        uint32_t po = mypre, ph = hpre;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          S.own[NH * lane + h] = make_uint4(m[h], po, hm[h], ph);
          po += (uint32_t)__popc(m[h]);
          ph += (uint32_t)__popc(hm[h]);
        }
      }
      {  // segment table: start and rank of every segment g >= 1
        uint32_t g = hpre + 1;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          uint32_t hh = hm[h];
          while (hh) {
            const uint32_t k = 32 * h + (uint32_t)(__ffs(hh) - 1);
            hh &= hh - 1;
            uint32_t Rk = mypre + (uint32_t)__popc(m[h] & lowmask(k % 32));
            if (h == 1) Rk += (uint32_t)__popc(m[0]);
            if (g <= (uint32_t)Cfg::MAXSEG) {
              S.seg_a[g] = (uint16_t)(i0 + k);
              S.seg_R[g] = (uint16_t)Rk;
            }
            if (g == 1) {
              S.s1 = (int32_t)(i0 + k);
              S.Rs1 = (int32_t)Rk;
            }
            if (g == nseg - 1) {
              S.am = (int32_t)(i0 + k);
              S.Ram = (int32_t)Rk;
            }
            ++g;
          }
        }
      }
      __syncwarp();  // own[], segment table

      // ---------------- constants of the tile's regions (every lane; lane r keeps region r)
      const bool segtab = nseg <= (uint32_t)Cfg::MAXSEG;  // warp-uniform
      const int32_t s1 = S.s1, am = S.am, Rs1 = S.Rs1, Ram = S.Ram;
      const int32_t z0 = s1 - Rs1, o0 = Rs1;
      const int32_t om = (int32_t)tot - Ram, zm = ((int32_t)len - am) - om;
      // HBM destinations (mod 2^32 arithmetic; the results are positions < n)
      const uint32_t D0z = T0 - P + tabF.x;
      const uint32_t D0o = P + tabF.y;
      const uint32_t Dmz = T0 + (uint32_t)am - P - (uint32_t)Ram + tabL.x;
      const uint32_t Dmo = P + (uint32_t)Ram + tabL.y;
      auto rup = [](int32_t x) { return (x + A - 1) / A * A; };
      const int32_t b1 = (int32_t)(D0z & (A - 1));
      const int32_t b2 = rup(b1 + z0) + (int32_t)(D0o & (A - 1));
      const int32_t b3 = rup(MARGIN + am) + (int32_t)(Dmz & (A - 1));
      const int32_t b4 = rup(b3 + zm) + (int32_t)(Dmo & (A - 1));
      const int32_t K0F = b1, K1F = b2, K0L = b3 - am + Ram, K1L = b4 - Ram;
      // the five regions (warp-uniform): identity, first zeros, first ones, last zeros, last ones
      const int32_t rb[LV_NREG] = {MARGIN + s1, b1, b2, b3, b4};
      const int32_t rl[LV_NREG] = {am - s1, z0, o0, zm, om};
      const uint32_t rD[LV_NREG] = {T0 + (uint32_t)s1, D0z, D0o, Dmz, Dmo};  // HBM destination of rb[r]
      // symbols of side region r with rank < ksplit_r land in destination tile
      // floor(D_r / TILE), the rest in the next tile
      if (segtab) {
        if (lane == 0) S.kt[0] = make_uint2(sa(K0F), sa(K1F));
        if (lane == 1) S.kt[nseg - 1] = make_uint2(sa(K0L), sa(K1L));
        // interior segment g (1 <= g <= nseg-2) lies wholly inside the tile: its
        // stage positions are its own positions, zeros first then ones:
        //   b = 0: q - R(q) + R(a_g) + MARGIN     b = 1: R(q) + a_{g+1} - R(a_{g+1}) + MARGIN
        for (uint32_t g = lane + 1; g + 1 < nseg; g += 32)
          S.kt[g] = make_uint2(sa((int32_t)S.seg_R[g] + MARGIN),
                               sa((int32_t)S.seg_a[g + 1] - (int32_t)S.seg_R[g + 1] + MARGIN));
      }

      // ---------------- next-level ones per (region, destination tile), lane-owned symbols
      uint32_t mycnt = 0;  // lane k < LV_NKEY: count of key k = 2 r + half
#ifndef WT_EXP_SKIP_COUNT
      if constexpr (!BITS) {
        // count of nbm bits among the set bits of M, split at rank k (the set
        // bits of M have ranks rank0, rank0+1, ... in position order).  Only
        // the lane holding rank k searches for its k-th set bit.
        auto split = [&](const uint32_t(&M)[NH], int32_t rank0, int32_t k, uint32_t& lo, uint32_t& hi) {
          if constexpr (NH == 2) {
            const uint64_t M64 = M[0] | ((uint64_t)M[1] << 32), N64 = nbm[0] | ((uint64_t)nbm[1] << 32);
            const uint32_t tot = (uint32_t)__popcll(N64 & M64);
            const int32_t nM = __popcll(M64);
            if (rank0 + nM <= k) lo = tot;
            else if (rank0 >= k) lo = 0;
            else {  // lowest (k - rank0) set bits of M
              const int32_t j = k - rank0;
              uint32_t p = 0;
#pragma unroll
              for (uint32_t st = 32; st; st >>= 1)
                if (__popcll(M64 & ((1ull << (p + st)) - 1)) <= j) p += st;
              lo = (uint32_t)__popcll(N64 & M64 & ((1ull << p) - 1));
            }
            hi = tot - lo;
          } else {
            const uint32_t tot = (uint32_t)__popc(nbm[0] & M[0]);
            const int32_t nM = __popc(M[0]);
            if (rank0 + nM <= k) lo = tot;
            else if (rank0 >= k) lo = 0;
            else {
              const int32_t j = k - rank0;
              uint32_t p = 0;
#pragma unroll
              for (uint32_t st = 16; st; st >>= 1)
                if (__popc(M[0] & ((1u << (p + st)) - 1)) <= j) p += st;
              lo = (uint32_t)__popc(nbm[0] & M[0] & ((1u << p) - 1));
            }
            hi = tot - lo;
          }
        };
        auto put2 = [&](int key, uint32_t lo, uint32_t hi) {  // keys (key, key+1) in one reduction
          const uint32_t sum = __reduce_add_sync(FULL, lo | (hi << 16));
          if (lane == (uint32_t)key) mycnt = sum & 0xffffu;
          if (lane == (uint32_t)key + 1) mycnt = sum >> 16;
        };
        uint32_t M[NH], lo, hi;
        {
          uint32_t fm[NH], lm[NH];
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            fm[h] = lowmask((uint32_t)min(max(s1 - (int32_t)i0 - 32 * h, 0), 32)) & vm[h];
            lm[h] = vm[h] & ~lowmask((uint32_t)min(max(am - (int32_t)i0 - 32 * h, 0), 32));
          }
          uint32_t c0 = 0;
#pragma unroll
          for (int h = 0; h < NH; ++h) c0 += (uint32_t)__popc(nbm[h] & vm[h] & ~fm[h] & ~lm[h]);
          put2(0, c0, 0u);
#pragma unroll
          for (int h = 0; h < NH; ++h) M[h] = fm[h] & ~m[h];
          split(M, (int32_t)(i0 - mypre), ksplit(D0z, z0), lo, hi);
          put2(2, lo, hi);
#pragma unroll
          for (int h = 0; h < NH; ++h) M[h] = fm[h] & m[h];
          split(M, (int32_t)mypre, ksplit(D0o, o0), lo, hi);
          put2(4, lo, hi);
          const int32_t qs = max((int32_t)i0, am);
          const int32_t Rq = ((int32_t)i0 < am) ? Ram : (int32_t)mypre;  // tile-local ones before qs
#pragma unroll
          for (int h = 0; h < NH; ++h) M[h] = lm[h] & ~m[h];
          split(M, (qs - am) - (Rq - Ram), ksplit(Dmz, zm), lo, hi);
          put2(6, lo, hi);
#pragma unroll
          for (int h = 0; h < NH; ++h) M[h] = lm[h] & m[h];
          split(M, Rq - Ram, ksplit(Dmo, om), lo, hi);
          put2(8, lo, hi);
        }
      }
#endif
      // ---------------- progressive counting: level-(l+2) node sizes, i.e. the
      // symbols of each level-l node by their (level-l, level-(l+1)) bit pair
#ifndef WT_EXP_SKIP_PCOUNT
      if (nvalid) {  // the lane's pieces: maximal runs of its symbols inside one node
        // (two node counts per 64-bit atomic: each stays < 2^32, no carry)
        auto piece = [&](uint32_t node, uint32_t c00, uint32_t c01, uint32_t c10, uint32_t c11) {
          unsigned long long* dst = reinterpret_cast<unsigned long long*>(cnt_next + 4u * node);
          const unsigned long long lo = (unsigned long long)c00 | ((unsigned long long)c01 << 32);
          const unsigned long long hi = (unsigned long long)c10 | ((unsigned long long)c11 << 32);
          if (lo) atomicAdd(dst, lo);
          if (hi) atomicAdd(dst + 1, hi);
        };
        if constexpr (NH == 2) {
          const uint64_t M = m[0] | ((uint64_t)m[1] << 32), NB = nbm[0] | ((uint64_t)nbm[1] << 32);
          const uint64_t V = vm[0] | ((uint64_t)vm[1] << 32), H = hm[0] | ((uint64_t)hm[1] << 32);
          uint64_t starts = (H | 1ull) & V;
          while (starts) {
            const int p = __ffsll((long long)starts) - 1;
            starts &= starts - 1;
            const int pend = starts ? __ffsll((long long)starts) - 1 : 64;
            const uint64_t pm = V & ((pend >= 64 ? ~0ull : ((1ull << pend) - 1)) & ~((1ull << p) - 1));
            const uint64_t z = pm & ~M, o = pm & M;
            piece((uint32_t)B[i0 + p] >> nsh, __popcll(z & ~NB), __popcll(z & NB), __popcll(o & ~NB),
                  __popcll(o & NB));
          }
        } else {
          const uint32_t M = m[0], NB = nbm[0], V = vm[0];
          uint32_t starts = (hm[0] | 1u) & V;
          while (starts) {
            const int p = __ffs(starts) - 1;
            starts &= starts - 1;
            const int pend = starts ? __ffs(starts) - 1 : 32;
            const uint32_t pm = V & lowmask((uint32_t)pend) & ~((1u << p) - 1u);
            const uint32_t z = pm & ~M, o = pm & M;
            piece((uint32_t)B[i0 + p] >> nsh, __popc(z & ~NB), __popc(z & NB), __popc(o & ~NB), __popc(o & NB));
          }
        }
      }
#endif
      if (segtab) __syncwarp();  // kt[]

      // ---------------- phase D: every symbol from the input buffer to its stage position
#ifndef WT_EXP_SKIP_D
      {
        if (segtab) {  // segment table in shared memory
          const uint32_t kt_base = smem_u32(S.kt);
          // word w = lane + 32 k: segment g of its first symbol, stage by kt[g]
          auto seg_word = [&](int k, bool check) {
            const uint32_t w = lane + 32 * k;
            const uint32_t q0 = w * SPW;
            const uint4 ow = own[NH * (w / XW)];
            const uint32_t R = ow.y + (uint32_t)__popc(ow.x & submask);
            uint32_t g = ow.w + (uint32_t)__popc(ow.z & subhead);  // segment of the word's first symbol
            const uint32_t m4 = ow.x >> sub;
            const uint32_t x = Win[w];
            if constexpr (SPW == 1) {
              const uint2 kk = ld_shared_u2(kt_base + 8u * g);
              word_one_segment(x, q0, R, m4, kk.x, kk.y, make_uint2(0, 0));
            } else {
              const uint32_t h4 = (ow.z >> sub) & ((1u << SPW) - 2u);  // heads inside the word
              const uint32_t nv = check ? min((uint32_t)SPW, len - q0) : (uint32_t)SPW;
              if (nv == (uint32_t)SPW && h4 == 0) {
                const uint2 kk = ld_shared_u2(kt_base + 8u * g);
                word_one_segment(x, q0, R, m4, kk.x, kk.y, lut_of(m4));
              } else {
                word_split(x, q0, R, m4, h4, nv, [&](int j, uint32_t, uint32_t h) {
                  g += (h >> j) & 1u;
                  return ld_shared_u2(kt_base + 8u * g);
                });
              }
            }
          };
          if (SPW == 1 && len == (uint32_t)TILE) {  // warp-uniform; batches of BK words, loads first
            constexpr int BK = 4;
#pragma unroll
            for (int k0 = 0; k0 < XW; k0 += BK) {
              uint32_t xs[BK], Rs[BK], gs[BK], bs[BK];
              uint2 ks[BK];
#pragma unroll
              for (int k = 0; k < BK; ++k) {
                const uint32_t w = lane + 32 * (k0 + k);
                const uint4 ow = own[NH * (w / XW)];
                xs[k] = Win[w];
                Rs[k] = ow.y + (uint32_t)__popc(ow.x & submask);
                gs[k] = ow.w + (uint32_t)__popc(ow.z & subhead);
                bs[k] = (ow.x >> sub) & 1u;
              }
#pragma unroll
              for (int k = 0; k < BK; ++k) ks[k] = ld_shared_u2(kt_base + 8u * gs[k]);
#pragma unroll
              for (int k = 0; k < BK; ++k)
                word_one_segment(xs[k], lane + 32 * (k0 + k), Rs[k], bs[k], ks[k].x, ks[k].y, make_uint2(0, 0));
            }
          } else if (len == (uint32_t)TILE) {
#pragma unroll
            for (int k = 0; k < XW; ++k) seg_word(k, false);
          } else {
#pragma unroll
            for (int k = 0; k < XW; ++k) {
              if ((lane + 32 * k) * SPW >= len) break;
              seg_word(k, true);
            }
          }
        } else {  // too many segments for the table: node tables from global memory
          auto consts = [&](uint32_t v) -> uint2 {
            if (v == vF) return make_uint2(sa(K0F), sa(K1F));
            if (v == vL) return make_uint2(sa(K0L), sa(K1L));
            // interior node: stage position = HBM destination - T0 + MARGIN
            const uint2 t = __ldg(&tab[v]);
            return make_uint2(sa((int32_t)(t.x - P) + MARGIN), sa((int32_t)(t.y + P - T0) + MARGIN));
          };
#pragma unroll
          for (int k = 0; k < XW; ++k) {
            const uint32_t w = lane + 32 * k;
            const uint32_t q0 = w * SPW;
            if (q0 >= len) break;
            const uint4 ow = own[NH * (w / XW)];
            const uint32_t R = ow.y + (uint32_t)__popc(ow.x & submask);
            const uint32_t m4 = ow.x >> sub;
            const uint32_t h4 = SPW == 1 ? 0u : (ow.z >> sub) & ((1u << SPW) - 2u);
            const uint32_t x = Win[w];
            const uint32_t nv = min((uint32_t)SPW, len - q0);
            if (nv == (uint32_t)SPW && h4 == 0) {
              const uint2 kk = consts(sym_in_word<T>(x, 0) >> nsh);
              word_one_segment(x, q0, R, m4, kk.x, kk.y, lut_of(m4));
            } else {
              word_split(x, q0, R, m4, h4, nv, [&](int, uint32_t sym, uint32_t) { return consts(sym >> nsh); });
            }
          }
        }
      }
#endif
      fence_proxy_async_smem();
      __syncwarp();  // stage partitioned (and the input buffer fully read)
      if constexpr (BITS) {
        emit_bits(LV_NREG, rb, rl, rD);
      } else {
      // ---------------- phase E: TMA bulk stores of the aligned bodies, element stores of the edges
      auto emit_region = [&](int32_t b, int32_t l, uint32_t D) {  // stage [b, b+l) -> HBM [D, D+l)
        if (l <= 0) return;  // warp-uniform
        const int32_t end = b + l;
        const int32_t fs = (b + A - 1) / A * A, fe = end / A * A;
        T* const go = out + D - b;  // HBM address of stage position q: go + q
        if (lane == 0 && fe > fs) bulk_s2g(go + fs, S.buf[ob] + fs, (uint32_t)(fe - fs) * (uint32_t)sizeof(T));
        // head edge [b, min(fs, end)) and tail edge [max(fe, that), end), each < A symbols
        const int32_t hend = min(fs, end), tst = max(fe, hend);
        const int32_t q = (lane < (uint32_t)A) ? b + (int32_t)lane : tst + (int32_t)lane - A;
        if (lane < (uint32_t)(2 * A) && ((lane < (uint32_t)A) ? (q < hend) : (q < end))) go[q] = S.buf[ob][q];
      };
      if constexpr (sizeof(T) == 1) {  // (A = 16: one region's two edges fill the warp)
#pragma unroll
        for (int r = 0; r < LV_NREG; ++r) emit_region(rb[r], rl[r], rD[r]);
        bulk_commit();  // every lane commits (empty groups too): a uniform wait below, no divergence
      } else {
        // lane r < LV_NREG: region r's bulk store; then all regions' edge
        // symbols (<= 2A each) as one lane-parallel list of slots
        const uint32_t r_ = min(lane, (uint32_t)(LV_NREG - 1));
        int32_t b = rb[0], l = rl[0];
        uint32_t D = rD[0];
#pragma unroll
        for (int k = 1; k < LV_NREG; ++k)
          if (r_ == (uint32_t)k) b = rb[k], l = rl[k], D = rD[k];
        if (lane >= (uint32_t)LV_NREG) l = 0;
        const int32_t end = b + l, fs = (b + A - 1) / A * A, fe = end / A * A;
        const uint32_t Dmb = D - (uint32_t)b;  // HBM position of stage position q: Dmb + q
        if (l > 0 && fe > fs) bulk_s2g(out + (Dmb + (uint32_t)fs), S.buf[ob] + fs, (uint32_t)(fe - fs) * (uint32_t)sizeof(T));
        bulk_commit();  // every lane (empty groups too): no divergence
        const int32_t hend = l > 0 ? min(fs, end) : b, tst = max(fe, hend), endv = l > 0 ? end : b;
#pragma unroll
        for (uint32_t base = 0; base < (uint32_t)(2 * A * LV_NREG); base += 32) {
          const uint32_t slot = base + lane;
          const int rs = (int)min(slot / (2 * A), (uint32_t)(LV_NREG - 1));
          const uint32_t e = slot % (2 * A);
          const int32_t b_ = __shfl_sync(FULL, b, rs), hend_ = __shfl_sync(FULL, hend, rs);
          const int32_t tst_ = __shfl_sync(FULL, tst, rs), end_ = __shfl_sync(FULL, endv, rs);
          const uint32_t Dmb_ = __shfl_sync(FULL, Dmb, rs);
          const int32_t q = (e < (uint32_t)A) ? b_ + (int32_t)e : tst_ + (int32_t)e - A;
          if (slot < (uint32_t)(2 * A * LV_NREG) && ((e < (uint32_t)A) ? (q < hend_) : (q < end_)))
            out[Dmb_ + (uint32_t)q] = S.buf[ob][q];
        }
      }
      if (lane < (uint32_t)LV_NKEY && mycnt) {  // next-level ones per destination tile
        const int r = (int)(lane >> 1);
        uint32_t D = r == 1 ? D0z : D0o;
        D = r == 3 ? Dmz : r == 4 ? Dmo : D;
        atomicAdd(&agg_next[r == 0 ? tile : D / TILE + (lane & 1)], mycnt);
      }
      }  // !BITS
    }
    // the previous tile's output buffer: once its bulk stores have read it, load a new tile into it
    bulk_wait_read<1>();  // each lane waits for its own groups (lanes without bulk stores: empty)
    __syncwarp();
    if (lane == 0 && it >= 1) issue(it + NB - 2);
  }
  pdl_trigger();  // (at the tail: the next launch's CTAs do not crowd the pass)
  if (SCATTER) {
    cc_flush();
    bulk_wait<0>();
  }
}

}  // namespace wt
