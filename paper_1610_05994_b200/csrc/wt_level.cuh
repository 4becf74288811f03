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
// Execution model (B200-first, not the paper's thread-per-level):
//   * persistent CTAs of 256 threads, several per SM; tiles of 8 KiB of
//     symbols (a multiple of 512 positions: every bitmap word and superblock
//     belongs to one tile), assigned round-robin; LV_STAGES tiles in flight per
//     CTA with cp.async.bulk (TMA bulk copy) into shared memory on mbarriers;
//   * NO look-back: the ones of level l in every tile (agg_l[t]) were counted by
//     the pass that wrote T_l (the histogram pass for l = 0) and a tiny scan
//     turned them into pre_l[t], so the tiles of a pass are independent;
//   * phase A/B (thread owns 32 consecutive bytes): SWAR bit extraction, the
//     bitmap word(s), warp + block scan of popcounts -> tile-local rank R(q),
//     superblocks SB[t] = r(512 t);
//   * the tile's symbols are partitioned IN PLACE in the shared stage buffer.
//     Nodes are sorted along T_l, so the tile is: a first segment (node vF,
//     may start before the tile), interior nodes (wholly inside the tile, so
//     by node locality their destinations are exactly their own positions:
//     an identity region), and a last segment (node vL, may run past the
//     tile).  Interior symbols go to (dest - T0); the first and last
//     segments' zeros/ones runs go to four side regions, each staged at an
//     offset congruent to its HBM destination modulo 16 bytes;
//   * phase D (thread handles 8 words, word w = tid + 256 k: lanes touch
//     consecutive 32-bit words, so the byte stores are bank-conflict free)
//     writes every symbol to its stage position;
//   * phase E: one thread issues <= 5 TMA bulk stores (cp.async.bulk
//     shared->global) for the 16-byte-aligned body of each region; threads
//     store the <= 10 partial edge chunks and count, per destination tile, the
//     next level's bit of the written symbols (agg_{l+1}), aggregated in
//     shared memory and flushed with <= 10 global atomics per tile.
#pragma once
#include "wt_device.cuh"

namespace wt {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------ configuration
constexpr int LV_THREADS = 256;
constexpr int LV_WARPS = LV_THREADS / 32;
constexpr int LV_NREG = 5;    // regions: identity, first zeros/ones, last zeros/ones
constexpr int LV_NKEY = 2 * LV_NREG;

template <typename T>
struct LvTile {
  static constexpr int W = (int)sizeof(T);
  static constexpr int E = (W == 4) ? 16 : 32;     // symbols per thread in phase A
  static constexpr int TILE = LV_THREADS * E;      // symbols per tile: 8192 / 8192 / 4096
  static constexpr int A = 16 / W;                 // symbols per 16-byte chunk
  static constexpr int SPW = 4 / W;                // symbols per 32-bit word
  static constexpr int XW = E * W / 4;             // 32-bit words per phase-A thread (8 / 16 / 16)
  static constexpr int WPT = TILE / SPW / LV_THREADS;  // words per thread in phase D (== XW)
  static constexpr int TPW = 32 / E;               // threads per bitmap word (1, 1, 2)
  static constexpr int MARGIN = 4 * A;             // side-region slack before/after the tile
  static constexpr int BUF = TILE + 2 * MARGIN;    // ring buffer (symbols)
  static constexpr int NB = (W == 1) ? 5 : 4;      // ring buffers per CTA
  static constexpr int MINB = (W == 1) ? 4 : 3;    // CTAs per SM the register budget is sized for
  // segment table capacity (u8 scatter levels have <= 64 nodes); tiles with
  // more segments look the node tables up in global memory instead
  static constexpr int MAXSEG = (W == 1) ? 128 : 512;
  static_assert(TILE % 512 == 0, "tiles hold whole superblocks");
  static_assert(WPT == XW && LV_THREADS % XW == 0, "phase D word / owner layout");
};

template <typename T>
struct LevelSmem {
  using C = LvTile<T>;
  alignas(128) T buf[C::NB][C::BUF];      // ring: input tiles land at buf[b][MARGIN], outputs are staged
  uint4 own[LV_THREADS];                  // per phase-A thread: {bit mask, ones | heads << 16 before, head mask, -}
  uint16_t seg_a[C::MAXSEG + 1];          // segment g starts at tile position seg_a[g] (g >= 1)
  uint16_t seg_R[C::MAXSEG + 1];          // tile-local ones before seg_a[g]
  short2 kt[C::MAXSEG];                   // segment g: stage offsets {K0, K1} relative to the output buffer
  uint32_t lut[16];                       // in-word stable partition selectors (partition_lut_entry)
  uint32_t warp_tot[LV_WARPS];
  int32_t s1, am, Rs1, Ram;               // first-segment end, last-segment start, ranks there
  int32_t K[4];                           // K0F, K1F, K0L, K1L (relative to the output buffer, in symbols)
  int32_t rbase[LV_NREG], rlen[LV_NREG], ksplit[LV_NREG];
  long long gofs[LV_NREG];                // HBM position of stage position q: q + gofs[r]
  unsigned long long dtile[LV_NKEY];      // destination tile of each (region, half) key
  uint32_t cnt[LV_NKEY];                  // next-level ones per key
  alignas(8) unsigned long long bar[C::NB];
};

template <typename T>
constexpr size_t level_smem_bytes() {
  return sizeof(LevelSmem<T>);
}

// ------------------------------------------------------------ SWAR helpers
template <typename T>
__device__ __forceinline__ uint32_t bitmask32(uint32_t bit) {  // `bit` of every symbol packed in a 32-bit word
  if (sizeof(T) == 1) return 0x01010101u << bit;
  if (sizeof(T) == 2) return 0x00010001u << bit;
  return 1u << bit;
}

// bit `sh` of the symbols held in xw[NW] (little-endian), symbol k -> bit k.
template <typename T, int NW>
__device__ __forceinline__ uint32_t swar_bits(const uint32_t (&xw)[NW], uint32_t sh) {
  uint32_t m = 0;
  if (sizeof(T) == 1) {
    // gather bit sh of the 4 bytes of a word with one multiply:
    // (x & 0x01010101<<sh) * (1 + 2^7 + 2^14 + 2^21) puts byte j's bit at 21+sh+j
    const uint32_t msk = 0x01010101u << sh;
#pragma unroll
    for (int k = 0; k < NW; ++k) m |= ((((xw[k] & msk) * 0x00204081u) >> (21 + sh)) & 0xfu) << (4 * k);
  } else if (sizeof(T) == 2) {
    const uint32_t msk = 0x00010001u << sh;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const uint32_t t = xw[k] & msk;
      m |= (((t >> sh) | (t >> (sh + 15))) & 3u) << (2 * k);
    }
  } else {
#pragma unroll
    for (int k = 0; k < NW; ++k) m |= ((xw[k] >> sh) & 1u) << k;
  }
  return m;
}

template <typename T, int NW>
__device__ __forceinline__ uint32_t sym_of(const uint32_t (&xw)[NW], int k) {
  if (sizeof(T) == 1) return (xw[k >> 2] >> (8 * (k & 3))) & 0xffu;
  if (sizeof(T) == 2) return (xw[k >> 1] >> (16 * (k & 1))) & 0xffffu;
  return xw[k];
}

// st.shared of the low sizeof(T) bytes of v at shared byte address a + OFF
template <typename T, int OFF = 0>
__device__ __forceinline__ void st_shared(uint32_t a, uint32_t v) {
  if (sizeof(T) == 1) asm volatile("st.shared.u8 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF));
  else if (sizeof(T) == 2) asm volatile("st.shared.u16 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF));
  else asm volatile("st.shared.u32 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF));
}

// Stable in-word partition of the SPW symbols of a 32-bit word by their bits
// (bit j of `bits` = bit of symbol j): a PRMT selector that moves the zero
// symbols to the low end (in order) and the one symbols after them (in
// order), plus the number of zeros in bits 16..18.
template <typename T>
__host__ __device__ constexpr uint32_t partition_lut_entry(uint32_t bits) {
  uint32_t sel = 0, k = 0, nz = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (uint32_t j = 0; j < 4 / sizeof(T); ++j)
      if (((bits >> j) & 1u) == (uint32_t)pass) {
        for (uint32_t byte = 0; byte < sizeof(T); ++byte) sel |= (j * sizeof(T) + byte) << (4 * (k * sizeof(T) + byte));
        ++k;
        nz += pass == 0;
      }
  return sel | (nz << 16);
}

template <typename T>
__device__ __forceinline__ uint32_t sym_in_word(uint32_t x, int j) {
  if (sizeof(T) == 1) return (x >> (8 * j)) & 0xffu;
  if (sizeof(T) == 2) return (x >> (16 * j)) & 0xffffu;
  return x;
}

__device__ __forceinline__ uint32_t lowmask(uint32_t k) { return k >= 32 ? 0xffffffffu : ((1u << k) - 1u); }

// ------------------------------------------------------------ the kernel
template <typename T, bool SCATTER>
__global__ void __launch_bounds__(LV_THREADS, LvTile<T>::MINB)
    k_level(const T* __restrict__ in, T* __restrict__ out, uint64_t n, uint32_t sh,
            const ulonglong2* __restrict__ tab, uint32_t* __restrict__ bits, uint64_t words_per_level,
            unsigned long long* __restrict__ sb, uint64_t nsb, const unsigned long long* __restrict__ pre,
            uint32_t* __restrict__ agg_next, const int32_t* __restrict__ flag) {
  using Cfg = LvTile<T>;
  constexpr int TILE = Cfg::TILE, A = Cfg::A, E = Cfg::E, TPW = Cfg::TPW, SPW = Cfg::SPW, WPT = Cfg::WPT;
  constexpr int MARGIN = Cfg::MARGIN, NB = Cfg::NB, XW = Cfg::XW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LevelSmem<T>& S = *reinterpret_cast<LevelSmem<T>*>(smem_raw);

  if (*flag) return;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t nsh = sh + 1;  // node id = symbol >> nsh
  const uint32_t i0 = tid * E;  // first tile position of this thread (phase A)

  // Ring of NB buffers: tile `it` (the CTA's it-th) is loaded into buf[it % NB];
  // with SCATTER its partitioned output is staged in buf[(it - 1) % NB] (the
  // previous tile's input, free once that tile's phase D is done), whose
  // bulk stores are read-complete one iteration later, when the buffer is
  // refilled.  Without SCATTER every buffer is an input stage.
  auto tile_of = [&](uint32_t it) -> uint64_t { return (uint64_t)blockIdx.x + (uint64_t)it * gridDim.x; };
  auto issue = [&](uint32_t it) {  // thread 0: bulk-copy the CTA's it-th tile into buf[it % NB]
    const uint64_t t = tile_of(it);
    if (t >= ntiles) return;
    const int b = (int)(it % NB);
    const uint64_t T0 = t * (uint64_t)TILE;
    const uint64_t len = min((uint64_t)TILE, n - T0);
    const uint32_t bytes = (uint32_t)(len * sizeof(T)) & ~15u;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&S.bar[b], bytes);
    if (bytes) bulk_g2s(S.buf[b] + MARGIN, in + T0, bytes, &S.bar[b]);
  };

  if (tid == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&S.bar[b], 1);
    fence_mbar_init();
    for (int b = 0; b < (SCATTER ? NB - 1 : NB); ++b) issue((uint32_t)b);
  }
  if (SCATTER && tid < LV_NKEY) S.cnt[tid] = 0;
  if (SCATTER && tid < 16) S.lut[tid] = partition_lut_entry<T>(tid);
  __syncthreads();

  for (uint32_t it = 0;; ++it) {
    const uint64_t tile = tile_of(it);
    if (tile >= ntiles) break;
    const int ib = (int)(it % NB), ob = (int)((it + NB - 1) % NB);
    const uint64_t T0 = tile * (uint64_t)TILE;
    const uint32_t len = (uint32_t)min((uint64_t)TILE, n - T0);
    const unsigned long long P = __ldg(&pre[tile]);  // ones of this level before the tile
    T* const B = S.buf[ib] + MARGIN;                 // tile position q lives at B[q]
    mbar_wait(&S.bar[ib], (it / NB) & 1u);
    if (len < TILE) {  // tail bytes the 16-byte bulk copy did not cover
      const uint32_t done = ((len * (uint32_t)sizeof(T)) & ~15u) / (uint32_t)sizeof(T);
      for (uint32_t i = done + tid; i < len; i += LV_THREADS) B[i] = in[T0 + i];
      __syncthreads();
    }

    // ---------------- phase A: the thread's E symbols -> E bits, bitmap word(s)
    uint32_t vF = 0, vL = 0;
    if (SCATTER) {
      vF = (uint32_t)B[0] >> nsh;
      vL = (uint32_t)B[len - 1] >> nsh;
    }
    uint32_t xw[XW];
    {
      const uint4* src = reinterpret_cast<const uint4*>(B + i0);
#pragma unroll
      for (int v = 0; v < XW / 4; ++v) {
        const uint4 q = src[v];
        xw[4 * v] = q.x, xw[4 * v + 1] = q.y, xw[4 * v + 2] = q.z, xw[4 * v + 3] = q.w;
      }
    }
    const uint32_t nvalid = (i0 >= len) ? 0u : min((uint32_t)E, len - i0);
    const uint32_t vmask = lowmask(nvalid);
    const uint32_t m = swar_bits<T>(xw, sh) & vmask;
    const uint32_t nbm = SCATTER ? (swar_bits<T>(xw, sh - 1) & vmask) : 0u;  // next level's bits
    {
      uint32_t w = m;
      if (TPW > 1) {
        w = m << (E * (lane % TPW));
#pragma unroll
        for (int o = 1; o < TPW; o <<= 1) w |= __shfl_xor_sync(FULL, w, o);
      }
      const uint64_t gw = (T0 + i0) / 32;
      if ((lane % TPW) == 0 && gw < words_per_level) bits[gw] = w;
    }
    // segment heads: positions q > 0 of the tile whose node differs from q-1's
    uint32_t hm = 0;
    if (SCATTER && vF != vL) {  // block-uniform
      uint32_t prev = tid ? ((uint32_t)B[i0 - 1] >> nsh) : vF;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const uint32_t nd = sym_of<T>(xw, q) >> nsh;
        hm |= (nd != prev ? 1u : 0u) << q;
        prev = nd;
      }
      hm &= vmask;
    }
    const uint32_t c = ((uint32_t)__popc(hm) << 16) | (uint32_t)__popc(m);  // packed heads | ones
    const uint32_t incl = warp_incl_scan_u32(c);
    if (lane == 31) S.warp_tot[warp] = incl;
    ulonglong2 tabF = make_ulonglong2(0, 0), tabL = make_ulonglong2(0, 0);
    if (SCATTER && warp == 0) {
      tabF = __ldg(&tab[vF]);
      tabL = __ldg(&tab[vL]);
    }
    __syncthreads();  // B1: warp totals

    if (!SCATTER) {
      if (tid == 0) issue(it + NB);  // every read of this buffer is done
    } else if (tid < LV_NKEY) {      // flush the previous tile's next-level counts
      const uint32_t v = S.cnt[tid];
      if (v) {
        atomicAdd(&agg_next[S.dtile[tid]], v);
        S.cnt[tid] = 0;
      }
    }
    // block prefix: every warp scans the LV_WARPS warp totals itself
    uint32_t wpre, totp;
    {
      const uint32_t wt = (lane < (uint32_t)LV_WARPS) ? S.warp_tot[lane] : 0u;
      const uint32_t wi = warp_incl_scan_u32(wt);
      wpre = __shfl_sync(FULL, wi - wt, warp);
      totp = __shfl_sync(FULL, wi, LV_WARPS - 1);
    }
    const uint32_t prep = wpre + incl - c;
    const uint32_t mypre = prep & 0xffffu, hpre = prep >> 16;
    const uint32_t tot = totp & 0xffffu, nseg = (totp >> 16) + 1;
    if ((i0 & 511u) == 0 && T0 + i0 < n) sb[(T0 + i0) >> 9] = P + mypre;
    if (tid == 0 && T0 + TILE >= n) sb[nsb - 1] = P + tot;
    if (!SCATTER) continue;

    S.own[tid] = make_uint4(m, prep, hm, 0u);
    {  // segment table: start and rank of every segment g >= 1
      uint32_t h = hm, g = hpre + 1;
      while (h) {
        const uint32_t k = (uint32_t)(__ffs(h) - 1);
        h &= h - 1;
        const int32_t a_ = (int32_t)(i0 + k), R_ = (int32_t)(mypre + __popc(m & lowmask(k)));
        if (g <= (uint32_t)Cfg::MAXSEG) {
          S.seg_a[g] = (uint16_t)a_;
          S.seg_R[g] = (uint16_t)R_;
        }
        if (g == 1) {
          S.s1 = a_;
          S.Rs1 = R_;
        }
        if (g == nseg - 1) {
          S.am = a_;
          S.Ram = R_;
        }
        ++g;
      }
    }
    __syncthreads();  // B2: own[], segment table

    const bool segtab = nseg <= (uint32_t)Cfg::MAXSEG;  // block-uniform
    // ---------------- constants of the tile's regions (warp 0, lane r writes region r)
    if (warp == 0) {
      const bool one = (nseg == 1);
      const int32_t s1 = one ? (int32_t)len : S.s1, am = one ? (int32_t)len : S.am;
      const int32_t Rs1 = one ? (int32_t)tot : S.Rs1, Ram = one ? (int32_t)tot : S.Ram;
      const int32_t z0 = s1 - Rs1, o0 = Rs1;
      const int32_t om = (int32_t)tot - Ram, zm = ((int32_t)len - am) - om;
      const long long D0z = (long long)T0 - (long long)P + (long long)tabF.x;
      const long long D0o = (long long)P + (long long)tabF.y;
      const long long Dmz = (long long)T0 + am - (long long)P - Ram + (long long)tabL.x;
      const long long Dmo = (long long)P + Ram + (long long)tabL.y;
      auto rup = [](int32_t x) { return (x + A - 1) / A * A; };
      const int32_t b1 = (int32_t)(D0z & (A - 1));
      const int32_t b2 = rup(b1 + z0) + (int32_t)(D0o & (A - 1));
      const int32_t b3 = rup(MARGIN + am) + (int32_t)(Dmz & (A - 1));
      const int32_t b4 = rup(b3 + zm) + (int32_t)(Dmo & (A - 1));
      const int32_t K0L = b3 - am + Ram, K1L = b4 - Ram;
      if (lane < 4) S.K[lane] = lane == 0 ? b1 : lane == 1 ? b2 : lane == 2 ? K0L : K1L;
      if (segtab) {
        if (lane == 0) S.kt[0] = make_short2((short)b1, (short)b2);
        if (lane == 1 && !one) S.kt[nseg - 1] = make_short2((short)K0L, (short)K1L);
      }
      if (lane == 5) {
        S.s1 = s1;
        S.am = am;
        S.Ram = Ram;
      }
      if (lane < (uint32_t)LV_NREG) {
        const int r = (int)lane;
        const int32_t base = r == 0 ? MARGIN + s1 : r == 1 ? b1 : r == 2 ? b2 : r == 3 ? b3 : b4;
        const int32_t rl = r == 0 ? am - s1 : r == 1 ? z0 : r == 2 ? o0 : r == 3 ? zm : om;
        const long long D = r == 0 ? (long long)T0 + s1 : r == 1 ? D0z : r == 2 ? D0o : r == 3 ? Dmz : Dmo;
        S.rbase[r] = base;
        S.rlen[r] = rl;
        S.gofs[r] = D - base;  // HBM destination of stage position q: q + gofs
        const unsigned long long t0 = (unsigned long long)D / TILE;
        S.dtile[2 * r] = (r == 0) ? tile : t0;
        S.dtile[2 * r + 1] = t0 + 1;
        // region symbols with rank < ksplit land in destination tile t0, the rest in t0 + 1
        S.ksplit[r] = (r == 0) ? 0x7fffffff : (int32_t)min((long long)rl, (long long)(t0 + 1) * TILE - D);
      }
    } else if (segtab) {
      // interior segment g (1 <= g <= nseg-2) lies wholly inside the tile: its
      // stage positions are its own positions, zeros first then ones:
      //   b = 0: q - R(q) + R(a_g) + MARGIN     b = 1: R(q) + a_{g+1} - R(a_{g+1}) + MARGIN
      for (uint32_t g = tid - 31; g + 1 < nseg; g += LV_THREADS - 32)
        S.kt[g] = make_short2((short)(S.seg_R[g] + MARGIN), (short)(S.seg_a[g + 1] - S.seg_R[g + 1] + MARGIN));
    }
    __syncthreads();  // B3: constants

    // ---------------- next-level ones per (region, destination tile), thread-owned symbols
    {
      // count of nbm bits among the set bits of M, split at rank k (the set
      // bits of M have ranks rank0, rank0+1, ... in position order)
      auto split = [&](uint32_t M, int32_t rank0, int32_t k, uint32_t& lo, uint32_t& hi) {
        const int32_t nM = __popc(M);
        uint32_t Mlo;
        if (rank0 + nM <= k) Mlo = M;
        else if (rank0 >= k) Mlo = 0;
        else {  // the one thread per region holding the split: lowest (k - rank0) set bits of M
          const int32_t j = k - rank0;
          uint32_t p = 0;
#pragma unroll
          for (uint32_t st = 16; st; st >>= 1)
            if (__popc(M & lowmask(p + st)) <= j) p += st;
          Mlo = M & lowmask(p);
        }
        lo = (uint32_t)__popc(nbm & Mlo);
        hi = (uint32_t)__popc(nbm & M & ~Mlo);
      };
      uint32_t cnt[LV_NKEY];
      if (nseg == 1) {  // block-uniform: one segment, only the first-segment runs
        split(vmask & ~m, (int32_t)(i0 - mypre), S.ksplit[1], cnt[2], cnt[3]);
        split(m, (int32_t)mypre, S.ksplit[2], cnt[4], cnt[5]);
#pragma unroll
        for (int key = 2; key < 6; ++key) {
          const uint32_t sum = __reduce_add_sync(FULL, cnt[key]);
          if (lane == 0 && sum) atomicAdd(&S.cnt[key], sum);
        }
      } else {
        const int32_t s1 = S.s1, am = S.am, Ram = S.Ram;
        const uint32_t fm = lowmask((uint32_t)min(max(s1 - (int32_t)i0, 0), E));           // first segment
        const uint32_t lm = vmask & ~lowmask((uint32_t)min(max(am - (int32_t)i0, 0), E));  // last segment
        const uint32_t im = vmask & ~fm & ~lm;                                             // interior
        cnt[0] = (uint32_t)__popc(nbm & im);
        cnt[1] = 0;
        split(fm & ~m, (int32_t)(i0 - mypre), S.ksplit[1], cnt[2], cnt[3]);
        split(fm & m, (int32_t)mypre, S.ksplit[2], cnt[4], cnt[5]);
        const int32_t qs = max((int32_t)i0, am);
        const int32_t Rq = ((int32_t)i0 >= am) ? (int32_t)mypre : Ram;
        split(lm & ~m, (qs - am) - (Rq - Ram), S.ksplit[3], cnt[6], cnt[7]);
        split(lm & m, Rq - Ram, S.ksplit[4], cnt[8], cnt[9]);
#pragma unroll
        for (int key = 0; key < LV_NKEY; ++key) {
          if (key == 1) continue;
          if (key > 1 && S.rlen[key >> 1] == 0) continue;  // block-uniform
          const uint32_t sum = __reduce_add_sync(FULL, cnt[key]);
          if (lane == 0 && sum) atomicAdd(&S.cnt[key], sum);
        }
      }
    }

    // ---------------- phase D: every symbol from the input buffer to its stage position
    {
      const int32_t sbuf = (int32_t)(smem_u32(S.buf[ob]) / (uint32_t)sizeof(T));  // in symbols
      const uint32_t* Win = reinterpret_cast<const uint32_t*>(B);
      const uint32_t sub = (tid % (uint32_t)XW) * SPW;  // word w = tid + 256 k: owner w / XW, offset (w % XW) * SPW
      const uint32_t submask = lowmask(sub), subhead = lowmask(sub + 1);
      // stores the SPW symbols of word x (tile position q0, R ones before it,
      // bits m4) into segment (K0, K1) (stage offsets relative to the buffer)
      auto lut_of = [&](uint32_t m4) -> uint32_t { return SPW == 1 ? 0u : S.lut[m4 & ((1u << SPW) - 1u)]; };
      auto word_one_segment = [&](uint32_t x, uint32_t q0, uint32_t R, uint32_t m4, int32_t K0, int32_t K1,
                                  uint32_t e) {
        const int32_t az = sbuf + (int32_t)(q0 - R) + K0;
        if (SPW == 1) {
          st_shared<T>((uint32_t)((m4 & 1u) ? sbuf + (int32_t)R + K1 : az) * (uint32_t)sizeof(T), x);
        } else {
          const uint32_t y = __byte_perm(x, 0u, e);
          const int32_t nz = (int32_t)(e >> 16);
          const int32_t a1 = sbuf + (int32_t)R + K1 - nz;  // the ones go to a1 + k for k >= nz
          const uint32_t A0 = (uint32_t)az * (uint32_t)sizeof(T), A1 = (uint32_t)a1 * (uint32_t)sizeof(T);
          st_shared<T, 0>(nz > 0 ? A0 : A1, y);
          if (SPW > 1) st_shared<T, sizeof(T)>(nz > 1 ? A0 : A1, y >> (8 * sizeof(T)));
          if (SPW > 2) {
            st_shared<T, 2 * sizeof(T)>(nz > 2 ? A0 : A1, y >> 16);
            st_shared<T, 3 * sizeof(T)>(nz > 3 ? A0 : A1, y >> 24);
          }
        }
      };
      if (nseg == 1 && len == (uint32_t)TILE) {  // block-uniform: one segment, full tile
        const int32_t K0F = S.K[0], K1F = S.K[1];
        // all shared loads first (independent), then the stores
        uint32_t xs[WPT], Rs[WPT], ms[WPT], es[WPT];
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
          const uint32_t w = tid + LV_THREADS * k;
          const uint2 ow = *reinterpret_cast<const uint2*>(&S.own[w / XW]);
          xs[k] = Win[w];
          Rs[k] = (ow.y & 0xffffu) + (uint32_t)__popc(ow.x & submask);
          ms[k] = ow.x >> sub;
        }
#pragma unroll
        for (int k = 0; k < WPT; ++k) es[k] = lut_of(ms[k]);
#pragma unroll
        for (int k = 0; k < WPT; ++k)
          word_one_segment(xs[k], (tid + LV_THREADS * k) * SPW, Rs[k], ms[k], K0F, K1F, es[k]);
      } else if (segtab) {  // segment table in shared memory
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
          const uint32_t w = tid + LV_THREADS * k;
          const uint32_t q0 = w * SPW;
          if (q0 >= len) break;
          const uint4 ow = S.own[w / XW];
          const uint32_t R = (ow.y & 0xffffu) + (uint32_t)__popc(ow.x & submask);
          uint32_t g = (ow.y >> 16) + (uint32_t)__popc(ow.z & subhead);  // segment of the word's first symbol
          const uint32_t m4 = ow.x >> sub;
          const uint32_t h4 = (ow.z >> sub) & ((1u << SPW) - 2u);         // heads inside the word
          const uint32_t x = Win[w];
          const uint32_t nv = min((uint32_t)SPW, len - q0);
          if (nv == (uint32_t)SPW && h4 == 0) {
            const short2 kk = S.kt[g];
            word_one_segment(x, q0, R, m4, kk.x, kk.y, lut_of(m4));
          } else {
#pragma unroll
            for (int j = 0; j < SPW; ++j) {
              if ((uint32_t)j < nv) {
                g += (h4 >> j) & 1u;
                const short2 kk = S.kt[g];
                const uint32_t Rj = R + (uint32_t)__popc(m4 & lowmask(j));
                const uint32_t b = (m4 >> j) & 1u;
                st_shared<T>((uint32_t)(sbuf + (b ? (int32_t)Rj + kk.y : (int32_t)(q0 + j - Rj) + kk.x)) *
                                 (uint32_t)sizeof(T),
                             sym_in_word<T>(x, j));
              }
            }
          }
        }
      } else {  // too many segments for the table: node tables from global memory
        const int32_t K0F = S.K[0], K1F = S.K[1], K0L = S.K[2], K1L = S.K[3];
        auto consts = [&](uint32_t v, int32_t& K0, int32_t& K1) {
          if (v == vF) {
            K0 = K0F;
            K1 = K1F;
          } else if (v == vL) {
            K0 = K0L;
            K1 = K1L;
          } else {  // interior node: stage position = HBM destination - T0 + MARGIN
            const ulonglong2 t = __ldg(&tab[v]);
            K0 = (int32_t)((long long)t.x - (long long)P) + MARGIN;
            K1 = (int32_t)((long long)t.y + (long long)P - (long long)T0) + MARGIN;
          }
        };
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
          const uint32_t w = tid + LV_THREADS * k;
          const uint32_t q0 = w * SPW;
          if (q0 >= len) break;
          const uint4 ow = S.own[w / XW];
          const uint32_t R = (ow.y & 0xffffu) + (uint32_t)__popc(ow.x & submask);
          const uint32_t m4 = ow.x >> sub;
          const uint32_t h4 = (ow.z >> sub) & ((1u << SPW) - 2u);
          const uint32_t x = Win[w];
          const uint32_t nv = min((uint32_t)SPW, len - q0);
          if (nv == (uint32_t)SPW && h4 == 0) {
            int32_t K0, K1;
            consts(sym_in_word<T>(x, 0) >> nsh, K0, K1);
            word_one_segment(x, q0, R, m4, K0, K1, lut_of(m4));
          } else {
#pragma unroll
            for (int j = 0; j < SPW; ++j) {
              if ((uint32_t)j < nv) {
                const uint32_t sym = sym_in_word<T>(x, j);
                int32_t K0, K1;
                consts(sym >> nsh, K0, K1);
                const uint32_t Rj = R + (uint32_t)__popc(m4 & lowmask(j));
                const uint32_t b = (m4 >> j) & 1u;
                st_shared<T>((uint32_t)(sbuf + (b ? (int32_t)Rj + K1 : (int32_t)(q0 + j - Rj) + K0)) *
                                 (uint32_t)sizeof(T),
                             sym);
              }
            }
          }
        }
      }
    }
    fence_proxy_async_smem();
    __syncthreads();  // B4: stage partitioned (and the input buffer fully read)

    // ---------------- phase E: TMA bulk stores of the aligned bodies, element stores of the edges
    if (tid < (uint32_t)LV_NREG) {  // lane r of warp 0: region r's 16-byte-aligned body
      const int32_t b = S.rbase[tid], l = S.rlen[tid];
      const int32_t fs = (b + A - 1) / A * A, fe = (b + l) / A * A;
      if (l > 0 && fe > fs)
        bulk_s2g(out + (S.gofs[tid] + fs), S.buf[ob] + fs, (uint32_t)(fe - fs) * (uint32_t)sizeof(T));
      bulk_commit();
    }
    if (tid < (uint32_t)(2 * A * LV_NREG)) {
      const int r = (int)(tid / (2 * A)), e = (int)(tid % (2 * A));
      const int32_t b = S.rbase[r], l = S.rlen[r], end = b + l;
      const int32_t fs = (b + A - 1) / A * A, fe = (b + l) / A * A;
      const int32_t hend = min(fs, end);                             // head edge [b, hend), < A symbols
      const int32_t q = (e < A) ? b + e : max(fe, hend) + (e - A);  // tail edge [max(fe, hend), end), < A
      if (l > 0 && ((e < A) ? (q < hend) : (q < end))) out[S.gofs[r] + q] = S.buf[ob][q];
    }
    // the previous tile's output buffer: once its bulk stores have read it, load a new tile into it
    if (warp == 0) {
      if (lane < (uint32_t)LV_NREG) bulk_wait_read<1>();  // each lane's own bulk groups
      __syncwarp();
      if (lane == 0 && it >= 1) issue(it + NB - 2);
    }
  }
  if (SCATTER) {
    __syncthreads();
    if (tid < LV_NKEY) {
      const uint32_t v = S.cnt[tid];
      if (v) atomicAdd(&agg_next[S.dtile[tid]], v);
    }
    if (tid < (uint32_t)LV_NREG) bulk_wait<0>();
  }
}

}  // namespace wt
