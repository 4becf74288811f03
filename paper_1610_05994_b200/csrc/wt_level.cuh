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
  static_assert(TILE % 512 == 0, "tiles hold whole superblocks");
  static_assert(WPT == XW && LV_THREADS % XW == 0, "phase D word / owner layout");
};

template <typename T>
struct LevelSmem {
  using C = LvTile<T>;
  alignas(128) T buf[C::NB][C::BUF];      // ring: input tiles land at buf[b][MARGIN], outputs are staged
  uint2 own[LV_THREADS];                  // per phase-A thread: {bit mask, tile-local ones before}
  uint32_t warp_tot[LV_WARPS];
  int32_t s1, am, Rs1, Ram;               // first-segment end, last-segment start, ranks there
  int32_t K[4];                           // K0F, K1F, K0L, K1L (shared addresses in symbols)
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

// st.shared of the low sizeof(T) bytes of v at shared byte address a
template <typename T>
__device__ __forceinline__ void st_shared(uint32_t a, uint32_t v) {
  if (sizeof(T) == 1) asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
  else if (sizeof(T) == 2) asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v));
  else asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
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
    const uint32_t c = (uint32_t)__popc(m);
    const uint32_t incl = warp_incl_scan_u32(c);
    if (lane == 31) S.warp_tot[warp] = incl;

    uint32_t vF = 0, vL = 0;
    ulonglong2 tabF = make_ulonglong2(0, 0), tabL = make_ulonglong2(0, 0);
    uint32_t nfirst = 0, nlast = 0;
    if (SCATTER) {
      vF = (uint32_t)B[0] >> nsh;
      vL = (uint32_t)B[len - 1] >> nsh;
      if (tid == 0) {
        tabF = __ldg(&tab[vF]);
        tabL = __ldg(&tab[vL]);
      }
      if (vF != vL) {
        nfirst = tid ? ((uint32_t)B[i0 - 1] >> nsh) : vF;  // node just before the thread's range
#pragma unroll
        for (int q = 0; q < E; ++q)
          if ((uint32_t)q + 1 == nvalid) nlast = sym_of<T>(xw, q) >> nsh;
      }
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
    uint32_t wpre, tot;
    {
      const uint32_t wt = (lane < (uint32_t)LV_WARPS) ? S.warp_tot[lane] : 0u;
      const uint32_t wi = warp_incl_scan_u32(wt);
      wpre = __shfl_sync(FULL, wi - wt, warp);
      tot = __shfl_sync(FULL, wi, LV_WARPS - 1);
    }
    const uint32_t mypre = wpre + incl - c;
    if ((i0 & 511u) == 0 && T0 + i0 < n) sb[(T0 + i0) >> 9] = P + mypre;
    if (tid == 0 && T0 + TILE >= n) sb[nsb - 1] = P + tot;
    if (!SCATTER) continue;

    S.own[tid] = make_uint2(m, mypre);
    if (vF != vL && nvalid > 0) {  // segment finders (nodes are non-decreasing along T_l)
      // monotone nodes: the boundary's offset in the thread's range is the
      // number of its symbols before it (no dynamic register indexing)
      if (nfirst == vF && nlast != vF) {
        uint32_t k = 0;
#pragma unroll
        for (int q = 0; q < E; ++q) k += ((uint32_t)q < nvalid && (sym_of<T>(xw, q) >> nsh) == vF) ? 1u : 0u;
        S.s1 = (int32_t)(i0 + k);
        S.Rs1 = (int32_t)(mypre + __popc(m & lowmask(k)));
      }
      if (nfirst != vL && nlast == vL) {
        uint32_t k = 0;
#pragma unroll
        for (int q = 0; q < E; ++q) k += ((uint32_t)q < nvalid && (sym_of<T>(xw, q) >> nsh) != vL) ? 1u : 0u;
        S.am = (int32_t)(i0 + k);
        S.Ram = (int32_t)(mypre + __popc(m & lowmask(k)));
      }
    }
    __syncthreads();  // B2: own[], finder results

    // ---------------- constants of the tile's regions (one thread)
    if (tid == 0) {
      const bool one = (vF == vL);
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
      const int32_t base[LV_NREG] = {MARGIN + s1, b1, b2, b3, b4};
      const int32_t rl[LV_NREG] = {am - s1, z0, o0, zm, om};
      const long long go[LV_NREG] = {(long long)T0 - MARGIN, D0z - b1, D0o - b2, Dmz - b3, Dmo - b4};
      const int32_t sbuf = (int32_t)(smem_u32(S.buf[ob]) / (uint32_t)sizeof(T));  // in symbols
      S.K[0] = sbuf + b1;
      S.K[1] = sbuf + b2;
      S.K[2] = sbuf + b3 - am + Ram;
      S.K[3] = sbuf + b4 - Ram;
      S.s1 = s1;
      S.am = am;
      S.Ram = Ram;
#pragma unroll
      for (int r = 0; r < LV_NREG; ++r) {
        S.rbase[r] = base[r];
        S.rlen[r] = rl[r];
        S.gofs[r] = go[r];
        const long long d0 = (long long)base[r] + go[r];  // HBM destination of the region's first symbol
        const unsigned long long t0 = (unsigned long long)d0 / TILE;
        S.dtile[2 * r] = (r == 0) ? tile : t0;
        S.dtile[2 * r + 1] = t0 + 1;
        // region symbols with rank < ksplit land in destination tile t0, the rest in t0 + 1
        S.ksplit[r] = (r == 0) ? 0x7fffffff : (int32_t)min((long long)rl[r], (long long)(t0 + 1) * TILE - d0);
      }
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
        else {  // the one thread per region holding the split
          Mlo = 0;
          uint32_t x = M;
          for (int32_t j = k - rank0; j > 0; --j) {
            Mlo |= x & (0u - x);
            x &= x - 1;
          }
        }
        lo = (uint32_t)__popc(nbm & Mlo);
        hi = (uint32_t)__popc(nbm & M & ~Mlo);
      };
      uint32_t cnt[LV_NKEY];
      if (vF == vL) {  // block-uniform: one segment, only the first-segment runs
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
      const int32_t K0F = S.K[0], K1F = S.K[1], K0L = S.K[2], K1L = S.K[3];
      const int32_t sbufM = (int32_t)(smem_u32(S.buf[ob]) / (uint32_t)sizeof(T)) + MARGIN;
      const uint32_t* Win = reinterpret_cast<const uint32_t*>(B);
      auto consts = [&](uint32_t v, int32_t& K0, int32_t& K1) {
        if (v == vF) {
          K0 = K0F;
          K1 = K1F;
        } else if (v == vL) {
          K0 = K0L;
          K1 = K1L;
        } else {  // interior node: stage position = HBM destination - T0 + MARGIN
          const ulonglong2 t = __ldg(&tab[v]);
          K0 = (int32_t)((long long)t.x - (long long)P) + sbufM;
          K1 = (int32_t)((long long)t.y + (long long)P - (long long)T0) + sbufM;
        }
      };
      const uint32_t sub = (tid % (uint32_t)XW) * SPW;  // word w = tid + 256 k: owner w / XW, offset (w % XW) * SPW
      const uint32_t submask = lowmask(sub);
      if (vF == vL && len == (uint32_t)TILE) {  // block-uniform: one segment, full tile
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
          const uint32_t w = tid + LV_THREADS * k;
          const uint2 ow = S.own[w / XW];
          const uint32_t R = ow.y + (uint32_t)__popc(ow.x & submask);
          const uint32_t m4 = ow.x >> sub;
          const uint32_t x = Win[w];
          int32_t az = (int32_t)(w * SPW - R) + K0F, ao = (int32_t)R + K1F;
#pragma unroll
          for (int j = 0; j < SPW; ++j) {
            const bool b = (m4 >> j) & 1u;
            st_shared<T>((uint32_t)(b ? ao : az) * (uint32_t)sizeof(T), x >> (8 * sizeof(T) * j));
            if (b) ++ao;
            else ++az;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
          const uint32_t w = tid + LV_THREADS * k;
          const uint32_t q0 = w * SPW;
          if (q0 >= len) break;
          const uint2 ow = S.own[w / XW];
          const uint32_t R = ow.y + (uint32_t)__popc(ow.x & submask);
          const uint32_t m4 = (ow.x >> sub) & ((1u << SPW) - 1u);
          const uint32_t x = Win[w];
          const uint32_t nv = min((uint32_t)SPW, len - q0);
          const uint32_t v0 = sym_in_word<T>(x, 0) >> nsh;
          const uint32_t vl = sym_in_word<T>(x, SPW - 1) >> nsh;
          if (nv == (uint32_t)SPW && v0 == vl) {
            int32_t K0, K1;
            consts(v0, K0, K1);
            int32_t az = (int32_t)(q0 - R) + K0, ao = (int32_t)R + K1;
#pragma unroll
            for (int j = 0; j < SPW; ++j) {
              const bool b = (m4 >> j) & 1u;
              st_shared<T>((uint32_t)(b ? ao : az) * (uint32_t)sizeof(T), x >> (8 * sizeof(T) * j));
              if (b) ++ao;
              else ++az;
            }
          } else {
#pragma unroll
            for (int j = 0; j < SPW; ++j) {
              if ((uint32_t)j < nv) {
                const uint32_t sym = sym_in_word<T>(x, j);
                int32_t K0, K1;
                consts(sym >> nsh, K0, K1);
                const uint32_t Rj = R + (uint32_t)__popc(m4 & lowmask(j));
                const uint32_t b = (m4 >> j) & 1u;
                st_shared<T>((uint32_t)(b ? (int32_t)Rj + K1 : (int32_t)(q0 + j - Rj) + K0) * (uint32_t)sizeof(T),
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
    if (tid == 0) {
#pragma unroll
      for (int r = 0; r < LV_NREG; ++r) {
        const int32_t b = S.rbase[r], l = S.rlen[r];
        const int32_t fs = (b + A - 1) / A * A, fe = (b + l) / A * A;
        if (l > 0 && fe > fs)
          bulk_s2g(out + (S.gofs[r] + fs), S.buf[ob] + fs, (uint32_t)(fe - fs) * (uint32_t)sizeof(T));
      }
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
    if (tid == 0) {
      bulk_wait_read<1>();
      if (it >= 1) issue(it + NB - 2);
    }
  }
  if (SCATTER) {
    __syncthreads();
    if (tid < LV_NKEY) {
      const uint32_t v = S.cnt[tid];
      if (v) atomicAdd(&agg_next[S.dtile[tid]], v);
    }
    if (tid == 0) bulk_wait<0>();
  }
}

}  // namespace wt
