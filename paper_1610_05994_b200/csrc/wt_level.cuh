// wt_level.cuh -- a3/a4: the per-level stable segmented bit-partition (sm_100a).
//
// One pass over T_l produces B_l (bitmap words), SB_l (superblocks) and, for
// l < L-1, T_{l+1} = T_l stably partitioned inside every level-l node by bit
// sh = L-1-l (Alg. 1 lines 8-13, with the "C[node]++" cursors
// replaced by closed-form ranks; node of s at level l is s >> (sh+1),
// Proposition 1).
//
// Execution model (B200-first, not the paper's per-level thread):
//   * persistent CTAs (2 per SM), tiles of 16 KiB assigned round-robin; each
//     CTA keeps LV_STAGES tiles in flight with cp.async.bulk (TMA bulk copy)
//     into shared memory, completion on mbarriers;
//   * NO look-back: the ones of level l in every tile (agg_l[t]) were counted
//     by the pass that wrote T_l (the histogram pass for l = 0), and a tiny
//     scan turned them into pre_l[t] before this pass, so tiles are
//     independent.  While writing T_{l+1} this pass counts agg_{l+1};
//   * phase A  -- ballot: warp w turns 32 consecutive positions into one
//                 bitmap word with __ballot_sync (bit = (s >> sh) & 1) and, in
//                 the same sweep, a "segment head" word (node changes);
//   * phase B  -- popcounts -> warp scan -> block scan + pre_l[tile] give the
//                 global rank r(j); bitmap words and SB[t] = r(512 t) go
//                 straight to HBM;
//   * phase C  -- the tile's node segments become <= 2 runs each (zeros run ->
//                 left child, ones run -> right child); every run gets a
//                 shared-memory staging window whose start is congruent to its
//                 HBM destination modulo 16 bytes;
//   * phase D  -- every symbol is stored into its run's staging window
//                 (stable: position inside the run = zeros/ones before it);
//   * phase E  -- the staging windows are written out as aligned 16-byte
//                 vectors (partial vectors only at run edges), counting the
//                 next level's bit per destination tile (agg_{l+1}).
//   Tiles with more than LV_MAXSEG node segments (very deep levels with tiny
//   nodes) scatter each symbol directly instead of phases C-E.
//
// Global destinations (ob[v] = ones of level l before node v, Zn[v] = zeros
// of level l before node v+1; both from the node tables built from C):
//   b = 0: dest = (j - r(j)) + ob[v]        b = 1: dest = r(j) + Zn[v]
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
__device__ __forceinline__ uint32_t lanemask_le() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

// ------------------------------------------------------------ configuration
constexpr int LV_THREADS = 512;
constexpr int LV_WARPS = LV_THREADS / 32;
constexpr int LV_STAGES = 3;
constexpr int LV_MAXSEG = 256;
constexpr int LV_MAXRUN = 2 * LV_MAXSEG;
static_assert(LV_MAXRUN <= LV_THREADS, "one thread per run in phase C");

// Every thread owns 32 consecutive bytes of the tile: E symbols.  For uint8 a
// thread's E bits are exactly one 32-bit bitmap word.
template <typename T>
struct LvTile {
  static constexpr int E = 32 / (int)sizeof(T);        // symbols per thread
  static constexpr int TILE = LV_THREADS * E;          // 16 KiB, a multiple of 512 positions
  static constexpr int A = 16 / (int)sizeof(T);        // symbols per 16-byte vector
  static constexpr int TPW = 32 / E;                   // threads per bitmap word (1, 2, 4)
  static constexpr int OUTCAP = TILE + A * LV_MAXRUN + A;
};

template <typename T>
struct LevelSmem {
  using C = LvTile<T>;
  alignas(128) T in[LV_STAGES][C::TILE];
  alignas(16) T out[C::OUTCAP];
  uint32_t tmask[LV_THREADS];  // bit k = bit sh of the thread's k-th symbol
  uint32_t tpre[LV_THREADS];   // tile-local exclusive prefix per thread, packed (heads << 16) | ones
  uint32_t seg_start[LV_MAXSEG + 1];
  int32_t run_base[LV_MAXRUN];  // staging base of run r (see phase D)
  uint32_t run_s[LV_MAXRUN];    // staging start (symbols)
  uint32_t run_len[LV_MAXRUN];
  uint32_t run_chunk0[LV_MAXRUN + 1];
  unsigned long long run_d[LV_MAXRUN];
  uint32_t warp_tot[LV_WARPS];
  uint32_t warp_tot2[LV_WARPS];
  uint32_t total;
  alignas(8) unsigned long long bar[LV_STAGES];
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

// bit `sh` of the E symbols held in xw[8] (32 bytes), symbol k -> bit k.
template <typename T>
__device__ __forceinline__ uint32_t swar_bits(const uint32_t (&xw)[8], uint32_t sh) {
  uint32_t m = 0;
  if (sizeof(T) == 1) {
    // gather bit sh of the 4 bytes of a word with one multiply:
    // (x & 0x01010101<<sh) * (1 + 2^7 + 2^14 + 2^21) puts byte j's bit at 21+sh+j
    const uint32_t msk = 0x01010101u << sh;
#pragma unroll
    for (int k = 0; k < 8; ++k) m |= ((((xw[k] & msk) * 0x00204081u) >> (21 + sh)) & 0xfu) << (4 * k);
  } else if (sizeof(T) == 2) {
    const uint32_t msk = 0x00010001u << sh;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t t = xw[k] & msk;
      m |= (((t >> sh) | (t >> (sh + 15))) & 3u) << (2 * k);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) m |= ((xw[k] >> sh) & 1u) << k;
  }
  return m;
}

template <typename T>
__device__ __forceinline__ uint32_t sym_of(const uint32_t (&xw)[8], int k) {
  if (sizeof(T) == 1) return (xw[k >> 2] >> (8 * (k & 3))) & 0xffu;
  if (sizeof(T) == 2) return (xw[k >> 1] >> (16 * (k & 1))) & 0xffffu;
  return xw[k];
}

// Adds `cnt` to agg[tau] once per group of lanes (in `mask`) that share tau.
__device__ __forceinline__ void agg_add(uint32_t* agg, uint32_t mask, uint32_t tau, uint32_t cnt) {
  const uint32_t grp = __match_any_sync(mask, tau);
  const uint32_t tot = __reduce_add_sync(grp, cnt);
  if (tot && (threadIdx.x & 31) == (uint32_t)(__ffs(grp) - 1)) atomicAdd(&agg[tau], tot);
}

// ------------------------------------------------------------ the kernel
template <typename T, bool SCATTER>
__global__ void __launch_bounds__(LV_THREADS, 2)
    k_level(const T* __restrict__ in, T* __restrict__ out, uint64_t n, uint32_t sh,
            const ulonglong2* __restrict__ tab, uint32_t* __restrict__ bits, uint64_t words_per_level,
            unsigned long long* __restrict__ sb, uint64_t nsb, const unsigned long long* __restrict__ pre,
            uint32_t* __restrict__ agg_next, const int32_t* __restrict__ flag) {
  using Cfg = LvTile<T>;
  constexpr int TILE = Cfg::TILE, A = Cfg::A, E = Cfg::E, TPW = Cfg::TPW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LevelSmem<T>& S = *reinterpret_cast<LevelSmem<T>*>(smem_raw);

  if (*flag) return;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t nb_mask = SCATTER ? bitmask32<T>(sh - 1) : 0u;  // next level's bit
  const uint32_t i0 = tid * E;                                  // first tile position of this thread

  auto tile_of = [&](uint32_t it) -> uint64_t { return (uint64_t)blockIdx.x + (uint64_t)it * gridDim.x; };
  auto issue = [&](int s, uint64_t t) {  // thread 0: bulk-copy tile t into stage s
    const uint64_t T0 = t * (uint64_t)TILE;
    const uint64_t len = min((uint64_t)TILE, n - T0);
    const uint32_t bytes = (uint32_t)(len * sizeof(T)) & ~15u;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&S.bar[s], bytes);
    if (bytes) bulk_g2s(S.in[s], in + T0, bytes, &S.bar[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < LV_STAGES; ++s) mbar_init(&S.bar[s], 1);
    fence_mbar_init();
    for (int s = 0; s < LV_STAGES; ++s)
      if (tile_of(s) < ntiles) issue(s, tile_of(s));
  }
  __syncthreads();

  for (uint32_t it = 0;; ++it) {
    const int s = (int)(it % LV_STAGES);
    const uint64_t tile = tile_of(it);
    if (tile >= ntiles) break;
    const uint64_t T0 = tile * (uint64_t)TILE;
    const uint32_t len = (uint32_t)min((uint64_t)TILE, n - T0);
    const uint64_t P = pre[tile];  // ones of this level before the tile
    mbar_wait(&S.bar[s], (it / LV_STAGES) & 1u);
    const T* xin = S.in[s];
    if (len < TILE) {  // tail bytes the 16-byte bulk copy did not cover
      const uint32_t done = ((len * (uint32_t)sizeof(T)) & ~15u) / (uint32_t)sizeof(T);
      for (uint32_t i = done + tid; i < len; i += LV_THREADS) S.in[s][i] = in[T0 + i];
      __syncthreads();
    }

    // ---------------- phase A: the thread's 32 bytes -> E bits (+ segment heads)
    uint32_t xw[8];
    {
      const uint4* src = reinterpret_cast<const uint4*>(xin) + 2 * tid;
      const uint4 va = src[0], vb = src[1];
      xw[0] = va.x, xw[1] = va.y, xw[2] = va.z, xw[3] = va.w;
      xw[4] = vb.x, xw[5] = vb.y, xw[6] = vb.z, xw[7] = vb.w;
    }
    const uint32_t nvalid = (i0 >= len) ? 0u : min((uint32_t)E, len - i0);
    const uint32_t vmask = (nvalid >= 32) ? 0xffffffffu : ((1u << nvalid) - 1u);
    const uint32_t m = swar_bits<T>(xw, sh) & vmask;
    uint32_t hm = 0;
    if (SCATTER) {
      const uint32_t nf = sym_of<T>(xw, 0) >> (sh + 1);
      const uint32_t nl = sym_of<T>(xw, E - 1) >> (sh + 1);
      uint32_t prev = __shfl_up_sync(FULL, nl, 1);
      if (lane == 0) prev = (tid > 0) ? ((uint32_t)xin[i0 - 1] >> (sh + 1)) : nf;
      if (nvalid < (uint32_t)E || nf != nl || nf != prev) {
        uint32_t p = prev;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const uint32_t nd = sym_of<T>(xw, k) >> (sh + 1);
          if (nd != p) hm |= 1u << k;
          p = nd;
        }
        if (tid == 0) hm &= ~1u;  // the tile start is not a head
        hm &= vmask;
      }
    }
    // bitmap word(s): TPW threads per 32-bit word
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
    // ---------------- phase B: tile-local ranks (packed heads/ones), superblocks
    const uint32_t c = ((uint32_t)__popc(hm) << 16) | (uint32_t)__popc(m);
    const uint32_t incl = warp_incl_scan_u32(c);
    if (lane == 31) S.warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t wtot = (lane < (uint32_t)LV_WARPS) ? S.warp_tot[lane] : 0u;
      const uint32_t wi = warp_incl_scan_u32(wtot);
      if (lane < (uint32_t)LV_WARPS) S.warp_tot2[lane] = wi - wtot;
      if (lane == 31) S.total = wi;
    }
    __syncthreads();
    const uint32_t tot = S.total;
    const uint32_t tot_ones = tot & 0xffffu;
    const uint32_t nseg = (tot >> 16) + 1;
    const uint32_t mypre = S.warp_tot2[warp] + incl - c;
    if ((i0 & 511u) == 0 && T0 + i0 < n) sb[(T0 + i0) >> 9] = P + (mypre & 0xffffu);
    if (tid == 0 && T0 + TILE >= n) sb[nsb - 1] = P + tot_ones;

    if (SCATTER) {
      if (nseg <= (uint32_t)LV_MAXSEG) {
        S.tmask[tid] = m;
        S.tpre[tid] = mypre;
        if (hm) {  // segment starts
          uint32_t h = hm, g = (mypre >> 16) + 1;
          while (h) {
            const int b = __ffs(h) - 1;
            h &= h - 1;
            S.seg_start[g++] = i0 + (uint32_t)b;
          }
        }
        if (tid == 0) {
          S.seg_start[0] = 0;
          S.seg_start[nseg] = len;
        }
        __syncthreads();
        // tile-local exclusive rank of position x in [0, len]
        auto Rloc = [&](uint32_t x) -> uint32_t {
          if (x >= len) return tot_ones;
          const uint32_t t = x / E, r = x % E;
          return (S.tpre[t] & 0xffffu) + (uint32_t)__popc(S.tmask[t] & ((1u << r) - 1u));
        };
        // ---------------- phase C: runs (2 per segment), staging windows
        const uint32_t nrun = 2 * nseg;
        uint32_t a = 0, Ra = 0;
        if (tid < nrun) {
          const uint32_t g = tid >> 1;
          a = S.seg_start[g];
          const uint32_t e = S.seg_start[g + 1];
          Ra = Rloc(a);
          const uint32_t Re = Rloc(e);
          const uint32_t v = (uint32_t)xin[a] >> (sh + 1);
          const ulonglong2 te = __ldg(&tab[v]);
          if (tid & 1) {
            S.run_len[tid] = Re - Ra;
            S.run_d[tid] = P + Ra + te.y;
          } else {
            S.run_len[tid] = (e - Re) - (a - Ra);
            S.run_d[tid] = (T0 - P) + (a - Ra) + te.x;
          }
        }
        __syncthreads();
        uint32_t packed = 0, pad = 0;
        if (tid < nrun) {
          const uint32_t L_ = S.run_len[tid];
          const unsigned long long D_ = S.run_d[tid];
          const uint32_t prev_end = tid ? (uint32_t)((S.run_d[tid - 1] + S.run_len[tid - 1]) & (A - 1)) : 0u;
          pad = ((uint32_t)(D_ & (A - 1)) - prev_end) & (A - 1);
          const uint32_t nch = L_ ? (uint32_t)((D_ + L_ + A - 1) / A - D_ / A) : 0u;
          packed = (nch << 16) | (pad + L_);
        }
        const uint32_t pin = warp_incl_scan_u32(packed);
        if (lane == 31) S.warp_tot[warp] = pin;
        __syncthreads();
        if (warp == 0) {
          const uint32_t wtot = (lane < (uint32_t)LV_WARPS) ? S.warp_tot[lane] : 0u;
          const uint32_t wi = warp_incl_scan_u32(wtot);
          if (lane < (uint32_t)LV_WARPS) S.warp_tot2[lane] = wi - wtot;
          if (lane == 31) S.run_chunk0[nrun] = wi >> 16;
        }
        __syncthreads();
        if (tid < nrun) {
          const uint32_t ex = S.warp_tot2[warp] + pin - packed;
          const uint32_t sstart = (ex & 0xffffu) + pad;
          S.run_s[tid] = sstart;
          S.run_chunk0[tid] = ex >> 16;
          // zeros run: pos = sstart + (i - R(i)) - (a - Ra);  ones run: pos = sstart + R(i) - Ra
          S.run_base[tid] = (tid & 1) ? (int32_t)sstart - (int32_t)Ra : (int32_t)sstart - (int32_t)(a - Ra);
        }
        __syncthreads();
        // ---------------- phase D: symbols into their staging windows
        {
          uint32_t g = mypre >> 16;
          uint32_t R = mypre & 0xffffu;
          int32_t po = S.run_base[2 * g + 1] + (int32_t)R;
          int32_t pz = S.run_base[2 * g] + (int32_t)(i0 - R);
          if (hm == 0 && nvalid == (uint32_t)E) {
#pragma unroll
            for (int k = 0; k < E; ++k) {
              const uint32_t b = (m >> k) & 1u;
              S.out[b ? po : pz] = (T)sym_of<T>(xw, k);
              po += (int32_t)b;
              pz += 1 - (int32_t)b;
            }
          } else {
#pragma unroll
            for (int k = 0; k < E; ++k) {
              if ((uint32_t)k < nvalid) {
                if ((hm >> k) & 1u) {
                  ++g;
                  const uint32_t Rk = R + (uint32_t)__popc(m & ((1u << k) - 1u));
                  po = S.run_base[2 * g + 1] + (int32_t)Rk;
                  pz = S.run_base[2 * g] + (int32_t)(i0 + k - Rk);
                }
                const uint32_t b = (m >> k) & 1u;
                S.out[b ? po : pz] = (T)sym_of<T>(xw, k);
                po += (int32_t)b;
                pz += 1 - (int32_t)b;
              }
            }
          }
        }
        __syncthreads();
        // ---------------- phase E: aligned 16-byte write-out + next-level tile counts
        const uint32_t nch_total = S.run_chunk0[nrun];
        for (uint32_t base = 0; base < nch_total; base += LV_THREADS) {
          const uint32_t ch = base + tid;
          uint32_t tau = 0xffffffffu, cnt = 0;
          if (ch < nch_total) {
            uint32_t lo = 0, hi = nrun;  // largest r with run_chunk0[r] <= ch
            while (hi - lo > 1) {
              const uint32_t mid = (lo + hi) >> 1;
              if (S.run_chunk0[mid] <= ch) lo = mid;
              else hi = mid;
            }
            const unsigned long long Dr = S.run_d[lo];
            const uint32_t Lr = S.run_len[lo], sr = S.run_s[lo];
            const unsigned long long D = (Dr / A) * A + (unsigned long long)(ch - S.run_chunk0[lo]) * A;
            const long long off = (long long)D - (long long)Dr;
            tau = (uint32_t)(D / TILE);
            if (off >= 0 && off + A <= (long long)Lr) {
              const uint4 v = *reinterpret_cast<const uint4*>(&S.out[sr + off]);
              *reinterpret_cast<uint4*>(out + D) = v;
              cnt = (uint32_t)(__popc(v.x & nb_mask) + __popc(v.y & nb_mask) + __popc(v.z & nb_mask) +
                               __popc(v.w & nb_mask));
            } else {
#pragma unroll
              for (int q = 0; q < A; ++q) {
                const long long o = off + q;
                if (o >= 0 && o < (long long)Lr) {
                  const T x = S.out[sr + o];
                  out[D + q] = x;
                  cnt += ((uint32_t)x >> (sh - 1)) & 1u;
                }
              }
            }
          }
          agg_add(agg_next, FULL, tau, cnt);
        }
      } else {
        // deep level, many tiny nodes: scatter every symbol straight to HBM
        uint64_t r = P + (mypre & 0xffffu);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          uint32_t tau = 0xffffffffu, cnt = 0;
          if ((uint32_t)k < nvalid) {
            const uint32_t x = sym_of<T>(xw, k);
            const uint32_t b = (m >> k) & 1u;
            const ulonglong2 e = __ldg(&tab[x >> (sh + 1)]);
            const uint64_t dest = b ? (r + e.y) : (T0 + i0 + k - r + e.x);
            out[dest] = (T)x;
            r += b;
            tau = (uint32_t)(dest / TILE);
            cnt = (x >> (sh - 1)) & 1u;
          }
          agg_add(agg_next, FULL, tau, cnt);
        }
      }
    }
    __syncthreads();  // stage s and the staging buffer are free again
    if (tid == 0 && tile_of(it + LV_STAGES) < ntiles) issue(s, tile_of(it + LV_STAGES));
  }
}

}  // namespace wt
