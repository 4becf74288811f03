// wt_pair2.cuh -- the level pass of a two-level tree of 1-byte symbols
// (sigma 3 or 4: the DNA-like workload, the paper's rna.* datasets,
// P:889-895), specialised.
//
// With L = 2 (Alg. 1; Prop. 1) level 0 is one node, so
//   B_0 = bit 1 of every symbol, in S order;
//   B_1 = bit 0 of the symbols whose bit 1 is 0, in S order (positions
//         [0, Z), Z = the zeros of level 0), then bit 0 of those whose bit 1 is
//         1 (positions [Z, n)).
// The pass over S before it (k_prologue) counted every tile's level-0 ones and
// their total (so Z = n - ones0), and a scan turned them into the tile
// prefixes pre[t].  So every tile is independent: its zeros' bits go to B_1 at
// T0 - pre[t], its ones' bits at Z + pre[t].
//
// This is the general fused pair (k_level<., 2>) with everything L = 2 does
// not need taken out -- node tables, segments, the TMA ring, progressive
// counting: a warp takes 2048-symbol tiles round-robin (the level pass's
// tiles, whose prefixes the scan produced) through its own ring of TMA
// buffers, every lane 64 consecutive symbols.  The lane's symbols are compacted 4 at a time: one
// multiply gathers their 8 bits into a byte, a 256-entry table gives their
// level-0 bits and their zeros' and ones' bit-0 strings, whose appends are
// multiply-adds.  Each lane's two strings (<= 64 bits) are stored straight to
// B_1: words wholly inside the lane's run plain, the run's first and last
// words (shared with neighbouring lanes and tiles: the paper's atomic
// boundary words) OR-ed into the zero-filled level.
#pragma once
#include <cuda.h>

#include "wt_device.cuh"
#include "wt_ptx.cuh"

namespace wt {

constexpr int P2_TILE = 2048;  // = LvTile<uint8_t>::TILE (the tile prefixes' granularity)
constexpr int P2_MINB = 32;    // warps (CTAs) per SM the register budget is sized for (every slot: latency hiding)

// 256-entry table, index = the (bit 0, bit 1) pairs of 4 symbols (bit 2j =
// bit 0 of symbol j, bit 2j+1 = its bit 1):
//   .x = [3:0] bit 0 of the symbols with bit 1 = 0, in order (the zeros' string)
//        [19:16] bit 1 of the four symbols (their level-0 bits)
//        [31:28] bit 0 of the symbols with bit 1 = 1 (the ones' string: one
//        shift extracts it)
//   .y = [7:0] 2^(their zeros), [15:8] 2^(their ones): the strings' position multipliers
__device__ __forceinline__ uint2 p2_lut_entry(uint32_t idx) {
  uint32_t zb = 0, nz = 0, ob = 0, no = 0, m1 = 0;
  for (uint32_t j = 0; j < 4; ++j) {
    const uint32_t b0 = (idx >> (2 * j)) & 1u, b1 = (idx >> (2 * j + 1)) & 1u;
    m1 |= b1 << j;
    if (b1) ob |= b0 << no++;
    else zb |= b0 << nz++;
  }
  return make_uint2(zb | (m1 << 16) | (ob << 28), (1u << nz) | ((1u << no) << 8));
}

// 32 consecutive symbols (8 words), the first `valid` real: level-0 word m,
// zeros' string Z, ones' string O.
__device__ __forceinline__ void p2_quarter(const uint32_t* w, uint32_t valid, const uint2* lut, uint32_t& m,
                                           uint32_t& Z, uint32_t& O) {
  m = Z = O = 0;
  if (valid == 32) {
    uint32_t pz = 1, po = 1;
#pragma unroll
    for (int wi = 0; wi < 8; ++wi) {
      // byte j's two bits to 24 + 2j: x * (2^24 + 2^18 + 2^12 + 2^6) (symbols < 4: the
      // pass over S checked the range; no carries reach the top byte)
      const uint2 e = lut[(w[wi] * 0x01041040u) >> 24];
      m |= ((e.x >> 16) & 15u) << (4 * wi);
      Z += (e.x & 15u) * pz;
      O += (e.x >> 28) * po;
      pz *= e.y & 0xffu;
      po *= e.y >> 8;
    }
    return;
  }
  uint32_t nz = 0, no = 0;
  uint32_t ww[8];  // (a copy: the dynamic index below must not pull the caller's registers into memory)
#pragma unroll
  for (int k = 0; k < 8; ++k) ww[k] = w[k];
  for (uint32_t j = 0; j < valid; ++j) {
    const uint32_t s = (ww[j >> 2] >> (8 * (j & 3))) & 0xffu;
    const uint32_t b1 = (s >> 1) & 1u, b0 = s & 1u;
    m |= b1 << j;
    if (b1) O |= b0 << no++;
    else Z |= b0 << nz++;
  }
}

// nb <= 64 bits of v (v[0] low) at global bit position pos of `bits`: the
// words wholly inside [pos, pos + nb) stored, the partial first / last OR-ed
__device__ __forceinline__ void p2_put(uint32_t* bits, uint64_t pos, const uint32_t (&v)[2], uint32_t nb) {
  if (nb == 0) return;
  const uint64_t j = pos >> 5;
  const uint32_t off = (uint32_t)(pos & 31u), end = off + nb;  // bit range [off, end) of words j, j+1, j+2
  const uint32_t w0 = v[0] << off;
  const uint32_t w1 = __funnelshift_lc(v[0], v[1], off);
  const uint32_t w2 = __funnelshift_lc(v[1], 0u, off);
  if (off == 0 && end >= 32) bits[j] = w0;
  else atomicOr(&bits[j], w0);
  if (end > 32) {
    if (end >= 64) bits[j + 1] = w1;
    else atomicOr(&bits[j + 1], w1);
  }
  if (end > 64) {
    if (end == 96) bits[j + 2] = w2;
    else atomicOr(&bits[j + 2], w2);
  }
}

// nb <= 128 bits of v (v[0] low) at global bit position pos of `bits`: the
// words wholly inside [pos, pos + nb) stored, the partial first / last OR-ed
__device__ __forceinline__ void p2_put4(uint32_t* bits, uint64_t pos, const uint32_t (&v)[4], uint32_t nb) {
  const uint64_t j = pos >> 5;
  const uint32_t off = (uint32_t)(pos & 31u), end = off + nb;  // bit range [off, end) of words j ..
#pragma unroll
  for (uint32_t k = 0; k < 5; ++k) {
    if (32 * k >= end) break;
    const uint32_t lo = k ? v[k - 1] : 0u, hi = k < 4 ? v[k] : 0u;
    const uint32_t wk = __funnelshift_lc(lo, hi, off);
    if ((k > 0 || off == 0) && 32 * k + 32 <= end) bits[j + k] = wk;
    else atomicOr(&bits[j + k], wk);
  }
}

constexpr int P2_WARPS = 4;   // independent warps per CTA (they share the table)
#ifndef WT_P2_NB
#define WT_P2_NB 2
#endif
constexpr int P2_NB = WT_P2_NB;  // per-warp ring of input tiles
constexpr int P2_WT = 4096;      // bytes (symbols) per warp tile: one 128-byte row per lane, two level tiles

struct P2Smem {
  alignas(1024) uint4 ring[P2_WARPS][P2_NB][P2_WT / 16];  // 32 rows of 128 bytes per tile, 128-byte swizzle
  uint2 lut[256];
  alignas(8) unsigned long long bar[P2_WARPS][P2_NB];
};
constexpr size_t p2_smem_bytes() { return sizeof(P2Smem) + 1024; }

// 2-D tensor-map bulk copy (rows of 128 bytes, SWIZZLE_128B) into shared memory
__device__ __forceinline__ void p2_tma(void* dst, const void* tmap, int32_t row, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(0), "r"(row), "r"(smem_u32(bar))
      : "memory");
}

// B_0, SB_0 and B_1 (which must be zero on entry) of a two-level tree of n
// 1-byte symbols.  P2_WARPS independent warps per CTA (no block barrier after
// the table is built); warp tiles of 4096 symbols (two level tiles, whose
// prefixes pre[t] the scan produced) round-robin over all warps.  Each warp
// streams its tiles through a ring of P2_NB buffers filled by TMA tensor
// copies (S as rows of 128 bytes, 128-byte swizzle): lane l owns row l, 128
// consecutive symbols, and reads its eight 16-byte chunks in an order in which
// the lanes of a load hit distinct banks.  The lane's two strings (<= 128 bits
// each) are stored with their inner words plain, the first / last OR-ed.
__global__ void __launch_bounds__(32 * P2_WARPS, 6)
    k_pair2(const uint8_t* __restrict__ S, uint64_t n, uint32_t ntiles, const uint32_t* __restrict__ pre,
            const unsigned long long* __restrict__ ones0, uint32_t* __restrict__ B0,
            unsigned long long* __restrict__ SB0, uint64_t nsb, uint32_t* __restrict__ B1,
            const int32_t* __restrict__ flag, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ unsigned char p2_raw[];
  // (an offset from the __shared__ array, not an integer round trip: the
  // compiler keeps the shared address space -- LDS / STS instead of generic loads)
  P2Smem& sm = *reinterpret_cast<P2Smem*>(p2_raw + ((1024u - (smem_u32(p2_raw) & 1023u)) & 1023u));
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < 256; i += 32 * P2_WARPS) sm.lut[i] = p2_lut_entry(i);
  if (lane == 0) {
    for (int b = 0; b < P2_NB; ++b) mbar_init(&sm.bar[wid][b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t gw = blockIdx.x * P2_WARPS + wid, nw = gridDim.x * P2_WARPS;  // this warp, all warps
  const uint32_t nwt = (uint32_t)((n + P2_WT - 1) / P2_WT);                   // warp tiles
  const uint64_t full_bytes = n & ~127ull;  // the tensor map's whole rows
#ifndef WT_P2_ROUND_ROBIN
  // a contiguous chunk of warp tiles per warp: its runs of B_1 are contiguous,
  // so most boundary words are shared with the warp's own next tile instead of
  // with another SM's at the same moment (pair 0.305 -> 0.298 ms on cfg2; a
  // chunk per CTA with its warps round-robin inside it: 0.304; the general
  // k_pairn measured slower with chunks and keeps round-robin tiles)
  const uint32_t chunk = (nwt + nw - 1) / nw;
#endif
  auto issue = [&](uint32_t it) {           // lane 0: the warp's it-th tile into ring slot it % P2_NB
#ifndef WT_P2_ROUND_ROBIN
    const uint32_t tile = it < chunk ? gw * chunk + it : 0xffffffffu;
#else
    const uint32_t tile = gw + it * nw;
#endif
    if (tile >= nwt) return;
    const int b = (int)(it % P2_NB);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&sm.bar[wid][b], P2_WT);  // (rows past the tensor's end are zero-filled)
    p2_tma(sm.ring[wid][b], &tmap, (int32_t)(tile * (P2_WT / 128)), &sm.bar[wid][b]);
  };
  pdl_wait();  // the tile prefixes, ones0, the zero-filled B_1 (and no range error)
  if (*flag) return;
  if (lane == 0)
    for (uint32_t b = 0; b < P2_NB; ++b) issue(b);
  const uint64_t Z = n - *ones0;  // the zeros of level 0: B_1's ones' run starts here
  const uint32_t swz = lane & 7u;
  for (uint32_t it = 0;; ++it) {
#ifndef WT_P2_ROUND_ROBIN
    const uint32_t tile = it < chunk ? gw * chunk + it : 0xffffffffu;
#else
    const uint32_t tile = gw + it * nw;
#endif
    if (tile >= nwt) break;
    const int b = (int)(it % P2_NB);
    const uint64_t T0 = (uint64_t)tile * P2_WT;
    const uint64_t p0 = T0 + 128ull * lane;
    const uint32_t pt = 2 * tile + (lane >> 4);                // the lane's level tile
    const uint32_t P = pt < ntiles ? __ldg(&pre[pt]) : 0u;     // level-0 ones before it
    mbar_wait(&sm.bar[wid][b], (it / P2_NB) & 1u);
    unsigned char* const buf = reinterpret_cast<unsigned char*>(sm.ring[wid][b]);
    if (T0 + P2_WT > full_bytes && full_bytes < n) {  // the partial last row: into its swizzled place
      for (uint64_t g = full_bytes + lane; g < n; g += 32) {
        const uint32_t off = (uint32_t)(g - T0), r = off >> 7, c = (off >> 4) & 7u;
        buf[r * 128 + ((c ^ (r & 7u)) << 4) + (off & 15u)] = S[g];
      }
      __syncwarp();
    }
    const uint32_t nvalid = p0 >= n ? 0u : (uint32_t)min((uint64_t)128, n - p0);
    uint32_t m[4];
    uint64_t zc[2], oc[2];
    uint32_t nzh[2], noh[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // the lane's two 64-symbol halves
      uint32_t w[16];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t c = 4 * (uint32_t)h + (uint32_t)k;
        const uint4 q = *reinterpret_cast<const uint4*>(buf + lane * 128 + ((c ^ swz) << 4));
        w[4 * k] = q.x, w[4 * k + 1] = q.y, w[4 * k + 2] = q.z, w[4 * k + 3] = q.w;
      }
      const uint32_t hv = nvalid > 64u * h ? min(nvalid - 64u * h, 64u) : 0u;
      uint32_t Zs[2], Os[2];
      p2_quarter(w, min(hv, 32u), sm.lut, m[2 * h], Zs[0], Os[0]);
      p2_quarter(w + 8, hv > 32 ? hv - 32 : 0u, sm.lut, m[2 * h + 1], Zs[1], Os[1]);
      const uint32_t o0 = (uint32_t)__popc(m[2 * h]);
      const uint32_t z0 = min(hv, 32u) - o0;
      noh[h] = o0 + (uint32_t)__popc(m[2 * h + 1]);
      nzh[h] = hv - noh[h];
      zc[h] = (uint64_t)Zs[0] | ((uint64_t)Zs[1] << z0);
      oc[h] = (uint64_t)Os[0] | ((uint64_t)Os[1] << o0);
    }
    __syncwarp();  // every lane has read the slot: refill it
    if (lane == 0) issue(it + P2_NB);
    // level-0 words (the last tile's padding words: zero)
    if (p0 < ((n + 511) & ~511ull)) *reinterpret_cast<uint4*>(B0 + p0 / 32) = make_uint4(m[0], m[1], m[2], m[3]);
    const uint32_t no = noh[0] + noh[1];
    const uint32_t inc = warp_incl_scan_u32(no);
    const uint32_t h15 = __shfl_sync(FULL, inc, 15);
    const uint32_t hb = (lane >> 4) ? h15 : 0u;  // (lanes 16..31: the second level tile)
    const uint32_t R = inc - no - hb;  // level-0 ones before the lane, inside its level tile
    const uint32_t P0 = __shfl_sync(FULL, P, 0);
    if ((lane & 3u) == 0 && p0 < n) SB0[p0 / 512] = P + R;
    if (tile + 1 == nwt && lane == 31) SB0[nsb - 1] = P0 + inc;
    // the lane's two strings of <= 128 bits: half 1's bits after half 0's
    uint32_t Zv[4], Ov[4];
    {
      const uint64_t lo = zc[0] | (nzh[0] >= 64 ? 0ull : (zc[1] << nzh[0]));
      const uint64_t hi = nzh[0] == 0 ? 0ull : (nzh[0] >= 64 ? zc[1] : (zc[1] >> (64 - nzh[0])));
      Zv[0] = (uint32_t)lo, Zv[1] = (uint32_t)(lo >> 32), Zv[2] = (uint32_t)hi, Zv[3] = (uint32_t)(hi >> 32);
    }
    {
      const uint64_t lo = oc[0] | (noh[0] >= 64 ? 0ull : (oc[1] << noh[0]));
      const uint64_t hi = noh[0] == 0 ? 0ull : (noh[0] >= 64 ? oc[1] : (oc[1] >> (64 - noh[0])));
      Ov[0] = (uint32_t)lo, Ov[1] = (uint32_t)(lo >> 32), Ov[2] = (uint32_t)hi, Ov[3] = (uint32_t)(hi >> 32);
    }
    const uint32_t nzl = nvalid - no;
    if (nzl) p2_put4(B1, p0 - P - R, Zv, nzl);   // zeros before the lane: positions - ones
    if (no) p2_put4(B1, Z + P + R, Ov, no);
  }
  pdl_trigger();
}

}  // namespace wt
