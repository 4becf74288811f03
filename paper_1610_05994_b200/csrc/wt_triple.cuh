// wt_triple.cuh -- the fused final three levels of a tree (a5 with k = 3 at
// the bottom, Alg. 1 lines 8-13 for levels L-3, L-2, L-1): one pass
// over T_{L-3} writes B_{L-3}, SB_{L-3}, B_{L-2} and B_{L-1}; T_{L-2} and
// T_{L-1} never exist and no symbol moves.
//
// T_{L-3} is S stably sorted by the top L-3 bits (Prop. 1).  A
// symbol s at position j of level-(L-3) node v (v = s >> 3) has the class
// (b2, b1) of its bits 2 and 1; its level-(L-1) node is 4v + (2 b2 + b1) and,
// the order inside every node being stable, its position there is that node's
// start plus the symbols of the same class in v before j.  So B_{L-1} holds,
// per level-(L-1) node, the bit 0 of that class's symbols in T_{L-3} order,
// and B_{L-2}, per level-(L-2) node 2v + b2, their bit 1 (the no-move pair of
// wt_pairn.cuh one level up).  A lane's run of symbols inside one node thus
// sends six bit strings to six contiguous destinations:
//   B_{L-2}: bit 1 of its b2 = 0 / b2 = 1 symbols (zeros' / ones' of level L-3)
//   B_{L-1}: bit 0 of its class 00 / 01 / 10 / 11 symbols.
// Destinations need, besides the level-(L-3) tile prefixes and node table
// {ob, Zn}, the class-01 and class-11 symbols before the run (G01, G11: tile
// prefixes of per-tile counts) and before its node (node table tab3), and the
// class sizes of every node (cls) -- counted by k_cls3, one read-only pass
// over T_{L-3} before (the counters Alg. 1 lines 5-6 keep per level, P:539-540,
// taken two levels ahead).
//
// Strings per 32 symbols (a unit): stage 1 reads the 4-symbol table of
// wt_pair2.cuh twice per 4 symbols -- indexed by the bit pairs (2, 1) and
// (2, 0) -- giving the b2 nibble and the bit-1 and bit-0 strings of the b2 = 0
// and b2 = 1 symbols (equal lengths, position order); stage 2 splits each
// (bit-1, bit-0) string pair by bit 1 with a second table (index: 4 bits of
// each) into the class strings.  Execution as k_pairn: 4 KiB warp tiles
// (two level tiles) through a TMA tensor ring, one 128-byte row per lane.
#pragma once
#include <cuda.h>

#include "wt_device.cuh"
#include "wt_pair2.cuh"
#include "wt_pairn.cuh"
#include "wt_ptx.cuh"

namespace wt {

// the bit pair (2, 1) (MODE 1) or (2, 0) (MODE 2) of every symbol of a word
// moved to bits (1, 0) of the symbol
template <int W, int MODE>
__device__ __forceinline__ uint32_t tr_word(uint32_t x) {
  constexpr uint32_t M0 = W == 1 ? 0x01010101u : W == 2 ? 0x00010001u : 1u;
  if constexpr (MODE == 1) return x >> 1;
  else return (x & M0) | ((x >> 1) & (M0 << 1));
}

// table index (bit 2j = low bit, bit 2j+1 = high bit of symbol j) of the
// symbols 4g .. 4g+3 of a lane for the bit pair of MODE
template <typename T, int MODE>
__device__ __forceinline__ uint32_t tr_index(const uint32_t (&w)[16], int g) {
  if constexpr (sizeof(T) == 1) {
    return ((tr_word<1, MODE>(w[g]) & 0x03030303u) * 0x01041040u) >> 24;
  } else if constexpr (sizeof(T) == 2) {
    const uint32_t x = (tr_word<2, MODE>(w[2 * g]) & 0x00030003u) | ((tr_word<2, MODE>(w[2 * g + 1]) & 0x00030003u) << 4);
    return (x | (x >> 14)) & 0xffu;
  } else {
    uint32_t a, b, x;  // the four low bytes into one word, then as for bytes
    asm("prmt.b32 %0, %1, %2, 0x0040;" : "=r"(a) : "r"(w[4 * g]), "r"(w[4 * g + 1]));
    asm("prmt.b32 %0, %1, %2, 0x0040;" : "=r"(b) : "r"(w[4 * g + 2]), "r"(w[4 * g + 3]));
    asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(x) : "r"(a), "r"(b));
    return ((tr_word<1, MODE>(x) & 0x03030303u) * 0x01041040u) >> 24;
  }
}

// stage-2 table, index (hi nibble << 4 | lo nibble) of 4 symbols' (bit 1, bit
// 0): the p2 entry of the interleaved pairs (bit 0 of the bit-1 = 0 symbols,
// bit 0 of the bit-1 = 1 symbols, the strings' position multipliers)
__device__ __forceinline__ uint2 tr_lutc_entry(uint32_t i) {
  uint32_t idx = 0;
  for (uint32_t j = 0; j < 4; ++j) idx |= (((i >> j) & 1u) << (2 * j)) | (((i >> (4 + j)) & 1u) << (2 * j + 1));
  return p2_lut_entry(idx);
}

// One unit: up to 32 consecutive symbols (UG groups of 4) of a lane, nv of them
// real.  m: bit 2 (position order); Z1/Z0: bit 1 / bit 0 of the b2 = 0
// symbols, O1/O0: of the b2 = 1 symbols; nz, no their counts.
template <typename T, int UG>
__device__ __forceinline__ void tr_stage1(const uint32_t (&w)[16], int g0, uint32_t j0, uint32_t nv,
                                          const uint2* lut, uint32_t& m, uint32_t& Z1, uint32_t& Z0, uint32_t& O1,
                                          uint32_t& O0, uint32_t& nz, uint32_t& no) {
  m = Z1 = Z0 = O1 = O0 = 0;
  if (nv == 4u * UG) {
    uint32_t pz = 1, po = 1;
#pragma unroll
    for (int g = 0; g < UG; ++g) {
      const uint2 a = lut[tr_index<T, 1>(w, g0 + g)];
      const uint2 b = lut[tr_index<T, 2>(w, g0 + g)];
      m |= ((a.x >> 16) & 15u) << (4 * g);
      Z1 += (a.x & 15u) * pz;
      Z0 += (b.x & 15u) * pz;
      O1 += (a.x >> 28) * po;
      O0 += (b.x >> 28) * po;
      pz *= a.y & 0xffu;
      po *= a.y >> 8;
    }
    no = (uint32_t)__popc(m);
    nz = 4u * UG - no;
    return;
  }
  nz = no = 0;
  for (uint32_t j = 0; j < nv; ++j) {
    const uint32_t s = pn_sym<T>(w, j0 + j);
    const uint32_t b2 = (s >> 2) & 1u, b1 = (s >> 1) & 1u, b0 = s & 1u;
    m |= b2 << j;
    if (b2) {
      O1 |= b1 << no;
      O0 |= b0 << no++;
    } else {
      Z1 |= b1 << nz;
      Z0 |= b0 << nz++;
    }
  }
}

// stage 2: the (bit 1, bit 0) strings H, Lo of n symbols split by bit 1: the
// bit-0 strings of the bit-1 = 0 symbols (c0) and of the bit-1 = 1 ones (c1)
template <int UG>
__device__ __forceinline__ void tr_stage2(uint32_t H, uint32_t Lo, uint32_t n, const uint2* lutc, uint32_t& c0,
                                          uint32_t& c1) {
  c0 = c1 = 0;
  uint32_t p0 = 1, p1 = 1;
  // (a partial last chunk: its padding symbols are (0, 0), appended after the
  // real ones, past the lengths the caller uses)
#pragma unroll
  for (int k = 0; k < UG; ++k) {
    if (4 * k >= (int)n) break;
    const uint2 e = lutc[(((H >> (4 * k)) & 15u) << 4) | ((Lo >> (4 * k)) & 15u)];
    c0 += (e.x & 15u) * p0;
    c1 += (e.x >> 28) * p1;
    p0 *= e.y & 0xffu;
    p1 *= e.y >> 8;
  }
}

// a lane's string of up to 4 units (each <= 32 bits, lengths l[u]) as 128 bits
template <int NU>
__device__ __forceinline__ void tr_cat(const uint32_t (&s)[NU], const uint32_t (&l)[NU], uint32_t (&v)[4],
                                       uint32_t& len) {
  uint64_t lo = 0, hi = 0;
  len = 0;
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    const uint64_t x = s[u];
    if (len < 64) {
      lo |= x << len;
      if (len > 32) hi |= x >> (64 - len);
    } else {
      hi |= x << (len - 64);
    }
    len += l[u];
  }
  v[0] = (uint32_t)lo, v[1] = (uint32_t)(lo >> 32), v[2] = (uint32_t)hi, v[3] = (uint32_t)(hi >> 32);
}

// the per-level-(L-3)-node constants of the six destinations
struct TrNode {
  uint32_t ob, zb;       // ones / zeros of level L-3 before the node
  uint32_t n01, n11;     // class-01 / 11 symbols before the node (G01, G11 at its start)
  uint32_t Zn, ob1;      // zeros up to its end, ones before the next node
  uint32_t s01, s11;     // class sizes
};
__device__ __forceinline__ TrNode tr_node(const uint2* __restrict__ tab, const uint2* __restrict__ tab3,
                                          const uint2* __restrict__ cls, uint32_t v, uint32_t nv, uint32_t n) {
  TrNode d;
  const uint2 t = __ldg(&tab[v]);
  d.ob = t.x;
  d.Zn = t.y;
  d.zb = v ? __ldg(&tab[v - 1]).y : 0u;
  d.ob1 = (v + 1 < nv) ? __ldg(&tab[v + 1]).x : n - t.y;  // (the last node ends at n)
  const uint2 g = __ldg(&tab3[v]);
  d.n01 = g.x;
  d.n11 = g.y;
  const uint2 c = __ldg(&cls[v]);
  d.s01 = c.x;
  d.s11 = c.y;
  return d;
}

// the six strings of a run of node v starting at global position j with
// r = ones of level L-3 before j and G01 / G11 = class-01 / 11 symbols before
// j (all mod 2^32: positions < n < 2^32); strings as 128-bit values (NW words)
template <int NW, typename Put>
__device__ __forceinline__ void tr_put_run(const TrNode& d, uint32_t j, uint32_t r, uint32_t G01, uint32_t G11,
                                           uint32_t* __restrict__ B2, uint32_t* __restrict__ B1, Put put,
                                           const uint32_t (&z1)[4], uint32_t lz, const uint32_t (&o1)[4], uint32_t lo,
                                           const uint32_t (&c00)[4], uint32_t l00, const uint32_t (&c01)[4],
                                           uint32_t l01, const uint32_t (&c10)[4], uint32_t l10,
                                           const uint32_t (&c11)[4], uint32_t l11) {
  const uint32_t zj = j - r;                  // zeros of level L-3 before j
  const uint32_t sv = d.zb + d.ob;            // the node's first position
  const uint32_t zv = d.Zn - d.zb, ov = d.ob1 - d.ob;  // its zeros / ones
  const uint32_t a01 = G01 - d.n01, a11 = G11 - d.n11;  // class 01 / 11 of the node before j
  const uint32_t a00 = (zj - d.zb) - a01, a10 = (r - d.ob) - a11;
  put(B2, zj + d.ob, z1, lz);                         // level L-2, node 2v: zeros' bit-1 string
  put(B2, r + d.Zn, o1, lo);                          // node 2v+1
  const uint32_t N10 = sv + zv;
  put(B1, sv + a00, c00, l00);                        // level L-1, node 4v
  put(B1, sv + (zv - d.s01) + a01, c01, l01);         // node 4v+1
  put(B1, N10 + a10, c10, l10);                       // node 4v+2
  put(B1, N10 + (ov - d.s11) + a11, c11, l11);        // node 4v+3
}

template <typename T>
struct TrCfg {
  static constexpr int W = (int)sizeof(T);
  static constexpr int E = 128 / W;   // symbols per lane (one 128-byte row)
  static constexpr int WT = 32 * E;   // symbols per warp tile (two level tiles)
  static constexpr int UG = E >= 64 ? 8 : E / 8;  // groups of 4 symbols per unit (32 / 32 / 16 symbols)
  static constexpr int US = 4 * UG;   // symbols per unit
  static constexpr int NU = E / US;   // units per lane (4 / 2 / 2)
};

struct TrSmem {
  alignas(1024) uint4 ring[PN_WARPS][PN_NB][PN_WT / 16];
  uint2 lut[256];
  uint2 lutc[256];
  alignas(8) unsigned long long bar[PN_WARPS][PN_NB];
};
constexpr size_t tr_smem_bytes() { return sizeof(TrSmem) + 1024; }

// Counting pass over T_{L-3}: per level tile the class-01 and class-11
// symbols (agg01, agg11), per level-(L-3) node its class-01 and class-11 sizes
// (cls[v] = {01, 11}, zero on entry).  One warp per level tile, 64 bytes per
// lane.
template <typename T>
__global__ void __launch_bounds__(256) k_cls3(const T* __restrict__ in, uint32_t n, uint32_t ntiles,
                                              uint32_t* __restrict__ agg01, uint32_t* __restrict__ agg11,
                                              uint2* __restrict__ cls, const int32_t* __restrict__ flag) {
  constexpr int EH = 64 / (int)sizeof(T), LT = 32 * EH;
  pdl_wait();
  if (*flag) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * 8 + (threadIdx.x >> 5), nwarps = gridDim.x * 8;
  // the lane's 64 bytes of tile t (symbols past n read as 0, masked out below)
  auto load = [&](uint32_t t, uint32_t(&w)[16]) {
    const uint64_t p0 = (uint64_t)t * LT + (uint64_t)EH * lane;
    const uint32_t nv = p0 >= n ? 0u : (uint32_t)min((uint64_t)EH, n - p0);
    if (nv == (uint32_t)EH) {
      const uint4* src = reinterpret_cast<const uint4*>(in + p0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint4 q = ldg_nc_v4(src + k);
        w[4 * k] = q.x, w[4 * k + 1] = q.y, w[4 * k + 2] = q.z, w[4 * k + 3] = q.w;
      }
    } else {
      constexpr uint32_t SPW = 4 / sizeof(T);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        uint32_t x = 0;
#pragma unroll
        for (uint32_t q = 0; q < SPW; ++q) {
          const uint32_t j = (uint32_t)k * SPW + q;
          if (j < nv) x |= (uint32_t)in[p0 + j] << (8 * sizeof(T) * q);
        }
        w[k] = x;
      }
    }
  };
  uint32_t wn[16];
  if (warp < ntiles) load(warp, wn);
  for (uint32_t t = warp; t < ntiles; t += nwarps) {
    const uint64_t p0 = (uint64_t)t * LT + (uint64_t)EH * lane;
    const uint32_t nv = p0 >= n ? 0u : (uint32_t)min((uint64_t)EH, n - p0);
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = wn[k];
    if (t + nwarps < ntiles) load(t + nwarps, wn);  // the next tile's loads in flight while this one is counted
    // bits 2 and 1 in position order
    uint64_t M2, M1;
    if constexpr (EH == 64) {
      M2 = swar_bits<T, 8, 0>(w, 2u) | ((uint64_t)swar_bits<T, 8, 8>(w, 2u) << 32);
      M1 = swar_bits<T, 8, 0>(w, 1u) | ((uint64_t)swar_bits<T, 8, 8>(w, 1u) << 32);
    } else {
      M2 = swar_bits<T, 16, 0>(w, 2u);
      M1 = swar_bits<T, 16, 0>(w, 1u);
    }
    const uint64_t V = nv >= 64 ? ~0ull : ((1ull << nv) - 1ull);
    M2 &= V;
    M1 &= V;
    const uint32_t c01 = (uint32_t)__popcll(~M2 & M1 & V), c11 = (uint32_t)__popcll(M2 & M1);
    const uint32_t t01 = __reduce_add_sync(FULL, c01), t11 = __reduce_add_sync(FULL, c11);
    if (lane == 0) {
      agg01[t] = t01;
      agg11[t] = t11;
    }
    // node sizes by class
    const uint32_t vf = nv ? pn_sym_c<T, 0>(w) >> 3 : 0u;
    const uint32_t vl = (nv == (uint32_t)EH ? pn_sym_c<T, EH - 1>(w) : nv ? pn_sym<T>(w, nv - 1) : 0u) >> 3;
    const uint32_t wf = __shfl_sync(FULL, vf, 0);  // (lane 0 holds a real symbol)
    if (__all_sync(FULL, nv == 0 || (vf == wf && vl == wf))) {  // the tile inside one node: one atomic
      if (lane == 0 && (t01 | t11))
        atomicAdd(reinterpret_cast<unsigned long long*>(&cls[wf]),
                  (unsigned long long)t01 | ((unsigned long long)t11 << 32));
    } else if (nv) {  // the lane's runs inside one node
      uint64_t heads = 0;
      if (vf != vl) {
        uint32_t prev = vf;
        for (uint32_t j = 1; j < nv; ++j) {
          const uint32_t nd = pn_sym<T>(w, j) >> 3;
          heads |= (uint64_t)(nd != prev) << j;
          prev = nd;
        }
      }
      uint32_t a = 0, v = vf;
      for (;;) {
        const uint32_t e = heads ? (uint32_t)(__ffsll((long long)heads) - 1) : nv;
        const uint64_t pm = (e >= 64 ? ~0ull : ((1ull << e) - 1ull)) & ~((1ull << a) - 1ull);
        const uint32_t r01 = (uint32_t)__popcll(~M2 & M1 & pm), r11 = (uint32_t)__popcll(M2 & M1 & pm);
        if (r01 | r11)
          atomicAdd(reinterpret_cast<unsigned long long*>(&cls[v]),
                    (unsigned long long)r01 | ((unsigned long long)r11 << 32));
        if (e >= nv) break;
        a = e;
        v = pn_sym<T>(w, e) >> 3;
        heads &= heads - 1;
      }
    }
  }
  pdl_trigger();
}

// B_{L-3} (bits3), SB_{L-3} and B_{L-2}, B_{L-1} (both zero on entry) from
// T_{L-3} (n < 2^32 symbols), its tile prefixes pre / pre01 / pre11 (ones of
// level L-3, class-01 and class-11 symbols before every level tile), the node
// tables tab = {ob, Zn} (level L-3, nv nodes), tab3 = {class 01, 11 before the
// node} and the class sizes cls.
#ifndef WT_TR_MINB
#define WT_TR_MINB 4
#endif
template <typename T>
__global__ void __launch_bounds__(32 * PN_WARPS, WT_TR_MINB)
    k_triple(const T* __restrict__ in, uint32_t n, uint32_t ntiles, const uint32_t* __restrict__ pre,
             const uint32_t* __restrict__ pre01, const uint32_t* __restrict__ pre11, const uint2* __restrict__ tab,
             uint32_t nvn, const uint2* __restrict__ tab3, const uint2* __restrict__ cls, uint32_t* __restrict__ bits3,
             unsigned long long* __restrict__ sb, uint32_t nsb, uint32_t* __restrict__ B2, uint32_t* __restrict__ B1,
             const int32_t* __restrict__ flag, const __grid_constant__ CUtensorMap tmap) {
  using C = TrCfg<T>;
  constexpr int E = C::E, EH = E / 2, WT = C::WT, UG = C::UG, US = C::US, NU = C::NU;
  extern __shared__ unsigned char tr_raw[];
  // (an offset from the __shared__ array, not an integer round trip: the
  // compiler keeps the shared address space -- LDS / STS instead of generic loads)
  TrSmem& sm = *reinterpret_cast<TrSmem*>(tr_raw + ((1024u - (smem_u32(tr_raw) & 1023u)) & 1023u));
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < 256; i += 32 * PN_WARPS) {
    sm.lut[i] = p2_lut_entry(i);
    sm.lutc[i] = tr_lutc_entry(i);
  }
  if (lane == 0) {
    for (int b = 0; b < PN_NB; ++b) mbar_init(&sm.bar[wid][b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t gw = blockIdx.x * PN_WARPS + wid, nw = gridDim.x * PN_WARPS;
  const uint32_t nwt = (uint32_t)(((uint64_t)n + WT - 1) / WT);
  const uint64_t nbytes = (uint64_t)n * sizeof(T);
  const uint64_t full_bytes = nbytes & ~127ull;
  auto issue = [&](uint32_t it) {
    const uint32_t tile = gw + it * nw;
    if (tile >= nwt) return;
    const int b = (int)(it % PN_NB);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&sm.bar[wid][b], PN_WT);
    p2_tma(sm.ring[wid][b], &tmap, (int32_t)(tile * (PN_WT / 128)), &sm.bar[wid][b]);
  };
  pdl_wait();
  if (*flag) return;
  if (lane == 0)
    for (uint32_t b = 0; b < PN_NB; ++b) issue(b);
  const uint32_t swz = lane & 7u;
  const uint64_t padded = ((uint64_t)n + 511) & ~511ull;
  const unsigned char* inb = reinterpret_cast<const unsigned char*>(in);
  auto put4 = [](uint32_t* bits, uint32_t pos, const uint32_t(&v)[4], uint32_t nb) {
    if (nb) p2_put4(bits, (uint64_t)pos, v, nb);
  };
  for (uint32_t it = 0;; ++it) {
    const uint32_t tile = gw + it * nw;
    if (tile >= nwt) break;
    const int b = (int)(it % PN_NB);
    const uint64_t T0 = (uint64_t)tile * WT;
    const uint64_t p0 = T0 + (uint32_t)E * lane;
    const uint32_t lt = 2 * tile + (lane >> 4);
    const bool ltv = lt < ntiles;
    const uint32_t P = ltv ? __ldg(&pre[lt]) : 0u;
    const uint32_t P01 = ltv ? __ldg(&pre01[lt]) : 0u, P11 = ltv ? __ldg(&pre11[lt]) : 0u;
    mbar_wait(&sm.bar[wid][b], (it / PN_NB) & 1u);
    unsigned char* const buf = reinterpret_cast<unsigned char*>(sm.ring[wid][b]);
    const uint64_t B0 = T0 * sizeof(T);
    if (B0 + PN_WT > full_bytes && full_bytes < nbytes) {
      for (uint64_t g = full_bytes + lane; g < nbytes; g += 32) {
        const uint32_t off = (uint32_t)(g - B0), r = off >> 7, c = (off >> 4) & 7u;
        buf[r * 128 + ((c ^ (r & 7u)) << 4) + (off & 15u)] = inb[g];
      }
      __syncwarp();
    }
    const uint32_t nvalid = p0 >= n ? 0u : (uint32_t)min((uint64_t)E, n - p0);
    uint32_t w0[16], w1[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 q0 = *reinterpret_cast<const uint4*>(buf + lane * 128 + (((uint32_t)k ^ swz) << 4));
      const uint4 q1 = *reinterpret_cast<const uint4*>(buf + lane * 128 + (((uint32_t)(k + 4) ^ swz) << 4));
      w0[4 * k] = q0.x, w0[4 * k + 1] = q0.y, w0[4 * k + 2] = q0.z, w0[4 * k + 3] = q0.w;
      w1[4 * k] = q1.x, w1[4 * k + 1] = q1.y, w1[4 * k + 2] = q1.z, w1[4 * k + 3] = q1.w;
    }
    __syncwarp();  // every lane has read the slot: refill it
    if (lane == 0) issue(it + PN_NB);
    // the lane's units: strings and counts
    uint32_t m[NU], Z1[NU], O1[NU], lz[NU], lo[NU], c00[NU], c01[NU], c10[NU], c11[NU];
    uint32_t l00[NU], l01[NU], l10[NU], l11[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const uint32_t s0 = (uint32_t)u * US;  // the unit's first symbol in the lane
      const uint32_t nvu = nvalid > s0 ? min(nvalid - s0, (uint32_t)US) : 0u;
      const int g0 = (int)((s0 % EH) / 4);
      uint32_t Z0, O0;
      if (s0 < (uint32_t)EH) tr_stage1<T, UG>(w0, g0, s0 % EH, nvu, sm.lut, m[u], Z1[u], Z0, O1[u], O0, lz[u], lo[u]);
      else tr_stage1<T, UG>(w1, g0, s0 % EH, nvu, sm.lut, m[u], Z1[u], Z0, O1[u], O0, lz[u], lo[u]);
      tr_stage2<UG>(Z1[u], Z0, lz[u], sm.lutc, c00[u], c01[u]);
      tr_stage2<UG>(O1[u], O0, lo[u], sm.lutc, c10[u], c11[u]);
      l01[u] = (uint32_t)__popc(Z1[u]);
      l00[u] = lz[u] - l01[u];
      l11[u] = (uint32_t)__popc(O1[u]);
      l10[u] = lo[u] - l11[u];
    }
    // B_{L-3} words (the last tile's padding words: zero)
    if (p0 < padded) {
      if constexpr (US == 32 && NU == 4) *reinterpret_cast<uint4*>(bits3 + p0 / 32) = make_uint4(m[0], m[1], m[2], m[3]);
      else if constexpr (US == 32) *reinterpret_cast<uint2*>(bits3 + p0 / 32) = make_uint2(m[0], m[1]);
      else bits3[p0 / 32] = m[0] | (m[1] << 16);
    }
    uint32_t ones = 0, x01 = 0, x11 = 0;
#pragma unroll
    for (int u = 0; u < NU; ++u) ones += lo[u], x01 += l01[u], x11 += l11[u];
    const uint32_t inc = warp_incl_scan_u32(ones);
    const uint32_t incx = warp_incl_scan_u32(x01 | (x11 << 16));  // (<= 2048 per level tile: no carry)
    const uint32_t h15 = __shfl_sync(FULL, inc, 15), h15x = __shfl_sync(FULL, incx, 15);
    const uint32_t R = inc - ones - ((lane >> 4) ? h15 : 0u);
    const uint32_t Q = incx - (x01 | (x11 << 16)) - ((lane >> 4) ? h15x : 0u);
    const uint32_t P0 = __shfl_sync(FULL, P, 0);
    if ((p0 & 511u) == 0 && p0 < n) sb[p0 / 512] = P + R;
    if (tile + 1 == nwt && lane == 31) sb[nsb - 1] = P0 + inc;
    if (nvalid) {
      const uint32_t r0 = P + R, g01 = P01 + (Q & 0xffffu), g11 = P11 + (Q >> 16);
      const uint32_t v = pn_sym_c<T, 0>(w0) >> 3;
      const uint32_t vlast =
          (nvalid > (uint32_t)EH ? pn_sym<T>(w1, nvalid - EH - 1) : pn_sym<T>(w0, nvalid - 1)) >> 3;
      if (v == vlast) {  // the lane inside one node: six whole strings
        const TrNode d = tr_node(tab, tab3, cls, v, nvn, n);
        uint32_t sz[4], so[4], s00[4], s01[4], s10[4], s11[4], kz, ko, k00, k01, k10, k11;
        tr_cat<NU>(Z1, lz, sz, kz);
        tr_cat<NU>(O1, lo, so, ko);
        tr_cat<NU>(c00, l00, s00, k00);
        tr_cat<NU>(c01, l01, s01, k01);
        tr_cat<NU>(c10, l10, s10, k10);
        tr_cat<NU>(c11, l11, s11, k11);
        tr_put_run<4>(d, (uint32_t)p0, r0, g01, g11, B2, B1, put4, sz, kz, so, ko, s00, k00, s01, k01, s10, k10, s11,
                      k11);
      } else {  // per unit, per run of one node
        uint32_t j = (uint32_t)p0, r = r0, a01 = g01, a11 = g11;  // before the unit
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const uint32_t s0 = (uint32_t)u * US;
          const uint32_t nvu = nvalid > s0 ? min(nvalid - s0, (uint32_t)US) : 0u;
          if (nvu == 0) break;
          const uint32_t(&w)[16] = s0 < (uint32_t)EH ? w0 : w1;
          const uint32_t jb = s0 % EH;  // the unit's first symbol in its half
          // bit 1 in position order, node changes
          uint32_t m1 = 0, heads = 0;
          uint32_t prev = pn_sym<T>(w, jb) >> 3, vv = prev;
          for (uint32_t q = 0; q < nvu; ++q) {
            const uint32_t sym = pn_sym<T>(w, jb + q);
            m1 |= ((sym >> 1) & 1u) << q;
            const uint32_t nd = sym >> 3;
            heads |= (uint32_t)(nd != prev) << q;
            prev = nd;
          }
          const uint32_t m2 = m[u];
          uint32_t a = 0;
          for (;;) {
            const uint32_t e = heads ? (uint32_t)(__ffs(heads) - 1) : nvu;
            const uint32_t ma = lowmask(a), me = lowmask(e);
            // counts before a inside the unit: b2 zeros / ones, classes
            const uint32_t oa = (uint32_t)__popc(m2 & ma), za = a - oa;
            const uint32_t q01 = (uint32_t)__popc(~m2 & m1 & ma), q11 = (uint32_t)__popc(m2 & m1 & ma);
            const uint32_t q00 = za - q01, q10 = oa - q11;
            const uint32_t oe = (uint32_t)__popc(m2 & me), ze = e - oe;
            const uint32_t e01 = (uint32_t)__popc(~m2 & m1 & me), e11 = (uint32_t)__popc(m2 & m1 & me);
            const uint32_t e00 = ze - e01, e10 = oe - e11;
            auto sub = [](uint32_t x, uint32_t from, uint32_t k, uint32_t(&out)[4]) {
              out[0] = (from >= 32 ? 0u : x >> from) & lowmask(k);
              out[1] = out[2] = out[3] = 0u;
            };
            uint32_t sz[4], so[4], s00[4], s01[4], s10[4], s11[4];
            sub(Z1[u], za, ze - za, sz);
            sub(O1[u], oa, oe - oa, so);
            sub(c00[u], q00, e00 - q00, s00);
            sub(c01[u], q01, e01 - q01, s01);
            sub(c10[u], q10, e10 - q10, s10);
            sub(c11[u], q11, e11 - q11, s11);
            const TrNode d = tr_node(tab, tab3, cls, vv, nvn, n);
            tr_put_run<1>(d, j + a, r + oa, a01 + q01, a11 + q11, B2, B1, put4, sz, ze - za, so, oe - oa, s00,
                          e00 - q00, s01, e01 - q01, s10, e10 - q10, s11, e11 - q11);
            if (e >= nvu) break;
            a = e;
            vv = pn_sym<T>(w, jb + e) >> 3;
            heads &= heads - 1;
          }
          j += nvu;
          r += lo[u];
          a01 += l01[u];
          a11 += l11[u];
        }
      }
    }
  }
  pdl_trigger();
}

// (k_leaf3 is in wt_kernels.cuh, beside k_leaf_offsets)

}  // namespace wt
