// wt_pairn.cuh -- the fused final pair of any tree with L >= 2: pass L-2 over
// T_{L-2} writes B_{L-2}, SB_{L-2} and B_{L-1} (a5 with k = 2 at the bottom
// of the tree; Alg. 1 lines 8-13 for levels L-2 and L-1).
//
// T_{L-2} is S stably sorted by the top L-2 bits (Prop. 1), so a
// position j of node v (v = s >> 2) with level-(L-2) bit b1 = bit 1 of s goes
// to T_{L-1} position
//   b1 = 0: j - r(j) + ob[v]        b1 = 1: r(j) + Zn[v]
// (r(j) = level-(L-2) ones before j; {ob, Zn} = the node table the prep built,
// the closed form of Alg. 1's C[node]++ cursors), and B_{L-1} at that position
// is bit 0 of s.  No symbol moves: a lane's run of symbols inside one node
// sends its zeros' bit-0 string (in order) to one destination and its ones'
// bit-0 string to another, both contiguous.
//
// This is k_pair2's execution (wt_pair2.cuh) made general: per warp a ring of
// two 4 KiB TMA tensor copies of T_{L-2} (rows of 128 bytes, 128-byte swizzle;
// two of the level pass's tiles, so its tile prefixes pre[t] apply, one per
// half warp); lane l owns row l (E symbols), compacted as two 64-byte halves,
// 4 symbols at a time, by the 256-entry table (bit 0 / bit 1 of 4 symbols ->
// their level-(L-2) bits, the zeros' and ones' bit-0 strings and the strings'
// position multipliers).  A lane inside one node stores its two strings whole;
// node changes inside a lane split each half's strings into per-node
// substrings (the strings are in position order, so node g's part is the bits
// between the zeros / ones before g's first symbol and after its last).  Every
// string is stored with its interior words plain and its first / last word
// OR-ed into the zero-filled B_{L-1} (the paper's atomic boundary words,
// P:814-821).  No leaves are counted: C comes from B_{L-1}'s superblocks
// afterwards (k_leaf_offsets).  The wavelet matrix (one global node per level)
// runs the same kernel with the node index masked to 0.
#pragma once
#include <cuda.h>

#include "wt_device.cuh"
#include "wt_pair2.cuh"
#include "wt_ptx.cuh"

namespace wt {

template <typename T>
struct PnCfg {
  static constexpr int W = (int)sizeof(T);
  static constexpr int EH = 64 / W;         // symbols per half lane (64 bytes)
  static constexpr int E = 2 * EH;          // symbols per lane: one 128-byte row
  static constexpr int LT = 16 * E;         // symbols per level tile (= LvTile<T>::TILE, 2 KiB): 16 lanes
  static constexpr int WT = 32 * E;         // symbols per warp tile (4 KiB): two level tiles
  static constexpr int G = EH / 4;          // groups of 4 symbols per half
  static constexpr int NH = EH > 32 ? 2 : 1;  // 32-symbol words of a half's bits
  static constexpr int GH = G / NH;         // groups per word
};
constexpr int PN_WARPS = 4;  // independent warps per CTA (they share the table)
constexpr int PN_NB = 2;     // per-warp ring of input tiles
constexpr int PN_WT = 4096;  // bytes per warp tile

struct PnSmem {
  alignas(1024) uint4 ring[PN_WARPS][PN_NB][PN_WT / 16];  // 32 rows of 128 bytes per tile, 128-byte swizzle
  uint2 lut[256];
  alignas(8) unsigned long long bar[PN_WARPS][PN_NB];
};
constexpr size_t pn_smem_bytes() { return sizeof(PnSmem) + 1024; }

// the (bit 0, bit 1) pairs of symbols 4g .. 4g+3 of a lane (w: its 16 words)
// as the table index (bit 2j = bit 0 of symbol j, bit 2j+1 = its bit 1)
template <typename T>
__device__ __forceinline__ uint32_t pn_index(const uint32_t (&w)[16], int g) {
  if constexpr (sizeof(T) == 1) {
    // byte j's two bits to 24 + 2j (masked to 2 bits: no carries into the top byte)
    return ((w[g] & 0x03030303u) * 0x01041040u) >> 24;
  } else if constexpr (sizeof(T) == 2) {
    const uint32_t x = (w[2 * g] & 0x00030003u) | ((w[2 * g + 1] & 0x00030003u) << 4);
    return (x | (x >> 14)) & 0xffu;
  } else {
    // the four low bytes into one word (three byte permutes), then as for bytes
    uint32_t a, b, x;
    asm("prmt.b32 %0, %1, %2, 0x0040;" : "=r"(a) : "r"(w[4 * g]), "r"(w[4 * g + 1]));      // [w0.b0, w1.b0, ..]
    asm("prmt.b32 %0, %1, %2, 0x0040;" : "=r"(b) : "r"(w[4 * g + 2]), "r"(w[4 * g + 3]));  // [w2.b0, w3.b0, ..]
    asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(x) : "r"(a), "r"(b));                       // [w0, w1, w2, w3].b0
    return ((x & 0x03030303u) * 0x01041040u) >> 24;
  }
}

// symbol j of a lane (j may be a run-time value: the word is selected from
// the registers, so the lane's words stay out of local memory)
template <typename T>
__device__ __forceinline__ uint32_t pn_sym(const uint32_t (&w)[16], uint32_t j) {
  constexpr uint32_t SPW = 4 / sizeof(T);
  const uint32_t k = j / SPW;
  uint32_t x = w[0];
#pragma unroll
  for (uint32_t i = 1; i < 16; ++i) x = (k == i) ? w[i] : x;
  if constexpr (sizeof(T) == 1) return (x >> (8 * (j & 3))) & 0xffu;
  else if constexpr (sizeof(T) == 2) return (x >> (16 * (j & 1))) & 0xffffu;
  else return x;
}
// symbol j of a lane, j a compile-time index
template <typename T, int J>
__device__ __forceinline__ uint32_t pn_sym_c(const uint32_t (&w)[16]) {
  if constexpr (sizeof(T) == 1) return (w[J >> 2] >> (8 * (J & 3))) & 0xffu;
  else if constexpr (sizeof(T) == 2) return (w[J >> 1] >> (16 * (J & 1))) & 0xffffu;
  else return w[J];
}
// bit j of the lane: symbol j's node differs from symbol j-1's (j >= 1)
template <typename T, int J, int E>
__device__ __forceinline__ uint64_t pn_heads(const uint32_t (&w)[16], uint32_t prev) {
  if constexpr (J >= E) {
    return 0ull;
  } else {
    const uint32_t nd = pn_sym_c<T, J>(w) >> 2;
    return ((uint64_t)(nd != prev) << J) | pn_heads<T, J + 1, E>(w, nd);
  }
}

// nb <= 32 bits of v at global bit position pos of `bits`: a word wholly
// inside [pos, pos + nb) stored, a partial one OR-ed
__device__ __forceinline__ void pn_put32(uint32_t* bits, uint64_t pos, uint32_t v, uint32_t nb) {
  if (nb == 0) return;
  const uint64_t j = pos >> 5;
  const uint32_t off = (uint32_t)(pos & 31u), end = off + nb;
  const uint32_t w0 = v << off;
  if (off == 0 && end == 32) bits[j] = w0;
  else atomicOr(&bits[j], w0);
  if (end > 32) atomicOr(&bits[j + 1], v >> (32 - off));  // (off > 0 here; end < 64)
}

// bits [a, a + k) of a 64-bit string as two words (k <= 64)
__device__ __forceinline__ void pn_sub(uint64_t s, uint32_t a, uint32_t k, uint32_t (&v)[2]) {
  const uint64_t x = (a >= 64 ? 0ull : (s >> a)) & (k >= 64 ? ~0ull : ((1ull << k) - 1ull));
  v[0] = (uint32_t)x;
  v[1] = (uint32_t)(x >> 32);
}

// one half lane (64 bytes, EH symbols, `nv` of them real): level-(L-2) bits m
// (position order), the zeros' / ones' bit-0 strings and their lengths
template <typename T>
__device__ __forceinline__ void pn_half(const uint32_t (&w)[16], uint32_t nv, const uint2* lut,
                                        uint32_t (&m)[PnCfg<T>::NH], uint64_t& zc, uint64_t& oc, uint32_t& nz,
                                        uint32_t& no) {
  using C = PnCfg<T>;
  constexpr int EH = C::EH, NH = C::NH, GH = C::GH;
  zc = oc = 0;
  nz = no = 0;
  if (nv == (uint32_t)EH) {
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      uint32_t mm = 0, Zs = 0, Os = 0, pz = 1, po = 1;
#pragma unroll
      for (int g = 0; g < GH; ++g) {
        const uint2 e = lut[pn_index<T>(w, h * GH + g)];
        mm |= ((e.x >> 16) & 15u) << (4 * g);
        Zs += (e.x & 15u) * pz;
        Os += (e.x >> 28) * po;
        pz *= e.y & 0xffu;
        po *= e.y >> 8;
      }
      m[h] = mm;
      const uint32_t o = (uint32_t)__popc(mm), z = (uint32_t)(4 * GH) - o;
      zc |= (uint64_t)Zs << nz;
      oc |= (uint64_t)Os << no;
      nz += z;
      no += o;
    }
  } else {
#pragma unroll
    for (int h = 0; h < NH; ++h) m[h] = 0;
    for (uint32_t j = 0; j < nv; ++j) {
      const uint32_t s = pn_sym<T>(w, j);
      const uint32_t b1 = (s >> 1) & 1u, b0 = s & 1u;
      if (NH == 1 || j < 32) m[0] |= b1 << (j & 31);
      else m[NH - 1] |= b1 << (j & 31);
      if (b1) oc |= (uint64_t)b0 << no++;
      else zc |= (uint64_t)b0 << nz++;
    }
  }
}

// nb bits (<= 2 EH <= 128) of the concatenation of two strings a (na bits) and
// b at global bit position pos
template <int EH>
__device__ __forceinline__ void pn_put_cat(uint32_t* bits, uint64_t pos, uint64_t a, uint32_t na, uint64_t b,
                                           uint32_t nb) {
  if (na + nb == 0) return;
  if constexpr (EH == 64) {  // 128-bit strings
    const uint64_t lo = a | (na >= 64 ? 0ull : (b << na));
    const uint64_t hi = na == 0 ? 0ull : (na >= 64 ? b : (b >> (64 - na)));
    const uint32_t v[4] = {(uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32)};
    p2_put4(bits, pos, v, na + nb);
  } else if constexpr (EH == 32) {  // 64-bit strings
    const uint64_t x = a | (b << na);
    const uint32_t v[2] = {(uint32_t)x, (uint32_t)(x >> 32)};
    p2_put(bits, pos, v, na + nb);
  } else {  // 32-bit strings
    pn_put32(bits, pos, (uint32_t)a | ((uint32_t)b << na), na + nb);
  }
}

// B_{L-2} (bits), its superblocks and B_{L-1} (must be zero on entry) from
// T_{L-2} (n symbols, n < 2^32), the level-(L-2) tile prefixes pre[t] and node
// table tab[v] = {ob[v], Zn[v]}.  Warp tiles of 4 KiB (two level tiles); lane
// l owns row l (128 bytes), processed as two 64-byte halves.  A lane inside
// one node stores its two strings whole; a lane that spans nodes splits each
// half's strings at the node changes.
template <typename T>
__global__ void __launch_bounds__(32 * PN_WARPS, 6)
    k_pairn(const T* __restrict__ in, uint32_t n, uint32_t ntiles, const uint32_t* __restrict__ pre,
            const uint2* __restrict__ tab, uint32_t* __restrict__ bits, uint32_t words,
            unsigned long long* __restrict__ sb, uint32_t nsb, uint32_t* __restrict__ B1, uint32_t vmask,
            const int32_t* __restrict__ flag, const __grid_constant__ CUtensorMap tmap) {
  // vmask: all ones for the tree (node v = s >> 2); 0 for the wavelet matrix,
  // whose levels are one global node each (tab[0] = {0, Z_{L-2}})
  using C = PnCfg<T>;
  constexpr int E = C::E, EH = C::EH, WT = C::WT, NH = C::NH;
  extern __shared__ unsigned char pn_raw[];
  // (an offset from the __shared__ array, not an integer round trip: the
  // compiler keeps the shared address space -- LDS / STS instead of generic loads)
  PnSmem& sm = *reinterpret_cast<PnSmem*>(pn_raw + ((1024u - (smem_u32(pn_raw) & 1023u)) & 1023u));
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < 256; i += 32 * PN_WARPS) sm.lut[i] = p2_lut_entry(i);
  if (lane == 0) {
    for (int b = 0; b < PN_NB; ++b) mbar_init(&sm.bar[wid][b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t gw = blockIdx.x * PN_WARPS + wid, nw = gridDim.x * PN_WARPS;
  const uint32_t nwt = (uint32_t)(((uint64_t)n + WT - 1) / WT);  // warp tiles
  const uint64_t nbytes = (uint64_t)n * sizeof(T);
  const uint64_t full_bytes = nbytes & ~127ull;  // the tensor map's whole rows
  auto issue = [&](uint32_t it) {
    const uint32_t tile = gw + it * nw;
    if (tile >= nwt) return;
    const int b = (int)(it % PN_NB);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&sm.bar[wid][b], PN_WT);  // (rows past the tensor's end are zero-filled)
    p2_tma(sm.ring[wid][b], &tmap, (int32_t)(tile * (PN_WT / 128)), &sm.bar[wid][b]);
  };
  pdl_wait();  // T_{L-2}, the tile prefixes, the node table, the zero-filled B_{L-1}
  if (*flag) return;
  if (lane == 0)
    for (uint32_t b = 0; b < PN_NB; ++b) issue(b);
  const uint32_t swz = lane & 7u;
  const uint64_t padded = ((uint64_t)n + 511) & ~511ull;
  const unsigned char* inb = reinterpret_cast<const unsigned char*>(in);
  for (uint32_t it = 0;; ++it) {
    const uint32_t tile = gw + it * nw;
    if (tile >= nwt) break;
    const int b = (int)(it % PN_NB);
    const uint64_t T0 = (uint64_t)tile * WT;
    const uint64_t p0 = T0 + (uint32_t)E * lane;  // the lane's first position
    const uint32_t lt = 2 * tile + (lane >> 4);  // its level tile
    const uint32_t P = lt < ntiles ? __ldg(&pre[lt]) : 0u;
    mbar_wait(&sm.bar[wid][b], (it / PN_NB) & 1u);
    unsigned char* const buf = reinterpret_cast<unsigned char*>(sm.ring[wid][b]);
    const uint64_t B0 = T0 * sizeof(T);
    if (B0 + PN_WT > full_bytes && full_bytes < nbytes) {  // the partial last row: into its swizzled place
      for (uint64_t g = full_bytes + lane; g < nbytes; g += 32) {
        const uint32_t off = (uint32_t)(g - B0), r = off >> 7, c = (off >> 4) & 7u;
        buf[r * 128 + ((c ^ (r & 7u)) << 4) + (off & 15u)] = inb[g];
      }
      __syncwarp();
    }
    const uint32_t nvalid = p0 >= n ? 0u : (uint32_t)min((uint64_t)E, n - p0);
    const uint32_t nv0 = min(nvalid, (uint32_t)EH), nv1 = nvalid - nv0;
    uint32_t w0[16], w1[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 q0 = *reinterpret_cast<const uint4*>(buf + lane * 128 + (((uint32_t)k ^ swz) << 4));
      const uint4 q1 = *reinterpret_cast<const uint4*>(buf + lane * 128 + (((uint32_t)(k + 4) ^ swz) << 4));
      w0[4 * k] = q0.x, w0[4 * k + 1] = q0.y, w0[4 * k + 2] = q0.z, w0[4 * k + 3] = q0.w;
      w1[4 * k] = q1.x, w1[4 * k + 1] = q1.y, w1[4 * k + 2] = q1.z, w1[4 * k + 3] = q1.w;
    }
    uint32_t m0[NH], m1[NH];
    uint64_t zc0, oc0, zc1, oc1;
    uint32_t nz0, no0, nz1, no1;
    pn_half<T>(w0, nv0, sm.lut, m0, zc0, oc0, nz0, no0);
    pn_half<T>(w1, nv1, sm.lut, m1, zc1, oc1, nz1, no1);
    // bitmap words of level L-2 (the last tile's padding words: zero)
    if (p0 < padded) {
      if constexpr (EH == 64) *reinterpret_cast<uint4*>(bits + p0 / 32) = make_uint4(m0[0], m0[1], m1[0], m1[1]);
      else if constexpr (EH == 32) *reinterpret_cast<uint2*>(bits + p0 / 32) = make_uint2(m0[0], m1[0]);
      else bits[p0 / 32] = m0[0] | (m1[0] << 16);
    }
    const uint32_t ones = no0 + no1;
    const uint32_t inc = warp_incl_scan_u32(ones);
    const uint32_t h15 = __shfl_sync(FULL, inc, 15);
    const uint32_t R = inc - ones - ((lane >> 4) ? h15 : 0u);  // ones before the lane, inside its level tile
    const uint32_t P0 = __shfl_sync(FULL, P, 0);
    if ((p0 & 511u) == 0 && p0 < n) sb[p0 / 512] = P + R;
    if (tile + 1 == nwt && lane == 31) sb[nsb - 1] = P0 + inc;
    if (nvalid) {
      const uint32_t v = (pn_sym_c<T, 0>(w0) >> 2) & vmask;
      const uint32_t vlast =
          ((nv1 == (uint32_t)EH ? pn_sym_c<T, EH - 1>(w1) : nv1 ? pn_sym<T>(w1, nv1 - 1) : pn_sym<T>(w0, nv0 - 1)) >> 2) &
          vmask;
      const uint32_t pr = (uint32_t)p0 - P - R;  // zeros before the lane (mod 2^32: positions < n < 2^32)
      if (v == vlast) {  // the lane inside one node: both strings whole
        const uint2 tv = __ldg(&tab[v]);
        pn_put_cat<EH>(B1, (uint64_t)(uint32_t)(pr + tv.x), zc0, nz0, zc1, nz1);
        pn_put_cat<EH>(B1, (uint64_t)(uint32_t)(P + R + tv.y), oc0, no0, oc1, no1);
      } else {
        // each half: its runs of one node [a, e) with node vv
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t nvh = h ? nv1 : nv0;
          if (nvh == 0) continue;
          const uint32_t(&w)[16] = h ? w1 : w0;
          const uint32_t(&m)[NH] = h ? m1 : m0;
          const uint64_t zc = h ? zc1 : zc0, oc = h ? oc1 : oc0;
          const uint32_t ph = (uint32_t)p0 + (h ? (uint32_t)EH : 0u);  // the half's first position
          const uint32_t Rh = P + R + (h ? no0 : 0u);                  // level-(L-2) ones before it
          uint32_t vv = (pn_sym_c<T, 0>(w) >> 2) & vmask;
          uint64_t heads = pn_heads<T, 1, EH>(w, vv) & (nvh >= 64 ? ~0ull : ((1ull << nvh) - 1ull));
          const uint64_t m64 = (uint64_t)m[0] | (NH == 2 ? ((uint64_t)m[NH - 1] << 32) : 0ull);
          uint32_t a = 0, oa = 0;  // run start, ones before it in the half
          for (;;) {
            const uint32_t e = heads ? (uint32_t)(__ffsll((long long)heads) - 1) : nvh;
            const uint64_t em = e >= 64 ? ~0ull : ((1ull << e) - 1ull);
            const uint32_t oe = (uint32_t)__popcll(m64 & em);
            const uint2 tv = __ldg(&tab[vv]);
            const uint64_t dz = (uint32_t)(ph + a - Rh - oa + tv.x), d1 = (uint32_t)(Rh + oa + tv.y);
            const uint32_t kz = (e - a) - (oe - oa), ko = oe - oa;
            if constexpr (EH == 64) {
              uint32_t sz[2], so[2];
              pn_sub(zc, a - oa, kz, sz);
              pn_sub(oc, oa, ko, so);
              p2_put(B1, dz, sz, kz);
              p2_put(B1, d1, so, ko);
            } else {  // strings of <= 32 bits
              const uint32_t za = a - oa;
              pn_put32(B1, dz, (za >= 32 ? 0u : (uint32_t)zc >> za) & lowmask(kz), kz);
              pn_put32(B1, d1, (oa >= 32 ? 0u : (uint32_t)oc >> oa) & lowmask(ko), ko);
            }
            if (e >= nvh) break;
            a = e;
            oa = oe;
            {  // node of symbol e of the half: its bytes in the (swizzled) ring slot
              const uint32_t off = (uint32_t)(E * lane + (h ? EH : 0) + e) * (uint32_t)sizeof(T);
              const uint32_t r = off >> 7, c = (off >> 4) & 7u;
              vv = ((uint32_t)*reinterpret_cast<const T*>(buf + r * 128 + ((c ^ (r & 7u)) << 4) + (off & 15u)) >> 2) &
                   vmask;
            }
            heads &= heads - 1;
          }
        }
      }
    }
    __syncwarp();  // every lane is done with the slot: refill it
    if (lane == 0) issue(it + PN_NB);
  }
  pdl_trigger();
}

}  // namespace wt
