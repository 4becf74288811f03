// wt_l2.cuh -- a tree of two levels (sigma <= 4: the DNA-like workload, the
// paper's rna.* datasets) built in ONE pass over S.
//
// With L = 2 the levels are (Alg. 1, Prop. 1):
//   B_0 = bit 1 of every symbol, in S order (level 0 is one node);
//   B_1 = bit 0 of the symbols whose bit 1 is 0, in S order (node 0 of level
//         1, positions [0, Z)), then bit 0 of those whose bit 1 is 1 (node 1,
//         positions [Z, n)), Z = the zeros of level 0.
// So B_1 is two stream compactions of S's bit-0 plane.  A tile's zeros'
// bits go to B_1 at (T0 - P) -- P = the ones of level 0 before the tile -- and
// its ones' bits at Z + P.  P comes from a decoupled look-back over the
// tiles (published right after the tile's counts, waited for after its
// compaction work); Z is only known once every tile is counted, so the ones'
// bits go to a one-stream buffer at P and a second small kernel moves the
// stream to bit Z of B_1 (one read + one write of n/16 bytes on DNA-like
// input, instead of a second read of S).  Words shared by two tiles' runs
// (the paper's atomic boundary words) are written by the tile that
// holds the word's first bit; the others' bits go to a per-tile side word
// that k_l2_side ORs in.  B_0's superblocks are written by the pass (P known),
// B_1's by the final scan from the finished bitmap.
//
// Tiles: 256 threads x 8 chunks of 16 bytes (chunk c = k*256 + t, coalesced
// loads), 32768 / 16384 / 8192 symbols for 1 / 2 / 4-byte symbols.  1-byte
// symbols compact 4 symbols per table lookup: the 2 bits of 4 symbols are
// gathered into one byte by one multiply, and a 256-entry table gives their
// level-0 bits and both compacted strings.
#pragma once
#include "wt_prologue.cuh"

namespace wt {

constexpr int L2_THREADS = 256;
constexpr int L2_VEC = 8;  // 16-byte chunks per thread

template <typename T>
struct L2Tile {
  static constexpr int A = 16 / (int)sizeof(T);         // symbols per chunk
  static constexpr int TS = L2_THREADS * L2_VEC * A;    // symbols per tile
  static constexpr int SW = TS / 32 + 4;                // stage words per stream
  static_assert(TS % 512 == 0, "tiles hold whole superblocks");
};

struct L2Args {
  uint32_t* B0;                // level 0 bitmap words
  uint32_t* B1;                // level 1 bitmap words (the zeros' run written here)
  uint32_t* ost;               // the ones' run of level 1, from bit 0 (workspace)
  unsigned long long* SB0;     // level 0 superblocks
  uint32_t* side;              // per tile: first partial word of the zeros' run, of the ones' run
  unsigned long long* cnt;     // leaf counts, packed {H0 | H1 << 32, H2 | H3 << 32}
  uint32_t* ticket;
  int32_t* flag;
  LookbackState lb;
  uint64_t n, sigma, ntiles, nsb;
};

// 256-entry table for 1-byte symbols: index = the (bit 0, bit 1) pairs of 4
// symbols (bit 2j = bit 0 of symbol j, bit 2j+1 = its bit 1).  Entry:
// [3:0] bit 0 of the symbols with bit 1 = 0, in order; [6:4] their number;
// [11:8] bit 0 of the symbols with bit 1 = 1; [14:12] their number;
// [19:16] bit 1 of the four symbols (level-0 bits).
__device__ __forceinline__ uint32_t l2_lut_entry(uint32_t idx) {
  uint32_t zb = 0, nz = 0, ob = 0, no = 0, m1 = 0;
  for (uint32_t j = 0; j < 4; ++j) {
    const uint32_t b0 = (idx >> (2 * j)) & 1u, b1 = (idx >> (2 * j + 1)) & 1u;
    m1 |= b1 << j;
    if (b1) ob |= b0 << no++;
    else zb |= b0 << nz++;
  }
  return zb | (nz << 4) | (ob << 8) | (no << 12) | (m1 << 16);
}

template <typename T>
__device__ __forceinline__ uint32_t l2_sym(const uint4& q, int j) {
  const uint32_t w = j * (int)sizeof(T) / 4;
  const uint32_t x = w == 0 ? q.x : w == 1 ? q.y : w == 2 ? q.z : q.w;
  if (sizeof(T) == 1) return (x >> (8 * (j & 3))) & 0xffu;
  if (sizeof(T) == 2) return (x >> (16 * (j & 1))) & 0xffffu;
  return x;
}

// One chunk: level-0 bits m1 (A bits), the zeros' bit-0 string Z (nz bits)
// and the ones' bit-0 string O (no bits), of its first nvalid symbols.
template <typename T>
__device__ __forceinline__ void l2_chunk(const uint4& q, uint32_t nvalid, const uint32_t* lut, uint32_t& m1,
                                         uint32_t& Z, uint32_t& nz, uint32_t& O, uint32_t& no) {
  constexpr int A = L2Tile<T>::A;
  m1 = Z = nz = O = no = 0;
  if (sizeof(T) == 1 && nvalid == (uint32_t)A) {
    const uint32_t xs[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int wi = 0; wi < 4; ++wi) {
      // (x & 0x03030303) * (2^24 + 2^18 + 2^12 + 2^6): byte j's two bits land at
      // 24 + 2j (no carries into the top byte)
      const uint32_t idx = ((xs[wi] & 0x03030303u) * 0x01041040u) >> 24;
      const uint32_t e = lut[idx];
      m1 |= ((e >> 16) & 15u) << (4 * wi);
      Z |= (e & 15u) << nz;
      nz += (e >> 4) & 7u;
      O |= ((e >> 8) & 15u) << no;
      no += (e >> 12) & 7u;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < A; ++j) {
    if ((uint32_t)j < nvalid) {
      const uint32_t s = l2_sym<T>(q, j);
      const uint32_t b1 = (s >> 1) & 1u, b0 = s & 1u;
      m1 |= b1 << j;
      if (b1) O |= b0 << no++;
      else Z |= b0 << nz++;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(L2_THREADS, 2) k_l2(const T* __restrict__ S, L2Args a) {
  using Cfg = L2Tile<T>;
  constexpr int A = Cfg::A, TS = Cfg::TS, SW = Cfg::SW, NW = L2_THREADS / 32;
  __shared__ uint32_t lut[256];
  __shared__ uint32_t zst[SW], ost[SW];
  __shared__ uint32_t wsum[NW][L2_VEC];  // per warp and k: ones (then their exclusive prefix over warps)
  __shared__ uint32_t ksum[L2_VEC + 1];  // per k: the tile's ones of chunk row k, exclusive prefix over k
  __shared__ uint32_t s_red[NW][2];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_P;
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (sizeof(T) == 1) lut[t] = l2_lut_entry(t);
  for (uint32_t i = t; i < (uint32_t)SW; i += L2_THREADS) zst[i] = 0, ost[i] = 0;
  pdl_wait();  // (the control block is zeroed by a memset before this launch)
  if (t == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t T0 = tile * (uint64_t)TS;
  const uint64_t n = a.n;
  // ---- loads (chunk c = k * 256 + t: a warp reads 512 consecutive bytes per k)
  uint4 v[L2_VEC];
  uint32_t nv[L2_VEC];
#pragma unroll
  for (int k = 0; k < L2_VEC; ++k) {
    const uint64_t pos = T0 + (uint64_t)(k * L2_THREADS + t) * A;
    nv[k] = pos >= n ? 0u : (uint32_t)min((uint64_t)A, n - pos);
    if (nv[k] == (uint32_t)A) {
      v[k] = ldg_nc_v4(S + pos);
    } else {
      uint32_t w[4] = {0, 0, 0, 0};
      for (uint32_t j = 0; j < nv[k]; ++j)
        w[j * sizeof(T) / 4] |= (uint32_t)S[pos + j] << (8 * sizeof(T) * (j % (4 / sizeof(T))));
      v[k] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  // ---- range check, per chunk: level-0 bits and the two bit-0 strings
  const bool pow2 = (a.sigma & (a.sigma - 1)) == 0;
  const uint32_t badm = ~(msb_mask32<T>(0) * 3u);  // (sigma = 4: any bit above the two)
  bool bad = false;
  uint32_t m1[L2_VEC], Zc[L2_VEC], nz[L2_VEC], Oc[L2_VEC], no[L2_VEC];
  uint32_t h1 = 0, h3 = 0;  // symbols 1 and 3 (the ones in the two strings)
#pragma unroll
  for (int k = 0; k < L2_VEC; ++k) {
    bad |= any_ge<T>(v[k].x, a.sigma, pow2, badm) | any_ge<T>(v[k].y, a.sigma, pow2, badm) |
           any_ge<T>(v[k].z, a.sigma, pow2, badm) | any_ge<T>(v[k].w, a.sigma, pow2, badm);
    l2_chunk<T>(v[k], nv[k], lut, m1[k], Zc[k], nz[k], Oc[k], no[k]);
    h1 += (uint32_t)__popc(Zc[k]);
    h3 += (uint32_t)__popc(Oc[k]);
  }
  if (__any_sync(FULL, bad) && lane == 0) *a.flag = 2;  // WT_ERR_SYMBOL_RANGE
  // ---- level-0 bitmap words: 32 / A consecutive lanes hold one word (chunks c, c+1, ...)
#pragma unroll
  for (int k = 0; k < L2_VEC; ++k) {
    uint32_t w = m1[k] << (A * (lane % (32 / A)));
#pragma unroll
    for (int o = 1; o < 32 / A; o <<= 1) w |= __shfl_xor_sync(FULL, w, o);
    const uint64_t pos = T0 + (uint64_t)(k * L2_THREADS + t) * A;
    if (lane % (32 / A) == 0 && pos < ((n + 511) & ~511ull)) a.B0[pos / 32] = w;  // (padding words: zero)
  }
  // ---- ones (= the ones' string lengths) per chunk: exclusive prefix in position order
  uint32_t inc[L2_VEC / 2];
#pragma unroll
  for (int p = 0; p < L2_VEC / 2; ++p) inc[p] = warp_incl_scan_u32(no[2 * p] | (no[2 * p + 1] << 16));
  if (lane == 31) {
#pragma unroll
    for (int p = 0; p < L2_VEC / 2; ++p) wsum[warp][2 * p] = inc[p] & 0xffffu, wsum[warp][2 * p + 1] = inc[p] >> 16;
  }
  {  // leaf counts of symbols 1 and 3, per warp then per tile
    uint32_t x = h1, y = h3;
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o), y += __shfl_xor_sync(FULL, y, o);
    if (lane == 0) s_red[warp][0] = x, s_red[warp][1] = y;
  }
  __syncthreads();
  if (t < (uint32_t)L2_VEC) {  // thread k: exclusive prefix over warps of row k, and the row total
    uint32_t acc = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t x = wsum[w][t];
      wsum[w][t] = acc;
      acc += x;
    }
    ksum[t] = acc;
  }
  __syncthreads();
  uint32_t Otile = 0;
  if (t == 0) {  // rows' exclusive prefix, the tile's ones; publish them (look-back aggregate)
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < L2_VEC; ++k) {
      const uint32_t x = ksum[k];
      ksum[k] = acc;
      acc += x;
    }
    ksum[L2_VEC] = acc;
    Otile = acc;
    lb_publish(a.lb, tile, tile == 0 ? ST_PREFIX : ST_AGG, 1, acc);
    uint32_t x = 0, y = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) x += s_red[w][0], y += s_red[w][1];
    const uint64_t valid = min((uint64_t)TS, n - T0);
    const uint32_t Ztile = (uint32_t)valid - acc;
    atomicAdd(a.cnt, (unsigned long long)(Ztile - x) | ((unsigned long long)x << 32));
    atomicAdd(a.cnt + 1, (unsigned long long)(acc - y) | ((unsigned long long)y << 32));
  }
  __syncthreads();
  // ---- the strings into the tile's two bit stages (tile-relative bit positions)
  uint32_t preo[L2_VEC];
#pragma unroll
  for (int k = 0; k < L2_VEC; ++k) {
    const uint32_t wi = (k & 1) ? (inc[k >> 1] >> 16) : (inc[k >> 1] & 0xffffu);
    preo[k] = ksum[k] + wsum[warp][k] + wi - no[k];
    const uint32_t c = (uint32_t)(k * L2_THREADS) + t;
    const uint32_t prez = c * A - preo[k];  // (chunks before c are full)
    if (nz[k]) {
      const uint32_t j = prez >> 5, o = prez & 31u;
      atomicOr(&zst[j], Zc[k] << o);
      if (o && (Zc[k] >> (32 - o))) atomicOr(&zst[j + 1], Zc[k] >> (32 - o));
    }
    if (no[k]) {
      const uint32_t j = preo[k] >> 5, o = preo[k] & 31u;
      atomicOr(&ost[j], Oc[k] << o);
      if (o && (Oc[k] >> (32 - o))) atomicOr(&ost[j + 1], Oc[k] >> (32 - o));
    }
  }
  // ---- the tile's prefix P (ones of level 0 before it)
  if (warp == 0) {
    const uint64_t P = lookback(a.lb, tile, __shfl_sync(FULL, Otile, 0), 1, true);
    if (lane == 0) s_P = P;
  }
  __syncthreads();
  const uint64_t P = s_P;
  const uint32_t Ot = ksum[L2_VEC];
  const uint64_t valid = min((uint64_t)TS, n - T0);
  const uint32_t Zt = (uint32_t)valid - Ot;
  // level-0 superblocks: every 32 chunks (512 symbols of 1 byte; generally 512 / A chunks)
#pragma unroll
  for (int k = 0; k < L2_VEC; ++k) {
    const uint32_t c = (uint32_t)(k * L2_THREADS) + t;
    const uint64_t pos = T0 + (uint64_t)c * A;
    if ((c * A) % 512 == 0 && pos < n) a.SB0[pos / 512] = P + preo[k];
  }
  if (tile + 1 == a.ntiles && t == 0) a.SB0[a.nsb - 1] = P + Ot;
  // ---- the two runs: words whose first bit lies in the run are stored, the
  // first word (if it starts before the run) goes to the side word
  auto emit = [&](const uint32_t* st, uint64_t start, uint32_t len, uint32_t* dst, uint32_t* side) {
    const uint32_t base = (uint32_t)(start & 31u);
    const uint64_t w0 = start >> 5;
    const uint32_t nw = len ? (base + len + 31) / 32 : 0;
    for (uint32_t j = t; j < nw; j += L2_THREADS) {
      const uint32_t lo = st[j], pv = j ? st[j - 1] : 0u;
      const uint32_t word = base ? ((lo << base) | (pv >> (32 - base))) : lo;
      if (j == 0 && base) *side = word;
      else dst[w0 + j] = word;
    }
    if (t == 0 && (nw == 0 || base == 0)) *side = 0;
  };
  emit(zst, T0 - P, Zt, a.B1, a.side + 2 * tile);
  emit(ost, P, Ot, a.ost, a.side + 2 * tile + 1);
  pdl_trigger();
}

// The side words: a run's first word when another tile holds its first bit.
template <int TS>
__global__ void k_l2_side(const uint32_t* __restrict__ side, const unsigned long long* __restrict__ SB0,
                          uint64_t ntiles, uint32_t* __restrict__ B1, uint32_t* __restrict__ ost,
                          const int32_t* __restrict__ flag) {
  pdl_wait();
  const uint64_t tile = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tile < ntiles && !*flag) {
    const uint64_t T0 = tile * (uint64_t)TS, P = SB0[T0 / 512];
    const uint32_t z = side[2 * tile], o = side[2 * tile + 1];
    if (z) atomicOr(&B1[(T0 - P) >> 5], z);
    if (o) atomicOr(&ost[P >> 5], o);
  }
  pdl_trigger();
}

// The ones' run moved behind the zeros' run: B_1 bit Z + q = one-stream bit
// q, q < O; B_1 words from Z / 32 to the level's end (zero padding included).
// One thread per two words.
__global__ void k_l2_shift(const uint32_t* __restrict__ ost, const unsigned long long* __restrict__ SB0, uint64_t n,
                           uint64_t nsb, uint64_t W, uint32_t* __restrict__ B1, const int32_t* __restrict__ flag) {
  pdl_wait();
  if (*flag) return;
  const uint64_t O = SB0[nsb - 1], Z = n - O;
  const uint64_t wz = Z >> 5;
  const uint32_t s = (uint32_t)(Z & 31u);
  const uint64_t owords = (O + 31) >> 5;  // one-stream words holding bits
  const uint64_t i0 = 2 * ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x);
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    const uint64_t i = i0 + d;  // B_1 word wz + i
    if (wz + i >= W) break;
    const uint32_t cur = i < owords ? ost[i] : 0u;
    uint32_t word;
    if (s == 0) {
      word = cur;
    } else {
      const uint32_t prev = (i >= 1 && i - 1 < owords) ? ost[i - 1] : 0u;
      word = (cur << s) | (i ? prev >> (32 - s) : 0u);
      if (i == 0) word |= B1[wz] & ((1u << s) - 1u);  // the zeros' last bits share the word
    }
    B1[wz + i] = word;
  }
  pdl_trigger();
}

}  // namespace wt
