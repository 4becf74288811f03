// wt_quad.cuh -- a5: the interior fused group of k = 2 levels (sm_100a).
//
// One pass over T_l (l + 2 <= L - 2) does the work of Alg. 1's sweeps l and
// l+1: it writes B_l and SB_l, the bits of level l+1 (B_{l+1}, in
// T_{l+1} order, into a zero-filled level; its superblocks come from a scan
// afterwards) and T_{l+2} -- T_l stably partitioned inside every level-l node
// v by the PAIR of bits (sh, sh-1), sh = L-1-l, i.e. into the four level-(l+2)
// nodes 4v..4v+3 (Proposition 1).  T_{l+1} is never materialised.
//
// Closed-form destinations.  With c = 2 b_l + b_{l+1} the class of a symbol,
// g_c(v) the size of level-(l+2) node 4v+c, P_c(v) the class-c symbols of the
// nodes before v and G_c(j) the class-c symbols of T_l[0, j), the symbol at
// position j of node v (start N(v)) goes to
//     T_{l+2}:  N(v) + sum_{c' < c} g_c'(v) + (G_c(j) - P_c(v))
//     its B_{l+1} bit (T_{l+1} position): N(v) + (b_l ? g_0 + g_1 : 0)
//               + (ranks of its b_l class in v before j)
// so a tile needs only G_c at its first position (tile prefixes of the class
// counts, scanned by the k_prep before it from the counts the previous pass
// made: "progressive counting") and the node tables g, P (the
// level-(l+2) node sizes the previous pass counted; <= 64 nodes, held in
// shared memory for the whole kernel).
//
// Execution: persistent 256-thread CTAs, 8 KiB tiles through a double-buffered
// TMA bulk ring; every thread owns 32 consecutive bytes.
//   1. masks of bits sh, sh-1 (SWAR), B_l words, warp scans of the class counts;
//   2. tile-exclusive class ranks, SB_l, class ranks at the segment (node) starts;
//   3. (one warp) the run layout: per segment 4 symbol runs and 2 bit strings,
//      each run staged congruent mod 16 bytes to its HBM destination;
//   4. every symbol stored to its stage slot, every thread's B_{l+1}
//      substrings OR-ed into a bit stage aligned to the global words;
//   5. runs copied out as aligned 16-byte vectors (+ edge elements), counting
//      the next pass's per-tile ones (and class pairs) on the way; the bit
//      strings' words stored (their first and last words OR-ed: shared with
//      neighbouring strings and tiles -- the paper's atomic boundary words,
//      P:814-821);
//   6. per run: the tile counts and the next level's node sizes flushed as
//      global atomics (a handful per run).
#pragma once
#include "wt_device.cuh"
#include "wt_ptx.cuh"
#include "wt_level.cuh"

namespace wt {

#ifndef WT_Q_THREADS
#define WT_Q_THREADS 256
#endif
#ifndef WT_Q_MINB
#define WT_Q_MINB 4
#endif
constexpr uint32_t Q_THREADS = WT_Q_THREADS;   // (experiment builds override the geometry)
constexpr uint32_t Q_WARPS = Q_THREADS / 32;
constexpr uint32_t Q_TILE_BYTES = 32 * Q_THREADS;  // 32 bytes per thread
constexpr uint32_t Q_MAXL = 6;                 // quads run at levels l <= Q_MAXL (2^l nodes)
constexpr uint32_t Q_MAXSEG = 1u << Q_MAXL;    // segments (nodes) per tile
constexpr uint32_t Q_MAXRUN = 4 * Q_MAXSEG;
constexpr uint32_t Q_MAXSTR = 2 * Q_MAXSEG;
constexpr uint32_t Q_MINB = WT_Q_MINB;         // CTAs per SM

template <typename T>
struct QCfg {
  static constexpr uint32_t TILE = Q_TILE_BYTES / sizeof(T);  // symbols per tile
  static constexpr uint32_t E = TILE / Q_THREADS;             // symbols per thread: 32 / 16 / 8
  static constexpr uint32_t CT = LvTile<T>::TILE;             // count tile (the k_prep prefixes' granularity)
  static constexpr uint32_t V16 = 16 / sizeof(T);             // symbols per 16-byte chunk
  static constexpr uint32_t STAGE = TILE + V16 * Q_MAXRUN;    // staged symbols (+ alignment slack per run)
  static constexpr uint32_t BSW = TILE / 32 + 2 * Q_MAXSTR;   // bit-stage words
  static constexpr uint32_t MAXPIECE = TILE / CT + 2 * Q_MAXRUN;
  static_assert(TILE % CT == 0 && CT % 512 == 0, "tiles hold whole count tiles and superblocks");
  static_assert(E * sizeof(T) == 32, "32 bytes per thread");
};

template <typename T>
struct QSmem {
  alignas(128) uint8_t in[2][Q_TILE_BYTES];
  alignas(16) T stage[QCfg<T>::STAGE];
  uint32_t bst[QCfg<T>::BSW];
  uint2 pc[QCfg<T>::MAXPIECE];  // per (run, destination count tile): {ones of bit sh-2, c01 | c11 << 16 of bits sh-2, sh-3}
  uint32_t wsA[Q_WARPS], wsB[Q_WARPS];
  // node table (the whole kernel): level-(l+2) sizes g, class prefixes P, starts N
  uint4 ng[Q_MAXSEG], nP[Q_MAXSEG];
  uint32_t nstart[Q_MAXSEG + 1];
  // segments of the current tile (double-buffered by tile parity)
  uint32_t nseg[2];
  uint32_t seg_a[2][Q_MAXSEG + 1], seg_v[2][Q_MAXSEG];
  uint4 segpre[Q_MAXSEG + 1];  // class counts of the tile before each segment start
  // runs (segment-major, class-minor) and strings (segment-major, b_l-minor)
  uint32_t r_dest[Q_MAXRUN], r_len[Q_MAXRUN], r_sb[Q_MAXRUN], r_cb[Q_MAXRUN + 1], r_pb[Q_MAXRUN + 1];
  uint32_t r_eb[Q_MAXRUN + 1], r_fc[Q_MAXRUN], r_he[Q_MAXRUN], r_ts[Q_MAXRUN];  // edge prefix, first chunk, head end, tail start
  uint2 lut[256];  // B_{l+1} string compaction, 4 symbols per entry (q_lut_entry)
  uint32_t s_pos[Q_MAXSTR], s_len[Q_MAXSTR], s_sw[Q_MAXSTR], s_wb[Q_MAXSTR + 1];
  alignas(8) unsigned long long bar[2];
};
template <typename T>
constexpr size_t quad_smem_bytes() {
  return sizeof(QSmem<T>);
}

// largest i in [0, cnt) with a[i] <= x (a[0] <= x, a ascending)
__device__ __forceinline__ uint32_t q_upper(const uint32_t* a, uint32_t cnt, uint32_t x) {
  uint32_t lo = 0, hi = cnt;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

// nb <= 32 bits of v at bit position pos of the bit stage (OR)
__device__ __forceinline__ void q_put_bits(uint32_t* bst, uint32_t pos, uint32_t v, uint32_t nb) {
  if (nb == 0) return;
  const uint32_t w = pos >> 5, o = pos & 31u;
  atomicOr(&bst[w], v << o);
  if (o + nb > 32) atomicOr(&bst[w + 1], v >> (32 - o));
}

// 256-entry table, index = the level-l bits of 4 symbols (low nibble) and their
// level-(l+1) bits (high nibble):
//   .x = [3:0] level-(l+1) bits of the symbols with level-l bit 0, in order;
//        [11:8] those of the symbols with level-l bit 1
//   .y = [7:0] 2^(#zeros), [15:8] 2^(#ones): the strings' position multipliers
__device__ __forceinline__ uint2 q_lut_entry(uint32_t idx) {
  uint32_t zb = 0, nz = 0, ob = 0, no = 0;
  for (uint32_t j = 0; j < 4; ++j) {
    const uint32_t b0 = (idx >> j) & 1u, b1 = (idx >> (4 + j)) & 1u;
    if (b0) ob |= b1 << no++;
    else zb |= b1 << nz++;
  }
  return make_uint2(zb | (ob << 8), (1u << nz) | ((1u << no) << 8));
}

// Parameters of one quad launch.
struct QuadArgs {
  uint32_t n, ntq, sh, nodes;  // nodes = 2^l
  const uint32_t* pre1;        // count-tile prefixes of T_l: ones of bit sh
  const uint32_t* pre01;       //   class 01 (bit sh = 0, bit sh-1 = 1)
  const uint32_t* pre11;       //   class 11
  const uint32_t* gcnt;        // level-(l+2) node sizes, 4 per level-l node
  uint32_t* bits;              // B_l
  unsigned long long* sb;      // SB_l
  uint32_t nsb, words;
  uint32_t* bits1;             // B_{l+1} (zero on entry)
  uint32_t* agg_next;          // ones of bit sh-2 per count tile of T_{l+2}
  uint32_t* agg01_next;        // (D = 2) class counts of bits sh-2, sh-3 per count tile
  uint32_t* agg11_next;
  uint32_t* cnt_next;          // D = 1: level-(l+3) node sizes; D = 2: level-(l+4)
  uint32_t D;
  const int32_t* flag;
};

template <typename T>
__global__ void __launch_bounds__(Q_THREADS, Q_MINB) k_quad(const T* __restrict__ in, T* __restrict__ out,
                                                            QuadArgs a) {
  using C = QCfg<T>;
  constexpr uint32_t TILE = C::TILE, E = C::E, CT = C::CT, V16 = C::V16;
  extern __shared__ __align__(128) uint8_t q_raw[];  // (no runtime realignment: the compiler keeps the shared space)
  QSmem<T>& s = *reinterpret_cast<QSmem<T>*>(q_raw);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t sh = a.sh;
  const uint32_t p0 = tid * E;  // the thread's first symbol in the tile

  if (tid == 0) {
    mbar_init(&s.bar[0], 1);
    mbar_init(&s.bar[1], 1);
    fence_mbar_init();
  }
  for (uint32_t i = tid; i < C::BSW; i += Q_THREADS) s.bst[i] = 0;
  for (uint32_t i = tid; i < C::MAXPIECE; i += Q_THREADS) s.pc[i] = make_uint2(0, 0);
  for (uint32_t i = tid; i < 256; i += Q_THREADS) s.lut[i] = q_lut_entry(i);
  pdl_wait();
  if (*a.flag) return;
  // node table: exclusive prefixes of the level-(l+2) sizes over the level-l nodes
  if (warp == 0) {
    uint4 carry = make_uint4(0, 0, 0, 0);
    for (uint32_t v0 = 0; v0 < a.nodes; v0 += 32) {
      const uint32_t v = v0 + lane;
      const uint4 g = v < a.nodes ? *reinterpret_cast<const uint4*>(a.gcnt + 4 * v) : make_uint4(0, 0, 0, 0);
      const uint4 i = make_uint4(warp_incl_scan_u32(g.x), warp_incl_scan_u32(g.y), warp_incl_scan_u32(g.z),
                                 warp_incl_scan_u32(g.w));
      if (v < a.nodes) {
        const uint4 P = make_uint4(carry.x + i.x - g.x, carry.y + i.y - g.y, carry.z + i.z - g.z, carry.w + i.w - g.w);
        s.ng[v] = g;
        s.nP[v] = P;
        s.nstart[v] = P.x + P.y + P.z + P.w;
      }
      carry.x += __shfl_sync(FULL, i.x, 31);
      carry.y += __shfl_sync(FULL, i.y, 31);
      carry.z += __shfl_sync(FULL, i.z, 31);
      carry.w += __shfl_sync(FULL, i.w, 31);
    }
    if (lane == 0) s.nstart[a.nodes] = a.n;
  }
  __syncthreads();

  const uint32_t n = a.n;
  auto issue = [&](uint32_t t, uint32_t b) {  // TMA of tile t's whole 16-byte chunks into buffer b
    const uint32_t j0 = t * TILE;
    const uint32_t cnt = min(TILE, n - j0);
    const uint32_t bytes = (cnt * (uint32_t)sizeof(T)) & ~15u;
    mbar_arrive_expect_tx(&s.bar[b], bytes);
    if (bytes) bulk_g2s(s.in[b], in + j0, bytes, &s.bar[b]);
  };
  if (tid == 0 && blockIdx.x < a.ntq) issue(blockIdx.x, 0);

  uint32_t it = 0;
  for (uint32_t t = blockIdx.x; t < a.ntq; t += gridDim.x, ++it) {
    const uint32_t b = it & 1u, sp = it & 1u;
    const uint32_t j0 = t * TILE;
    const uint32_t cnt = min(TILE, n - j0);
    if (tid == 0 && t + gridDim.x < a.ntq) issue(t + gridDim.x, b ^ 1u);
    // ---- segments of the tile (warp 0): the level-l nodes it intersects
    if (warp == 0) {
      uint32_t base = 0;
      for (uint32_t v0 = 0; v0 < a.nodes; v0 += 32) {
        const uint32_t v = v0 + lane;
        bool hit = false;
        uint32_t st = 0;
        if (v < a.nodes) {
          st = s.nstart[v];
          const uint32_t en = s.nstart[v + 1];
          hit = en > st && en > j0 && st < j0 + cnt;
        }
        const uint32_t bm = __ballot_sync(FULL, hit);
        if (hit) {
          const uint32_t k = base + __popc(bm & lanemask_lt());
          s.seg_a[sp][k] = st > j0 ? st - j0 : 0u;
          s.seg_v[sp][k] = v;
        }
        base += __popc(bm);
      }
      if (lane == 0) {
        s.nseg[sp] = base;
        s.seg_a[sp][base] = cnt;
      }
    }
    // ---- phase 1: masks, B_l, warp scans of the class counts
    mbar_wait(&s.bar[b], (it >> 1) & 1u);
    const uint32_t tma_el = ((cnt * (uint32_t)sizeof(T)) & ~15u) / (uint32_t)sizeof(T);
    if (cnt > tma_el && p0 + E > tma_el && p0 < cnt) {  // the tail past the last whole chunk (last tile)
      T* ib = reinterpret_cast<T*>(s.in[b]);
      for (uint32_t e = max(p0, tma_el); e < min(p0 + E, cnt); ++e) ib[e] = in[j0 + e];
    }
    // the thread's 32 bytes (read again in phase 4: not kept live across the barriers)
    auto load_words = [&](uint32_t (&w)[8]) {
      const uint4* src = reinterpret_cast<const uint4*>(s.in[b] + 32 * tid);
      const uint32_t h = (tid >> 2) & 1u;  // rotated halves: conflict-free 16-byte loads
      const uint4 x0 = src[h], x1 = src[h ^ 1u];
      const uint4 lo = h ? x1 : x0, hi = h ? x0 : x1;
      w[0] = lo.x, w[1] = lo.y, w[2] = lo.z, w[3] = lo.w, w[4] = hi.x, w[5] = hi.y, w[6] = hi.z, w[7] = hi.w;
    };
    const uint32_t vm = p0 >= cnt ? 0u : lowmask(min(E, cnt - p0));
    uint32_t m0, m1;
    {
      uint32_t w[8];
      load_words(w);
      m0 = swar_bits<T, 8>(w, sh) & vm;
      m1 = swar_bits<T, 8>(w, sh - 1) & vm;
    }
    const uint32_t c11 = __popc(m0 & m1), c01 = __popc(~m0 & m1), c1 = __popc(m0);
    {  // B_l words (LSB-first)
      uint32_t word = m0;
      if constexpr (E == 16) word |= __shfl_down_sync(FULL, m0, 1) << 16;
      if constexpr (E == 8)
        word |= (__shfl_down_sync(FULL, m0, 1) << 8) | (__shfl_down_sync(FULL, m0, 2) << 16) |
                (__shfl_down_sync(FULL, m0, 3) << 24);
      const uint32_t gw = (j0 + p0) / 32;
      if ((p0 % 32) == 0 && gw < a.words) a.bits[gw] = word;
    }
    const uint32_t vA = c01 | (c11 << 16), vB = c1 - c11;  // (01, 11), 10
    const uint32_t iA = warp_incl_scan_u32(vA), iB = warp_incl_scan_u32(vB);
    if (lane == 31) {
      s.wsA[warp] = iA;
      s.wsB[warp] = iB;
    }
    __syncthreads();  // ---- sync 1
    // ---- phase 2: tile-exclusive class ranks, SB_l, ranks at the segment starts
    uint32_t eA = iA - vA, eB = iB - vB, tA = 0, tB = 0;
#pragma unroll
    for (uint32_t k = 0; k < Q_WARPS; ++k) {
      const uint32_t xa = s.wsA[k], xb = s.wsB[k];
      if (k < warp) eA += xa, eB += xb;
      tA += xa, tB += xb;
    }
    const uint32_t e01 = eA & 0xffffu, e11 = eA >> 16, e10 = eB;
    const uint32_t pv = min(p0, cnt);
    const uint32_t e00 = pv - e01 - e11 - e10;
    const uint32_t ct0 = (TILE / CT) * t;  // the tile's first count tile
    const uint32_t pre1 = a.pre1[ct0];
    if ((p0 % 512) == 0 && j0 + p0 < n) a.sb[(j0 + p0) / 512] = pre1 + e10 + e11;
    const uint32_t t01 = tA & 0xffffu, t11 = tA >> 16, t10 = tB;
    const uint32_t t00 = cnt - t01 - t11 - t10;
    if (tid == 0 && t + 1 == a.ntq) a.sb[a.nsb - 1] = pre1 + t10 + t11;
    const uint32_t nseg = s.nseg[sp];
    const uint32_t* seg_a = s.seg_a[sp];
    const uint32_t mc00 = ~m0 & ~m1 & vm, mc01 = ~m0 & m1, mc10 = m0 & ~m1, mc11 = m0 & m1;
    uint32_t sf = 0;  // the segment holding the thread's first symbol
    if (p0 < cnt) {
      sf = q_upper(seg_a, nseg, p0);
      for (uint32_t k = (seg_a[sf] == p0 ? sf : sf + 1); k < nseg && seg_a[k] < p0 + E; ++k) {
        const uint32_t lm = lowmask(seg_a[k] - p0);
        s.segpre[k] = make_uint4(e00 + __popc(mc00 & lm), e01 + __popc(mc01 & lm), e10 + __popc(mc10 & lm),
                                 e11 + __popc(mc11 & lm));
      }
    }
    if (tid == 0) s.segpre[nseg] = make_uint4(t00, t01, t10, t11);
    __syncthreads();  // ---- sync 2
    // ---- phase 3 (warp 0): run and string layout
    if (warp == 0) {
      const uint32_t G01 = a.pre01[ct0], G11 = a.pre11[ct0], G10 = pre1 - G11;
      const uint32_t G00 = j0 - G01 - G10 - G11;
      // carries of the packed prefix sums: X = stage symbols | full chunks << 16,
      // Y = pieces | bit-stage words << 16, Z = edge symbols
      uint32_t cX = 0, cY = 0, cZ = 0;
      for (uint32_t s0 = 0; s0 < nseg; s0 += 32) {
        const uint32_t k = s0 + lane;
        uint32_t len[4] = {0, 0, 0, 0}, dst[4] = {0, 0, 0, 0};
        uint32_t zpos = 0, zlen = 0, opos = 0, olen = 0, zw = 0, ow = 0;
        uint32_t sX = 0, sY = 0, sZ = 0;
        if (k < nseg) {
          const uint32_t v = s.seg_v[sp][k];
          const uint4 g = s.ng[v], P = s.nP[v];
          const uint32_t N = s.nstart[v];
          const uint4 q0 = s.segpre[k], q1 = s.segpre[k + 1];
          len[0] = q1.x - q0.x, len[1] = q1.y - q0.y, len[2] = q1.z - q0.z, len[3] = q1.w - q0.w;
          const uint32_t r00 = G00 + q0.x - P.x, r01 = G01 + q0.y - P.y, r10 = G10 + q0.z - P.z,
                         r11 = G11 + q0.w - P.w;  // class ranks in v before the segment start
          dst[0] = N + r00;
          dst[1] = N + g.x + r01;
          dst[2] = N + g.x + g.y + r10;
          dst[3] = N + g.x + g.y + g.z + r11;
          zpos = N + r00 + r01, zlen = len[0] + len[1];
          opos = N + g.x + g.y + r10 + r11, olen = len[2] + len[3];
          zw = zlen ? ((zpos & 31u) + zlen + 31) / 32 : 0u;
          ow = olen ? ((opos & 31u) + olen + 31) / 32 : 0u;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t e = dst[c] + len[c];
            const uint32_t fc0 = (dst[c] + V16 - 1) / V16, fc1 = e / V16;
            const uint32_t nf = fc1 > fc0 ? fc1 - fc0 : 0u;
            const uint32_t he = min(fc0 * V16, e), ts = max(fc1 * V16, he);
            const uint32_t npc = len[c] ? (e - 1) / CT - dst[c] / CT + 1 : 0u;
            sX += (len[c] + V16) | (nf << 16);
            sY += npc;
            sZ += (he - dst[c]) + (e - ts);
          }
          sY += (zw + ow) << 16;
        }
        uint32_t xX = cX, xY = cY, xZ = cZ;
        if (nseg > 1) {
          xX += warp_incl_scan_u32(sX) - sX;
          xY += warp_incl_scan_u32(sY) - sY;
          xZ += warp_incl_scan_u32(sZ) - sZ;
        }
        if (k < nseg) {
          uint32_t oS = xX & 0xffffu, oC = xX >> 16, oP = xY & 0xffffu, oE = xZ;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t r = 4 * k + c;
            const uint32_t e = dst[c] + len[c];
            const uint32_t fc0 = (dst[c] + V16 - 1) / V16, fc1 = e / V16;
            const uint32_t nf = fc1 > fc0 ? fc1 - fc0 : 0u;
            const uint32_t he = min(fc0 * V16, e), ts = max(fc1 * V16, he);
            s.r_dest[r] = dst[c];
            s.r_len[r] = len[c];
            s.r_sb[r] = oS + ((dst[c] - oS) & (V16 - 1));  // congruent to the destination mod 16 bytes
            s.r_cb[r] = oC;
            s.r_pb[r] = oP;
            s.r_eb[r] = oE;
            s.r_fc[r] = fc0;
            s.r_he[r] = he;
            s.r_ts[r] = ts;
            oS += len[c] + V16;
            oC += nf;
            oP += len[c] ? (e - 1) / CT - dst[c] / CT + 1 : 0u;
            oE += (he - dst[c]) + (e - ts);
          }
          const uint32_t xW = xY >> 16;
          s.s_pos[2 * k] = zpos, s.s_len[2 * k] = zlen, s.s_sw[2 * k] = xW, s.s_wb[2 * k] = xW;
          s.s_pos[2 * k + 1] = opos, s.s_len[2 * k + 1] = olen, s.s_sw[2 * k + 1] = xW + zw,
                      s.s_wb[2 * k + 1] = xW + zw;
        }
        if (nseg > 1) {
          cX = __shfl_sync(FULL, xX + sX, 31);
          cY = __shfl_sync(FULL, xY + sY, 31);
          cZ = __shfl_sync(FULL, xZ + sZ, 31);
        } else {
          cX = xX + sX, cY = xY + sY, cZ = xZ + sZ;
        }
      }
      if (lane == 0) {
        s.r_cb[4 * nseg] = cX >> 16;
        s.r_pb[4 * nseg] = cY & 0xffffu;
        s.r_eb[4 * nseg] = cZ;
        s.s_wb[2 * nseg] = cY >> 16;
      }
    }
    __syncthreads();  // ---- sync 3
    // ---- phase 4: stage every symbol, OR the B_{l+1} substrings
    if (p0 < cnt) {
      const T* ib = reinterpret_cast<const T*>(s.in[b]);
      const uint32_t stage0 = smem_u32(s.stage);
      for (uint32_t k = sf; k < nseg && seg_a[k] < p0 + E; ++k) {
        const uint32_t lo = seg_a[k] > p0 ? seg_a[k] - p0 : 0u;
        const uint32_t hi = min(seg_a[k + 1] - p0, E);
        const uint32_t lm = lowmask(lo);
        const uint4 q = s.segpre[k];
        // the thread's first stage slot of each class in this segment
        const uint32_t r0 = s.r_sb[4 * k + 0] + e00 + __popc(mc00 & lm) - q.x;
        const uint32_t r1 = s.r_sb[4 * k + 1] + e01 + __popc(mc01 & lm) - q.y;
        const uint32_t r2 = s.r_sb[4 * k + 2] + e10 + __popc(mc10 & lm) - q.z;
        const uint32_t r3 = s.r_sb[4 * k + 3] + e11 + __popc(mc11 & lm) - q.w;
        // B_{l+1} substrings' offsets: zeros / ones of the segment before
        const uint32_t zo = r0 - s.r_sb[4 * k] + r1 - s.r_sb[4 * k + 1];
        const uint32_t oo = r2 - s.r_sb[4 * k + 2] + r3 - s.r_sb[4 * k + 3];
        uint32_t Z = 0, O = 0, nz, no;
        if (lo == 0 && hi == E) {
          // stage cursors: shared-window byte addresses (< 2^16: the CTA's
          // shared memory is < 64 KiB) packed as 16-bit fields
          constexpr uint32_t W = sizeof(T);
          constexpr bool ABS = sizeof(QSmem<T>) + 2048 <= 65536;  // (else cursors relative to the stage)
          const uint32_t sb0 = ABS ? stage0 : 0u;
          uint32_t P01 = (sb0 + W * r0) | ((sb0 + W * r1) << 16);
          uint32_t P23 = (sb0 + W * r2) | ((sb0 + W * r3) << 16);
          uint32_t w[8];
          load_words(w);
#pragma unroll
          for (uint32_t i = 0; i < E; ++i) {
            const bool p0b = (m0 >> i) & 1u, p1b = (m1 >> i) & 1u;
            const uint32_t P = p0b ? P23 : P01;
            const uint32_t pos = __byte_perm(P, 0u, p1b ? 0x4432u : 0x4410u);
            // (st.shared.u8 / u16 stores the low bits: no masking of the symbol)
            const uint32_t x = W == 4 ? w[i] : w[(i * W) / 4] >> (8 * ((i * W) % 4));
            st_shared<T>(ABS ? pos : stage0 + pos, x);
            const uint32_t inc = p1b ? (W << 16) : W;
            P23 += p0b ? inc : 0u;
            P01 += p0b ? 0u : inc;
          }
          // the strings, 4 symbols per table lookup (multiply-add appends)
          uint32_t pz = 1, po = 1;
#pragma unroll
          for (uint32_t g = 0; g < E / 4; ++g) {
            const uint2 e = s.lut[((m0 >> (4 * g)) & 15u) | (((m1 >> (4 * g)) & 15u) << 4)];
            Z += (e.x & 15u) * pz;
            O += ((e.x >> 8) & 15u) * po;
            pz *= e.y & 0xffu;
            po *= e.y >> 8;
          }
          nz = __popc(~m0 & vm);
          no = __popc(m0);
        } else {
          uint32_t c0 = r0, c1 = r1, c2 = r2, c3 = r3;
          nz = no = 0;
          for (uint32_t i = lo; i < hi; ++i) {
            const uint32_t x = (uint32_t)ib[p0 + i];
            const uint32_t b0 = (m0 >> i) & 1u, b1 = (m1 >> i) & 1u;
            const uint32_t pos = b0 ? (b1 ? c3 : c2) : (b1 ? c1 : c0);
            s.stage[pos] = (T)x;
            if (b0) {
              O |= b1 << no;
              ++no;
              if (b1) ++c3;
              else ++c2;
            } else {
              Z |= b1 << nz;
              ++nz;
              if (b1) ++c1;
              else ++c0;
            }
          }
        }
        q_put_bits(s.bst, 32 * s.s_sw[2 * k] + (s.s_pos[2 * k] & 31u) + zo, Z, nz);
        q_put_bits(s.bst, 32 * s.s_sw[2 * k + 1] + (s.s_pos[2 * k + 1] & 31u) + oo, O, no);
      }
    }
    __syncthreads();  // ---- sync 4
    // ---- phase 5: runs out (whole 16-byte chunks as vectors, then the edge
    // symbols), next-level counts per piece; bit strings out
    {
      const uint32_t nruns = 4 * nseg;
      const uint32_t sh2 = sh - 2;
      const uint32_t M2 = bitmask32<T>(sh2);
      const bool D2 = a.D == 2;
      const uint32_t nch = s.r_cb[nruns];
      // each thread a contiguous range of chunks (one run lookup, then a walk)
      const uint32_t per = (nch + Q_THREADS - 1) / Q_THREADS;
      const uint32_t qb = min(nch, tid * per), qe = min(nch, qb + per);
      uint32_t r = qb < qe ? q_upper(s.r_cb, nruns, qb) : 0u;  // (runs without chunks share r_cb with the next: the last wins)
      for (uint32_t qi = qb; qi < qe; ++qi) {
        while (s.r_cb[r + 1] <= qi) ++r;
        const uint32_t dst = s.r_dest[r];
        const uint32_t kc = s.r_fc[r] + (qi - s.r_cb[r]);
        const uint32_t e0 = kc * V16;
        const uint4 x = *reinterpret_cast<const uint4*>(&s.stage[s.r_sb[r] + (e0 - dst)]);
        *reinterpret_cast<uint4*>(out + e0) = x;
        const uint32_t piece = s.r_pb[r] + e0 / CT - dst / CT;
        const uint32_t ones = __popc(x.x & M2) + __popc(x.y & M2) + __popc(x.z & M2) + __popc(x.w & M2);
        if (ones) atomicAdd(&s.pc[piece].x, ones);
        if (D2) {  // bit sh-3 moved onto bit sh-2 of the same symbol
          const uint32_t yx = (x.x << 1) & M2, yy = (x.y << 1) & M2, yz = (x.z << 1) & M2, yw = (x.w << 1) & M2;
          const uint32_t p11 = __popc(x.x & yx) + __popc(x.y & yy) + __popc(x.z & yz) + __popc(x.w & yw);
          const uint32_t p01 = __popc(yx) + __popc(yy) + __popc(yz) + __popc(yw) - p11;
          if (p01 | p11) atomicAdd(&s.pc[piece].y, p01 | (p11 << 16));
        }
      }
      const uint32_t ned = s.r_eb[nruns];
      for (uint32_t qi = tid; qi < ned; qi += Q_THREADS) {
        const uint32_t r = q_upper(s.r_eb, nruns, qi);
        const uint32_t dst = s.r_dest[r], he = s.r_he[r];
        const uint32_t k = qi - s.r_eb[r];
        const uint32_t e = k < he - dst ? dst + k : s.r_ts[r] + (k - (he - dst));
        const uint32_t x = (uint32_t)s.stage[s.r_sb[r] + (e - dst)];
        out[e] = (T)x;
        const uint32_t piece = s.r_pb[r] + e / CT - dst / CT;
        const uint32_t b2 = (x >> sh2) & 1u;
        if (b2) atomicAdd(&s.pc[piece].x, 1u);
        if (D2 && ((x >> (sh2 - 1)) & 1u)) atomicAdd(&s.pc[piece].y, b2 ? 0x10000u : 1u);
      }
      const uint32_t nstr = 2 * nseg, nw = s.s_wb[nstr];
      for (uint32_t wi = tid; wi < nw; wi += Q_THREADS) {
        const uint32_t k = q_upper(s.s_wb, nstr, wi);
        const uint32_t i = wi - s.s_wb[k];
        const uint32_t nwk = s.s_wb[k + 1] - s.s_wb[k];
        const uint32_t v = s.bst[s.s_sw[k] + i];
        s.bst[s.s_sw[k] + i] = 0;
        uint32_t* g = a.bits1 + (s.s_pos[k] >> 5) + i;
        if (i == 0 || i + 1 == nwk) {
          if (v) atomicOr(g, v);
        } else {
          *g = v;
        }
      }
    }
    __syncthreads();  // ---- sync 5
    // ---- phase 6: per run, the count tiles' counts and the next level's node sizes
    {
      const uint32_t nruns = 4 * nseg;
      const bool D2 = a.D == 2;
      for (uint32_t r = tid; r < nruns; r += Q_THREADS) {
        const uint32_t len = s.r_len[r];
        if (len == 0) continue;
        const uint32_t dst = s.r_dest[r];
        const uint32_t pb = s.r_pb[r], pe = s.r_pb[r + 1];
        uint32_t ones = 0, p01 = 0, p11 = 0;
        for (uint32_t p = pb; p < pe; ++p) {
          const uint2 c = s.pc[p];
          s.pc[p] = make_uint2(0, 0);
          const uint32_t ct = dst / CT + (p - pb);
          if (c.x) atomicAdd(a.agg_next + ct, c.x);
          if (D2) {
            if (c.y & 0xffffu) atomicAdd(a.agg01_next + ct, c.y & 0xffffu);
            if (c.y >> 16) atomicAdd(a.agg11_next + ct, c.y >> 16);
          }
          ones += c.x, p01 += c.y & 0xffffu, p11 += c.y >> 16;
        }
        const uint32_t x = 4 * s.seg_v[sp][r / 4] + (r & 3u);  // the run's level-(l+2) node
        if (D2) {
          const uint32_t q00 = len - ones - p01, q10 = ones - p11;
          uint32_t* cn = a.cnt_next + 4 * x;
          if (q00) atomicAdd(cn + 0, q00);
          if (p01) atomicAdd(cn + 1, p01);
          if (q10) atomicAdd(cn + 2, q10);
          if (p11) atomicAdd(cn + 3, p11);
        } else {
          if (len - ones) atomicAdd(a.cnt_next + 2 * x, len - ones);
          if (ones) atomicAdd(a.cnt_next + 2 * x + 1, ones);
        }
      }
    }
  }
  pdl_trigger();
}

}  // namespace wt
