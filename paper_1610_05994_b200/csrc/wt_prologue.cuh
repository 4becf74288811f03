// wt_prologue.cuh -- a1: the one pass over S before the level passes.
//
// Alg. 1 counts symbols per level node (lines 5-6) before each
// level's sweep.  Here no full histogram of S is taken: by Proposition 1
// the size of a level-(l+2) node is the number of symbols of its
// level-l parent node with a given pair of bits (l-th and (l+1)-th MSB), and
// the pass over T_l -- which is sorted by the top l bits -- counts exactly
// that (wt_level.cuh), "progressively".  What is left for the pass over S:
//   * the symbol-range check (any S[j] >= sigma -> WT_ERR_SYMBOL_RANGE);
//   * agg0[t] = symbols of level tile t whose bit L-1 is set (the per-tile
//     ones of B_0, so level 0 needs no look-back);
//   * ones0 = the total of agg0, i.e. the size of level-1 node 1;
//   * with Q (the first pass is a quad, wt_quad.cuh): also per tile the
//     symbols whose top two bits are 01 and 11 (agg01, agg11), and the four
//     level-2 node sizes (hist4, the quad's node table).
// One warp per level tile (2 KiB = 4 x 16 bytes per lane), two tiles in
// flight per warp, no block synchronisation.
#pragma once
#include "wt_device.cuh"
#include "wt_level.cuh"

namespace wt {

constexpr int PRO_THREADS = 256;

template <typename T>
__device__ __forceinline__ uint32_t msb_mask32(uint32_t bit) {
  if (sizeof(T) == 1) return 0x01010101u << bit;
  if (sizeof(T) == 2) return 0x00010001u << bit;
  return 1u << bit;
}

// any symbol of word x (little-endian, sizeof(T) bytes each) >= sigma
template <typename T>
__device__ __forceinline__ bool any_ge(uint32_t x, uint64_t sigma, bool pow2, uint32_t badm) {
  if (pow2) return (x & badm) != 0;  // sigma = 2^L: a mask test
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 4 / (int)sizeof(T); ++j) {
    const uint32_t s = (sizeof(T) == 4) ? x : (x >> (8 * sizeof(T) * j)) & ((1u << (8 * sizeof(T))) - 1u);
    bad |= (uint64_t)s >= sigma;
  }
  return bad;
}

template <typename T, bool Q = false>
__global__ void __launch_bounds__(PRO_THREADS) k_prologue(const T* __restrict__ S, uint64_t n, uint64_t sigma,
                                                          uint32_t L, uint32_t* __restrict__ agg0,
                                                          unsigned long long* __restrict__ ones0,
                                                          int32_t* __restrict__ flag,
                                                          uint32_t* __restrict__ agg01 = nullptr,
                                                          uint32_t* __restrict__ agg11 = nullptr,
                                                          uint32_t* __restrict__ hist4 = nullptr) {
  constexpr uint32_t PER = 16 / sizeof(T);
  constexpr uint32_t TILE = LvTile<T>::TILE;
  constexpr uint32_t VL = TILE / PER / 32;  // 16-byte vectors per lane per tile (4)
  static_assert(VL * PER * 32 == TILE, "tile layout");
  pdl_trigger();  // (launched normally, after the control-block memset) the first k_prep may start waiting
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t)blockIdx.x * (PRO_THREADS / 32) + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * (PRO_THREADS / 32);
  const uint32_t m32 = L ? msb_mask32<T>(L - 1) : 0u;
  const bool pow2 = (sigma & (sigma - 1)) == 0;
  const uint32_t symbits = (8 * sizeof(T) >= 32) ? 0xffffffffu : ((1u << (8 * sizeof(T))) - 1u);
  const uint32_t lowbits = L >= 32 ? 0xffffffffu : ((1u << L) - 1u);
  const uint32_t badm = ~(msb_mask32<T>(0) * (lowbits & symbits));
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const uint64_t nvec = n / PER;
  bool bad = false;
  unsigned long long mine = 0;  // ones of this warp's tiles (lane 0)
  uint32_t h[4] = {0, 0, 0, 0};  // (Q) class totals of this warp's tiles (lane 0)
  for (uint64_t t0 = warp; t0 < ntiles; t0 += 2 * nwarps) {
    uint4 v[2][VL];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int k = 0; k < (int)VL; ++k) {
        const uint64_t idx = (t0 + (uint64_t)u * nwarps) * (TILE / PER) + (uint64_t)k * 32 + lane;
        v[u][k] = (idx < nvec) ? ldg_nc_v4(S + idx * PER) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t t = t0 + (uint64_t)u * nwarps;
      if (t >= ntiles) break;  // warp-uniform
      uint32_t ones = 0, q01 = 0, q11 = 0;
#pragma unroll
      for (int k = 0; k < (int)VL; ++k) {
        ones += (uint32_t)(__popc(v[u][k].x & m32) + __popc(v[u][k].y & m32) + __popc(v[u][k].z & m32) +
                           __popc(v[u][k].w & m32));
        if constexpr (Q) {  // bit L-2 moved onto bit L-1 of the same symbol (L >= 4: no carry across symbols)
          const uint32_t xs[4] = {v[u][k].x, v[u][k].y, v[u][k].z, v[u][k].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t lo = (xs[j] << 1) & m32;
            q11 += __popc(xs[j] & lo);
            q01 += __popc(~xs[j] & lo);
          }
        }
        bad |= any_ge<T>(v[u][k].x, sigma, pow2, badm) | any_ge<T>(v[u][k].y, sigma, pow2, badm) |
               any_ge<T>(v[u][k].z, sigma, pow2, badm) | any_ge<T>(v[u][k].w, sigma, pow2, badm);
      }
      if (t == ntiles - 1) {  // symbols past the last whole vector
        for (uint64_t j = nvec * PER + lane; j < n; j += 32) {
          const uint32_t x = (uint32_t)S[j];
          bad |= (uint64_t)x >= sigma;
          ones += L ? (x >> (L - 1)) & 1u : 0u;
          if constexpr (Q) {
            const uint32_t b1 = (x >> (L - 2)) & 1u, b0 = (x >> (L - 1)) & 1u;
            q11 += b0 & b1;
            q01 += (b0 ^ 1u) & b1;
          }
        }
      }
      const uint32_t tot = __reduce_add_sync(FULL, ones);
      if (lane == 0 && agg0) {
        agg0[t] = tot;
        mine += tot;
      }
      if constexpr (Q) {
        const uint32_t t01 = __reduce_add_sync(FULL, q01), t11 = __reduce_add_sync(FULL, q11);
        if (lane == 0) {
          agg01[t] = t01;
          agg11[t] = t11;
          const uint32_t syms = (uint32_t)min((uint64_t)TILE, n - t * TILE);
          h[0] += syms - tot - t01;
          h[1] += t01;
          h[2] += tot - t11;
          h[3] += t11;
        }
      }
    }
  }
  if (lane == 0 && mine) atomicAdd(ones0, mine);
  if constexpr (Q) {
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (h[c]) atomicAdd(hist4 + c, h[c]);
  }
  if (__any_sync(FULL, bad) && lane == 0) *flag = 2;  // WT_ERR_SYMBOL_RANGE
}

}  // namespace wt
