// wt_hist.cuh -- a1: one pass over S computing
//   * H[c] = #{j : S[j] = c}, c < 2^L, accumulated into node_offsets (then
//     scanned in place into C).  Alg. 1 counts per level (lines 5-6,
//     P:539-540); by Proposition 1 every level's counters are a
//     coarsening of H, so this one pass serves all levels;
//   * agg0[t] = number of symbols of level-0 tile t whose bit L-1 is set (the
//     per-tile ones of B_0, so level 0 never needs a look-back);
//   * the symbol-range flag (any S[j] >= sigma -> WT_ERR_SYMBOL_RANGE).
// Three counting strategies by alphabet size: u32 shared-memory bins
// (2^L <= 4096, several copies), packed u16 shared-memory bins (2^L <= 65536)
// and run-aggregated global atomics (larger alphabets).
#pragma once
#include "wt_device.cuh"
#include "wt_level.cuh"

namespace wt {

constexpr int HIST_G = 8;  // level tiles per block iteration

template <typename T>
__device__ __forceinline__ uint32_t msb_mask32(uint32_t bit) {
  if (sizeof(T) == 1) return 0x01010101u << bit;
  if (sizeof(T) == 2) return 0x00010001u << bit;
  return 1u << bit;
}

// Block-cooperative sweep over S in groups of HIST_G level tiles.  vec(v,
// valid) is called warp-uniformly for each 16-byte vector (lanes of a warp
// hold 32 consecutive vectors, always inside one level tile); scal(x) for the
// < 16 bytes past the last whole vector.  red: shared scratch [HIST_G].
template <typename T, int B, class VecFn, class ScalarFn>
__device__ __forceinline__ void hist_tiles(const T* __restrict__ S, uint64_t n, uint32_t L,
                                           uint32_t* __restrict__ agg0, uint32_t* red, VecFn vec, ScalarFn scal) {
  constexpr uint32_t PER = 16 / sizeof(T);
  constexpr uint32_t TILE = LvTile<T>::TILE;
  constexpr uint32_t VT = TILE / PER;  // vectors per level tile
  constexpr int K = HIST_G * (int)VT / B;
  static_assert(K * B == HIST_G * (int)VT && VT % 32 == 0, "group layout");
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t bit = L ? L - 1 : 0;
  const uint32_t m32 = L ? msb_mask32<T>(bit) : 0u;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const uint64_t ngroups = (ntiles + HIST_G - 1) / HIST_G;
  const uint64_t nvec = n / PER;
  const uint64_t last_tile = ntiles ? ntiles - 1 : 0;
  if (agg0 && tid < HIST_G) red[tid] = 0;
  __syncthreads();
  for (uint64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const uint64_t v0 = g * HIST_G * VT;
    uint4 v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = v0 + (uint64_t)k * B + tid;
      v[k] = (idx < nvec) ? ldg_nc_v4(S + idx * PER) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = v0 + (uint64_t)k * B + tid;
      const bool valid = idx < nvec;
      uint32_t ones = 0;
      if (valid)
        ones = (uint32_t)(__popc(v[k].x & m32) + __popc(v[k].y & m32) + __popc(v[k].z & m32) +
                          __popc(v[k].w & m32));
      if (agg0) {
        const uint32_t w = __reduce_add_sync(FULL, ones);
        if (lane == 0 && w) atomicAdd(&red[(k * B + (int)warp * 32) / (int)VT], w);
      }
      vec(v[k], valid);
    }
    if (v0 + HIST_G * VT > nvec) {  // this group holds the scalar tail (all inside the last tile)
      uint32_t tail = 0;
      for (uint64_t j = nvec * PER + tid; j < n; j += B) {
        const uint32_t x = (uint32_t)S[j];
        tail += (x >> bit) & 1u;
        scal(x);
      }
      if (agg0 && L && tail) atomicAdd(&red[last_tile - g * HIST_G], tail);
    }
    if (agg0) {
      __syncthreads();
      if (tid < HIST_G) {
        const uint64_t t = g * HIST_G + tid;
        if (t < ntiles) agg0[t] = red[tid];
        red[tid] = 0;
      }
      __syncthreads();
    }
  }
}

// ---- tiny alphabets (L <= 2, sigma <= 4): no bins at all.  Per 32-bit word,
// SWAR lane accumulators count symbols with bit 0 set, bit 1 set and both;
// H[0..3] follow by inclusion-exclusion.  Symbols outside [0, 2^L) are
// caught by a mask test, values in [sigma, 2^L) by their counts.
template <typename T>
__global__ void __launch_bounds__(512) k_hist_bits(const T* __restrict__ S, uint64_t n, uint64_t sigma, uint32_t L,
                                                   unsigned long long* __restrict__ H, uint32_t* __restrict__ agg0,
                                                   int32_t* __restrict__ flag) {
  __shared__ uint32_t red[HIST_G];
  __shared__ unsigned long long tot[4];
  if (threadIdx.x < 4) tot[threadIdx.x] = 0;
  constexpr uint32_t PER = 16 / sizeof(T);
  const uint32_t lo = msb_mask32<T>(0);                                   // bit 0 of every symbol
  const uint32_t badm = ~(lo * ((1u << L) - 1u));                         // bits no symbol < 2^L has
  const uint32_t msk2 = L >= 2 ? lo : 0u;
  unsigned long long c1 = 0, c2 = 0, c3 = 0, cnt = 0;
  uint32_t badbits = 0;
  auto lanesum = [](uint32_t a) -> uint32_t {  // sum of the per-symbol lanes of a
    if (sizeof(T) == 1) return (a * 0x01010101u) >> 24;
    if (sizeof(T) == 2) return (a * 0x00010001u) >> 16;
    return a;
  };
  hist_tiles<T, 512>(S, n, L, agg0, red,
                     [&](const uint4& v, bool valid) {
                       if (!valid) return;
                       const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                       uint32_t a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
                       for (int k = 0; k < 4; ++k) {
                         badbits |= w[k] & badm;
                         const uint32_t b = w[k] & lo, t = (w[k] >> 1) & msk2;
                         a1 += b;
                         a2 += t;
                         a3 += b & t;
                       }
                       c1 += lanesum(a1);
                       c2 += lanesum(a2);
                       c3 += lanesum(a3);
                       cnt += PER;
                     },
                     [&](uint32_t x) {
                       badbits |= (x >> L);
                       c1 += x & 1u;
                       c2 += (x >> 1) & (L >= 2 ? 1u : 0u);
                       c3 += x & (x >> 1) & (L >= 2 ? 1u : 0u);
                       cnt += 1;
                     });
  // block totals of H[0..3]
  unsigned long long h[4] = {cnt - c1 - c2 + c3, c1 - c3, c2 - c3, c3};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    unsigned long long x = h[k];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&tot[k], x);
  }
  if (__syncthreads_or(badbits != 0)) {
    if (threadIdx.x == 0) *flag = 2;  // WT_ERR_SYMBOL_RANGE
  }
  if (threadIdx.x < (1u << L)) {
    const unsigned long long x = tot[threadIdx.x];
    if (x) {
      atomicAdd(&H[threadIdx.x], x);
      if (threadIdx.x >= sigma) *flag = 2;
    }
  }
}

// ---- small alphabets: u32 shared bins, `copies` copies (warp w uses w % copies)
template <typename T>
__global__ void __launch_bounds__(512) k_hist_smem(const T* __restrict__ S, uint64_t n, uint64_t sigma, uint32_t L,
                                                   uint32_t copies, unsigned long long* __restrict__ H,
                                                   uint32_t* __restrict__ agg0, int32_t* __restrict__ flag) {
  extern __shared__ uint32_t sh_hist[];
  __shared__ uint32_t red[HIST_G];
  const uint32_t nbins = 1u << L;
  for (uint32_t i = threadIdx.x; i < copies * nbins; i += blockDim.x) sh_hist[i] = 0;
  __syncthreads();
  uint32_t* my = sh_hist + ((threadIdx.x >> 5) % copies) * nbins;
  bool bad = false;
  auto one = [&](uint32_t x) {
    if (x < sigma) atomicAdd(&my[x], 1u);
    else bad = true;
  };
  hist_tiles<T, 512>(S, n, L, agg0, red,
                     [&](const uint4& v, bool valid) {
                       if (!valid) return;
                       const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
                       for (uint32_t k = 0; k < 16 / sizeof(T); ++k) one((uint32_t)e[k]);
                     },
                     one);
  if (bad) *flag = 2;  // WT_ERR_SYMBOL_RANGE
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) {
    uint32_t s = 0;
    for (uint32_t c = 0; c < copies; ++c) s += sh_hist[c * nbins + i];
    if (s) atomicAdd(&H[i], (unsigned long long)s);
  }
}

// ---- medium alphabets: packed 16-bit shared bins (two per word).  A bin
// reaching 0x8000 moves 0x8000 to the global count, so a half never carries
// into its neighbour.
template <typename T>
__global__ void __launch_bounds__(1024) k_hist_smem16(const T* __restrict__ S, uint64_t n, uint64_t sigma,
                                                      uint32_t L, unsigned long long* __restrict__ H,
                                                      uint32_t* __restrict__ agg0, int32_t* __restrict__ flag) {
  extern __shared__ uint32_t sh16[];
  __shared__ uint32_t red[HIST_G];
  const uint32_t nbins = 1u << L;
  for (uint32_t i = threadIdx.x; i < (nbins + 1) / 2; i += blockDim.x) sh16[i] = 0;
  __syncthreads();
  bool bad = false;
  auto one = [&](uint32_t x) {
    if (x < sigma) {
      const uint32_t shv = (x & 1u) * 16u;
      const uint32_t old = atomicAdd(&sh16[x >> 1], 1u << shv);
      if (((old >> shv) & 0xffffu) == 0x7fffu) {
        atomicAdd(&H[x], 0x8000ull);
        atomicSub(&sh16[x >> 1], 0x8000u << shv);
      }
    } else {
      bad = true;
    }
  };
  hist_tiles<T, 1024>(S, n, L, agg0, red,
                      [&](const uint4& v, bool valid) {
                        if (!valid) return;
                        const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
                        for (uint32_t k = 0; k < 16 / sizeof(T); ++k) one((uint32_t)e[k]);
                      },
                      one);
  if (bad) *flag = 2;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < (nbins + 1) / 2; i += blockDim.x) {
    const uint32_t w = sh16[i];
    if (w & 0xffffu) atomicAdd(&H[2 * i], (unsigned long long)(w & 0xffffu));
    if (w >> 16) atomicAdd(&H[2 * i + 1], (unsigned long long)(w >> 16));
  }
}

// ---- large alphabets: global atomics, one per run of equal symbols inside
// each warp's 32 consecutive vectors (runs are common in integer data).
template <typename T>
__global__ void __launch_bounds__(512) k_hist_global(const T* __restrict__ S, uint64_t n, uint64_t sigma,
                                                     uint32_t L, unsigned long long* __restrict__ H,
                                                     uint32_t* __restrict__ agg0, int32_t* __restrict__ flag) {
  __shared__ uint32_t red[HIST_G];
  constexpr uint32_t PER = 16 / sizeof(T);
  const uint32_t lane = threadIdx.x & 31;
  bool bad = false;
  auto vec = [&](const uint4& v, bool valid) {
    uint32_t x[PER];
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (uint32_t k = 0; k < PER; ++k) x[k] = valid ? (uint32_t)e[k] : 0xffffffffu;
    uint32_t prev = __shfl_up_sync(FULL, x[PER - 1], 1);
    if (lane == 0) prev = ~x[0];
    uint32_t headmask = 0;
#pragma unroll
    for (uint32_t k = 0; k < PER; ++k) {
      const uint32_t p = (k == 0) ? prev : x[k - 1];
      if (x[k] != p) headmask |= 1u << k;
    }
    const uint32_t first_head = headmask ? (uint32_t)(__ffs(headmask) - 1) : PER;
    const uint32_t lanes_with_head = __ballot_sync(FULL, headmask != 0);
    const uint32_t later = lanes_with_head & ~((2u << lane) - 1u);
    const uint32_t next_lane = later ? (uint32_t)(__ffs(later) - 1) : 32u;
    const uint32_t nl_first = __shfl_sync(FULL, first_head, next_lane & 31);
    const uint32_t next_lane_pos = (next_lane < 32) ? next_lane * PER + nl_first : 32 * PER;
    if (!valid) return;
#pragma unroll
    for (uint32_t k = 0; k < PER; ++k) {
      if (headmask & (1u << k)) {
        const uint32_t rest = headmask & ~((2u << k) - 1u);
        const uint32_t nxt = rest ? lane * PER + (uint32_t)(__ffs(rest) - 1) : next_lane_pos;
        // past-the-end lanes hold 0xffffffff, a distinct run head, so a run never extends into them
        if (x[k] < sigma) atomicAdd(&H[x[k]], (unsigned long long)(nxt - (lane * PER + k)));
        else bad = true;
      }
    }
  };
  auto one = [&](uint32_t x) {
    if (x < sigma) atomicAdd(&H[x], 1ull);
    else bad = true;
  };
  hist_tiles<T, 512>(S, n, L, agg0, red, vec, one);
  if (bad) *flag = 2;
}

}  // namespace wt
