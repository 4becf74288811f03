// wt_kernels.cuh -- the hot path of the levelwise wavelet-tree build (sm_100a).
//
// Steps (PAPER.md = P:n):
//   a1 k_hist_*      H[c] = #{j : S[j] = c} plus the symbol-range flag.  Alg. 1
//                    counts per level (lines 5-6); by Prop. 1
//                     every level's counters are a coarsening of H,
//                    so one pass over S serves all levels.
//   a2 k_scan        C = exclusive_scan(H) (line 7), in place in the
//                    caller's node_offsets; then the per-level node tables.
//   a3 k_level<.,1>  level l < L-1: stable segmented bit-partition of T_l:
//                    bitmap words by ballot, rank by warp/block scan +
//                    decoupled look-back, superblocks, scatter to T_{l+1}.
//   a4 k_level<.,0>  level L-1: bitmap + superblocks only.
#pragma once
#include "wt_device.cuh"

namespace wt {

// ============================================================ a1 histogram

// Small alphabets (2^L bins fit in shared memory): per-warp-group private
// shared-memory histograms, merged into the global counts at block exit.
template <typename T>
__global__ void __launch_bounds__(512) k_hist_smem(const T* __restrict__ S, uint64_t n, uint64_t sigma,
                                                   uint32_t nbins, uint32_t copies,
                                                   unsigned long long* __restrict__ H,
                                                   int32_t* __restrict__ flag) {
  extern __shared__ uint32_t sh_hist[];
  for (uint32_t i = threadIdx.x; i < copies * nbins; i += blockDim.x) sh_hist[i] = 0;
  __syncthreads();
  uint32_t* my = sh_hist + ((threadIdx.x >> 5) % copies) * nbins;
  bool bad = false;
  constexpr uint32_t PER = 16 / sizeof(T);
  const uint64_t nvec = n / PER;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nvec; q += stride) {
    const uint4 v = ldg_nc_v4(S + q * PER);
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (uint32_t k = 0; k < PER; ++k) {
      const uint32_t x = (uint32_t)e[k];
      if (x < sigma) atomicAdd(&my[x], 1u);
      else bad = true;
    }
  }
  for (uint64_t j = nvec * PER + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const uint32_t x = (uint32_t)S[j];
    if (x < sigma) atomicAdd(&my[x], 1u);
    else bad = true;
  }
  if (bad) *flag = 2;  // WT_ERR_SYMBOL_RANGE
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) {
    uint32_t s = 0;
    for (uint32_t c = 0; c < copies; ++c) s += sh_hist[c * nbins + i];
    if (s) atomicAdd(&H[i], (unsigned long long)s);
  }
}

// Large alphabets: global atomics, aggregated over runs of equal symbols
// inside each warp's 32 x 16-byte chunk (runs are common in integer data).
template <typename T>
__global__ void __launch_bounds__(256) k_hist_global(const T* __restrict__ S, uint64_t n, uint64_t sigma,
                                                     unsigned long long* __restrict__ H,
                                                     int32_t* __restrict__ flag) {
  constexpr uint32_t PER = 16 / sizeof(T);
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nvec = n / PER;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t wid = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  bool bad = false;
  const uint64_t nchunks = (nvec + 31) / 32;
  for (uint64_t ch = wid; ch < nchunks; ch += warps) {
    const uint64_t q = ch * 32 + lane;
    uint32_t x[PER];
    const bool valid = q < nvec;
    if (valid) {
      const uint4 v = ldg_nc_v4(S + q * PER);
      const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (uint32_t k = 0; k < PER; ++k) x[k] = (uint32_t)e[k];
    } else {
#pragma unroll
      for (uint32_t k = 0; k < PER; ++k) x[k] = 0xffffffffu;
    }
    // run heads inside the chunk; the element before this lane's first is the
    // previous lane's last.
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
    // position (within the chunk) of the first head in the next lane that has one
    const uint32_t later = lanes_with_head & ~((2u << lane) - 1u);
    uint32_t next_lane = later ? (uint32_t)(__ffs(later) - 1) : 32u;
    const uint32_t nl_first = __shfl_sync(FULL, first_head, next_lane & 31);
    const uint32_t next_lane_pos = (next_lane < 32) ? next_lane * PER + nl_first : 32 * PER;
    if (valid) {
#pragma unroll
      for (uint32_t k = 0; k < PER; ++k) {
        if (headmask & (1u << k)) {
          const uint32_t rest = headmask & ~((2u << k) - 1u);
          const uint32_t nxt = rest ? lane * PER + (uint32_t)(__ffs(rest) - 1) : next_lane_pos;
          const uint32_t cnt = nxt - (lane * PER + k);
          // invalid (past-the-end) lanes hold 0xffffffff, a distinct run head,
          // so a run never extends into them
          if (x[k] < sigma) atomicAdd(&H[x[k]], (unsigned long long)cnt);
          else bad = true;
        }
      }
    }
  }
  for (uint64_t j = nvec * PER + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = (uint32_t)S[j];
    if (x < sigma) atomicAdd(&H[x], 1ull);
    else bad = true;
  }
  if (bad) *flag = 2;
}

// ================================================================ a2 scans

constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// Exclusive scan of uint64 values over [0, count) with a decoupled look-back.
// Op supplies load(i) and store(i, exclusive, value).
template <class Op>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan(Op op, uint64_t count, uint64_t* status,
                                                       uint32_t* tile_counter, uint32_t epoch,
                                                       const int32_t* __restrict__ flag) {
  __shared__ uint64_t s_warp[SCAN_THREADS / 32];
  __shared__ uint64_t s_P;
  __shared__ uint32_t s_tile;
  if (*flag) return;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
  uint64_t v[SCAN_ITEMS];
  uint64_t tsum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = (base + k < count) ? op.load(base + k) : 0;
    tsum += v[k];
  }
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t incl = warp_incl_scan_u64(tsum);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint64_t w = (lane < SCAN_THREADS / 32) ? s_warp[lane] : 0;
    const uint64_t wi = warp_incl_scan_u64(w);
    const uint64_t total = __shfl_sync(FULL, wi, 31);
    if (lane < SCAN_THREADS / 32) s_warp[lane] = wi - w;
    const uint64_t P = lookback(status, tile, total, epoch);
    if (lane == 0) s_P = P;
  }
  __syncthreads();
  uint64_t run = s_P + s_warp[warp] + incl - tsum;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < count) op.store(base + k, run, v[k]);
    run += v[k];
  }
}

// C = exclusive_scan(H), in place; C[count] = total.
struct OpNodeOffsets {
  unsigned long long* C;
  uint64_t count;
  __device__ uint64_t load(uint64_t i) const { return C[i]; }
  __device__ void store(uint64_t i, uint64_t excl, uint64_t val) const {
    C[i] = excl;
    if (i + 1 == count) C[count] = excl + val;
  }
};

// Node tables.  Level l (0 <= l <= L-2), node v, s = L - l; entry k = 2^l - 1 + v.
//   leftsize(v) = C[(2v+1) << (s-1)] - C[2v << (s-1)]   (left child size)
//   Zn[v] = sum_{v' <= v} leftsize(v')  (zeros of level l before node v+1)
//   ob[v] = C[v << s] - (Zn[v] - leftsize(v))  (ones of level l before node v)
// The scan below runs over all levels concatenated and stores the global
// inclusive value; k_tables_fix subtracts the level's base.
__device__ __forceinline__ void level_of(uint64_t k, uint32_t& l, uint64_t& v) {
  l = 63u - (uint32_t)__clzll((long long)(k + 1));
  v = k + 1 - (1ull << l);
}
struct OpTables {
  const unsigned long long* C;
  ulonglong2* tab;
  unsigned long long* lvlbase;  // lvlbase[l+1] = global inclusive at the end of level l
  uint32_t L;
  __device__ uint64_t load(uint64_t k) const {
    uint32_t l;
    uint64_t v;
    level_of(k, l, v);
    const uint32_t s = L - l;
    return C[(2 * v + 1) << (s - 1)] - C[(2 * v) << (s - 1)];
  }
  __device__ void store(uint64_t k, uint64_t excl, uint64_t val) const {
    uint32_t l;
    uint64_t v;
    level_of(k, l, v);
    tab[k].y = excl + val;
    if (v + 1 == (1ull << l)) lvlbase[l + 1] = excl + val;
  }
};

__global__ void __launch_bounds__(256) k_tables_fix(const unsigned long long* __restrict__ C,
                                                    ulonglong2* __restrict__ tab,
                                                    const unsigned long long* __restrict__ lvlbase,
                                                    uint32_t L, uint64_t count,
                                                    const int32_t* __restrict__ flag) {
  if (*flag) return;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t l;
    uint64_t v;
    level_of(k, l, v);
    const uint32_t s = L - l;
    const uint64_t left = C[(2 * v + 1) << (s - 1)] - C[(2 * v) << (s - 1)];
    const uint64_t zn = tab[k].y - (l ? lvlbase[l] : 0ull);
    const uint64_t ob = C[v << s] - (zn - left);
    tab[k] = make_ulonglong2(ob, zn);
  }
}

// ============================================================ a3/a4 levels
//
// One CTA = one tile of TILE consecutive positions of T_l (TILE*sizeof(T) =
// 16 KiB, a multiple of 512 positions, so every 32-bit bitmap word and every
// 512-bit superblock lies inside one tile).  Tile ids come from an atomic
// counter (in launch order) for the look-back's forward progress.
//   1. load the tile into shared memory (16-byte vector loads);
//   2. each warp forms its bitmap words with __ballot_sync over 32
//      consecutive positions (bit sh = L-1-l of each symbol);
//   3. popcounts -> warp scan -> block scan -> decoupled look-back give the
//      global exclusive rank r(j) at every position;
//   4. bitmap words and superblocks SB[t] = r(512 t) are stored;
//   5. (a3) scatter: with v = s >> (sh+1), b = bit sh,
//        b = 0: dest = (j - r(j)) + ob[v]     (zeros before j, minus zeros before
//                                              node v, plus node start)
//        b = 1: dest = r(j) + Zn[v]           (right child start + ones before j
//                                              inside v)
//      which is Alg. 1 lines 8-13 turned from "C[node]++" cursors
//      into closed-form ranks; the result is the stable partition of every node
//      (node locality: T_{l+1} keeps node v inside v's range).
template <typename T>
struct LevelCfg;
template <>
struct LevelCfg<uint8_t> {
  static constexpr int TILE = 16384, THREADS = 512;
};
template <>
struct LevelCfg<uint16_t> {
  static constexpr int TILE = 8192, THREADS = 512;
};
template <>
struct LevelCfg<uint32_t> {
  static constexpr int TILE = 4096, THREADS = 512;
};

template <typename T, bool SCATTER>
__global__ void __launch_bounds__(LevelCfg<T>::THREADS)
    k_level(const T* __restrict__ in, T* __restrict__ out, uint64_t n, uint32_t sh,
            const ulonglong2* __restrict__ tab, uint32_t* __restrict__ bits, uint64_t words_per_level,
            unsigned long long* __restrict__ sb, uint64_t nsb, uint64_t* status,
            uint32_t* tile_counter, uint32_t epoch, const int32_t* __restrict__ flag) {
  constexpr int TILE = LevelCfg<T>::TILE;
  constexpr int THREADS = LevelCfg<T>::THREADS;
  constexpr int WORDS = TILE / 32;
  constexpr int WARPS = THREADS / 32;
  constexpr int WPW = WORDS / WARPS;
  static_assert(WPW >= 1 && WPW <= 32, "words per warp");
  static_assert(TILE % 512 == 0, "tile must hold whole superblocks");
  __shared__ __align__(16) T s_in[TILE];
  __shared__ uint32_t s_warp[WARPS];
  __shared__ unsigned long long s_P;
  __shared__ uint32_t s_total;
  __shared__ uint32_t s_tile;

  if (*flag) return;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t T0 = tile * (uint64_t)TILE;
  const uint32_t len = (uint32_t)min((uint64_t)TILE, n - T0);

  // 1. load
  if (len == TILE) {
    constexpr int NV = TILE * (int)sizeof(T) / 16;
    const char* src = reinterpret_cast<const char*>(in + T0);
    uint4* dst = reinterpret_cast<uint4*>(s_in);
#pragma unroll
    for (int q = threadIdx.x; q < NV; q += THREADS) dst[q] = ldg_nc_v4(src + 16 * (size_t)q);
  } else {
    for (int i = threadIdx.x; i < TILE; i += THREADS) s_in[i] = (i < (int)len) ? in[T0 + i] : (T)0;
  }
  __syncthreads();

  // 2. ballot words: warp w owns words [w*WPW, (w+1)*WPW); lane kk keeps word kk
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t myword = 0;
#pragma unroll
  for (int kk = 0; kk < WPW; ++kk) {
    const int i = (warp * WPW + kk) * 32 + lane;
    const uint32_t b = (i < (int)len) ? ((uint32_t)(s_in[i] >> sh) & 1u) : 0u;
    const uint32_t w = __ballot_sync(FULL, b);
    if (lane == (uint32_t)kk) myword = w;
  }
  // 3. ranks
  const uint32_t c = (lane < (uint32_t)WPW) ? (uint32_t)__popc(myword) : 0u;
  const uint32_t incl = warp_incl_scan_u32(c);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t wt = (lane < (uint32_t)WARPS) ? s_warp[lane] : 0u;
    const uint32_t wi = warp_incl_scan_u32(wt);
    const uint32_t total = __shfl_sync(FULL, wi, 31);
    if (lane < (uint32_t)WARPS) s_warp[lane] = wi - wt;
    const uint64_t P = lookback(status, tile, total, epoch);
    if (lane == 0) {
      s_P = P;
      s_total = total;
    }
  }
  __syncthreads();
  const uint64_t P = s_P;
  const uint32_t mypre = s_warp[warp] + incl - c;  // tile-local exclusive rank of word (lane)
  // 4. bitmap words + superblocks
  if (lane < (uint32_t)WPW) {
    const uint32_t k = warp * WPW + lane;
    const uint64_t gw = T0 / 32 + k;
    if (gw < words_per_level) bits[gw] = myword;
    if ((k & 15u) == 0 && T0 + 32ull * k < n) sb[(T0 + 32ull * k) >> 9] = P + mypre;
  }
  if (threadIdx.x == 0 && T0 + TILE >= n) sb[nsb - 1] = P + s_total;

  // 5. scatter to T_{l+1}
  if (SCATTER) {
    const uint32_t lt = lanemask_lt();
#pragma unroll 4
    for (int kk = 0; kk < WPW; ++kk) {
      const uint32_t w = __shfl_sync(FULL, myword, kk);
      const uint32_t wpre = __shfl_sync(FULL, mypre, kk);
      const int i = (warp * WPW + kk) * 32 + lane;
      if (i < (int)len) {
        const T x = s_in[i];
        const uint32_t b = ((uint32_t)x >> sh) & 1u;
        const uint64_t v = (uint64_t)x >> (sh + 1);
        const uint64_t r = P + wpre + (uint32_t)__popc(w & lt);
        const ulonglong2 e = __ldg(&tab[v]);
        const uint64_t dest = b ? (r + e.y) : (T0 + (uint64_t)i - r + e.x);
        out[dest] = x;
      }
    }
  }
}

// ================================================================ queries

// ones in positions [0, q) of one level (superblock + word popcounts)
__device__ __forceinline__ uint64_t rank1(const uint32_t* __restrict__ B,
                                          const unsigned long long* __restrict__ SB, uint64_t q) {
  const uint64_t t = q >> 9;
  uint64_t r = SB[t];
  const uint32_t wi = (uint32_t)(q >> 5) & 15u, bi = (uint32_t)q & 31u;
  if (wi == 0 && bi == 0) return r;
  const uint32_t* blk = B + 16 * t;
  for (uint32_t w = 0; w < wi; ++w) r += (uint32_t)__popc(blk[w]);
  if (bi) r += (uint32_t)__popc(blk[wi] & ((1u << bi) - 1u));
  return r;
}

struct TreeView {
  const uint32_t* bitmaps;
  const unsigned long long* sb;
  const unsigned long long* C;
  uint64_t n, W, NSB;
  uint32_t L;
};

__global__ void k_access(TreeView t, const uint64_t* __restrict__ pos, uint64_t m,
                         uint32_t* __restrict__ sym, int32_t* status) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t i = pos[k];
  if (i >= t.n) {
    sym[k] = 0xffffffffu;
    if (status) *status = 3;
    return;
  }
  uint64_t lo = 0, p = i, v = 0;
  for (uint32_t l = 0; l < t.L; ++l) {
    const uint32_t* B = t.bitmaps + l * t.W;
    const unsigned long long* SB = t.sb + l * t.NSB;
    const uint64_t q = lo + p;
    const uint32_t b = (B[q >> 5] >> (q & 31)) & 1u;
    const uint64_t ones_before = rank1(B, SB, q) - rank1(B, SB, lo);
    p = b ? ones_before : p - ones_before;
    v = 2 * v + b;
    lo = t.C[v << (t.L - 1 - l)];
  }
  sym[k] = (uint32_t)v;
}

__global__ void k_rank(TreeView t, uint64_t sigma, const uint32_t* __restrict__ cs,
                       const uint64_t* __restrict__ pos, uint64_t m, unsigned long long* __restrict__ cnt,
                       int32_t* status) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t i = pos[k];
  const uint64_t c = cs[k];
  if (i >= t.n || c >= sigma) {
    cnt[k] = ~0ull;
    if (status) *status = 3;
    return;
  }
  uint64_t lo = 0, r = i + 1;
  for (uint32_t l = 0; l < t.L; ++l) {
    const uint32_t* B = t.bitmaps + l * t.W;
    const unsigned long long* SB = t.sb + l * t.NSB;
    const uint32_t b = (uint32_t)(c >> (t.L - 1 - l)) & 1u;
    const uint64_t ones = rank1(B, SB, lo + r) - rank1(B, SB, lo);
    r = b ? ones : r - ones;
    lo = t.C[(c >> (t.L - 1 - l)) << (t.L - 1 - l)];
  }
  cnt[k] = r;
}

// position of the `target`-th (1-based, global) bit equal to b in one level
__device__ uint64_t select_bit(const uint32_t* __restrict__ B, const unsigned long long* __restrict__ SB,
                               uint64_t n, uint64_t nsb, uint32_t b, uint64_t target) {
  // rank_b at superblock t
  auto rb = [&](uint64_t t) -> uint64_t {
    const uint64_t ones = SB[t];
    const uint64_t pos = min(t * 512, n);
    return b ? ones : pos - ones;
  };
  // largest t with rb(t) < target
  uint64_t lo = 0, hi = nsb - 1;  // rb(0) = 0 < target, rb(nsb-1) = total >= target
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (rb(mid) < target) lo = mid;
    else hi = mid;
  }
  uint64_t need = target - rb(lo);
  const uint32_t* blk = B + 16 * lo;
  for (uint32_t w = 0; w < 16; ++w) {
    uint32_t word = b ? blk[w] : ~blk[w];
    const uint32_t c = (uint32_t)__popc(word);
    if (need <= c) {
      for (uint64_t d = 1; d < need; ++d) word &= word - 1;  // drop need-1 lowest set bits
      return lo * 512 + 32 * w + (uint32_t)(__ffs(word) - 1);
    }
    need -= c;
  }
  return ~0ull;  // unreachable for valid input
}

__global__ void k_select(TreeView t, uint64_t sigma, const uint32_t* __restrict__ cs,
                         const uint64_t* __restrict__ js, uint64_t m, unsigned long long* __restrict__ out,
                         int32_t* status) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t c = cs[k], j = js[k];
  if (c >= sigma || j == 0 || t.C[c + 1] - t.C[c] < j) {
    out[k] = ~0ull;
    if (status) *status = 3;
    return;
  }
  uint64_t p = j - 1;  // index inside the leaf
  for (uint32_t l = t.L; l-- > 0;) {
    const uint32_t* B = t.bitmaps + l * t.W;
    const unsigned long long* SB = t.sb + l * t.NSB;
    const uint64_t v = c >> (t.L - l);
    const uint64_t lo = t.C[v << (t.L - l)];
    const uint32_t b = (uint32_t)(c >> (t.L - 1 - l)) & 1u;
    const uint64_t before = b ? rank1(B, SB, lo) : lo - rank1(B, SB, lo);
    const uint64_t q = select_bit(B, SB, t.n, t.NSB, b, before + p + 1);
    p = q - lo;
  }
  out[k] = p;
}

}  // namespace wt
