// wt_device.cuh -- device helpers shared by the wavelet-tree kernels (sm_100a).
// Nothing here is shared with oracle/ (the oracle is a separate plain-C program).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace wt {

constexpr uint32_t FULL = 0xffffffffu;

// ---------------------------------------------------------------- look-back
// Decoupled look-back (single-pass prefix scan across tiles).  Per tile a
// 32-bit status word ([31:30] flag, [7:0] epoch) and two 64-bit values (the
// tile aggregate and the inclusive prefix, separate so that publishing the
// prefix never changes a value a reader of the aggregate flag is about to
// read): the value is stored first (relaxed), then the status with release
// semantics; a reader acquires the status before reading the value.  The epoch tells the
// look-back launches of one build apart, so the status array is zeroed once
// per build instead of once per launch.  Values are full 64-bit.
enum : uint32_t { ST_INVALID = 0, ST_AGG = 1, ST_PREFIX = 2 };

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct LookbackState {
  uint32_t* status;  // [tiles]
  uint64_t* value;   // [2][tiles]: aggregates, then inclusive prefixes
  uint64_t tiles;
};

__device__ __forceinline__ void lb_publish(LookbackState lb, uint64_t tile, uint32_t flag, uint32_t epoch,
                                           uint64_t v) {
  st_relaxed_u64(&lb.value[(flag == ST_PREFIX ? lb.tiles : 0) + tile], v);
  st_release_u32(&lb.status[tile], (flag << 30) | (epoch & 0xffu));
}

// Called by all 32 lanes of ONE warp.  Publishes `aggregate` for `tile`,
// returns the exclusive prefix of all earlier tiles and publishes the
// inclusive prefix.  Tile ids must be handed out in launch order by an atomic
// counter (forward progress: every earlier tile is owned by a resident CTA).
__device__ __forceinline__ uint64_t lookback(LookbackState lb, uint64_t tile, uint64_t aggregate, uint32_t epoch) {
  const uint32_t lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) lb_publish(lb, 0, ST_PREFIX, epoch, aggregate);
    return 0;
  }
  if (lane == 0) lb_publish(lb, tile, ST_AGG, epoch, aggregate);
  uint64_t exclusive = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t idx = base - (int64_t)lane;
    uint32_t flag;
    uint64_t val;
    while (true) {
      if (idx >= 0) {
        const uint32_t w = ld_acquire_u32(&lb.status[idx]);
        flag = ((w & 0xffu) == (epoch & 0xffu)) ? (w >> 30) : ST_INVALID;
        val = (flag != ST_INVALID) ? ld_relaxed_u64(&lb.value[(flag == ST_PREFIX ? lb.tiles : 0) + idx]) : 0;
      } else {
        flag = ST_PREFIX;
        val = 0;
      }
      if (__all_sync(FULL, flag != ST_INVALID)) break;
      __nanosleep(20);
    }
    const uint32_t pm = __ballot_sync(FULL, flag == ST_PREFIX);
    const uint32_t stop = pm ? (uint32_t)(__ffs(pm) - 1) : 31u;
    uint64_t c = (lane <= stop) ? val : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    exclusive += c;
    if (pm) break;
    base -= 32;
  }
  if (lane == 0) lb_publish(lb, tile, ST_PREFIX, epoch, exclusive + aggregate);
  return exclusive;
}

// The same look-back by a whole CTA (blockDim.x = NT threads, all of them call
// it): thread j looks at tile (tile - 1 - j), so one round trip covers NT
// predecessors instead of 32 -- when the scan's CTAs start together (a grid of
// one wave: the per-level preps) every aggregate is published at about the same
// time and a 32-tile window walks tile / 32 dependent round trips back to the
// first inclusive prefix.  `aggregate` is the tile's total (thread 0's copy is
// used); s_sum / s_has: NT / 32 shared entries each.  Returns the exclusive
// prefix to every thread; contains block barriers.
template <int NT>
__device__ __forceinline__ uint64_t block_lookback(LookbackState lb, uint64_t tile, uint64_t aggregate, uint32_t epoch,
                                                   uint64_t* s_sum, uint32_t* s_has) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) lb_publish(lb, tile, tile ? ST_AGG : ST_PREFIX, epoch, aggregate);
  uint64_t exclusive = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {  // (block-uniform trip count)
    const int64_t idx = base - (int64_t)threadIdx.x;
    uint32_t flag = ST_PREFIX;  // (before tile 0: an empty inclusive prefix)
    uint64_t val = 0;
    if (idx >= 0) {
      while (true) {
        const uint32_t w = ld_acquire_u32(&lb.status[idx]);
        flag = ((w & 0xffu) == (epoch & 0xffu)) ? (w >> 30) : ST_INVALID;
        if (flag != ST_INVALID) break;
        __nanosleep(20);
      }
      val = ld_relaxed_u64(&lb.value[(flag == ST_PREFIX ? lb.tiles : 0) + idx]);
    }
    const uint32_t pm = __ballot_sync(FULL, flag == ST_PREFIX);
    const uint32_t stop = pm ? (uint32_t)(__ffs(pm) - 1) : 31u;
    uint64_t c = (lane <= stop) ? val : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if (lane == 0) {
      s_sum[warp] = c;
      s_has[warp] = pm ? 1u : 0u;
    }
    __syncthreads();
    bool found = false;
#pragma unroll 1
    for (int w = 0; w < NT / 32; ++w) {
      exclusive += s_sum[w];
      if (s_has[w]) {
        found = true;
        break;
      }
    }
    if (found) break;
    base -= NT;
    __syncthreads();  // (s_sum / s_has are rewritten)
  }
  if (threadIdx.x == 0 && tile) lb_publish(lb, tile, ST_PREFIX, epoch, exclusive + aggregate);
  return exclusive;
}

// ------------------------------------------------------------- warp scans
__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t x) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL, x, o);
    if (lane >= (uint32_t)o) x += t;
  }
  return x;
}
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t x) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(FULL, x, o);
    if (lane >= (uint32_t)o) x += t;
  }
  return x;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

}  // namespace wt
