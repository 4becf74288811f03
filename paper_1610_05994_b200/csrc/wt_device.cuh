// wt_device.cuh -- device helpers shared by the wavelet-tree kernels (sm_100a).
// Nothing here is shared with oracle/ (the oracle is a separate plain-C program).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace wt {

constexpr uint32_t FULL = 0xffffffffu;

// ---------------------------------------------------------------- look-back
// Decoupled look-back (single-pass prefix scan across tiles).  One 64-bit
// status word per tile: [63:62] flag, [61:54] epoch, [53:0] value.  The value
// travels inside the same word as the flag, so relaxed single-copy-atomic
// 64-bit loads/stores are sufficient (no separate payload to order).  The
// epoch distinguishes the look-back launches of one build, so the status
// array is zeroed once per build instead of once per launch.
enum : uint64_t { ST_INVALID = 0, ST_AGG = 1, ST_PREFIX = 2 };
constexpr uint64_t VALUE_MASK = (1ull << 54) - 1;

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t pack_status(uint64_t flag, uint32_t epoch, uint64_t value) {
  return (flag << 62) | ((uint64_t)(epoch & 0xff) << 54) | (value & VALUE_MASK);
}

// Called by all 32 lanes of ONE warp.  Publishes `aggregate` for `tile`,
// returns the exclusive prefix of all earlier tiles and publishes the
// inclusive prefix.  Tile ids must be handed out in launch order by an atomic
// counter (forward progress: every earlier tile is owned by a resident CTA).
__device__ __forceinline__ uint64_t lookback(uint64_t* status, uint64_t tile, uint64_t aggregate,
                                             uint32_t epoch) {
  const uint32_t lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(&status[0], pack_status(ST_PREFIX, epoch, aggregate));
    return 0;
  }
  if (lane == 0) st_relaxed_u64(&status[tile], pack_status(ST_AGG, epoch, aggregate));
  uint64_t exclusive = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t idx = base - (int64_t)lane;
    uint64_t flag, val;
    while (true) {
      if (idx >= 0) {
        const uint64_t w = ld_relaxed_u64(&status[idx]);
        const uint32_t ep = (uint32_t)(w >> 54) & 0xffu;
        flag = (ep == (epoch & 0xffu)) ? (w >> 62) : ST_INVALID;
        val = w & VALUE_MASK;
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
  if (lane == 0) st_relaxed_u64(&status[tile], pack_status(ST_PREFIX, epoch, exclusive + aggregate));
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
