// wt_ptx.cuh -- PTX wrappers (mbarrier, TMA bulk copies, proxy fences) and
// SWAR / shared-memory helpers of the level pass (sm_100a).
#pragma once
#include "wt_device.cuh"

namespace wt {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// Programmatic dependent launch (the build's kernels are launched with
// programmatic stream serialization): a kernel may start while its
// predecessor still runs; pdl_wait() blocks until the predecessor grid has
// completed and its writes are visible (a no-op when launched normally).
// pdl_trigger() lets the successor launch (it then waits in its pdl_wait()).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------ SWAR helpers
template <typename T>
__device__ __forceinline__ uint32_t bitmask32(uint32_t bit) {  // `bit` of every symbol packed in a 32-bit word
  if (sizeof(T) == 1) return 0x01010101u << bit;
  if (sizeof(T) == 2) return 0x00010001u << bit;
  return 1u << bit;
}

// bit `sh` of the symbols held in xw[NW] (little-endian), symbol k -> bit k.
template <typename T, int NW, int OFF = 0, int XN>
__device__ __forceinline__ uint32_t swar_bits(const uint32_t (&xa)[XN], uint32_t sh) {
  static_assert(OFF + NW <= XN, "word range");
  const uint32_t* xw = xa + OFF;
  uint32_t m = 0;
  if constexpr (sizeof(T) == 1) {
    // gather bit sh of the 4 bytes of a word with one multiply:
    // (x & 0x01010101<<sh) * (1 + 2^7 + 2^14 + 2^21) puts byte j's bit at 21+sh+j
    // gather bit sh of the 4 bytes of a word with one multiply: (x & 0x01010101<<sh)
    // * ((1 + 2^7 + 2^14 + 2^21) << (7-sh)) puts byte j's bit at 28+j (no carries);
    // a multiply-high moves the nibble to 4k.  2 ALU + 2 FMA-pipe ops per word.
    static_assert(NW <= 8, "u8: at most 8 words per 32-bit mask");
    const uint32_t msk = 0x01010101u << sh;
    if constexpr (NW % 2 == 0) {
      // two words per multiply: t holds word k's four bits and word k+1's four
      // bits 4 apart (at s + 8j and s + 4 + 8j, s = sh for sh <= 3, else sh - 4),
      // t * (0x00204081 << (3 - s)) puts them at 24..31 in symbol order (the
      // other products are single bits at distinct positions below 24 or past
      // bit 31: no carries); a multiply-high moves the byte to 8k.
      const bool lo = sh <= 3;
      const uint32_t magic = 0x00204081u << (lo ? 3 - sh : 7 - sh);
#pragma unroll
      for (int k = 0; k < NW / 2; ++k) {
        const uint32_t a = xw[2 * k] & msk, b = xw[2 * k + 1] & msk;
        const uint32_t t = lo ? a + b * 16u : (a >> 4) + b;
        const uint32_t p = t * magic;
        const uint32_t v = (k == 3) ? p : __umulhi(p, 1u << (8 + 8 * k));
        m |= v & (0xffu << (8 * k));
      }
    } else {
      const uint32_t magic = 0x00204081u << (7 - sh);
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        const uint32_t p = (xw[k] & msk) * magic;
        const uint32_t v = (k == 7) ? p : __umulhi(p, 1u << (4 + 4 * k));
        m |= v & (0xfu << (4 * k));
      }
    }
  } else if constexpr (sizeof(T) == 2) {
    // bits sh and 16+sh of the word -> bits 30, 31 by one multiply
    // (x & msk) * (2^(30-sh) + 2^(15-sh)), then a multiply-high to 2k.
    static_assert(NW <= 16, "u16: at most 16 words per 32-bit mask");
    const uint32_t msk = 0x00010001u << sh;
    if (NW % 2 == 0 && sh <= 13) {
      // two words per multiply: t = (x_k & msk) + 4 (x_{k+1} & msk) holds the
      // 4 symbols' bits at sh, sh+16, sh+2, sh+18; t * (2^(28-sh) + 2^(13-sh))
      // puts them at 28..31 in symbol order (the other products land at 13, 15
      // or past bit 31: no carries); a multiply-high moves the nibble to 4k.
      const uint32_t magic = (1u << (28 - sh)) | (1u << (13 - sh));
#pragma unroll
      for (int k = 0; k < NW / 2; ++k) {
        const uint32_t t = (xw[2 * k] & msk) + (xw[2 * k + 1] & msk) * 4u;
        const uint32_t p = t * magic;
        const uint32_t v = (k == 7) ? p : __umulhi(p, 1u << (4 + 4 * k));
        m |= v & (0xfu << (4 * k));
      }
    } else {
      const uint32_t magic = (1u << (30 - sh)) | (1u << (15 - sh));
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        const uint32_t p = (xw[k] & msk) * magic;
        const uint32_t v = (k == 15) ? p : __umulhi(p, 1u << (2 + 2 * k));
        m |= v & (3u << (2 * k));
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < NW; ++k) m |= ((xw[k] >> sh) & 1u) << k;
  }
  return m;
}

template <typename T, int NW>
__device__ __forceinline__ uint32_t sym_of(const uint32_t (&xw)[NW], int k) {
  if (sizeof(T) == 1) return (xw[k >> 2] >> (8 * (k & 3))) & 0xffu;
  if (sizeof(T) == 2) return (xw[k >> 1] >> (16 * (k & 1))) & 0xffffu;
  return xw[k];
}

// st.shared of the low sizeof(T) bytes of v at shared byte address a + OFF
template <typename T, int OFF = 0>
__device__ __forceinline__ void st_shared(uint32_t a, uint32_t v) {
  if (sizeof(T) == 1) asm volatile("st.shared.u8 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF));
  else if (sizeof(T) == 2) asm volatile("st.shared.u16 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF));
  else asm volatile("st.shared.u32 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF));
}

// Stable in-word partition of the SPW symbols of a 32-bit word by their bits
// (bit j of `bits` = bit of symbol j): a PRMT selector that moves the zero
// symbols to the low end (in order) and the one symbols after them (in
// order), plus the number of zeros in bits 16..18.
template <typename T>
__host__ __device__ constexpr uint32_t partition_lut_entry(uint32_t bits) {
  uint32_t sel = 0, k = 0, nz = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (uint32_t j = 0; j < 4 / sizeof(T); ++j)
      if (((bits >> j) & 1u) == (uint32_t)pass) {
        for (uint32_t byte = 0; byte < sizeof(T); ++byte) sel |= (j * sizeof(T) + byte) << (4 * (k * sizeof(T) + byte));
        ++k;
        nz += pass == 0;
      }
  return sel | (nz << 16);
}

template <typename T>
__device__ __forceinline__ uint32_t sym_in_word(uint32_t x, int j) {
  if (sizeof(T) == 1) return (x >> (8 * j)) & 0xffu;
  if (sizeof(T) == 2) return (x >> (16 * j)) & 0xffffu;
  return x;
}

__device__ __forceinline__ uint2 ld_shared_u2(uint32_t a) {  // shared byte address a (8-byte aligned)
  uint2 v;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

__device__ __forceinline__ uint32_t lowmask(uint32_t k) { return k >= 32 ? 0xffffffffu : ((1u << k) - 1u); }

}  // namespace wt
