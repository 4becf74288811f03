// Microbenchmark: achievable HBM bandwidth of the level pass's memory pattern
// (per-warp ring of bulk-loaded tiles, bulk stores of the staged output) with
// no compute, vs plain vectorized copy.  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o mb mb_tma_copy.cu ; run ./mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void fence_proxy() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void expect(unsigned long long* bar, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(b) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t b, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(d)),
               "l"(s), "r"(b), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void s2g(void* d, const void* s, uint32_t b) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(smem_u32(s)), "r"(b)
               : "memory");
}
__device__ __forceinline__ void wait(unsigned long long* bar, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(ph)
      : "memory");
}

// one warp per CTA, ring of NB buffers of TB bytes; output staged in the previous buffer
template <int TB, int NB, int SPLIT>
__global__ void __launch_bounds__(32) k_ring(const uint8_t* in, uint8_t* out, size_t n) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + NB * (TB + 128));
  const uint32_t lane = threadIdx.x;
  const size_t ntiles = n / TB;
  auto tile_of = [&](uint32_t it) { return (size_t)blockIdx.x + (size_t)it * gridDim.x; };
  auto issue = [&](uint32_t it) {
    size_t t = tile_of(it);
    if (t >= ntiles) return;
    int b = it % NB;
    fence_proxy();
    expect(&bar[b], TB);
    g2s(sm + b * (TB + 128) + 64, in + t * TB, TB, &bar[b]);
  };
  if (lane == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < NB - 1; ++b) issue(b);
  }
  __syncwarp();
  for (uint32_t it = 0;; ++it) {
    size_t t = tile_of(it);
    if (t >= ntiles) break;
    int ib = it % NB, ob = (it + NB - 1) % NB;
    wait(&bar[ib], (it / NB) & 1);
    // "phase D": copy input buffer to output buffer (word per lane)
    const uint32_t* src = reinterpret_cast<const uint32_t*>(sm + ib * (TB + 128) + 64);
    uint32_t* dst = reinterpret_cast<uint32_t*>(sm + ob * (TB + 128) + 64);
    for (int w = lane; w < TB / 4; w += 32) dst[w] = src[w];
    fence_proxy();
    __syncwarp();
    if (lane == 0) {
      // SPLIT stores: e.g. zeros part and ones part to two destinations
      const uint32_t part = TB / SPLIT;
      for (int p = 0; p < SPLIT; ++p)
        s2g(out + (p * (n / SPLIT)) + t * part, sm + ob * (TB + 128) + 64 + p * part, part);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      if (it >= 1) issue(it + NB - 2);
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_copy(const uint4* in, uint4* out, size_t nv) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

template <int TB, int NB, int SPLIT>
void run(const uint8_t* in, uint8_t* out, size_t n, int sms) {
  auto k = k_ring<TB, NB, SPLIT>;
  size_t smem = NB * (TB + 128) + 64;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, 32, smem);
  int grid = bps * sms;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<grid, 32, smem>>>(in, out, n);
  cudaEventRecord(a);
  const int R = 10;
  for (int i = 0; i < R; ++i) k<<<grid, 32, smem>>>(in, out, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= R;
  printf("ring TB=%5d NB=%d split=%d warps/SM=%2d: %.3f ms  %.0f GB/s (r+w)  err=%s\n", TB, NB, SPLIT, bps, ms,
         2.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  size_t n = 256ull << 20;
  uint8_t *in, *out;
  cudaMalloc(&in, n);
  cudaMalloc(&out, n);
  cudaMemset(in, 1, n);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k_copy<<<sms * 8, 256>>>((const uint4*)in, (uint4*)out, n / 16);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) k_copy<<<sms * 8, 256>>>((const uint4*)in, (uint4*)out, n / 16);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("plain copy: %.3f ms %.0f GB/s\n", ms / 10, 2.0 * n / (ms / 10) / 1e6);
  }
  run<2048, 3, 1>(in, out, n, sms);
  run<2048, 3, 2>(in, out, n, sms);
  run<2048, 4, 2>(in, out, n, sms);
  run<4096, 3, 2>(in, out, n, sms);
  run<4096, 4, 2>(in, out, n, sms);
  run<8192, 3, 2>(in, out, n, sms);
  run<8192, 4, 2>(in, out, n, sms);
  run<16384, 3, 2>(in, out, n, sms);
  return 0;
}
