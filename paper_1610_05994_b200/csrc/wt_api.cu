// wt_api.cu -- host side of libwt.so: argument checks, workspace carving and
// the launch sequence of the levelwise build.  The C ABI is declared (and
// documented, with the paper citations) in include/wt.h.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include <cudaTypedefs.h>

#include "wt.h"
#include "wt_kernels.cuh"

namespace {

thread_local std::string g_last_error;
thread_local wt_event_t* g_events = nullptr;
thread_local uint32_t g_event_count = 0;

wt_status fail(wt_status st, const char* what) {
  g_last_error = what;
  return st;
}
wt_status fail_cuda(cudaError_t e, const char* what) {
  g_last_error = (g_last_error.empty() ? std::string() : g_last_error + ": ") + what + ": " + cudaGetErrorString(e);
  return WT_ERR_CUDA;
}

constexpr size_t ALIGN = 256;
size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

uint32_t levels_of(uint64_t sigma) {
  uint32_t L = 0;
  while (L < 63 && (1ull << L) < sigma) ++L;
  return L;
}

uint64_t level_tile(uint32_t width) {
  switch (width) {
    case 1: return wt::LvTile<uint8_t>::TILE;
    case 2: return wt::LvTile<uint16_t>::TILE;
    default: return wt::LvTile<uint32_t>::TILE;
  }
}

// Per-device launch facts (a process may drive several GPUs): the SM count
// and, per level-kernel instantiation, the dynamic shared-memory opt-in and
// the resident CTAs per SM.  Filled once per device under a mutex.
constexpr int MAX_DEVICES = 64;
std::mutex g_dev_mu;

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAX_DEVICES) dev = 0;
  return dev;
}

int num_sms() {
  static int sms[MAX_DEVICES] = {};
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  if (sms[dev] == 0 &&
      (cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms[dev] <= 0))
    sms[dev] = 148;
  return sms[dev];
}

// opt in to > 48 KiB dynamic shared memory once per level-kernel instantiation
// and device, and size the persistent grid: every resident CTA slot of every SM.
template <typename T, int SC>
cudaError_t level_kernel_setup(int* blocks_per_sm) {
  static int bps[MAX_DEVICES] = {};
  static cudaError_t err[MAX_DEVICES] = {};
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  if (bps[dev] == 0) {
    cudaError_t e = cudaFuncSetAttribute(wt::k_level<T, SC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)wt::level_smem_bytes<T>());
    int b = 0;
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, wt::k_level<T, SC>, wt::LV_THREADS,
                                                        wt::level_smem_bytes<T>());
    err[dev] = e;
    bps[dev] = b < 1 ? 1 : b;
  }
  *blocks_per_sm = bps[dev];
  return err[dev];
}

constexpr int MAX_LOOKBACK_LAUNCHES = 128;

// Workspace carve (all offsets 256-byte aligned).  The control block
// [0, ctrl_bytes) is zeroed once per build: range flag, tile counters (one per
// look-back scan launch), ones0, look-back status words (shared by every
// look-back scan of the build, told apart by epoch) and the per-level,
// per-tile ones counts agg[l][t] (filled by the pass that writes T_l).  Then:
// the tile prefixes pre[t], the node tables {ob, Zn} of levels 0..L-2, the
// two ping-pong level-node count buffers cnt[2][2^L] (uint32: pass l counts
// the level-(l+2) node sizes into cnt[l % 2]) and the ping-pong sequences
// T_1, T_2, ...
struct Carve {
  uint32_t L = 0;
  uint64_t words = 0, nsb = 0, c_len = 0, ntiles = 0;
  uint64_t status_entries = 0, tab_entries = 0, cnt_entries = 0;
  size_t off_flag = 0, off_counters = 0, off_ones0 = 0, off_status = 0, off_value = 0, off_agg = 0, ctrl_bytes = 0;
  size_t off_status2 = 0, off_value2 = 0;  // a second look-back state (two scans per k_prep launch)
  size_t off_pre = 0, off_tab = 0, off_cnt = 0, off_bufA = 0, off_bufB = 0, total = 0;
  // a5 interior fused groups (k_quad): per-tile class counts (zeroed with the
  // control block), their prefixes, the level-2 node sizes for the first quad
  size_t off_agg01 = 0, off_agg11 = 0, off_hist4 = 0, off_pre01 = 0, off_pre11 = 0;
  size_t off_tr = 0;  // k_triple: agg01, agg11, pre01, pre11 (ntiles each), cls, tab3 (2^(L-3) each)
  // host-API extras (after total)
  size_t off_seq = 0, off_bits = 0, off_sb = 0, off_c = 0, host_total = 0;
  // segmented build (n > seg_max(): S is cut into k segments, each built with
  // the direct launch sequence into its own tree, then merged -- the paper's
  // dd on one GPU; keeps every in-kernel position of the level
  // passes 32-bit while the tree holds n >= 2^32 symbols)
  bool seg = false;
  uint32_t k = 0;
  uint64_t seg_len = 0;
  size_t off_sc_counters = 0, off_sc_status = 0, off_sc_value = 0, seg_ctrl = 0;
  size_t off_tree[wt::DD_MAX_SEGMENTS] = {}, off_segws = 0;
  uint64_t sc_tiles = 0;
};

// Longest segment of a segmented build (a multiple of 4096 symbols, < 2^32).
// WT_SEG_MAX overrides it (tests exercise the segmented path at small n).
uint64_t seg_max() {
  const char* v = std::getenv("WT_SEG_MAX");
  if (v && *v) {
    const uint64_t x = std::strtoull(v, nullptr, 10) / 4096 * 4096;
    if (x >= 4096 && x <= (1ull << 31)) return x;
  }
  return 1ull << 31;
}
// per-level sizes of a tree of n symbols
uint64_t words_of(uint64_t n) { return 16 * ((n + 511) / 512); }
uint64_t nsb_of(uint64_t n) { return (n + 511) / 512 + 1; }
size_t tree_bytes(uint64_t n, uint32_t L) {
  return align_up((size_t)L * words_of(n) * 4) + align_up((size_t)L * nsb_of(n) * 8) +
         align_up(((1ull << L) + 1) * 8);
}
// superblock scans over nblocks blocks: look-back tiles
uint64_t sb_scan_tiles(uint64_t nblocks) {
  return std::max<uint64_t>(1, (nblocks + wt::SCAN_TILE_MIN - 1) / wt::SCAN_TILE_MIN);
}

Carve carve_direct(uint64_t n, uint64_t sigma, uint32_t width);

// a5: interior fused groups of k = 2 levels (k_quad, wt_quad.cuh) at
// l = 0, 2, ..., 2 (nquad - 1): l <= Q_MAXL (the node table of <= 64 nodes) and
// l + 2 <= L - 2 (T_{l+2} feeds a later pass; the last two levels are the fused
// final pair).  Opt-in (WT_QUAD=1, read per call): measured on B200 the quad
// pass is slower than the two level passes it replaces.
bool quad_enabled() {
  const char* v = std::getenv("WT_QUAD");
  return v && *v && *v != '0';
}
uint32_t quad_levels(uint32_t L) {
  if (!quad_enabled() || L < 4) return 0;
  uint32_t q = 0;
  while (2 * q <= wt::Q_MAXL && 2 * q + 2 <= L - 2) ++q;
  return q;
}

Carve carve(uint64_t n, uint64_t sigma, uint32_t width) {
  const uint64_t sm = seg_max();
  if (n <= sm) return carve_direct(n, sigma, width);
  Carve c;
  c.seg = true;
  c.L = levels_of(sigma);
  c.words = words_of(n);
  c.nsb = nsb_of(n);
  c.c_len = (1ull << c.L) + 1;
  c.seg_len = sm;
  c.k = (uint32_t)((n + sm - 1) / sm);
  c.sc_tiles = sb_scan_tiles(c.nsb - 1);
  size_t o = 0;
  c.off_flag = o;
  o += ALIGN;
  c.off_sc_counters = o;
  o += align_up(64 * sizeof(uint32_t));
  c.off_sc_status = o;
  o += align_up(c.sc_tiles * sizeof(uint32_t));
  c.seg_ctrl = o;  // [0, seg_ctrl) zeroed once per build
  c.off_sc_value = o;
  o += align_up(2 * c.sc_tiles * sizeof(uint64_t));
  for (uint32_t g = 0; g < c.k; ++g) {
    c.off_tree[g] = o;
    o += tree_bytes(std::min(sm, n - (uint64_t)g * sm), c.L);
  }
  c.off_segws = o;
  o += carve_direct(sm, sigma, width).total;
  c.total = o;
  c.off_seq = o;
  o += align_up(n * width);
  c.off_bits = o;
  o += align_up((size_t)c.L * c.words * 4);
  c.off_sb = o;
  o += align_up((size_t)c.L * c.nsb * 8);
  c.off_c = o;
  o += align_up(c.c_len * 8);
  c.host_total = o;
  return c;
}

Carve carve_direct(uint64_t n, uint64_t sigma, uint32_t width) {
  Carve c;
  c.L = levels_of(sigma);
  c.words = 16 * ((n + 511) / 512);
  c.nsb = (n + 511) / 512 + 1;
  c.c_len = (1ull << c.L) + 1;
  c.ntiles = (n + level_tile(width) - 1) / level_tile(width);
  const uint64_t scan_tiles = ((1ull << c.L) + wt::SCAN_TILE_MIN - 1) / wt::SCAN_TILE_MIN;
  c.tab_entries = c.L >= 2 ? (1ull << (c.L - 1)) - 1 : 0;
  c.cnt_entries = c.L >= 2 ? (1ull << c.L) : 0;
  const uint64_t pre_tiles = (c.ntiles + wt::SCAN_TILE_MIN - 1) / wt::SCAN_TILE_MIN;
  const uint64_t sb_tiles = (c.nsb + wt::SCAN_TILE_MIN - 1) / wt::SCAN_TILE_MIN;  // last level's superblock scan
  c.status_entries = std::max<uint64_t>(1, std::max(std::max(pre_tiles, scan_tiles), sb_tiles));
  size_t o = 0;
  c.off_flag = o;
  o += ALIGN;
  c.off_counters = o;
  o += align_up(MAX_LOOKBACK_LAUNCHES * sizeof(uint32_t));
  c.off_ones0 = o;
  o += ALIGN;
  c.off_status = o;
  o += align_up(c.status_entries * sizeof(uint32_t));
  c.off_status2 = o;
  o += align_up(c.status_entries * sizeof(uint32_t));
  c.off_agg = o;
  o += align_up((size_t)c.L * c.ntiles * sizeof(uint32_t));
  const uint32_t qrows = quad_levels(c.L) ? 2 * quad_levels(c.L) - 1 : 0;  // rows l = 0 .. 2 (nquad - 1)
  c.off_agg01 = o;
  o += align_up((size_t)qrows * c.ntiles * sizeof(uint32_t));
  c.off_agg11 = o;
  o += align_up((size_t)qrows * c.ntiles * sizeof(uint32_t));
  c.off_hist4 = o;
  o += ALIGN;
  c.ctrl_bytes = o;
  c.off_value = o;  // look-back values: written before their status, never read stale
  o += align_up(2 * c.status_entries * sizeof(uint64_t));
  c.off_value2 = o;
  o += align_up(2 * c.status_entries * sizeof(uint64_t));
  c.off_pre = o;
  o += align_up(c.ntiles * sizeof(uint32_t));
  c.off_pre01 = o;
  if (qrows) o += align_up(c.ntiles * sizeof(uint32_t));
  c.off_pre11 = o;
  if (qrows) o += align_up(c.ntiles * sizeof(uint32_t));
  c.off_tab = o;
  o += align_up(c.tab_entries * sizeof(uint2));
  // k_triple (the fused final three levels): per-tile class counts and their
  // prefixes, per level-(L-3) node the class sizes and the classes before it
  if (c.L >= 3) {
    c.off_tr = o;
    o += 4 * align_up(c.ntiles * sizeof(uint32_t)) + 2 * align_up((1ull << (c.L - 3)) * sizeof(uint2));
  }
  c.off_cnt = o;
  o += 2 * align_up(c.cnt_entries * sizeof(uint32_t));
  const size_t seq_bytes = align_up(n * width);
  // T_1 .. T_{L-2} (the fused pass L-2 writes no T_{L-1})
  c.off_bufA = o;
  if (c.L >= 3) o += seq_bytes;  // T_1, T_3, ...
  c.off_bufB = o;
  if (c.L >= 4) o += seq_bytes;  // T_2, T_4, ...
  c.total = o;
  c.off_seq = o;
  o += seq_bytes;
  c.off_bits = o;
  o += align_up((size_t)c.L * c.words * 4);
  c.off_sb = o;
  o += align_up((size_t)c.L * c.nsb * 8);
  c.off_c = o;
  o += align_up(c.c_len * 8);
  c.host_total = o;
  return c;
}

wt_status check_args(uint64_t n, uint64_t sigma, uint32_t width) {
  (void)n;
  if (width != 1 && width != 2 && width != 4) return fail(WT_ERR_ARG, "width must be 1, 2 or 4");
  if (sigma == 0) return fail(WT_ERR_ARG, "sigma must be >= 1");
  if (sigma > (1ull << (8 * width))) return fail(WT_ERR_ARG, "sigma exceeds the symbol width");
  if (levels_of(sigma) > 30) return fail(WT_ERR_ARG, "more than 30 levels");
  if (n > (uint64_t)wt::DD_MAX_SEGMENTS * seg_max()) return fail(WT_ERR_ARG, "n exceeds 32 segments of seg_max()");
  return WT_OK;
}

// Records the thread-local profiling events (if any) around each launch.
// A failed record (e.g. an uncreated event handle) is reported, not hidden.
struct Launcher {
  cudaStream_t s;
  uint32_t k = 0;
  cudaError_t pre() {
    if (g_events && 2 * k + 1 < g_event_count) return cudaEventRecord((cudaEvent_t)g_events[2 * k], s);
    return cudaSuccess;
  }
  cudaError_t post() {
    cudaError_t e = cudaSuccess;
    if (g_events && 2 * k + 1 < g_event_count) e = cudaEventRecord((cudaEvent_t)g_events[2 * k + 1], s);
    if (e == cudaSuccess && debug_sync()) {  // WT_DEBUG_SYNC=1: locate a faulting launch
      e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) g_last_error = "launch " + std::to_string(k) + " faulted";
    }
    ++k;
    return e;
  }
  static bool debug_sync() {
    static const bool on = [] {
      const char* v = std::getenv("WT_DEBUG_SYNC");
      return v && *v && *v != '0';
    }();
    return on;
  }
};

// Kernel launch with programmatic stream serialization (PDL): the kernel may
// start while its predecessor finishes; it calls pdl_wait() before touching
// the predecessor's results.  WT_NO_PDL=1 launches normally (A/B, debugging).
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("WT_NO_PDL");
    return !(v && *v && *v != '0');
  }();
  return on;
}
// The final pair pass writes B_{L-1}'s runs with global OR-reductions when it
// reads S itself (L = 2, where the pass is ALU-bound);
// WT_PAIR_RED=0/1 forces it off/on (A/B).
// The specialised pass for two-level trees of 1-byte symbols (k_pair2);
// WT_NO_PAIR2=1 (read per call) uses the general fused pair instead (A/B, tests).
bool pair2_enabled() {
  const char* v = std::getenv("WT_NO_PAIR2");
  return !(v && *v && *v != '0');
}
cudaError_t pair2_setup(int* blocks_per_sm) {
  static int bps[MAX_DEVICES] = {};
  static cudaError_t err[MAX_DEVICES] = {};
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  if (bps[dev] == 0) {
    int b = 0;
    cudaError_t e = cudaFuncSetAttribute(wt::k_pair2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)wt::p2_smem_bytes());
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, wt::k_pair2, 32 * wt::P2_WARPS, wt::p2_smem_bytes());
    err[dev] = e;
    bps[dev] = b < 1 ? 1 : b;
  }
  *blocks_per_sm = bps[dev];
  return err[dev];
}
// The fused final pair of deeper trees (k_pairn, wt_pairn.cuh); WT_NO_PAIRN=1
// (read per call) uses the general fused pair k_level<T, 2> instead (A/B, tests).
bool pairn_enabled() {
  const char* v = std::getenv("WT_NO_PAIRN");
  return !(v && *v && *v != '0');
}
// The fused final three levels (k_triple, wt_triple.cuh): opt-in, WT_TRIPLE=1
// (read per call).  Measured on B200 slower than the level pass + k_pairn it
// replaces.
bool triple_enabled() {
  const char* w = std::getenv("WT_TRIPLE");
  return w && *w && *w != '0';
}
template <typename T>
cudaError_t triple_setup(int* blocks_per_sm) {
  static int bps[MAX_DEVICES] = {};
  static cudaError_t err[MAX_DEVICES] = {};
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  if (bps[dev] == 0) {
    int b = 0;
    cudaError_t e = cudaFuncSetAttribute(wt::k_triple<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)wt::tr_smem_bytes());
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, wt::k_triple<T>, 32 * wt::PN_WARPS, wt::tr_smem_bytes());
    err[dev] = e;
    bps[dev] = b < 1 ? 1 : b;
  }
  *blocks_per_sm = bps[dev];
  return err[dev];
}
template <typename T>
cudaError_t pairn_setup(int* blocks_per_sm) {
  static int bps[MAX_DEVICES] = {};
  static cudaError_t err[MAX_DEVICES] = {};
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  if (bps[dev] == 0) {
    int b = 0;
    cudaError_t e = cudaFuncSetAttribute(wt::k_pairn<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)wt::pn_smem_bytes());
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, wt::k_pairn<T>, 32 * wt::PN_WARPS, wt::pn_smem_bytes());
    err[dev] = e;
    bps[dev] = b < 1 ? 1 : b;
  }
  *blocks_per_sm = bps[dev];
  return err[dev];
}
template <typename T>
cudaError_t quad_setup(int* blocks_per_sm) {
  static int bps[MAX_DEVICES] = {};
  static cudaError_t err[MAX_DEVICES] = {};
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  if (bps[dev] == 0) {
    int b = 0;
    cudaError_t e = cudaFuncSetAttribute(wt::k_quad<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)wt::quad_smem_bytes<T>());
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, wt::k_quad<T>, wt::Q_THREADS, wt::quad_smem_bytes<T>());
    err[dev] = e;
    bps[dev] = b < 1 ? 1 : b;
  }
  *blocks_per_sm = bps[dev];
  return err[dev];
}
// S as a 2-D tensor of rows of 128 bytes (floor(n / 128) rows; the kernel
// copies the partial last row itself), boxes of one 2048-byte tile, 128-byte
// swizzle.  cuTensorMapEncodeTiled comes from the driver through the
// runtime's entry-point query (no -lcuda).
bool rows128_tensor_map(CUtensorMap* map, const void* seq, uint64_t bytes, uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode || bytes < 128) return false;
  const cuuint64_t dims[2] = {128, bytes / 128};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(seq), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
int pair_red_override() {
  static const int v = [] {
    const char* s = std::getenv("WT_PAIR_RED");
    return (s && *s) ? (*s != '0' ? 1 : 0) : -1;
  }();
  return v;
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), uint32_t grid, uint32_t block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

enum Kind : uint32_t {
  K_PRO = 1, K_SCAN = 2, K_TABLES = 3, K_LEVEL = 4, K_LAST = 5, K_TSCAN = 6, K_MEMSET = 7, K_PAIR = 8, K_SBSCAN = 9,
  K_PREP = 11, K_FINAL = 12, K_DD_OFFSETS = 13, K_DD_MERGE = 14, K_DD_SB = 15, K_FLAGS = 16, K_P2C = 17,
  K_QUAD = 18, K_CLS3 = 21, K_TRIPLE = 22
};

// The launch sequence, shared by wt_build_async and wt_launch_plan.
template <typename T>
wt_status enqueue(const T* seq, uint64_t n, uint64_t sigma, const wt_tree_t* out, char* ws, const Carve& c,
                  Launcher& lk, uint32_t* kinds, uint32_t cap, uint32_t* count,
                  unsigned long long* mzeros = nullptr) {
  const cudaStream_t stream = lk.s;
  // mzeros != nullptr: the wavelet matrix (NEXT-4): every level one global
  // node, per-level zeros to mzeros[l], no node offsets
  const bool matrix = mzeros != nullptr;
  const bool dry = (seq == nullptr && out == nullptr);
  uint32_t nk = 0;
  auto note = [&](uint32_t kind) {
    if (kinds && nk < cap) kinds[nk] = kind;
    ++nk;
  };
  int32_t* flag = reinterpret_cast<int32_t*>(ws + c.off_flag);
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + c.off_counters);
  unsigned long long* ones0 = reinterpret_cast<unsigned long long*>(ws + c.off_ones0);
  const wt::LookbackState status{reinterpret_cast<uint32_t*>(ws + c.off_status),
                                 reinterpret_cast<uint64_t*>(ws + c.off_value), c.status_entries};
  const wt::LookbackState status2{reinterpret_cast<uint32_t*>(ws + c.off_status2),
                                  reinterpret_cast<uint64_t*>(ws + c.off_value2), c.status_entries};
  uint2* tab = reinterpret_cast<uint2*>(ws + c.off_tab);
  uint32_t* agg = reinterpret_cast<uint32_t*>(ws + c.off_agg);
  uint32_t* pre = reinterpret_cast<uint32_t*>(ws + c.off_pre);
  uint32_t* cnt[2] = {reinterpret_cast<uint32_t*>(ws + c.off_cnt),
                      reinterpret_cast<uint32_t*>(ws + c.off_cnt + align_up(c.cnt_entries * sizeof(uint32_t)))};
  T* buf[2] = {reinterpret_cast<T*>(ws + c.off_bufA), reinterpret_cast<T*>(ws + c.off_bufB)};
  unsigned long long* C = (dry || matrix) ? nullptr : reinterpret_cast<unsigned long long*>(out->node_offsets);
  const uint32_t L = c.L;
  cudaError_t e;
  // a5: interior fused groups (k_quad) at l = 0, 2, ..., 2 (nquad - 1)
  const uint32_t nquad = matrix ? 0u : quad_levels(L);
  uint32_t* agg01 = reinterpret_cast<uint32_t*>(ws + c.off_agg01);
  uint32_t* agg11 = reinterpret_cast<uint32_t*>(ws + c.off_agg11);
  uint32_t* hist4 = reinterpret_cast<uint32_t*>(ws + c.off_hist4);
  uint32_t* pre01 = reinterpret_cast<uint32_t*>(ws + c.off_pre01);
  uint32_t* pre11 = reinterpret_cast<uint32_t*>(ws + c.off_pre11);

  if (!dry) {
    if ((e = cudaMemsetAsync(ws, 0, c.ctrl_bytes, stream)) != cudaSuccess) return fail_cuda(e, "memset ctrl");
    if (n == 0) {
      if (matrix) {
        if (L && (e = cudaMemsetAsync(mzeros, 0, (size_t)L * 8, stream)) != cudaSuccess)
          return fail_cuda(e, "memset zeros");
      } else if ((e = cudaMemsetAsync(C, 0, c.c_len * 8, stream)) != cudaSuccess) {
        return fail_cuda(e, "memset C");
      }
      if (L && (e = cudaMemsetAsync(out->superblocks, 0, (size_t)L * c.nsb * 8, stream)) != cudaSuccess)
        return fail_cuda(e, "memset sb");
      if (count) *count = 0;
      return WT_OK;
    }
  } else if (n == 0) {
    if (count) *count = 0;
    return WT_OK;
  }
  uint32_t epoch = 1, counter = 0;
  // one decoupled look-back scan launch
  auto scan = [&](auto op, uint64_t cnt_, const char* what) -> wt_status {
    if (!dry) {
      if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
      constexpr uint64_t ST = wt::scan_tile_of<decltype(op)>();
      const uint32_t g = (uint32_t)((cnt_ + ST - 1) / ST);
      wt::k_scan<decltype(op)><<<g, wt::scan_threads_of<decltype(op)>(), 0, stream>>>(op, cnt_, status, counters + counter, epoch, flag);
      if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, what);
      if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
    }
    ++epoch;
    ++counter;
    return WT_OK;
  };
  wt_status st;

  // a1: the pass over S: range check, level-0 tile ones agg0, ones0
  note(K_PRO);
  if (!dry) {
    if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
    const uint64_t tiles = (n + wt::LvTile<T>::TILE - 1) / wt::LvTile<T>::TILE;  // one warp per tile
    const uint32_t grid = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>((tiles + wt::PRO_THREADS / 32 - 1) / (wt::PRO_THREADS / 32), 8ull * num_sms()));
    if (nquad)
      wt::k_prologue<T, true><<<grid, wt::PRO_THREADS, 0, stream>>>(seq, n, sigma, L, agg, ones0, flag, agg01,
                                                                     agg11, hist4);
    else
      wt::k_prologue<T><<<grid, wt::PRO_THREADS, 0, stream>>>(seq, n, sigma, L, L ? agg : nullptr, ones0, flag);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_prologue");
    if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
  }
  // one k_prep launch: scan A (look-back state 1), scan B (state 2), zero fills
  auto prep = [&](uint32_t kind, auto opA, uint64_t na, auto opB, uint64_t nb, wt::ZeroFill z,
                  const char* what) -> wt_status {
    note(kind);
    if (!dry) {
      if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
      constexpr int NT = wt::scan_threads_of<decltype(opA)>();  // (k_prep: CTAs of the first scan's size)
      constexpr uint64_t STA = wt::scan_tile_of<decltype(opA), NT>(), STB = wt::scan_tile_of<decltype(opB), NT>();
      const uint64_t ga = (na + STA - 1) / STA, gb = (nb + STB - 1) / STB;
      const uint64_t zu = z.n0 + z.n1;
      const uint64_t gz = zu ? std::min<uint64_t>((zu + 4 * NT - 1) / (4 * NT),
                                                  4ull * num_sms())
                             : (ga + gb ? 0 : 1);
      e = launch_pdl(wt::k_prep<decltype(opA), decltype(opB)>, (uint32_t)(ga + gb + gz), (uint32_t)NT, 0, stream,
                     opA, na, status, counters + counter, epoch, opB, nb, status2, counters + counter + 1, epoch + 1, z,
                     (const int32_t*)flag);
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, what);
      if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
    }
    epoch += 2;
    counter += 2;
    return WT_OK;
  };
  const wt::ZeroFill nozero{nullptr, 0, nullptr, 0};

  if (L == 0 && matrix) {  // no levels, nothing but the range check
    if (count) *count = nk;
    return WT_OK;
  }
  if (L == 0) {  // sigma = 1: C = [0, n]
    note(K_SCAN);
    if ((st = scan(wt::OpLeafC{nullptr, C, 1, n, nullptr}, 1, "k_scan(C)")) != WT_OK) return st;
    if (count) *count = nk;
    return WT_OK;
  }

  // a3 / a4: one pass per level
  constexpr uint64_t TILE = wt::LvTile<T>::TILE;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const size_t lsmem = wt::level_smem_bytes<T>();
  int bps_sc = 1, bps_last = 1, bps_pair = 1;
  if (!dry) {
    if ((e = level_kernel_setup<T, 1>(&bps_sc)) != cudaSuccess) return fail_cuda(e, "k_level setup");
    if ((e = level_kernel_setup<T, 0>(&bps_last)) != cudaSuccess) return fail_cuda(e, "k_level setup");
    if ((e = level_kernel_setup<T, 2>(&bps_pair)) != cudaSuccess) return fail_cuda(e, "k_level setup");
  }
  const uint32_t grid_sc = (uint32_t)std::min<uint64_t>(ntiles, (uint64_t)bps_sc * (uint64_t)num_sms());
  const uint32_t grid_last = (uint32_t)std::min<uint64_t>(ntiles, (uint64_t)bps_last * (uint64_t)num_sms());
  const uint32_t grid_pair = (uint32_t)std::min<uint64_t>(ntiles, (uint64_t)bps_pair * (uint64_t)num_sms());
  // two levels of 1-byte symbols: the specialised pass (wt_pair2.cuh) replaces the fused pair
  const bool pair2 = (L == 2 && !matrix && sizeof(T) == 1 && n >= 128 && pair2_enabled());
  // any other tree: the general fused final pair without symbol moves (wt_pairn.cuh)
  const bool pairn = (!pair2 && n * sizeof(T) >= 128 && pairn_enabled());
  const bool triple = (!matrix && L >= 3 && n * sizeof(T) >= 128 && 2 * nquad <= L - 3 && triple_enabled());
  auto level = [&](uint32_t l, int mode) -> wt_status {
    note(mode == 0 ? K_LAST : mode == 2 ? K_PAIR : K_LEVEL);
    if (dry) return WT_OK;
    if (mode == 2 && pair2) {
      int bps = 1;
      if ((e = pair2_setup(&bps)) != cudaSuccess) return fail_cuda(e, "k_pair2 setup");
      if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
      const uint64_t nwt = (n + wt::P2_WT - 1) / wt::P2_WT;  // warp tiles
      const uint32_t grid = (uint32_t)std::min<uint64_t>((nwt + wt::P2_WARPS - 1) / wt::P2_WARPS,
                                                         (uint64_t)bps * num_sms());
      CUtensorMap tmap;
      if (!rows128_tensor_map(&tmap, seq, n, wt::P2_WT / 128)) return fail(WT_ERR_CUDA, "cuTensorMapEncodeTiled");
      e = launch_pdl(wt::k_pair2, grid, (uint32_t)(32 * wt::P2_WARPS), wt::p2_smem_bytes(), stream,
                     reinterpret_cast<const uint8_t*>(seq), n, (uint32_t)c.ntiles, (const uint32_t*)pre,
                     (const unsigned long long*)ones0, out->bitmaps,
                     reinterpret_cast<unsigned long long*>(out->superblocks), c.nsb, out->bitmaps + c.words,
                     (const int32_t*)flag, tmap);
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_pair2");
      if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
      return WT_OK;
    }
    const T* in = (l == 0) ? seq : buf[(l - 1) & 1];
    if (mode == 2 && pairn) {
      int bps = 1;
      if ((e = pairn_setup<T>(&bps)) != cudaSuccess) return fail_cuda(e, "k_pairn setup");
      if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
      const uint64_t nwt = (n + wt::PnCfg<T>::WT - 1) / wt::PnCfg<T>::WT;  // warp tiles
      const uint32_t grid = (uint32_t)std::min<uint64_t>((nwt + wt::PN_WARPS - 1) / wt::PN_WARPS,
                                                         (uint64_t)bps * num_sms());
      CUtensorMap tmap;
      if (!rows128_tensor_map(&tmap, in, n * sizeof(T), wt::PN_WT / 128))
        return fail(WT_ERR_CUDA, "cuTensorMapEncodeTiled");
      e = launch_pdl(wt::k_pairn<T>, grid, (uint32_t)(32 * wt::PN_WARPS), wt::pn_smem_bytes(), stream, in,
                     (uint32_t)n, (uint32_t)c.ntiles, (const uint32_t*)pre,
                     (const uint2*)(matrix ? tab + l : tab + ((1ull << l) - 1)), out->bitmaps + (uint64_t)l * c.words,
                     (uint32_t)c.words,
                     reinterpret_cast<unsigned long long*>(out->superblocks) + (uint64_t)l * c.nsb, (uint32_t)c.nsb,
                     out->bitmaps + (uint64_t)(L - 1) * c.words, matrix ? 0u : 0xffffffffu, (const int32_t*)flag,
                     tmap);
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_pairn");
      if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
      return WT_OK;
    }
    T* o = mode == 0 ? nullptr : mode == 2 ? reinterpret_cast<T*>(out->bitmaps + (uint64_t)(L - 1) * c.words)
                                           : buf[l & 1];
    const int red = pair_red_override();
    const bool red_runs = mode == 2 && (red < 0 ? l == 0 : red == 1);
    const uint32_t sh = (L - 1 - l) | (matrix ? wt::LV_MATRIX : 0u) | (red_runs ? wt::LV_RED : 0u);
    const uint2* t = mode == 0 ? nullptr : matrix ? tab + l : tab + ((1ull << l) - 1);
    uint32_t* bits = out->bitmaps + (uint64_t)l * c.words;
    unsigned long long* sb = reinterpret_cast<unsigned long long*>(out->superblocks) + (uint64_t)l * c.nsb;
    uint32_t* agg_next = mode == 1 ? agg + (uint64_t)(l + 1) * c.ntiles : nullptr;
    uint32_t* cn = mode == 0 ? nullptr : cnt[l & 1];
    if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
    const uint32_t n32 = (uint32_t)n, nt32 = (uint32_t)c.ntiles, w32 = (uint32_t)c.words, nsb32 = (uint32_t)c.nsb;
    const uint32_t* pre_c = pre;
    const int32_t* flag_c = flag;
    if (mode == 0)
      e = launch_pdl(wt::k_level<T, 0>, grid_last, wt::LV_THREADS, lsmem, stream, in, o, n32, nt32, sh, t, bits, w32,
                     sb, nsb32, pre_c, agg_next, cn, flag_c);
    else if (mode == 2)
      e = launch_pdl(wt::k_level<T, 2>, grid_pair, wt::LV_THREADS, lsmem, stream, in, o, n32, nt32, sh, t, bits, w32,
                     sb, nsb32, pre_c, agg_next, cn, flag_c);
    else
      e = launch_pdl(wt::k_level<T, 1>, grid_sc, wt::LV_THREADS, lsmem, stream, in, o, n32, nt32, sh, t, bits, w32,
                     sb, nsb32, pre_c, agg_next, cn, flag_c);
    if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_level");
    if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
    return WT_OK;
  };

  if (L == 1) {  // C from ones0, the tile prefixes of level 0, the single (last) level
    if (matrix) {
      if ((st = prep(K_PREP, wt::OpTilePrefix{agg, pre}, c.ntiles,
                     wt::OpMatrixTab{agg, tab, mzeros, n, c.ntiles}, c.ntiles, nozero, "k_prep")) != WT_OK)
        return st;
    } else if ((st = prep(K_PREP, wt::OpTilePrefix{agg, pre}, c.ntiles, wt::OpLeafC{nullptr, C, 2, n, ones0}, 2,
                          nozero, "k_prep")) != WT_OK) {
      return st;
    }
    if ((st = level(0, 0)) != WT_OK) return st;
    if (count) *count = nk;
    return WT_OK;
  }
#ifdef WT_EXP_LEVELS  // experiment builds: only the first level passes (timing studies)
  const uint32_t Lrun = std::min<uint32_t>(L - 1, WT_EXP_LEVELS);
#else
  const uint32_t Lrun = L - 1;
#endif
  // L >= 2: passes 0..L-3 write T_{l+1}; pass L-2 is fused with level L-1
  // (writes B_{L-1} directly, no T_{L-1})
  uint32_t* const lastbits = dry ? nullptr : out->bitmaps + (uint64_t)(L - 1) * c.words;
  // The quads first.  Quad q (level l = 2q) reads T_l and the level-(l+2)
  // node sizes (hist4 for q = 0) and writes T_{l+2} and the node sizes the
  // next pass needs into the buffers of parity (nquad - 1 - q) + 1, so that the
  // pass after the last quad (level 2 nquad) finds them where a level pass
  // expects its input: T in buf[1], counts in cnt[1].
  for (uint32_t q = 0; q < nquad && 2 * q < Lrun; ++q) {
    const uint32_t l = 2 * q;
    const uint32_t D = (q + 1 < nquad) ? 2u : 1u;  // node sizes for a following quad (l+4) or level pass (l+3)
    const uint32_t po = ((nquad - 1 - q) & 1u) ? 0u : 1u;
    const uint64_t nt = c.ntiles;
    uint32_t* bits1 = dry ? nullptr : out->bitmaps + (uint64_t)(l + 1) * c.words;
    wt::ZeroFill z{dry ? nullptr : reinterpret_cast<uint4*>(cnt[po]), 1ull << (l + D),
                   reinterpret_cast<uint4*>(bits1), c.words / 4};
    if ((st = prep(K_PREP, wt::OpTilePrefix2{agg01 + l * nt, agg11 + l * nt, pre01, pre11}, nt,
                   wt::OpTilePrefix{agg + l * nt, pre}, nt, z, "k_prep(quad)")) != WT_OK)
      return st;
    note(K_QUAD);
    if (!dry) {
      int bps = 1;
      if ((e = quad_setup<T>(&bps)) != cudaSuccess) return fail_cuda(e, "k_quad setup");
      if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
      constexpr uint64_t QT = wt::QCfg<T>::TILE;
      const uint64_t ntq = (n + QT - 1) / QT;
      const uint32_t grid = (uint32_t)std::min<uint64_t>(ntq, (uint64_t)bps * num_sms());
      wt::QuadArgs qa;
      qa.n = (uint32_t)n;
      qa.ntq = (uint32_t)ntq;
      qa.sh = L - 1 - l;
      qa.nodes = 1u << l;
      qa.pre1 = pre;
      qa.pre01 = pre01;
      qa.pre11 = pre11;
      qa.gcnt = l == 0 ? hist4 : cnt[po ^ 1u];
      qa.bits = out->bitmaps + (uint64_t)l * c.words;
      qa.sb = reinterpret_cast<unsigned long long*>(out->superblocks) + (uint64_t)l * c.nsb;
      qa.nsb = (uint32_t)c.nsb;
      qa.words = (uint32_t)c.words;
      qa.bits1 = bits1;
      qa.agg_next = agg + (l + 2) * nt;
      qa.agg01_next = D == 2 ? agg01 + (l + 2) * nt : nullptr;
      qa.agg11_next = D == 2 ? agg11 + (l + 2) * nt : nullptr;
      qa.cnt_next = cnt[po];
      qa.D = D;
      qa.flag = flag;
      const T* qin = l == 0 ? seq : buf[po ^ 1u];
      e = launch_pdl(wt::k_quad<T>, grid, wt::Q_THREADS, wt::quad_smem_bytes<T>(), stream, qin, buf[po], qa);
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_quad");
      if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
    }
    // superblocks of level l+1 from the bits the quad OR-ed in
    note(K_SBSCAN);
    if ((st = scan(wt::OpBitsPop{bits1, dry ? nullptr
                                            : reinterpret_cast<unsigned long long*>(out->superblocks) +
                                                  (uint64_t)(l + 1) * c.nsb,
                                 c.nsb - 1, 0},
                   c.nsb - 1, "k_scan(quad sb)")) != WT_OK)
      return st;
  }
  const uint32_t lstop = triple ? std::min<uint32_t>(Lrun, L - 3) : Lrun;
  for (uint32_t l = 2 * nquad; l < lstop; ++l) {
    const bool pair = (l + 2 == L);
    // pre_l (scan of agg_l), the node tables of level l (from the level-(l+1)
    // node sizes counted by pass l-1, or from ones0 for l = 0), and zero the
    // node-count buffer pass l fills (and B_{L-1}, OR-ed by the fused pass)
    // (k_pairn counts no leaves: no count buffer to zero before it)
    wt::ZeroFill z{dry ? nullptr : reinterpret_cast<uint4*>(cnt[l & 1]),
                   (pair && pairn) ? 0ull : matrix ? 1ull : 1ull << l,
                   pair && !dry ? reinterpret_cast<uint4*>(lastbits) : nullptr, pair ? c.words / 4 : 0};
    if (matrix) {  // the level's one-node table from the scan of its per-tile ones
      wt::OpMatrixTab tb{agg + (uint64_t)l * c.ntiles, tab + l, mzeros + l, n, c.ntiles};
      if ((st = prep(K_PREP, wt::OpTilePrefix{agg + (uint64_t)l * c.ntiles, pre}, c.ntiles, tb, c.ntiles, z,
                     "k_prep")) != WT_OK)
        return st;
    } else {
      wt::OpLevelTab tb = (l == 0) ? wt::OpLevelTab{nullptr, tab, n, ones0}
                                   : wt::OpLevelTab{dry ? nullptr : cnt[(l - 1) & 1], tab + ((1ull << l) - 1), n,
                                                    nullptr};
      if ((st = prep(K_PREP, wt::OpTilePrefix{agg + (uint64_t)l * c.ntiles, pre}, c.ntiles, tb, 1ull << l, z,
                     "k_prep")) != WT_OK)
        return st;
    }
    if ((st = level(l, pair ? 2 : 1)) != WT_OK) return st;
  }
  if (triple && Lrun == L - 1) {
    // the fused final three levels: the level-(L-3) prep (tile prefixes, node
    // table; zero the class sizes and B_{L-2}), the class counts, their
    // prefixes and node table (zero B_{L-1}), the pass, the superblocks of
    // B_{L-2} and B_{L-1}, C
    const uint32_t l = L - 3;
    const uint64_t nt = c.ntiles, nv3 = 1ull << l;
    char* tr = ws + c.off_tr;
    uint32_t* tagg01 = reinterpret_cast<uint32_t*>(tr);
    uint32_t* tagg11 = reinterpret_cast<uint32_t*>(tr + align_up(nt * 4));
    uint32_t* tpre01 = reinterpret_cast<uint32_t*>(tr + 2 * align_up(nt * 4));
    uint32_t* tpre11 = reinterpret_cast<uint32_t*>(tr + 3 * align_up(nt * 4));
    uint2* cls = reinterpret_cast<uint2*>(tr + 4 * align_up(nt * 4));
    uint2* tab3 = reinterpret_cast<uint2*>(tr + 4 * align_up(nt * 4) + align_up(nv3 * sizeof(uint2)));
    uint32_t* B2 = dry ? nullptr : out->bitmaps + (uint64_t)(L - 2) * c.words;
    uint32_t* B1 = lastbits;
    const uint2* tabl = tab + ((1ull << l) - 1);
    {
      wt::ZeroFill z{dry ? nullptr : reinterpret_cast<uint4*>(cls), (nv3 * sizeof(uint2) + 15) / 16,
                     dry ? nullptr : reinterpret_cast<uint4*>(B2), c.words / 4};
      wt::OpLevelTab tb = (l == 0) ? wt::OpLevelTab{nullptr, tab, n, ones0}
                                   : wt::OpLevelTab{dry ? nullptr : cnt[(l - 1) & 1], tab + ((1ull << l) - 1), n,
                                                    nullptr};
      if ((st = prep(K_PREP, wt::OpTilePrefix{agg + (uint64_t)l * c.ntiles, pre}, c.ntiles, tb, 1ull << l, z,
                     "k_prep")) != WT_OK)
        return st;
    }
    const T* in = (l == 0) ? seq : buf[(l - 1) & 1];
    note(K_CLS3);
    if (!dry) {
      if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
      const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((nt + 7) / 8, 8ull * num_sms()));
      e = launch_pdl(wt::k_cls3<T>, g, 256u, (size_t)0, stream, in, (uint32_t)n, (uint32_t)nt, tagg01, tagg11, cls,
                     (const int32_t*)flag);
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_cls3");
      if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
    }
    {
      wt::ZeroFill z{dry ? nullptr : reinterpret_cast<uint4*>(B1), c.words / 4, nullptr, 0};
      if ((st = prep(K_PREP, wt::OpTilePrefix2{tagg01, tagg11, tpre01, tpre11}, nt, wt::OpNodeCls{cls, tab3}, nv3, z,
                     "k_prep(classes)")) != WT_OK)
        return st;
    }
    note(K_TRIPLE);
    if (!dry) {
      int bps = 1;
      if ((e = triple_setup<T>(&bps)) != cudaSuccess) return fail_cuda(e, "k_triple setup");
      if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
      const uint64_t nwt = (n + wt::TrCfg<T>::WT - 1) / wt::TrCfg<T>::WT;
      const uint32_t grid = (uint32_t)std::min<uint64_t>((nwt + wt::PN_WARPS - 1) / wt::PN_WARPS,
                                                         (uint64_t)bps * num_sms());
      CUtensorMap tmap;
      if (!rows128_tensor_map(&tmap, in, n * sizeof(T), wt::PN_WT / 128))
        return fail(WT_ERR_CUDA, "cuTensorMapEncodeTiled");
      e = launch_pdl(wt::k_triple<T>, grid, (uint32_t)(32 * wt::PN_WARPS), wt::tr_smem_bytes(), stream, in,
                     (uint32_t)n, (uint32_t)nt, (const uint32_t*)pre, (const uint32_t*)tpre01,
                     (const uint32_t*)tpre11, tabl, (uint32_t)nv3, (const uint2*)tab3, (const uint2*)cls,
                     out->bitmaps + (uint64_t)l * c.words,
                     reinterpret_cast<unsigned long long*>(out->superblocks) + (uint64_t)l * c.nsb, (uint32_t)c.nsb,
                     B2, B1, (const int32_t*)flag, tmap);
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_triple");
      if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
    }
    unsigned long long* const sb2 =
        dry ? nullptr : reinterpret_cast<unsigned long long*>(out->superblocks) + (uint64_t)(L - 2) * c.nsb;
    unsigned long long* const sb1 =
        dry ? nullptr : reinterpret_cast<unsigned long long*>(out->superblocks) + (uint64_t)(L - 1) * c.nsb;
    if ((st = prep(K_FINAL, wt::OpBitsPop{B2, sb2, c.nsb - 1}, c.nsb - 1, wt::OpBitsPop{B1, sb1, c.nsb - 1},
                   c.nsb - 1, nozero, "k_prep(final)")) != WT_OK)
      return st;
    note(K_P2C);
    if (!dry) {
      if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
      const uint32_t g = (uint32_t)std::min<uint64_t>((nv3 + 255) / 256, 8ull * num_sms());
      e = launch_pdl(wt::k_leaf3, g, 256u, (size_t)0, stream, tabl, (const uint2*)tab3, (const uint2*)cls, L,
                     (const uint32_t*)B1, (const unsigned long long*)sb1, n, C, (const int32_t*)flag);
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_leaf3");
      if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
    }
  } else if (Lrun == L - 1) {
    // superblocks of level L-1 from the bitmap the fused pass wrote, and C
    // (exclusive scan of the leaf counts pass L-2 made)
    // superblocks of level L-1: one scan launch that reads B_{L-1} itself
    // (block popcounts taken coalesced per scan tile), and C
    unsigned long long* const sbl =
        dry ? nullptr : reinterpret_cast<unsigned long long*>(out->superblocks) + (uint64_t)(L - 1) * c.nsb;
    if (matrix) {
      if ((st = prep(K_FINAL, wt::OpBitsPopZ{lastbits, sbl, c.nsb - 1, mzeros + (L - 1), n}, c.nsb - 1, wt::OpNone{},
                     0, nozero, "k_prep(final)")) != WT_OK)
        return st;
    } else if (pair2 || pairn) {
      // B_{L-1}'s superblocks, then C from them (k_pair2 / k_pairn count no leaves)
      if ((st = prep(K_FINAL, wt::OpBitsPop{lastbits, sbl, c.nsb - 1}, c.nsb - 1, wt::OpNone{}, 0, nozero,
                     "k_prep(final)")) != WT_OK)
        return st;
      note(K_P2C);
      if (!dry) {
        if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
        const uint64_t nv = 1ull << (L - 2);  // one thread per level-(L-2) node
        const uint32_t g = (uint32_t)std::min<uint64_t>((nv + 255) / 256, 8ull * num_sms());
        e = launch_pdl(wt::k_leaf_offsets, g, 256u, (size_t)0, stream, (const uint2*)(tab + ((1ull << (L - 2)) - 1)),
                       L, (const uint32_t*)lastbits, (const unsigned long long*)sbl, n, C, (const int32_t*)flag);
        if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_leaf_offsets");
        if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
      }
    } else if ((st = prep(K_FINAL, wt::OpBitsPop{lastbits, sbl, c.nsb - 1}, c.nsb - 1,
                          wt::OpLeafC{dry ? nullptr : cnt[(L - 2) & 1], C, 1ull << L, n, nullptr}, 1ull << L, nozero,
                          "k_prep(final)")) != WT_OK) {
      return st;
    }
  }
  if (count) *count = nk;
  return WT_OK;
}

wt_status dispatch_direct(const void* seq, uint64_t n, uint64_t sigma, uint32_t width, const wt_tree_t* out,
                          char* ws, const Carve& c, Launcher& lk, uint32_t* kinds, uint32_t cap, uint32_t* count,
                          unsigned long long* mzeros = nullptr) {
  switch (width) {
    case 1: return enqueue<uint8_t>((const uint8_t*)seq, n, sigma, out, ws, c, lk, kinds, cap, count, mzeros);
    case 2: return enqueue<uint16_t>((const uint16_t*)seq, n, sigma, out, ws, c, lk, kinds, cap, count, mzeros);
    default:
      return enqueue<uint32_t>((const uint32_t*)seq, n, sigma, out, ws, c, lk, kinds, cap, count, mzeros);
  }
}

// One level of a dd merge over the word range [w_begin, w_end) of the merged
// level bitmap (into out[0 ..)), and the segments' node offsets / sources.
cudaError_t launch_merge_level(const wt::DdOffsets& sg, const wt::DdLevelSrc& src, uint32_t l,
                               const unsigned long long* C, uint64_t n, uint64_t w_begin, uint64_t w_end,
                               uint32_t* out, cudaStream_t s, const int32_t* flag = nullptr) {
  if (w_end <= w_begin) return cudaSuccess;
  const uint64_t threads = (w_end - w_begin + wt::DD_WPT - 1) / wt::DD_WPT;
  wt::k_dd_merge_level<<<(uint32_t)((threads + wt::DD_THREADS - 1) / wt::DD_THREADS), wt::DD_THREADS, 0, s>>>(
      sg, src, l, C, n, w_begin, w_end, out, flag);
  return cudaGetLastError();
}

// superblocks of nblocks 512-bit blocks of `bits` (plus the final total), each
// offset by `base`: one decoupled-look-back scan launch (counter + status
// zeroed by the caller, epoch distinguishes launches sharing them)
cudaError_t launch_superblocks(const uint32_t* bits, uint64_t nblocks, uint64_t base, unsigned long long* sb,
                               const wt::LookbackState& lb, uint32_t* counter, uint32_t epoch, const int32_t* noflag,
                               cudaStream_t s) {
  if (nblocks == 0) {  // one entry: the base
    wt::k_set_u64<<<1, 32, 0, s>>>(sb, base);
    return cudaGetLastError();
  }
  constexpr uint64_t ST = wt::scan_tile_of<wt::OpBitsPop>();
  const uint32_t tiles = (uint32_t)((nblocks + ST - 1) / ST);
  wt::k_scan<wt::OpBitsPop><<<tiles, wt::scan_threads_of<wt::OpBitsPop>(), 0, s>>>(wt::OpBitsPop{bits, sb, nblocks, base}, nblocks, lb,
                                                               counter, epoch, noflag);
  return cudaGetLastError();
}

// A segmented build (c.seg): every segment with the direct launch sequence
// into its own tree (the segment workspace reused), the segments' range flags
// kept, then the merge: C = sum of the segments' C, every level's node runs
// concatenated (k_dd_merge_level), superblocks rescanned, flags OR-ed.
wt_status dispatch_segmented(const void* seq, uint64_t n, uint64_t sigma, uint32_t width, const wt_tree_t* out,
                             char* ws, const Carve& c, Launcher& lk, uint32_t* kinds, uint32_t cap,
                             uint32_t* count) {
  const bool dry = (seq == nullptr && out == nullptr);
  const cudaStream_t s = lk.s;
  uint32_t nk = 0;
  auto note = [&](uint32_t kind) {
    if (kinds && nk < cap) kinds[nk] = kind;
    ++nk;
  };
  cudaError_t e;
  int32_t* const flag = reinterpret_cast<int32_t*>(ws + c.off_flag);  // OR of the segments' range flags
  if (!dry && (e = cudaMemsetAsync(ws, 0, c.seg_ctrl, s)) != cudaSuccess) return fail_cuda(e, "memset seg ctrl");
  wt::DdOffsets sg{};
  sg.k = c.k;
  sg.L = c.L;
  wt_tree_t segt[wt::DD_MAX_SEGMENTS];
  uint64_t segn[wt::DD_MAX_SEGMENTS];
  for (uint32_t g = 0; g < c.k; ++g) {
    segn[g] = std::min(c.seg_len, n - (uint64_t)g * c.seg_len);
    char* t = ws + c.off_tree[g];
    segt[g].bitmaps = reinterpret_cast<uint32_t*>(t);
    segt[g].superblocks = reinterpret_cast<uint64_t*>(t + align_up((size_t)c.L * words_of(segn[g]) * 4));
    segt[g].node_offsets = reinterpret_cast<uint64_t*>(t + align_up((size_t)c.L * words_of(segn[g]) * 4) +
                                                       align_up((size_t)c.L * nsb_of(segn[g]) * 8));
    sg.C[g] = reinterpret_cast<const unsigned long long*>(segt[g].node_offsets);
    const Carve cg = carve_direct(segn[g], sigma, width);
    const void* sq = dry ? nullptr : static_cast<const char*>(seq) + (uint64_t)g * c.seg_len * width;
    uint32_t sub = 0;
    wt_status st = dispatch_direct(sq, segn[g], sigma, width, dry ? nullptr : &segt[g], ws + c.off_segws, cg, lk,
                                   kinds ? kinds + std::min(nk, cap) : nullptr, cap > nk ? cap - nk : 0, &sub);
    if (st != WT_OK) return st;
    nk += sub;
    note(K_FLAGS);
    if (!dry) {
      wt::k_or_flag<<<1, 32, 0, s>>>(reinterpret_cast<const int32_t*>(ws + c.off_segws + cg.off_flag), flag);
      if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_or_flag");
    }
  }
  unsigned long long* C = dry ? nullptr : reinterpret_cast<unsigned long long*>(out->node_offsets);
  note(K_DD_OFFSETS);
  if (!dry) {
    if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
    wt::k_dd_sum_offsets<<<(uint32_t)std::min<uint64_t>((c.c_len + 255) / 256, 4ull * num_sms()), 256, 0, s>>>(
        sg, c.c_len, C, flag);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_dd_sum_offsets");
    if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
  }
  const wt::LookbackState lb{reinterpret_cast<uint32_t*>(ws + c.off_sc_status),
                             reinterpret_cast<uint64_t*>(ws + c.off_sc_value), c.sc_tiles};
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + c.off_sc_counters);
  for (uint32_t l = 0; l < c.L; ++l) {
    note(K_DD_MERGE);
    note(K_DD_SB);
    if (dry) continue;
    wt::DdLevelSrc src{};
    for (uint32_t g = 0; g < c.k; ++g) src.bits[g] = segt[g].bitmaps + (uint64_t)l * words_of(segn[g]);
    uint32_t* ob = out->bitmaps + (uint64_t)l * c.words;
    if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
    if ((e = launch_merge_level(sg, src, l, C, n, 0, c.words, ob, s, flag)) != cudaSuccess)
      return fail_cuda(e, "k_dd_merge_level");
    if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
    if ((e = lk.pre()) != cudaSuccess) return fail_cuda(e, "profile event record");
    unsigned long long* sbl = reinterpret_cast<unsigned long long*>(out->superblocks) + (uint64_t)l * c.nsb;
    if ((e = launch_superblocks(ob, c.nsb - 1, 0, sbl, lb, counters + l, l + 1, flag, s)) != cudaSuccess)
      return fail_cuda(e, "superblock scan");
    if ((e = lk.post()) != cudaSuccess) return fail_cuda(e, "profile event record");
  }
  if (count) *count = nk;
  return WT_OK;
}

wt_status dispatch(const void* seq, uint64_t n, uint64_t sigma, uint32_t width, const wt_tree_t* out, char* ws,
                   const Carve& c, Launcher& lk, uint32_t* kinds, uint32_t cap, uint32_t* count) {
  if (c.seg) return dispatch_segmented(seq, n, sigma, width, out, ws, c, lk, kinds, cap, count);
  return dispatch_direct(seq, n, sigma, width, out, ws, c, lk, kinds, cap, count);
}

wt::TreeView view_of(const wt_tree_t* t, uint64_t n, uint64_t sigma) {
  wt::TreeView v;
  v.bitmaps = t->bitmaps;
  v.sb = reinterpret_cast<const unsigned long long*>(t->superblocks);
  v.C = reinterpret_cast<const unsigned long long*>(t->node_offsets);
  v.n = n;
  v.W = 16 * ((n + 511) / 512);
  v.NSB = (n + 511) / 512 + 1;
  v.L = levels_of(sigma);
  return v;
}

}  // namespace

extern "C" {

wt_status wt_sizes(uint64_t n, uint64_t sigma, uint32_t width, wt_sizes_t* out) {
  if (!out) return fail(WT_ERR_ARG, "out is NULL");
  wt_status st = check_args(n, sigma, width);
  if (st != WT_OK) return st;
  const Carve c = carve(n, sigma, width);
  out->levels = c.L;
  out->width = width;
  out->words_per_level = c.words;
  out->sb_per_level = c.nsb;
  out->c_len = c.c_len;
  out->bitmap_bytes = (uint64_t)c.L * c.words * 4;
  out->superblock_bytes = (uint64_t)c.L * c.nsb * 8;
  out->node_offset_bytes = c.c_len * 8;
  out->workspace_bytes = c.total;
  out->host_workspace_bytes = c.host_total;
  return WT_OK;
}

wt_status wt_build_async(const void* d_seq, uint64_t n, uint64_t sigma, uint32_t width, const wt_tree_t* out,
                         void* d_workspace, size_t workspace_bytes, int32_t* d_status, wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = check_args(n, sigma, width);
  if (st != WT_OK) return st;
  if (!out || !out->node_offsets || (levels_of(sigma) > 0 && (!out->superblocks || (n > 0 && !out->bitmaps))))
    return fail(WT_ERR_ARG, "output pointers are NULL");
  if (n > 0 && !d_seq) return fail(WT_ERR_ARG, "d_seq is NULL");
  if (n > 0 && (reinterpret_cast<uintptr_t>(d_seq) & 15)) return fail(WT_ERR_ARG, "d_seq must be 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(out->bitmaps) & 15) || (reinterpret_cast<uintptr_t>(out->superblocks) & 7) ||
      (reinterpret_cast<uintptr_t>(out->node_offsets) & 7))
    return fail(WT_ERR_ARG, "bitmaps must be 16-byte aligned, superblocks and node_offsets 8-byte aligned");
  const Carve c = carve(n, sigma, width);
  if (!d_workspace || workspace_bytes < c.total) return fail(WT_ERR_WORKSPACE, "workspace too small");
  if (reinterpret_cast<uintptr_t>(d_workspace) & (ALIGN - 1))
    return fail(WT_ERR_ARG, "workspace must be 256-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  Launcher lk{s};
  st = dispatch(d_seq, n, sigma, width, out, ws, c, lk, nullptr, 0, nullptr);
  if (st != WT_OK) return st;
  if (d_status) {
    cudaError_t e = cudaMemcpyAsync(d_status, ws + c.off_flag, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return fail_cuda(e, "status copy");
  }
  return WT_OK;
}

wt_status wt_matrix_build_async(const void* d_seq, uint64_t n, uint64_t sigma, uint32_t width,
                                const wt_matrix_t* out, void* d_workspace, size_t workspace_bytes, int32_t* d_status,
                                wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = check_args(n, sigma, width);
  if (st != WT_OK) return st;
  const uint32_t L = levels_of(sigma);
  if (!out || (L > 0 && (!out->zeros || !out->superblocks || (n > 0 && !out->bitmaps))))
    return fail(WT_ERR_ARG, "output pointers are NULL");
  if (n > 0 && !d_seq) return fail(WT_ERR_ARG, "d_seq is NULL");
  if (n > 0 && (reinterpret_cast<uintptr_t>(d_seq) & 15)) return fail(WT_ERR_ARG, "d_seq must be 16-byte aligned");
  const Carve c = carve(n, sigma, width);
  if (c.seg) return fail(WT_ERR_ARG, "the wavelet matrix takes n <= seg_max() (2^31)");
  if (!d_workspace || workspace_bytes < c.total) return fail(WT_ERR_WORKSPACE, "workspace too small");
  if (reinterpret_cast<uintptr_t>(d_workspace) & (ALIGN - 1))
    return fail(WT_ERR_ARG, "workspace must be 256-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  wt_tree_t t{out->bitmaps, out->superblocks, nullptr};
  unsigned long long dummy = 0;  // (L = 0: no zeros array; the pointer only marks the matrix mode)
  unsigned long long* z = L ? reinterpret_cast<unsigned long long*>(out->zeros) : &dummy;
  Launcher lk{s};
  st = dispatch_direct(d_seq, n, sigma, width, &t, ws, c, lk, nullptr, 0, nullptr, z);
  if (st != WT_OK) return st;
  if (d_status) {
    cudaError_t e = cudaMemcpyAsync(d_status, ws + c.off_flag, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return fail_cuda(e, "status copy");
  }
  return WT_OK;
}

wt_status wt_matrix_access(const wt_matrix_t* mx, uint64_t n, uint64_t sigma, const uint64_t* d_pos, uint64_t m,
                           uint32_t* d_sym, int32_t* d_status, wt_stream_t stream) {
  g_last_error.clear();
  if (!mx || sigma == 0 || levels_of(sigma) > 30) return fail(WT_ERR_ARG, "bad matrix / sigma");
  if (m == 0) return WT_OK;
  if (!d_pos || !d_sym) return fail(WT_ERR_ARG, "NULL query pointer");
  wt_tree_t t{mx->bitmaps, mx->superblocks, nullptr};
  wt::TreeView v = view_of(&t, n, sigma);
  wt::k_matrix_access<<<(uint32_t)((m + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      v, reinterpret_cast<const unsigned long long*>(mx->zeros), d_pos, m, d_sym, d_status);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_matrix_access");
}

wt_status wt_matrix_rank(const wt_matrix_t* mx, uint64_t n, uint64_t sigma, const uint32_t* d_c,
                         const uint64_t* d_pos, uint64_t m, uint64_t* d_cnt, int32_t* d_status, wt_stream_t stream) {
  g_last_error.clear();
  if (!mx || sigma == 0 || levels_of(sigma) > 30) return fail(WT_ERR_ARG, "bad matrix / sigma");
  if (m == 0) return WT_OK;
  if (!d_c || !d_pos || !d_cnt) return fail(WT_ERR_ARG, "NULL query pointer");
  wt_tree_t t{mx->bitmaps, mx->superblocks, nullptr};
  wt::TreeView v = view_of(&t, n, sigma);
  wt::k_matrix_rank<<<(uint32_t)((m + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      v, reinterpret_cast<const unsigned long long*>(mx->zeros), sigma, d_c, d_pos, m,
      reinterpret_cast<unsigned long long*>(d_cnt), d_status);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_matrix_rank");
}

wt_status wt_build(const void* d_seq, uint64_t n, uint64_t sigma, uint32_t width, const wt_tree_t* out,
                   void* d_workspace, size_t workspace_bytes, wt_stream_t stream) {
  wt_status st = wt_build_async(d_seq, n, sigma, width, out, d_workspace, workspace_bytes, nullptr, stream);
  if (st != WT_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const Carve c = carve(n, sigma, width);
  int32_t h_flag = 0;
  cudaError_t e = cudaMemcpyAsync(&h_flag, static_cast<char*>(d_workspace) + c.off_flag, sizeof(int32_t),
                                  cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return fail_cuda(e, "flag readback");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail_cuda(e, "stream sync");
  if (h_flag) return fail(WT_ERR_SYMBOL_RANGE, "a symbol is >= sigma");
  return WT_OK;
}

wt_status wt_build_from_host_async(const void* h_seq, uint64_t n, uint64_t sigma, uint32_t width,
                                   const wt_tree_t* h_out, void* d_workspace, size_t workspace_bytes,
                                   int32_t* h_status, wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = check_args(n, sigma, width);
  if (st != WT_OK) return st;
  if (!h_out || !h_out->node_offsets || (n > 0 && !h_seq) || !h_status) return fail(WT_ERR_ARG, "NULL host pointer");
  const Carve c = carve(n, sigma, width);
  if (!d_workspace || workspace_bytes < c.host_total) return fail(WT_ERR_WORKSPACE, "workspace too small");
  if (reinterpret_cast<uintptr_t>(d_workspace) & (ALIGN - 1))
    return fail(WT_ERR_ARG, "workspace must be 256-byte aligned");
  char* ws = static_cast<char*>(d_workspace);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  wt_tree_t dtree;
  dtree.bitmaps = reinterpret_cast<uint32_t*>(ws + c.off_bits);
  dtree.superblocks = reinterpret_cast<uint64_t*>(ws + c.off_sb);
  dtree.node_offsets = reinterpret_cast<uint64_t*>(ws + c.off_c);
  cudaError_t e;
  if (n && (e = cudaMemcpyAsync(ws + c.off_seq, h_seq, n * width, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return fail_cuda(e, "H2D sequence");
  Launcher lk{s};
  st = dispatch(ws + c.off_seq, n, sigma, width, &dtree, ws, c, lk, nullptr, 0, nullptr);
  if (st != WT_OK) return st;
  const size_t bb = (size_t)c.L * c.words * 4, sbb = (size_t)c.L * c.nsb * 8, cb = c.c_len * 8;
  if (bb && (e = cudaMemcpyAsync(h_out->bitmaps, dtree.bitmaps, bb, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return fail_cuda(e, "D2H bitmaps");
  if (sbb && (e = cudaMemcpyAsync(h_out->superblocks, dtree.superblocks, sbb, cudaMemcpyDeviceToHost, s)) !=
                 cudaSuccess)
    return fail_cuda(e, "D2H superblocks");
  if ((e = cudaMemcpyAsync(h_out->node_offsets, dtree.node_offsets, cb, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return fail_cuda(e, "D2H node offsets");
  if ((e = cudaMemcpyAsync(h_status, ws + c.off_flag, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return fail_cuda(e, "status readback");
  return WT_OK;
}

wt_status wt_build_from_host(const void* h_seq, uint64_t n, uint64_t sigma, uint32_t width, const wt_tree_t* h_out,
                             void* d_workspace, size_t workspace_bytes, wt_stream_t stream) {
  int32_t h_flag = 0;
  wt_status st = wt_build_from_host_async(h_seq, n, sigma, width, h_out, d_workspace, workspace_bytes, &h_flag,
                                          stream);
  if (st != WT_OK) return st;
  cudaError_t e;
  if ((e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream))) != cudaSuccess)
    return fail_cuda(e, "stream sync");
  if (h_flag) return fail(WT_ERR_SYMBOL_RANGE, "a symbol is >= sigma");
  return WT_OK;
}

static wt_status query_args(const wt_tree_t* tree, uint64_t n, uint64_t sigma) {
  if (!tree || !tree->node_offsets) return fail(WT_ERR_ARG, "tree is NULL");
  if (sigma == 0 || levels_of(sigma) > 30) return fail(WT_ERR_ARG, "bad sigma");
  if (levels_of(sigma) > 0 && n > 0 && (!tree->bitmaps || !tree->superblocks))
    return fail(WT_ERR_ARG, "tree pointers are NULL");
  return WT_OK;
}

wt_status wt_access(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint64_t* d_pos, uint64_t m,
                    uint32_t* d_sym, int32_t* d_status, wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = query_args(tree, n, sigma);
  if (st != WT_OK) return st;
  if (m == 0) return WT_OK;
  if (!d_pos || !d_sym) return fail(WT_ERR_ARG, "NULL query pointer");
  const uint32_t grid = (uint32_t)((m + 255) / 256);
  wt::k_access<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(view_of(tree, n, sigma), d_pos, m, d_sym,
                                                                         d_status);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_access");
}

wt_status wt_rank(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint32_t* d_c, const uint64_t* d_pos,
                  uint64_t m, uint64_t* d_cnt, int32_t* d_status, wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = query_args(tree, n, sigma);
  if (st != WT_OK) return st;
  if (m == 0) return WT_OK;
  if (!d_c || !d_pos || !d_cnt) return fail(WT_ERR_ARG, "NULL query pointer");
  const uint32_t grid = (uint32_t)((m + 255) / 256);
  wt::k_rank<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      view_of(tree, n, sigma), sigma, d_c, d_pos, m, reinterpret_cast<unsigned long long*>(d_cnt), d_status);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_rank");
}

wt_status wt_select(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint32_t* d_c, const uint64_t* d_j,
                    uint64_t m, uint64_t* d_out, int32_t* d_status, wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = query_args(tree, n, sigma);
  if (st != WT_OK) return st;
  if (m == 0) return WT_OK;
  if (!d_c || !d_j || !d_out) return fail(WT_ERR_ARG, "NULL query pointer");
  const uint32_t grid = (uint32_t)((m + 255) / 256);
  wt::k_select<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      view_of(tree, n, sigma), sigma, d_c, d_j, m, reinterpret_cast<unsigned long long*>(d_out), d_status, nullptr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_select");
}

// ---------------------------------------------------------------- alphabet remap (NEXT-4)
namespace {
struct RemapCarve {
  uint64_t words = 0, tiles = 0;
  size_t off_flag = 0, off_counter = 0, off_total = 0, off_status = 0, ctrl = 0, off_value = 0, off_present = 0,
         off_rank = 0, total = 0;
};
RemapCarve remap_carve(uint64_t sigma) {
  RemapCarve r;
  r.words = (sigma + 31) / 32;
  constexpr uint64_t ST = wt::scan_tile_of<wt::OpPopPrefix>();
  r.tiles = std::max<uint64_t>(1, (r.words + ST - 1) / ST);
  size_t o = 0;
  r.off_flag = o;
  o += ALIGN;
  r.off_counter = o;
  o += ALIGN;
  r.off_total = o;
  o += ALIGN;
  r.off_status = o;
  o += align_up(r.tiles * sizeof(uint32_t));
  r.off_present = o;  // zeroed with the control block
  o += align_up(r.words * sizeof(uint32_t));
  r.ctrl = o;
  r.off_value = o;
  o += align_up(2 * r.tiles * sizeof(uint64_t));
  r.off_rank = o;
  o += align_up(r.words * sizeof(uint32_t));
  r.total = o;
  return r;
}
}  // namespace

size_t wt_remap_workspace_bytes(uint64_t sigma) { return (sigma == 0 || sigma > (1ull << 32)) ? 0 : remap_carve(sigma).total; }

wt_status wt_remap_alphabet(const void* d_seq, uint64_t n, uint64_t sigma, uint32_t width, void* d_out,
                            uint32_t* d_alphabet, uint64_t* d_sigma_out, void* d_workspace, size_t workspace_bytes,
                            int32_t* d_status, wt_stream_t stream) {
  g_last_error.clear();
  if (width != 1 && width != 2 && width != 4) return fail(WT_ERR_ARG, "width must be 1, 2 or 4");
  if (sigma == 0 || sigma > (1ull << (8 * width))) return fail(WT_ERR_ARG, "sigma out of range for the width");
  if (n >= (1ull << 32)) return fail(WT_ERR_ARG, "n must be < 2^32");
  if ((n > 0 && (!d_seq || !d_out)) || !d_alphabet || !d_sigma_out) return fail(WT_ERR_ARG, "NULL pointer");
  const RemapCarve r = remap_carve(sigma);
  if (!d_workspace || workspace_bytes < r.total) return fail(WT_ERR_WORKSPACE, "workspace too small");
  if (reinterpret_cast<uintptr_t>(d_workspace) & (ALIGN - 1))
    return fail(WT_ERR_ARG, "workspace must be 256-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  int32_t* flag = reinterpret_cast<int32_t*>(ws + r.off_flag);
  uint32_t* present = reinterpret_cast<uint32_t*>(ws + r.off_present);
  uint32_t* rank = reinterpret_cast<uint32_t*>(ws + r.off_rank);
  unsigned long long* total = reinterpret_cast<unsigned long long*>(ws + r.off_total);
  cudaError_t e;
  if ((e = cudaMemsetAsync(ws, 0, r.ctrl, s)) != cudaSuccess) return fail_cuda(e, "memset remap control");
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 8ull * num_sms()));
  auto launch_w = [&](auto tag) -> cudaError_t {
    using T = decltype(tag);
    wt::k_remap_mark<T><<<g, 256, 0, s>>>(static_cast<const T*>(d_seq), n, sigma, present, flag);
    return cudaGetLastError();
  };
  e = width == 1 ? launch_w(uint8_t{}) : width == 2 ? launch_w(uint16_t{}) : launch_w(uint32_t{});
  if (e != cudaSuccess) return fail_cuda(e, "k_remap_mark");
  const wt::LookbackState lb{reinterpret_cast<uint32_t*>(ws + r.off_status), reinterpret_cast<uint64_t*>(ws + r.off_value),
                             r.tiles};
  wt::k_scan<wt::OpPopPrefix><<<(uint32_t)r.tiles, wt::scan_threads_of<wt::OpPopPrefix>(), 0, s>>>(
      wt::OpPopPrefix{present, rank, r.words, total}, r.words, lb, reinterpret_cast<uint32_t*>(ws + r.off_counter), 1u,
      flag);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_scan(remap)");
  auto apply_w = [&](auto tag) -> cudaError_t {
    using T = decltype(tag);
    if (n) wt::k_remap_apply<T><<<g, 256, 0, s>>>(static_cast<const T*>(d_seq), n, present, rank, static_cast<T*>(d_out), flag);
    return cudaGetLastError();
  };
  e = width == 1 ? apply_w(uint8_t{}) : width == 2 ? apply_w(uint16_t{}) : apply_w(uint32_t{});
  if (e != cudaSuccess) return fail_cuda(e, "k_remap_apply");
  wt::k_remap_alphabet<<<(uint32_t)((r.words + 255) / 256), 256, 0, s>>>(present, rank, r.words, d_alphabet);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_remap_alphabet");
  if ((e = cudaMemcpyAsync(d_sigma_out, total, 8, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
    return fail_cuda(e, "sigma copy");
  if (d_status && (e = cudaMemcpyAsync(d_status, flag, 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
    return fail_cuda(e, "status copy");
  return WT_OK;
}

// ---------------------------------------------------------------- domain decomposition merge (NEXT-3)
namespace {
wt_status dd_offsets_of(uint32_t k, const uint64_t* const* seg_offsets, uint64_t sigma, wt::DdOffsets* sg) {
  if (k == 0 || k > (uint32_t)wt::DD_MAX_SEGMENTS || !seg_offsets) return fail(WT_ERR_ARG, "k must be 1..32");
  if (sigma == 0 || levels_of(sigma) > 30) return fail(WT_ERR_ARG, "bad sigma");
  *sg = wt::DdOffsets{};
  sg->k = k;
  sg->L = levels_of(sigma);
  for (uint32_t g = 0; g < k; ++g) {
    if (!seg_offsets[g]) return fail(WT_ERR_ARG, "NULL segment node offsets");
    sg->C[g] = reinterpret_cast<const unsigned long long*>(seg_offsets[g]);
  }
  return WT_OK;
}
struct HostCg {  // host accessor of the segments' node offsets
  const uint64_t* const* C;
  __host__ __device__ uint64_t operator()(uint32_t h, uint64_t i) const { return C[h][i]; }
};
}  // namespace

void wt_dd_part_blocks(uint64_t n, uint64_t parts, uint64_t part, uint64_t* block_begin, uint64_t* block_end) {
  uint64_t a = 0, b = 0;
  if (parts > 0 && part < parts) wt::dd_part_blocks(n, parts, part, &a, &b);
  if (block_begin) *block_begin = a;
  if (block_end) *block_end = b;
}

wt_status wt_dd_plan(uint32_t k, const uint64_t* const* h_seg_offsets, uint64_t sigma, uint64_t parts,
                     uint64_t* h_plan) {
  g_last_error.clear();
  wt::DdOffsets sg;
  wt_status st = dd_offsets_of(k, h_seg_offsets, sigma, &sg);
  if (st != WT_OK) return st;
  const uint32_t L = sg.L;
  if (parts == 0 || (!h_plan && L > 0)) return fail(WT_ERR_ARG, "parts = 0 or NULL plan");
  const HostCg cg{h_seg_offsets};
  uint64_t n = 0;
  for (uint32_t g = 0; g < k; ++g) n += h_seg_offsets[g][1ull << L];
  for (uint32_t l = 0; l < L; ++l)
    for (uint64_t p = 0; p < parts; ++p) {
      uint64_t b_lo, b_hi;
      wt::dd_part_blocks(n, parts, p, &b_lo, &b_hi);
      const uint64_t q_lo = std::min(n, 512 * b_lo), q_hi = std::min(n, 512 * b_hi);
      for (uint32_t g = 0; g < k; ++g) {
        uint64_t* e = h_plan + ((l * parts + p) * k + g) * 2;
        e[0] = wt::dd_src_before(cg, k, L, l, g, q_lo);
        e[1] = wt::dd_src_before(cg, k, L, l, g, q_hi);
      }
    }
  return WT_OK;
}

wt_status wt_dd_plan_async(uint32_t k, const uint64_t* const* d_seg_offsets, uint64_t sigma, uint64_t n,
                           uint64_t parts, uint64_t* d_plan, wt_stream_t stream) {
  g_last_error.clear();
  wt::DdOffsets sg;
  wt_status st = dd_offsets_of(k, d_seg_offsets, sigma, &sg);
  if (st != WT_OK) return st;
  if (parts == 0 || (!d_plan && sg.L > 0)) return fail(WT_ERR_ARG, "parts = 0 or NULL plan");
  const uint64_t t = (uint64_t)sg.L * parts * k;
  if (t == 0) return WT_OK;
  wt::k_dd_plan<<<(uint32_t)((t + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      sg, n, parts, reinterpret_cast<unsigned long long*>(d_plan));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_dd_plan");
}

wt_status wt_dd_offsets(uint32_t k, const uint64_t* const* d_seg_offsets, uint64_t sigma, uint64_t* d_offsets,
                        wt_stream_t stream) {
  g_last_error.clear();
  wt::DdOffsets sg;
  wt_status st = dd_offsets_of(k, d_seg_offsets, sigma, &sg);
  if (st != WT_OK) return st;
  if (!d_offsets) return fail(WT_ERR_ARG, "NULL output");
  const uint64_t clen = (1ull << sg.L) + 1;
  wt::k_dd_sum_offsets<<<(uint32_t)std::min<uint64_t>((clen + 255) / 256, 4ull * num_sms()), 256, 0,
                         reinterpret_cast<cudaStream_t>(stream)>>>(
      sg, clen, reinterpret_cast<unsigned long long*>(d_offsets), nullptr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_dd_sum_offsets");
}

wt_status wt_dd_merge_level(uint32_t k, const uint64_t* const* d_seg_offsets, const uint64_t* d_offsets,
                            uint64_t sigma, uint64_t n, uint32_t level, const uint32_t* const* d_src_bits,
                            const uint64_t* src_base, uint64_t word_begin, uint64_t word_end, uint32_t* d_out,
                            wt_stream_t stream) {
  g_last_error.clear();
  wt::DdOffsets sg;
  wt_status st = dd_offsets_of(k, d_seg_offsets, sigma, &sg);
  if (st != WT_OK) return st;
  if (level >= sg.L) return fail(WT_ERR_ARG, "level >= L");
  if (!d_offsets || !d_src_bits || word_end > words_of(n) || word_begin > word_end)
    return fail(WT_ERR_ARG, "bad merge arguments");
  if (word_end > word_begin && !d_out) return fail(WT_ERR_ARG, "NULL output");
  wt::DdLevelSrc src{};
  for (uint32_t g = 0; g < k; ++g) {
    src.bits[g] = d_src_bits[g];
    src.base[g] = src_base ? src_base[g] : 0;
    if (src.base[g] & 31) return fail(WT_ERR_ARG, "source base must be a multiple of 32");
  }
  cudaError_t e = launch_merge_level(sg, src, level, reinterpret_cast<const unsigned long long*>(d_offsets), n,
                                     word_begin, word_end, d_out, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_dd_merge_level");
}

size_t wt_superblocks_scratch_bytes(uint64_t nblocks) {
  const uint64_t tiles = sb_scan_tiles(nblocks);
  return 2 * ALIGN + align_up(tiles * 4) + align_up(2 * tiles * 8);
}

wt_status wt_superblocks(const uint32_t* d_bits, uint64_t nblocks, uint64_t base, uint64_t* d_sb, void* d_scratch,
                         size_t scratch_bytes, wt_stream_t stream) {
  g_last_error.clear();
  if (!d_sb || (nblocks && !d_bits)) return fail(WT_ERR_ARG, "NULL pointer");
  if (!d_scratch || scratch_bytes < wt_superblocks_scratch_bytes(nblocks))
    return fail(WT_ERR_WORKSPACE, "scratch too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* sc = static_cast<char*>(d_scratch);
  const uint64_t tiles = sb_scan_tiles(nblocks);
  // [0, ALIGN): ticket counter, then a zero word as the (unused) range flag
  const size_t off_status = 2 * ALIGN, off_value = off_status + align_up(tiles * 4);
  cudaError_t e = cudaMemsetAsync(sc, 0, off_value, s);
  if (e != cudaSuccess) return fail_cuda(e, "memset scratch");
  const wt::LookbackState lb{reinterpret_cast<uint32_t*>(sc + off_status), reinterpret_cast<uint64_t*>(sc + off_value),
                             tiles};
  e = launch_superblocks(d_bits, nblocks, base, reinterpret_cast<unsigned long long*>(d_sb), lb,
                         reinterpret_cast<uint32_t*>(sc), 1, reinterpret_cast<const int32_t*>(sc + ALIGN), s);
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "superblock scan");
}

size_t wt_dd_merge_scratch_bytes(uint64_t n) { return wt_superblocks_scratch_bytes((n + 511) / 512); }

wt_status wt_dd_merge(uint32_t k, const wt_tree_t* segs, const uint64_t* seg_n, uint64_t sigma,
                      const wt_tree_t* out, void* d_scratch, size_t scratch_bytes, wt_stream_t stream) {
  g_last_error.clear();
  if (k == 0 || k > (uint32_t)wt::DD_MAX_SEGMENTS || !segs || !seg_n || !out || !out->node_offsets)
    return fail(WT_ERR_ARG, "bad segment list or output");
  if (sigma == 0 || levels_of(sigma) > 30) return fail(WT_ERR_ARG, "bad sigma");
  const uint32_t L = levels_of(sigma);
  uint64_t n = 0;
  const uint64_t* offs[wt::DD_MAX_SEGMENTS];
  for (uint32_t g = 0; g < k; ++g) {
    if (!segs[g].node_offsets || (L && seg_n[g] && !segs[g].bitmaps)) return fail(WT_ERR_ARG, "NULL segment tree");
    offs[g] = segs[g].node_offsets;
    n += seg_n[g];
  }
  if (L && (!out->bitmaps || !out->superblocks)) return fail(WT_ERR_ARG, "NULL output");
  if (!d_scratch || scratch_bytes < wt_dd_merge_scratch_bytes(n)) return fail(WT_ERR_WORKSPACE, "scratch too small");
  wt_status st = wt_dd_offsets(k, offs, sigma, out->node_offsets, stream);
  if (st != WT_OK) return st;
  const uint64_t W = words_of(n), nsb = nsb_of(n);
  for (uint32_t l = 0; l < L; ++l) {
    const uint32_t* src[wt::DD_MAX_SEGMENTS];
    for (uint32_t g = 0; g < k; ++g) src[g] = segs[g].bitmaps + (uint64_t)l * words_of(seg_n[g]);
    if ((st = wt_dd_merge_level(k, offs, out->node_offsets, sigma, n, l, src, nullptr, 0, W,
                                out->bitmaps + (uint64_t)l * W, stream)) != WT_OK)
      return st;
    if ((st = wt_superblocks(out->bitmaps + (uint64_t)l * W, nsb - 1, 0, out->superblocks + (uint64_t)l * nsb,
                             d_scratch, scratch_bytes, stream)) != WT_OK)
      return st;
  }
  return WT_OK;
}

wt_status wt_rank1(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint32_t* d_level, const uint64_t* d_pos,
                   uint64_t m, uint64_t* d_out, wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = query_args(tree, n, sigma);
  if (st != WT_OK) return st;
  if (m == 0) return WT_OK;
  if (!d_level || !d_pos || !d_out) return fail(WT_ERR_ARG, "NULL query pointer");
  wt::k_rank1<<<(uint32_t)((m + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      tree->bitmaps, reinterpret_cast<const unsigned long long*>(tree->superblocks), words_of(n), nsb_of(n), d_level,
      reinterpret_cast<const unsigned long long*>(d_pos), m, reinterpret_cast<unsigned long long*>(d_out));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_rank1");
}

uint64_t wt_select_index_entries(uint64_t n, uint64_t sigma) {
  if (sigma == 0 || levels_of(sigma) > 30) return 0;
  return 2ull * levels_of(sigma) * wt::select_samples_per_level(n);
}

wt_status wt_select_index(const wt_tree_t* tree, uint64_t n, uint64_t sigma, uint32_t* d_samples,
                          wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = query_args(tree, n, sigma);
  if (st != WT_OK) return st;
  const uint32_t L = levels_of(sigma);
  if (n >= (1ull << 32)) return fail(WT_ERR_ARG, "the select index stores 32-bit positions (n < 2^32)");
  if (L == 0) return WT_OK;
  if (!d_samples) return fail(WT_ERR_ARG, "NULL samples pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const wt::TreeView v = view_of(tree, n, sigma);
  const uint64_t entries = wt_select_index_entries(n, sigma);
  wt::k_fill_u32<<<(uint32_t)std::min<uint64_t>((entries + 255) / 256, 4ull * num_sms()), 256, 0, s>>>(
      d_samples, entries, (uint32_t)n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, "k_fill_u32");
  const uint64_t blocks = (uint64_t)L * (v.NSB - 1);
  if (blocks) {
    wt::k_select_samples_fill<<<(uint32_t)((blocks + 255) / 256), 256, 0, s>>>(v, d_samples);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e, "k_select_samples_fill");
  }
  return WT_OK;
}

wt_status wt_select_indexed(const wt_tree_t* tree, uint64_t n, uint64_t sigma, const uint32_t* d_samples,
                            const uint32_t* d_c, const uint64_t* d_j, uint64_t m, uint64_t* d_out,
                            int32_t* d_status, wt_stream_t stream) {
  g_last_error.clear();
  wt_status st = query_args(tree, n, sigma);
  if (st != WT_OK) return st;
  if (m == 0) return WT_OK;
  if (!d_c || !d_j || !d_out || (levels_of(sigma) > 0 && !d_samples)) return fail(WT_ERR_ARG, "NULL pointer");
  if (n >= (1ull << 32)) return fail(WT_ERR_ARG, "the select index stores 32-bit positions (n < 2^32)");
  const uint32_t grid = (uint32_t)((m + 255) / 256);
  wt::k_select<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      view_of(tree, n, sigma), sigma, d_c, d_j, m, reinterpret_cast<unsigned long long*>(d_out), d_status,
      d_samples);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WT_OK : fail_cuda(e, "k_select");
}

uint32_t wt_launch_plan(uint64_t n, uint64_t sigma, uint32_t width, uint32_t* kinds, uint32_t cap) {
  if (check_args(n, sigma, width) != WT_OK) return 0;
  const Carve c = carve(n, sigma, width);
  uint32_t count = 0;
  Launcher lk{nullptr};
  dispatch(nullptr, n, sigma, width, nullptr, nullptr, c, lk, kinds, cap, &count);
  return count;
}

uint32_t wt_debug_offsets(uint64_t n, uint64_t sigma, uint32_t width, uint64_t* offsets, uint32_t cap) {
  if (check_args(n, sigma, width) != WT_OK) return 0;
  const Carve c = carve(n, sigma, width);
  const uint64_t v[] = {c.off_flag, c.off_ones0, c.off_agg, c.off_pre, c.off_tab, c.off_cnt,
                        align_up(c.cnt_entries * sizeof(uint32_t)), c.off_bufA, c.off_bufB, c.ntiles};
  const uint32_t k = (uint32_t)(sizeof(v) / sizeof(v[0]));
  for (uint32_t i = 0; i < k && i < cap; ++i) offsets[i] = v[i];
  return k;
}

void wt_set_profile_events(wt_event_t* events, uint32_t count) {
  g_events = events;
  g_event_count = events ? count : 0;
}

const char* wt_status_string(wt_status status) {
  switch (status) {
    case WT_OK: return "WT_OK";
    case WT_ERR_ARG: return "WT_ERR_ARG";
    case WT_ERR_SYMBOL_RANGE: return "WT_ERR_SYMBOL_RANGE";
    case WT_ERR_INDEX: return "WT_ERR_INDEX";
    case WT_ERR_CUDA: return "WT_ERR_CUDA";
    case WT_ERR_WORKSPACE: return "WT_ERR_WORKSPACE";
  }
  return "WT_ERR_UNKNOWN";
}

const char* wt_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
