/*
 * wt_oracle.c -- the CPU ORACLE for the levelwise wavelet tree of
 * Fuentes-Sepulveda, Elejalde, Ferres, Seco, "Parallel Construction of
 * Wavelet Trees on Multicore Architectures" (arXiv 1610.05994).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the reference the CUDA path is
 * checked against.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant generator with paper_1610_05994_b200/ and the
 * product library never links or calls it.
 *
 * Plain, slow, single-threaded C.  Citations "P:n" are lines of
 * /root/reference/PAPER.md (not available at run time; cited for review).
 *
 * Construction = Algorithm 1 (pwt) with every parfor replaced by
 * a sequential for, exactly as P:507-509 says ("the sequential version can
 * be obtained by replacing parfor instructions with sequential for
 * instructions").  Readings of the paper adopted here:
 *   R1 the bit test "(S[j] & 2^{L-i-1}) == 1" of Alg. 1 line 9 is read
 *      as "!= 0": level i stores bit (L-1-i) of the code, the (i+1)-th MSB
 *      (Fig. 3 caption).
 *   R2 the alphabet is [0, sigma) (worked example uses R=[0,15]).
 *   R3 L = ceil(lg sigma); L = 0 when sigma == 1.
 *   R4 the prefix sum of line 7 is EXCLUSIVE (node offsets).
 *   R5 bits are stored LSB-first in 32-bit words; a level occupies
 *      16*ceil(n/512) words, bits >= n are zero.
 *   R6 createRankSelect (line 14), rank part: one 64-bit
 *      cumulative count per 512-bit block, SB[t] = rank1(B, min(512t, n))
 *      exclusive, t = 0..ceil(n/512); the last entry is the level total.
 *   R7 rank_c(S, i) is INCLUSIVE of i ("i = rank1(B,24) - 1 = 7").
 *
 * Every function here is parity-pinned by tests/test_oracle_pins.py (golden
 * worked example P:337-375, brute-force stable sort, the recursive per-node
 * definition, closed forms).  Nothing here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
  OR_OK = 0,
  OR_ERR_ARG = 1,
  OR_ERR_SYMBOL_RANGE = 2,
  OR_ERR_INDEX = 3,
  OR_ERR_NOMEM = 6,
  OR_ERR_INTERNAL = 7
};

/* S[j] read as an unsigned little-endian integer of `width` bytes (1, 2, 4). */
static uint64_t sym_at(const void* S, uint32_t width, uint64_t j) {
  if (width == 1) return ((const uint8_t*)S)[j];
  if (width == 2) return ((const uint16_t*)S)[j];
  return ((const uint32_t*)S)[j];
}

/* R3: number of levels L = ceil(lg sigma). */
uint32_t oracle_levels(uint64_t sigma) {
  uint32_t L = 0;
  while (L < 64 && ((uint64_t)1 << L) < sigma) L++;
  return L;
}

/* R5 / R6 sizes. */
uint64_t oracle_words_per_level(uint64_t n) { return 16 * ((n + 511) / 512); }
uint64_t oracle_sb_per_level(uint64_t n) { return (n + 511) / 512 + 1; }

static int check_args(uint64_t n, uint64_t sigma, uint32_t width) {
  (void)n;
  if (width != 1 && width != 2 && width != 4) return OR_ERR_ARG;
  if (sigma == 0) return OR_ERR_ARG;
  if (sigma > ((uint64_t)1 << (8 * width))) return OR_ERR_ARG;
  return OR_OK;
}

/* Every symbol must lie in [0, sigma) (R2). */
int oracle_validate(const void* S, uint64_t n, uint64_t sigma, uint32_t width) {
  int st = check_args(n, sigma, width);
  if (st != OR_OK) return st;
  for (uint64_t j = 0; j < n; j++)
    if (sym_at(S, width, j) >= sigma) return OR_ERR_SYMBOL_RANGE;
  return OR_OK;
}

/*
 * node_offsets C[c] = #{ j : S[j] < c }, c in [0, 2^L]: the counting of
 * Alg. 1 lines 5-7 done at the leaf granularity (Proposition 1, P:485-490:
 * the node of s at level i is s >> (L-i), so every level's counters are a
 * coarsening of this one array).  Histogram, then exclusive prefix sum.
 */
int oracle_node_offsets(const void* S, uint64_t n, uint64_t sigma, uint32_t width,
                        uint64_t* C) {
  int st = oracle_validate(S, n, sigma, width);
  if (st != OR_OK) return st;
  uint32_t L = oracle_levels(sigma);
  uint64_t nb = (uint64_t)1 << L;
  uint64_t* H = (uint64_t*)calloc(nb, sizeof(uint64_t));
  if (!H) return OR_ERR_NOMEM;
  for (uint64_t j = 0; j < n; j++) H[sym_at(S, width, j)] += 1;
  uint64_t acc = 0;
  for (uint64_t c = 0; c < nb; c++) {
    C[c] = acc;
    acc += H[c];
  }
  C[nb] = acc;
  free(H);
  return OR_OK;
}

/*
 * One level i of Algorithm 1, sequential form:
 *   line 3     B is a bitarray of size n            -> B (words_per_level words)
 *   line 4     C is an integer array of size 2^i     -> Cl
 *   lines 5-6  for j: increment C[S[j] / 2^{L-i}]
 *   line 7     prefix sum over C (exclusive, R4)     -> node starts, copied to Nl
 *   lines 8-13 for j: bitmapSetBit(B, C[S[j]/2^{L-i}], bit); increment that C
 *   line 14    createRankSelect(B), rank part (R6)   -> SB
 * Nl (2^i + 1 entries: node starts plus n) may be NULL.
 */
int oracle_build_level(const void* S, uint64_t n, uint64_t sigma, uint32_t width,
                       uint32_t level, uint32_t* B, uint64_t* SB, uint64_t* Nl) {
  int st = check_args(n, sigma, width);
  if (st != OR_OK) return st;
  uint32_t L = oracle_levels(sigma);
  if (level >= L) return OR_ERR_ARG;
  uint64_t nodes = (uint64_t)1 << level;
  uint32_t shift_node = L - level;      /* S[j] / 2^{L-i}           */
  uint32_t shift_bit = L - level - 1;   /* bit 2^{L-i-1}, reading R1 */

  uint64_t* Cl = (uint64_t*)calloc(nodes, sizeof(uint64_t));
  if (!Cl) return OR_ERR_NOMEM;

  /* lines 5-6 */
  for (uint64_t j = 0; j < n; j++) {
    uint64_t s = sym_at(S, width, j);
    if (s >= sigma) { free(Cl); return OR_ERR_SYMBOL_RANGE; }
    Cl[s >> shift_node] += 1;
  }
  /* line 7: exclusive prefix sum (R4) */
  uint64_t acc = 0;
  for (uint64_t v = 0; v < nodes; v++) {
    uint64_t cnt = Cl[v];
    Cl[v] = acc;
    acc += cnt;
  }
  if (Nl) {
    for (uint64_t v = 0; v < nodes; v++) Nl[v] = Cl[v];
    Nl[nodes] = acc;
  }
  /* line 3: zeroed bitarray, padded per R5 */
  uint64_t W = oracle_words_per_level(n);
  memset(B, 0, W * sizeof(uint32_t));
  /* lines 8-13 */
  for (uint64_t j = 0; j < n; j++) {
    uint64_t s = sym_at(S, width, j);
    uint64_t v = s >> shift_node;
    uint64_t pos = Cl[v];
    if ((s >> shift_bit) & 1) B[pos >> 5] |= (uint32_t)1 << (pos & 31); /* bitmapSetBit(B,pos,1) */
    Cl[v] = pos + 1;                                                    /* increment            */
  }
  /* line 14, rank part: cumulative popcount per 512-bit block (R6) */
  uint64_t nsb = oracle_sb_per_level(n);
  uint64_t ones = 0;
  for (uint64_t t = 0; t < nsb; t++) {
    SB[t] = ones;
    for (uint64_t w = 16 * t; w < 16 * (t + 1) && w < W; w++)
      ones += (uint64_t)__builtin_popcount(B[w]);
  }
  free(Cl);
  return OR_OK;
}

/*
 * The whole tree (Alg. 1, every level), plus the leaf-granularity node
 * offsets C.  Two independent derivations of the node starts are compared:
 * level i's prefix-summed counters (line 7) must equal C[v << (L-i)].
 * bitmaps: L * words_per_level uint32; superblocks: L * sb_per_level uint64;
 * node_offsets: 2^L + 1 uint64.
 */
int oracle_build(const void* S, uint64_t n, uint64_t sigma, uint32_t width,
                 uint32_t* bitmaps, uint64_t* superblocks, uint64_t* node_offsets) {
  int st = oracle_node_offsets(S, n, sigma, width, node_offsets);
  if (st != OR_OK) return st;
  uint32_t L = oracle_levels(sigma);
  uint64_t W = oracle_words_per_level(n), NSB = oracle_sb_per_level(n);
  uint64_t* Nl = (uint64_t*)malloc((((uint64_t)1 << (L > 0 ? L - 1 : 0)) + 1) * sizeof(uint64_t));
  if (!Nl) return OR_ERR_NOMEM;
  for (uint32_t i = 0; i < L; i++) {
    st = oracle_build_level(S, n, sigma, width, i, bitmaps + (uint64_t)i * W,
                            superblocks + (uint64_t)i * NSB, Nl);
    if (st != OR_OK) { free(Nl); return st; }
    for (uint64_t v = 0; v <= ((uint64_t)1 << i); v++)
      if (Nl[v] != node_offsets[v << (L - i)]) { free(Nl); return OR_ERR_INTERNAL; }
  }
  free(Nl);
  return OR_OK;
}

/* ---------------------------------------------------------------- queries */

/* bit q of one level bitmap (R5). */
static uint32_t bit_at(const uint32_t* B, uint64_t q) { return (B[q >> 5] >> (q & 31)) & 1u; }

/* rank1(B, q): ones in positions [0, q) -- superblock sample plus word popcounts (R6). */
uint64_t oracle_rank1(const uint32_t* B, const uint64_t* SB, uint64_t q) {
  uint64_t t = q >> 9;
  uint64_t r = SB[t];
  for (uint64_t w = 16 * t; w < (q >> 5); w++) r += (uint64_t)__builtin_popcount(B[w]);
  if (q & 31) r += (uint64_t)__builtin_popcount(B[q >> 5] & (((uint32_t)1 << (q & 31)) - 1));
  return r;
}

/*
 * access(S, i): top-down traversal.  At each level read the bit
 * at the current position, replace the in-node index i by rank_b(B, i) - 1
 * within the node (inclusive rank, R7) and descend to child b.  In the
 * one-pointer-per-level layout the node start is C[v << (L-1-l)] and the
 * in-node rank is a difference of two bitmap ranks.
 * path (optional, L+1 entries): the in-node index before each level and the
 * leaf index -- for the printed example 24 -> 7 -> 4 -> 2.
 */
int oracle_access(const uint32_t* bitmaps, const uint64_t* superblocks, const uint64_t* C,
                  uint64_t n, uint64_t sigma, uint64_t i, uint64_t* sym, uint64_t* path) {
  if (i >= n) return OR_ERR_INDEX;
  uint32_t L = oracle_levels(sigma);
  uint64_t W = oracle_words_per_level(n), NSB = oracle_sb_per_level(n);
  uint64_t lo = 0, p = i, v = 0;
  for (uint32_t l = 0; l < L; l++) {
    const uint32_t* B = bitmaps + (uint64_t)l * W;
    const uint64_t* SB = superblocks + (uint64_t)l * NSB;
    if (path) path[l] = p;
    uint64_t q = lo + p;
    uint32_t b = bit_at(B, q);
    uint64_t ones_in_node_le_q = oracle_rank1(B, SB, q + 1) - oracle_rank1(B, SB, lo); /* rank1 inclusive */
    if (b) p = ones_in_node_le_q - 1;                       /* i = rank1(B,i) - 1 */
    else p = (p + 1 - ones_in_node_le_q) - 1;               /* i = rank0(B,i) - 1 */
    v = 2 * v + b;
    lo = C[v << (L - 1 - l)];
  }
  if (path) path[L] = p;
  *sym = v;
  return OR_OK;
}

/*
 * rank_c(S, i), inclusive (R7): the number of c in
 * S[0..i].  Descend along c's bits, keeping the count r of node members in
 * the node's prefix that corresponds to S[0..i].
 */
int oracle_rank(const uint32_t* bitmaps, const uint64_t* superblocks, const uint64_t* C,
                uint64_t n, uint64_t sigma, uint64_t c, uint64_t i, uint64_t* out) {
  if (i >= n || c >= sigma) return OR_ERR_INDEX;
  uint32_t L = oracle_levels(sigma);
  uint64_t W = oracle_words_per_level(n), NSB = oracle_sb_per_level(n);
  uint64_t lo = 0, r = i + 1;
  for (uint32_t l = 0; l < L; l++) {
    const uint32_t* B = bitmaps + (uint64_t)l * W;
    const uint64_t* SB = superblocks + (uint64_t)l * NSB;
    uint32_t b = (uint32_t)((c >> (L - 1 - l)) & 1);
    uint64_t ones = oracle_rank1(B, SB, lo + r) - oracle_rank1(B, SB, lo);
    r = b ? ones : r - ones;
    lo = C[(c >> (L - 1 - l)) << (L - 1 - l)];
  }
  *out = r;
  return OR_OK;
}

/* position of the k-th (1-based) bit equal to b in B[lo, hi), by linear scan; hi if absent. */
static uint64_t select_in_range(const uint32_t* B, uint64_t lo, uint64_t hi, uint32_t b, uint64_t k) {
  for (uint64_t q = lo; q < hi; q++)
    if (bit_at(B, q) == b && --k == 0) return q;
  return hi;
}

/*
 * select_c(S, j): position of the j-th (1-based)
 * occurrence of c.  Bottom-up: start at in-node index j-1 in c's leaf, and
 * at each level from L-1 up to 0 map the in-node index p of child b to the
 * position of the (p+1)-th b-bit of the parent node.
 */
int oracle_select(const uint32_t* bitmaps, const uint64_t* superblocks, const uint64_t* C,
                  uint64_t n, uint64_t sigma, uint64_t c, uint64_t j, uint64_t* out) {
  (void)superblocks;
  if (c >= sigma || j == 0) return OR_ERR_INDEX;
  uint32_t L = oracle_levels(sigma);
  uint64_t W = oracle_words_per_level(n);
  if (C[c + 1] - C[c] < j) return OR_ERR_INDEX;
  uint64_t p = j - 1;
  for (uint32_t l = L; l-- > 0;) {
    const uint32_t* B = bitmaps + (uint64_t)l * W;
    uint64_t v = c >> (L - l);                 /* node at level l (Prop. 1) */
    uint64_t lo = C[v << (L - l)], hi = C[(v + 1) << (L - l)];
    uint32_t b = (uint32_t)((c >> (L - 1 - l)) & 1);
    uint64_t q = select_in_range(B, lo, hi, b, p + 1);
    if (q >= hi) return OR_ERR_INTERNAL;
    p = q - lo;
  }
  *out = p;
  return OR_OK;
}
