// common.cuh — internal declarations of libspgemm (CUDA, sm_100a).  Not part of the ABI.
//
// Stage-2 size classes ("tiers") re-derived for B200.  The paper bins rows
// by the stage-1 bound u_i into 38 bins / 5 groups sized for 48-96 KB scratchpads
// ([P:214-260], [P:299] "the parameters of the binning depends on specifications ... of GPU
// architectures").  Here, with cap_i = min(u_i, n) >= nnz(c_i*):
//   T_EMPTY            u = 0                      nothing to compute ([P:216])
//   T_G1..T_G32        u <= G (G = 1..32)         G-lane group per row, products sorted in
//                                                 registers (slot of the paper's heap group 3)
//   T_W64..T_W2048     1.25·cap <= S              one warp per row, S-slot shared-memory hash
//                                                 (slot of the bitonic-ESC group 4)
//   T_C2048..T_C8192   cap <= H                   one CTA per row, order-preserving hash with
//                                                 H home slots in 2H smem slots
//   T_E2048..T_E8192   u <= U (cap > 1638)        one CTA per row, bucket ESC: products counting-
//                                                 sorted into buckets (monotone bucket function),
//                                                 each bucket sorted by (column, product index)
//   T_BW               u > 32, W <= 2^17,         one warp per row, dense bitmap over the row's
//                      min(u,W) <= 2048           column window [lo, lo+W) (the SPA of [P:142]
//                                                 restricted to the window), 2-level for sparse
//                                                 windows; W = max_j max(b_j*) - min_j min(b_j*) + 1
//   T_LONG             otherwise                  progressive global table + re-allocation
//                                                 (group 5, [P:286-297])
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spgemm.h"

namespace sg {

enum Tier : int {
  T_EMPTY = 0,
  T_G1 = 1, T_G2 = 2, T_G4 = 3, T_G8 = 4, T_G16 = 5, T_G32 = 6,
  T_W64 = 7, T_W128 = 8, T_W256 = 9, T_W512 = 10, T_W1024 = 11, T_W2048 = 12,
  T_C2048 = 13, T_C4096 = 14, T_C8192 = 15,
  T_E2048 = 16, T_E4096 = 17, T_E8192 = 18,
  T_BW = 19,
  T_LONG = 20,
  NUM_TIERS = 21
};
static_assert(NUM_TIERS == SPGEMM_NUM_TIERS, "tier count mismatch with the ABI header");

constexpr int kEmptyKey = -1;

// Window-bitmap class limits: column window W (bits per warp) and row length (values per warp).
constexpr int64_t kBwMaxW = int64_t(1) << 17;
constexpr int64_t kBwMaxV = 2048;
// precise strategy: the bound may reach kBwMaxVRelax — the exact length decides at re-binning
// (rows longer than kBwMaxV leave the class), so rows whose products repeat columns many times
// (Galerkin products: u of 3-8 Ki, nnz of a few hundred) keep the dense accumulator
constexpr int64_t kBwMaxVRelax = 8192;

__host__ __device__ inline bool bw_ok(int64_t cap, int64_t W, int64_t vmax = kBwMaxV) {
  return W > 0 && W <= kBwMaxW && (cap < W ? cap : W) <= vmax;
}

struct TierParams {
  int force_tier;         // -1 = off
  int64_t long_threshold; // rows with cap above go long (0 = default by smem)
  int64_t bk_min_w;       // precise long rows: window above which values take the bucket path
  int bw_relax;           // window rows by the relaxed bound (kBwMaxVRelax)
};

// Long rows, precise numeric: rows whose column window is wider than one bitmap tile of the
// rank kernel (W > bk_min_w) and whose products fit the bucket count take the bucket path
// (longbk.cu): a stable partition of the row's products by column range, then one CTA sort per
// bucket.  Products per bucket: ~kBkTarget on average, at most kBkCap (else the row falls back
// to the rank kernel).
constexpr int64_t kBkDefaultMinW = int64_t(1) << 18;
constexpr int kBkTarget = 2048;
constexpr int kBkCap = 4096;
constexpr int kBkMaxBuckets = 512;
__host__ __device__ inline bool bk_eligible(int64_t u, int64_t W, int64_t min_w) {
  // (windows up to 2^29 columns: the bucket sort's key + product-index composite fits 32 bits)
  return W > min_w && W <= (int64_t(1) << 29) && u <= int64_t(kBkTarget) * kBkMaxBuckets;
}
// buckets: NB = next power of two >= ceil(u / kBkTarget); bucket of column c = (c - lo) >> sh,
// sh = max(0, ceil(log2 W) - log2 NB); ((W - 1) >> sh) + 1 <= NB buckets are used
__host__ __device__ inline void bk_shape(int64_t u, int64_t W, int& sh, int& nbk) {
  int lnb = 0;
  while ((int64_t(kBkTarget) << lnb) < u) ++lnb;
  int lw = 0;
  while ((int64_t(1) << lw) < W) ++lw;
  sh = lw > lnb ? lw - lnb : 0;
  nbk = (int)(((W - 1) >> sh) + 1);
}

__host__ __device__ inline int tier_capacity_ok(int t, int64_t u, int64_t cap, int64_t W) {
  if (t == T_EMPTY) return u == 0;
  if (t == T_BW) return bw_ok(cap, W);
  if (t >= T_G1 && t <= T_G32) return u <= (int64_t(1) << (t - T_G1));
  if (t >= T_W64 && t <= T_W2048) {
    int64_t S = int64_t(64) << (t - T_W64);
    return 4 * S >= 5 * cap && u <= S;  // table load <= 0.8; the values' ESC holds >= S items
  }
  if (t >= T_C2048 && t <= T_C8192) return cap <= (int64_t(2048) << (t - T_C2048));
  if (t >= T_E2048 && t <= T_E8192) return u <= (int64_t(2048) << (t - T_E2048));
  return 1;  // T_LONG holds anything
}

__host__ __device__ inline int esc_class(int64_t u) {
  for (int t = T_E2048; t <= T_E8192; ++t)
    if (u <= (int64_t(2048) << (t - T_E2048))) return t;
  return -1;
}

// Stage-2 classification of one row (the B200 re-derivation of Algorithm 3 [P:226-260]).
// W: the row's column window (0 when u = 0).
__host__ __device__ inline int classify(int64_t u, int64_t n, TierParams p, int64_t W) {
  if (u == 0) return T_EMPTY;
  int64_t cap = u < n ? u : n;
  if (p.force_tier >= 0 && u >= 2 && tier_capacity_ok(p.force_tier, u, cap, W)) return p.force_tier;
  if (p.long_threshold > 0 && cap > p.long_threshold) return T_LONG;
  if (u <= 32) {
    int g = 0;
    while ((int64_t(1) << g) < u) ++g;
    return T_G1 + g;
  }
  if (bw_ok(cap, W, p.bw_relax ? kBwMaxVRelax : kBwMaxV)) return T_BW;
  for (int t = T_W64; t <= T_W2048; ++t)
    if (tier_capacity_ok(t, u, cap, W)) return t;
  const int e = esc_class(u);  // products fit one CTA's shared memory: bucket ESC
  if (e >= 0) return e;
  for (int t = T_C2048; t <= T_C8192; ++t)
    if (tier_capacity_ok(t, u, cap, W)) return t;
  return T_LONG;
}

// PRECISE numeric classes: the symbolic pass knows nnz(c_i*) exactly, so tables are sized
// by it (load <= 1/2) instead of by the bound min(u_i, n).
__host__ __device__ inline int tier_exact_ok(int t, int64_t u, int64_t nnz) {
  if (t == T_EMPTY) return u == 0;
  if (t == T_BW) return 0;  // only rows that were window rows in the symbolic pass (below)
  if (t >= T_G1 && t <= T_G32) return u <= (int64_t(1) << (t - T_G1));
  if (t >= T_W64 && t <= T_W2048) return (int64_t(64) << (t - T_W64)) >= 2 * nnz && u <= (int64_t(64) << (t - T_W64));  // S >= 2·nnz, u <= S (ESC items)
  if (t >= T_C2048 && t <= T_C8192) return nnz <= (int64_t(2048) << (t - T_C2048));
  if (t >= T_E2048 && t <= T_E8192) return u <= (int64_t(2048) << (t - T_E2048));
  return 1;
}

// sym_class: the row's symbolic class; warp classes in numeric need the sorted column set
// that only the symbolic warp classes (STRUCT) produce.
__host__ __device__ inline int classify_exact(int64_t u, int64_t nnz, int sym_class, TierParams p) {
  if (u == 0) return T_EMPTY;
  if (sym_class == T_BW && nnz <= kBwMaxV) return T_BW;  // longer rows (relaxed bound): ESC / CTA classes
  // warp classes: the numeric pass sorts the row's u <= 0.8·S products in one CTA (ESC)
  if (p.force_tier < 0 && sym_class >= T_W64 && sym_class <= T_W2048) return sym_class;
  // long rows stay on the bitmap path (ranks, no sort): c3b rows with u > 8192 but
  // nnz <= 8192 took 248 ps/product in the CTA hash vs 28 in the bitmap fill
  if (p.force_tier < 0 && sym_class == T_LONG) return T_LONG;
  const bool has_struct = sym_class >= T_W64 && sym_class <= T_W2048;
  if (p.force_tier >= 0 && u >= 2 && tier_exact_ok(p.force_tier, u, nnz) &&
      (has_struct || p.force_tier < T_W64 || p.force_tier > T_W2048) &&
      !(p.force_tier >= T_G1 && p.force_tier <= T_G32 && has_struct))
    return p.force_tier;
  if (p.long_threshold > 0 && nnz > p.long_threshold) return T_LONG;
  if (u <= 32 && !has_struct) {
    int g = 0;
    while ((int64_t(1) << g) < u) ++g;
    return T_G1 + g;
  }
  if (has_struct)
    for (int t = T_W64; t <= T_W2048; ++t)
      if ((int64_t(64) << (t - T_W64)) >= 2 * nnz && u <= (int64_t(64) << (t - T_W64))) return t;
  const int e = esc_class(u);
  if (e >= 0) return e;
  for (int t = T_C2048; t <= T_C8192; ++t)
    if (nnz <= (int64_t(2048) << (t - T_C2048))) return t;
  return T_LONG;
}

// Hybrid C~ capacity of a row ([P:224]: u_i for short rows; here min(u_i, n) which is
// still a safe bound since nnz(c_i*) <= n).  Long rows live in their own growing arena —
// except long rows with wide windows (bk_eligible), which take the bucket path (longbk.cu)
// into a C~ slice of the upper bound (these rows' products rarely repeat a column).
__host__ __device__ inline int64_t hybrid_capacity(int t, int64_t u, int64_t n, int64_t W, int64_t bk_min_w) {
  if (t == T_LONG && !bk_eligible(u, W, bk_min_w)) return 0;
  return u < n ? u : n;
}
// C~ capacity by strategy: CAP_HYBRID keeps whole rows (columns + values) in C~; CAP_PRECISE
// keeps only the structure of the window-bitmap rows (STRUCT -> DENSE), no other row needs C~
// in the precise strategy.  There the capacity is rounded up to even so every slice starts on
// 8 bytes: STRUCT writes a row as its list of nonzero bitmap words ((first column, bits) pairs,
// 8 B each) when that fits the slice, else as the sorted column set (4 B per entry).
enum CapMode : int { CAP_NONE = 0, CAP_HYBRID = 1, CAP_PRECISE = 2 };
__host__ __device__ inline int64_t ctil_capacity(int mode, int t, int64_t u, int64_t n, int64_t W, int64_t bk_min_w) {
  if (mode == CAP_HYBRID) return hybrid_capacity(t, u, n, W, bk_min_w);
  if (mode == CAP_PRECISE && t == T_BW) return ((u < n ? u : n) + 1) & ~int64_t(1);
  return 0;
}

struct CsrView {
  const int64_t* rp;
  const int32_t* ci;
  const double* val;
};

// COUNT: nnz(c_i*) only.  FILL: sorted row with values (C~ in hybrid, C in precise numeric).
// STRUCT (precise symbolic): nnz(c_i*) and the sorted column set of the row, written to
// out_col at out_off.  DENSE (precise numeric): values from the sorted column set of STRUCT,
// accumulated into a dense, already ordered array (no insertion, no sort).
enum Mode : int { MODE_COUNT = 0, MODE_FILL = 1, MODE_STRUCT = 2, MODE_DENSE = 3 };

// Value arithmetic of Algorithm 1 lines 6, 9, 11: products rounded separately (no FMA), sums
// in the order of the walk.  V = double (SpDGEMM, the default) or float (SpSGEMM,
// SPGEMM_FLAG_FP32 / spgemm_create_f32: the paper's single-precision runs [P:403], [P:663]).
template <typename V> struct Arith;
template <> struct Arith<double> {
  __device__ static __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct Arith<float> {
  __device__ static __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ static __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};
// Value arrays travel as double* through the argument structs; kernels instantiated for V
// reinterpret them (float arrays when the handle is FP32).
template <typename V> __host__ __device__ __forceinline__ const V* vcast(const double* p) {
  return reinterpret_cast<const V*>(p);
}
template <typename V> __host__ __device__ __forceinline__ V* vcast(double* p) { return reinterpret_cast<V*>(p); }

struct LongState;

struct Stage3Args {
  CsrView A, B;
  int64_t n;
  int64_t b_nnz;         // nnz(B): 32-bit entry offsets below 2^31
  const int32_t* perm;   // rows grouped by tier
  int64_t first;         // this tier's rows are perm[first, first + count)
  int64_t count;
  const int64_t* out_off;  // per-row output offset (C~ offsets or C row_ptr), by row id
  int32_t* out_col;
  double* out_val;
  int64_t* nnz_row;        // per-row nnz (written in both modes; may be NULL in numeric)
  int mode;
  const int64_t* row_len;     // DENSE: nnz(c_i*) by row when out_off holds capacities (hybrid C~)
  const int32_t* struct_col;  // DENSE: sorted column sets from STRUCT
  const int64_t* struct_off;  // DENSE: their per-row offsets
  int32_t* bw_nw;             // precise T_BW: per row, the number of (first column, bits) words
                              // STRUCT wrote (-1: the sorted column set instead); NULL: columns
  const int32_t* rlo;         // first column of each row's window (stage 1)
  const int32_t* rhi;         // last column of each row's window (stage 1)
  const int64_t* U;           // u_i of every row (stage 1)
  const int4* bwin;           // (first, last, nnz) of each row of B (stage 1)
  int64_t bw_wmax, bw_vmax;   // T_BW: largest window / row length of the class
  int64_t bw_bmax;            // T_BW numeric: most nonzero 1024-column blocks in a row
  int64_t* bw_bmax_out;       // T_BW STRUCT: device max of the above (summary entry)
  int32_t* bw_ovf_list;       // T_BW STRUCT: rows with more nonzero blocks than the slots
  int32_t* bw_ovf_cnt;        //   (re-run over the full-window bitmap; device counter)
  const int32_t* count_dev;   // if set, the kernel reads its row count here (rows = perm[0..))
  int* work_ctr;              // long rows: dynamic row counter (zeroed by the launcher)
  // bitmap FILL, progressive mode (hybrid long rows): work index r -> long row active[r];
  // output through the row's chunk table into the arena; a tile that does not fit the row's
  // capacity checkpoints the row into ovf_list
  LongState* lst;
  const int32_t* active;
  const int64_t* chunk_table;  // [nlong][kMaxChunks]
  int32_t* arena_col;
  double* arena_val;
  int log2c0;
  int32_t* ovf_list;
  int32_t* ovf_cnt;
  int f32;                     // values are float (SpSGEMM)
};
// Long-row bitmap tile width in 32-column words (spgemm_set_debug_long_tile; 0 = default).
extern int64_t g_long_tile_words;

// ---- host-side launchers (defined in the .cu files) --------------------------------
struct Stage12Ws {
  int64_t* U;          // [m]
  uint8_t* tier;       // [m]
  int32_t* perm;       // [m]
  int64_t* ctil_off;   // [m+1]
  int32_t* blk_tier;   // [nblk * NUM_TIERS]
  int64_t* blk_cap;    // [nblk]
  int64_t* blk_usum;   // [nblk]
  int64_t* blk_umax;   // [nblk]
  int64_t* summary;    // [kSumLen] device
  int4* bwin;          // [k] (first column, last column, nnz, 0) of each row of B
  int32_t* rlo;        // [m] first column of each row's window
  int32_t* rhi;        // [m] last column of each row's window
  int64_t nblk;
};
constexpr int kS12Threads = 256;
constexpr int kS12RowsPerThread = 8;
constexpr int64_t kS12RowsPerBlock = int64_t(kS12Threads) * kS12RowsPerThread;
// summary layout
constexpr int kSumCount = 0;                       // tier counts [NUM_TIERS]
constexpr int kSumOff = NUM_TIERS;                 // tier offsets [NUM_TIERS+1]
constexpr int kSumU = 2 * NUM_TIERS + 1;           // sum u
constexpr int kSumCap = kSumU + 1;                 // sum cap (C~ entries)
constexpr int kSumUMax = kSumU + 2;                // max u
constexpr int kSumWmax = kSumU + 3;              // max W over T_BW rows
constexpr int kSumVmax = kSumU + 4;              // max min(u, W) over T_BW rows (after re-binning:
                                                 // max nnz(c_i*))
constexpr int kSumBmax = kSumU + 5;              // max nonzero 1024-column blocks (T_BW STRUCT)
constexpr int kSumBkU = kSumU + 6;               // precise long rows on the bucket path: sum u
constexpr int kSumBkRows = kSumU + 7;            //   and their number
constexpr int kSumLen = kSumU + 8;

cudaError_t launch_stage1(int64_t m, int64_t k, int64_t n, CsrView A, CsrView B, TierParams tp,
                          int cap_mode, Stage12Ws& ws, cudaStream_t s);
cudaError_t launch_stage2(int64_t m, Stage12Ws& ws, int cap_mode, int64_t n, int64_t bk_min_w, cudaStream_t s);
// PRECISE: re-bin rows by (u_i, nnz(c_i*)) into ws.tier/perm (ws.U and nnz_row are inputs).
cudaError_t launch_rebin(int64_t m, int64_t n, const int64_t* nnz_row, TierParams tp, Stage12Ws& ws,
                         cudaStream_t s);

cudaError_t launch_stage3_tier(int tier, const Stage3Args& a, cudaStream_t s);
// warp classes T_W64..T_W2048 (warp.cu)
cudaError_t launch_warp_tier(int tier, const Stage3Args& a, cudaStream_t s);
// window-bitmap class T_BW (warp.cu)
cudaError_t launch_bw_tier(const Stage3Args& a, cudaStream_t s);
cudaError_t launch_bw_one(const Stage3Args& a, cudaStream_t s);
int num_sms();
// bucket-ESC classes (esc.cu)
cudaError_t launch_esc(int tier, const Stage3Args& a, cudaStream_t s);
// the same sort for the warp classes' rows in FILL mode: one CTA of S items per row
cudaError_t launch_esc_items(int S, const Stage3Args& a, cudaStream_t s);
// PRECISE long rows: bitmap over the column window (COUNT: nnz; FILL: ranks → C)
cudaError_t launch_long_bitmap(const Stage3Args& a, cudaStream_t s);
// long rows with wide windows, precise numeric: bucket partition + per-bucket sort (longbk.cu)
struct BkDesc {      // one bucket of one row
  int64_t off;       // its first item in the staging arrays
  int32_t size;      // items (products)
  int32_t blo;       // first column of its column range
  int32_t sh;        // key bits (the range is 2^sh columns)
  int32_t uniq;      // distinct columns (written by the sort)
};
struct BkRow {       // one row on the bucket path: buckets [desc0, desc0 + nbk)
  int32_t row, nbk;
  int64_t desc0;
};
struct BkWork {
  int32_t* stg_col;          // staging: sum u over the bucket rows
  double* stg_val;           //   (fp64, or fp32 reinterpreted)
  BkDesc* desc;
  BkRow* rows;
  unsigned long long* cur64; // [0] staging items used, [1] descriptors used
  int32_t* cur32;            // [0] bucket rows, [1] rows left to the rank kernel
  int32_t* fb_list;          // those rows
  int64_t min_w;             // bk_eligible window threshold
};
// rank_fallback: run the rank kernel on the rows left over (precise); else only list them
cudaError_t launch_long_buckets(const Stage3Args& a, const BkWork& bw, int64_t max_rows, bool rank_fallback,
                                cudaStream_t s);

// Exclusive scan of int64 values x[0..len) into y[0..len]; y[len] = total.  tmp must hold
// scan_tmp_elems(len) int64.
int64_t scan_tmp_elems(int64_t len);
cudaError_t launch_exclusive_scan(const int64_t* x, int64_t* y, int64_t len, int64_t* tmp,
                                  cudaStream_t s);

// Long-row (T_LONG) progressive path (hybrid strategy, [P:297]) ------------------------
// Every long row owns a growable slice of the long-row arena, addressed through a table of
// chunks: chunk 0 holds positions [0, C0), chunk g >= 1 positions [C0·2^(g-1), C0·2^g) (C0 a
// power of two), i.e. each 2x growth adds one chunk and nothing already written moves.  The
// table entry of chunk g is (arena offset of the chunk) - (its first position), so position
// p of the row lives at arena[table[chunk_of(p)] + p].
constexpr int kMaxChunks = 34;
__host__ __device__ inline int chunk_of(int64_t p, int log2c0) {
  const uint64_t q = uint64_t(p) >> log2c0;
  if (q == 0) return 0;
#ifdef __CUDA_ARCH__
  return 64 - __clzll((long long)q);
#else
  return 64 - __builtin_clzll(q);
#endif
}
__host__ __device__ inline int chunks_for(int64_t cap, int log2c0) {  // chunks covering [0, cap)
  return cap <= 0 ? 0 : chunk_of(cap - 1, log2c0) + 1;
}

struct LongState {
  int64_t next_col;  // checkpoint: first column of the next tile to compute ([P:297]); INT64_MIN = row start
  int64_t cap;       // current capacity in entries ("we use 2x each time" [P:297])
  int64_t capmax;    // min(u_i, n): never above the upper bound (reading Q8)
  int64_t count;     // entries written so far (the tiles before the checkpoint)
  int64_t need;      // at an overflow: count + the entries of the checkpointed tile; after growth: new cap
};

cudaError_t launch_long_init(LongState* st, const int32_t* perm, int64_t first, int64_t nlong, const int64_t* U,
                             int64_t n, int64_t cap0, int64_t* sizes, cudaStream_t s);
// overflowed rows in `list`: need -> new cap = cap·2^j >= need (capped at capmax); sizes[i] = new - old
cudaError_t launch_long_grow(LongState* st, const int32_t* list, int64_t nlist, int64_t* sizes, cudaStream_t s);
// chunk tables of the rows in `list` for positions [old cap, new cap) at arena offsets base + off[i]
cudaError_t launch_long_assign(LongState* st, const int32_t* list, int64_t nlist, const int64_t* off, int64_t base,
                               int64_t* table, int log2c0, cudaStream_t s);

// VMM arena (vmm.cu): reserved virtual range, physical memory mapped at its end on demand.
struct VmmArena {
  void* base = nullptr;
  size_t reserved = 0, mapped = 0, gran = 0;
  int device = 0;
  void* impl = nullptr;
};
cudaError_t vmm_reserve(VmmArena* a, size_t bytes);
cudaError_t vmm_ensure(VmmArena* a, size_t bytes);
void vmm_release(VmmArena* a);  // back to the per-device cache (at most 4 arenas kept)
void vmm_trim();                  // release the cached arenas

// Stage 4 -------------------------------------------------------------------------------
struct CopyArgs {
  int64_t m;
  const int32_t* perm;       // long rows are perm[long_first, long_first + nlong)
  int64_t long_first, nlong;
  const int64_t* c_rp;       // final row pointers [m+1]
  const int64_t* ctil_off;   // by row (C~ offsets; rows with an empty slice live in the arena)
  int64_t ctil_total;        // C~ entries (the end of the last row's slice)
  const uint8_t* tier;
  const int32_t* ctil_col;
  const double* ctil_val;
  const int64_t* chunk_table;  // long rows: [nlong][kMaxChunks] into the arena
  const int32_t* arena_col;
  const double* arena_val;
  int log2c0;
  int32_t* c_col;
  double* c_val;
  int f32;                     // values are float
};
cudaError_t launch_copy(const CopyArgs& a, cudaStream_t s);

// Library-owned stream-ordered pool (one per device, release threshold: keep everything, so
// warm multiplies allocate without OS calls).  The default device pool is left untouched;
// spgemm_trim_workspace_cache() returns the cached bytes.
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t s);

cudaError_t launch_validate(int64_t rows, int64_t cols, const int64_t* rp, const int32_t* ci,
                            int64_t nnz, int32_t* err, cudaStream_t s);

}  // namespace sg
