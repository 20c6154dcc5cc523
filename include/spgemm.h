/*
 * spgemm.h — C ABI of libspgemm.so: the four-stage CSR SpGEMM of Liu & Vinter,
 * "A Framework for General Sparse Matrix-Matrix Multiplication on GPUs and
 * Heterogeneous Processors" (arXiv 1504.05022), rebuilt for B200 (sm_100a).
 *
 * Citations: [P:n] = line n of the paper text, [S:n] = line n of SPEC.md.
 *
 * The operation ([P:44], [P:113-138]): A is m×k, B is k×n, C = A·B is m×n, all in CSR
 * (row pointer array of rows+1 offsets, column index array, value array [P:113]).
 * Storage here: int64 row pointers, int32 column indices, fp64 values ("32-bit index and
 * 64-bit value" [P:169]).  Result semantics: structural — C holds every (i,k) for which
 * some a_ij and b_jk are stored, explicit zeros and exact cancellations included ("does
 * not take into consideration cancellation" [P:169]); each row of C is sorted by column
 * and duplicate-free, like the paper's heap / ESC / merge outputs [P:266-295].
 *
 * Input preconditions: A and B are valid CSR with strictly ascending, duplicate-free
 * columns per row (the paper's assumption, footnote at [P:178]).  They are checked only
 * with SPGEMM_FLAG_VALIDATE (one extra kernel + sync); otherwise behaviour on invalid CSR
 * is undefined (no out-of-bounds writes are attempted for column indices in [0, n)).
 *
 * Stages (Figure "framework", [P:187-196]):
 *   1 upper bound u_i = sum_{a_ij} nnz(b_j*)            [P:198-212]
 *   2 binning of rows by u_i + hybrid C~ allocation      [P:214-260]
 *   3 per-bin row computation, long rows progressive     [P:262-297]
 *   4 arrange data: scan nnz(c_i*), compact C~ into C    [P:301]
 *
 * Pointers: every matrix pointer is a DEVICE pointer on the device that was current
 * when the handle was created, unless a function says "host".  No exception crosses
 * this ABI; every call returns a status.  On failure, output buffers are untouched and
 * the handle stays destroyable.
 */
#ifndef SPGEMM_H_
#define SPGEMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct spgemm_handle_s* spgemm_handle_t;
typedef void* spgemm_stream_t; /* a cudaStream_t; NULL = legacy default stream */

typedef enum {
  SPGEMM_SUCCESS = 0,
  SPGEMM_ERROR_INVALID_VALUE = 1, /* NULL handle/pointer where required, m/k/n/nnz < 0, bad flags  */
  SPGEMM_ERROR_INVALID_CSR = 2,   /* only with SPGEMM_FLAG_VALIDATE: row_ptr[0] != 0, decreasing
                                     row_ptr, row_ptr[rows] != nnz, column outside [0, cols),
                                     unsorted or duplicate columns in a row                        */
  SPGEMM_ERROR_INDEX_OVERFLOW = 3,/* m, k or n > INT32_MAX (column indices are int32)             */
  SPGEMM_ERROR_OUT_OF_MEMORY = 4, /* workspace, C~ or long-row growth allocation failed           */
  SPGEMM_ERROR_INVALID_STATE = 5, /* numeric before a successful symbolic                         */
  SPGEMM_ERROR_CUDA = 6,          /* any CUDA runtime error; text via spgemm_last_error()         */
  SPGEMM_ERROR_NCCL = 7,          /* dist_* entry points only                                     */
  SPGEMM_ERROR_INTERNAL = 8
} spgemm_status_t;

enum {
  SPGEMM_FLAG_VALIDATE = 1u << 0,          /* validate A and B on the device (one extra sync)     */
  SPGEMM_FLAG_INPUTS_REPLICATED = 1u << 1, /* dist only: every rank passes the full A and B       */
  SPGEMM_FLAG_PRECISE = 1u << 2,           /* two-pass "precise" strategy ([P:165]): symbolic runs
                                              a structure-only stage 3 and numeric recomputes the
                                              rows straight into C (no temporary C~).  Default is
                                              the paper's hybrid method ([P:224]): C~ + stage-4 copy */
  SPGEMM_FLAG_UPPER_BOUND = 1u << 3,       /* hybrid with the upper-bound allocation for long rows
                                              too (C~ row = min(u_i, n), no growth) [P:169]        */
  SPGEMM_FLAG_FP32 = 1u << 4               /* SpSGEMM: fp32 values (set by spgemm_create_f32)       */
};

/* Number of stage-2 size classes ("bins", re-derived for 228 KB smem/SM). */
#define SPGEMM_NUM_TIERS 21

typedef struct spgemm_stats {
  int64_t m, k, n, nnz_a, nnz_b;
  int64_t sum_u;            /* nnz(C^) = flops/2 [P:169], [P:433]                          */
  int64_t nnz_c;            /* nnz(C) (after symbolic)                                     */
  int64_t max_u;            /* largest u_i                                                 */
  int64_t tier_rows[SPGEMM_NUM_TIERS];
  int64_t ctil_entries;     /* C~ capacity in entries (hybrid; 0 for PRECISE)               */
  int64_t long_rows;        /* rows on the progressive long-row path                        */
  int64_t long_entries;     /* final long-row arena capacity in entries                     */
  int32_t growth_rounds;    /* re-allocation rounds of the long-row path ("2x each time" [P:297]) */
  int32_t flags;
  int64_t workspace_bytes;  /* device bytes held by the handle after symbolic (pool + mapped long-row arena) */
  float stage_ms[4];        /* CUDA-event times on the handle's stream: symbolic stage 1+2,
                               stage 3 (all classes incl. long rows), stage-4 scan; numeric  */
  float tier_ms[SPGEMM_NUM_TIERS];         /* stage-3 time per class (last symbolic;
                                              for PRECISE: last numeric)                    */
  int64_t tier_a_entries[SPGEMM_NUM_TIERS];/* sum nnz(a_i*) over the rows of each class     */
  int64_t tier_products[SPGEMM_NUM_TIERS]; /* sum u_i over the rows of each class           */
  int64_t tier_c_entries[SPGEMM_NUM_TIERS];/* sum nnz(c_i*) over the rows of each class     */
  int32_t launches_symbolic;               /* kernels launched by the last symbolic         */
  int32_t launches_numeric;                /* kernels launched by the last numeric          */
  float tier_ms_symbolic[SPGEMM_NUM_TIERS];/* stage-3 time per class in the last symbolic
                                              (PRECISE: the COUNT / STRUCT pass)             */
} spgemm_stats_t;

/* Create a handle for C = A·B.  No device work, no synchronisation (unless VALIDATE).
 * A: m×k, row_ptr[m+1], col_idx[a_nnz], val[a_nnz]; B: k×n likewise.  The handle keeps
 * the pointers (no copy): A and B must stay valid and unmodified until numeric's work
 * has completed on `stream`.  flags: SPGEMM_FLAG_*.  Errors: INVALID_VALUE,
 * INDEX_OVERFLOW, INVALID_CSR (VALIDATE only), CUDA, OUT_OF_MEMORY. */
spgemm_status_t spgemm_create(spgemm_handle_t* handle, int64_t m, int64_t k, int64_t n,
                              const int64_t* a_row_ptr, const int32_t* a_col_idx,
                              const double* a_val, int64_t a_nnz, const int64_t* b_row_ptr,
                              const int32_t* b_col_idx, const double* b_val, int64_t b_nnz,
                              spgemm_stream_t stream, uint32_t flags);

/* Stages 1-3 and the stage-4 scan on `stream` (Figure "framework" [P:187-196]).
 * Synchronises `stream` (the paper's host reads bin counters and sums nnz at the same
 * points [P:264], [P:301]) and writes nnz(C) to *c_nnz (HOST pointer).  May be called
 * again (recomputes, e.g. after A/B values change).  Errors: INVALID_VALUE, CUDA,
 * OUT_OF_MEMORY (handle stays destroyable). */
spgemm_status_t spgemm_symbolic(spgemm_handle_t handle, int64_t* c_nnz);

/* Stage 4 compaction ([P:301]) into caller-allocated C: c_row_ptr[m+1] (int64),
 * c_col_idx[c_nnz] (int32), c_val[c_nnz] (fp64), all device pointers.  Enqueued on the
 * handle's stream; returns without synchronising.  With SPGEMM_FLAG_PRECISE this
 * recomputes the rows (stage 3 with values) directly into C.  Errors: INVALID_STATE
 * (no successful symbolic), INVALID_VALUE, CUDA. */
spgemm_status_t spgemm_numeric(spgemm_handle_t handle, int64_t* c_row_ptr, int32_t* c_col_idx,
                               double* c_val);

/* SpSGEMM — the paper's single-precision runs ([P:403], [P:663]): the same four stages with
 * fp32 values (float a_val / b_val / c_val, DEVICE pointers); every product a_ij·b_jk is
 * rounded to fp32 and the sums run in fp32 in the same j-ascending order as the fp64 path.
 * Structure, row pointers and errors are those of spgemm_create / spgemm_numeric; the handle
 * must be finished with spgemm_numeric_f32 (spgemm_numeric on it fails with INVALID_VALUE,
 * and spgemm_numeric_f32 on an fp64 handle likewise).  Not available through dist_*. */
spgemm_status_t spgemm_create_f32(spgemm_handle_t* handle, int64_t m, int64_t k, int64_t n,
                                  const int64_t* a_row_ptr, const int32_t* a_col_idx,
                                  const float* a_val, int64_t a_nnz, const int64_t* b_row_ptr,
                                  const int32_t* b_col_idx, const float* b_val, int64_t b_nnz,
                                  spgemm_stream_t stream, uint32_t flags);
spgemm_status_t spgemm_numeric_f32(spgemm_handle_t handle, int64_t* c_row_ptr, int32_t* c_col_idx,
                                   float* c_val);

/* Frees all workspace.  NULL → no-op.  Synchronises the handle's stream. */
spgemm_status_t spgemm_destroy(spgemm_handle_t handle);

/* Statistics of the last symbolic/numeric (HOST out pointer). */
spgemm_status_t spgemm_get_stats(spgemm_handle_t handle, spgemm_stats_t* out);

/* Copies the stage-1 bound U (int64, m entries) and the stage-2 class of each row (int32,
 * m entries; may be NULL) into DEVICE buffers, for exact-integer tests.  Valid after
 * symbolic.  Enqueued on the handle's stream. */
spgemm_status_t spgemm_debug_get_u(spgemm_handle_t handle, int64_t* u, int32_t* tier);

/* Testing knobs (process-global, take effect at the next symbolic):
 *   force_tier >= 0: route every row with u_i >= 2 through stage-3 class `force_tier`
 *   when it can hold the row (else the normal class); -1 = off.
 *   long_initial_capacity > 0: initial long-row capacity in entries (default 16384); small
 *   values force the re-allocation path ([P:297]).  long_threshold > 0: rows with
 *   min(u_i, n) above it take the long-row path (default: when no shared-memory class fits).
 */
spgemm_status_t spgemm_set_debug(int32_t force_tier, int64_t long_initial_capacity,
                                 int64_t long_threshold);

/* Testing knob (process-global, next launch): the long-row bitmap kernels process a row's
 * column window in tiles of at most `tile_columns` columns (rounded up to the kernel's
 * multiple of 32-column words); 0 = the default, sized by shared memory (1 Mi columns for
 * counting, 256 Ki for values).  Small values force the multi-tile path on small inputs.
 * Errors: INVALID_VALUE (negative). */
spgemm_status_t spgemm_set_debug_long_tile(int64_t tile_columns);

/* Debug / test knob: precise numeric sends long rows whose column window is wider than
 * min_window columns (and whose u_i <= 2^20) to the bucket path — a stable partition of the
 * row's products by column range, then one CTA sort per bucket (the ESC of [P:277-284] over
 * column ranges) — instead of the bitmap rank kernel.  0 = default (2^18, one rank tile),
 * negative = never.  Takes effect at the next spgemm_symbolic.  Process-wide; not thread-safe. */
spgemm_status_t spgemm_set_debug_long_bucket(int64_t min_window);

/* Workspace comes from a library-owned stream-ordered memory pool per device that keeps
 * freed blocks cached (warm multiplies make no OS allocations; the device's default pool and
 * PyTorch's allocator are not touched); the hybrid long-row VMM arenas are cached likewise
 * (up to 4, with their mapped pages).  This releases every cached arena and returns pool
 * bytes above keep_bytes to the device (current device; synchronises it).  Errors: CUDA. */
spgemm_status_t spgemm_trim_workspace_cache(int64_t keep_bytes);

const char* spgemm_status_string(spgemm_status_t s);
/* Last error text of `handle` (NULL → this thread's last error). */
const char* spgemm_last_error(spgemm_handle_t handle);
/* Library build string (arch, version). */
const char* spgemm_version(void);

/* ---------------------------------------------------------------- multi-GPU ---------
 * One process per GPU; NCCL inside the library; torch.distributed only ships the id.
 * A is split into row blocks balanced by the prefix sum of u (the paper's load-balance
 * quantity, "the number of necessary arithmetic operations" [P:25]); B is replicated with
 * ncclBroadcast; C's row offsets are stitched with an ncclAllGather of per-rank nnz.
 * Every rank must call the dist_* functions in the same order. */
spgemm_status_t spgemm_nccl_get_unique_id(uint8_t id[128]);

/* A, B significant on rank 0 only unless flags has SPGEMM_FLAG_INPUTS_REPLICATED (then
 * every rank passes the full A and B and nothing but the nnz allgather crosses NVLink). */
spgemm_status_t spgemm_dist_create(spgemm_handle_t* handle, int rank, int nranks,
                                   const uint8_t id[128], int64_t m, int64_t k, int64_t n,
                                   const int64_t* a_row_ptr, const int32_t* a_col_idx,
                                   const double* a_val, int64_t a_nnz, const int64_t* b_row_ptr,
                                   const int32_t* b_col_idx, const double* b_val, int64_t b_nnz,
                                   spgemm_stream_t stream, uint32_t flags);

/* Sharded inputs (config 5: each rank generates its own share).  Rank r passes the rows
 * [a_row_begin, a_row_end) of A (the caller's partition, not re-balanced; blocks must cover
 * A's rows in rank order for the global CSR to be the concatenation) and the rows
 * [b_row_begin, b_row_end) of B; the B slices of all ranks must tile [0, k) in rank order.
 * Row pointer arrays have (rows + 1) entries and may start at any value: entry e of a block
 * is col_idx[e - row_ptr[0]] / val[e - row_ptr[0]].  B is replicated by an all-gather of the
 * slices (grouped ncclBroadcast, slices placed at their global entry offset, row pointers
 * rebased); B's values travel on a second stream during the structure-only symbolic pass of
 * SPGEMM_FLAG_PRECISE.  All pointers are DEVICE pointers and stay owned by the caller (valid
 * until dist_numeric's work completed).  Errors: INVALID_VALUE (ranges, NULL pointers,
 * INPUTS_REPLICATED), INDEX_OVERFLOW, NCCL, CUDA. */
spgemm_status_t spgemm_dist_create_sharded(spgemm_handle_t* handle, int rank, int nranks,
                                           const uint8_t id[128], int64_t m, int64_t k, int64_t n,
                                           int64_t a_row_begin, int64_t a_row_end,
                                           const int64_t* a_row_ptr, const int32_t* a_col_idx,
                                           const double* a_val, int64_t a_nnz, int64_t b_row_begin,
                                           int64_t b_row_end, const int64_t* b_row_ptr,
                                           const int32_t* b_col_idx, const double* b_val,
                                           int64_t b_nnz, spgemm_stream_t stream, uint32_t flags);

/* Partition + input movement + local stages 1-3 + allgather.  Rank owns rows
 * [*row_begin, *row_end) of C (HOST outs); *local_nnz / *global_nnz are HOST outs.
 * Synchronises the handle's stream. */
spgemm_status_t spgemm_dist_symbolic(spgemm_handle_t handle, int64_t* row_begin,
                                     int64_t* row_end, int64_t* local_nnz, int64_t* global_nnz);

/* Local stage 4 into the rank's block of C: c_row_ptr has row_end-row_begin+1 entries and
 * holds GLOBAL offsets, so concatenating rank blocks gives the single-GPU CSR. */
spgemm_status_t spgemm_dist_numeric(spgemm_handle_t handle, int64_t* c_row_ptr,
                                    int32_t* c_col_idx, double* c_val);

/* ---- host arithmetic of the dist protocol (all HOST pointers; used by dist_symbolic and
 * exported so that CPU tests drive the same code) ---- */

/* Partition rule: given the inclusive prefix sums of u over m rows, write nranks+1 split
 * points: s_0 = 0, s_P = m, s_r = min{ i : scan[i] >= ceil(r·total/P) } + 1 clamped
 * monotone (rank r owns rows [s_r, s_r+1): about Σu/P products each, [P:25]). */
spgemm_status_t spgemm_partition_rows(const int64_t* u_inclusive_scan, int64_t m, int nranks,
                                      int64_t* splits);

/* Entry ranges of the row blocks: rp_at_splits[r] = A.row_ptr[s_r] (nranks+1 values) ->
 * entry_bounds[2r], entry_bounds[2r+1] = first / one-past-last entry of rank r's block (the
 * col_idx / val ranges the root sends).  Errors: INVALID_VALUE, INVALID_CSR (decreasing). */
spgemm_status_t spgemm_dist_block_entries(const int64_t* rp_at_splits, int nranks,
                                          int64_t* entry_bounds);

/* Placement of sharded B slices: slice r = rows [row_begin[r], row_end[r]) with nnz[r]
 * entries; checks that the slices tile [0, k) in rank order and writes entry_base[r] (global
 * entry offset of slice r) and entry_base[nranks] = nnz(B).  Errors: INVALID_VALUE. */
spgemm_status_t spgemm_dist_slice_layout(const int64_t* row_begin, const int64_t* row_end,
                                         const int64_t* nnz, int nranks, int64_t k,
                                         int64_t* entry_base);

/* Stitching (stage 4's sum across ranks, [P:301]): from every rank's nnz, this rank's
 * global row-pointer offset and nnz(C). */
spgemm_status_t spgemm_dist_offsets(const int64_t* local_nnz, int nranks, int rank,
                                    int64_t* offset, int64_t* total);

/* Test hook: the DEVICE partition kernel of dist_symbolic on a DEVICE inclusive scan (m
 * entries) -> HOST splits (nranks+1), to hold it against spgemm_partition_rows. */
spgemm_status_t spgemm_debug_partition(const int64_t* u_inclusive_scan, int64_t m, int nranks,
                                       int64_t* splits);

#ifdef __cplusplus
}
#endif
#endif /* SPGEMM_H_ */
