// api.cu — the C ABI of libspgemm.so (include/spgemm.h): handle, workspace, and the
// host orchestration of the four stages (Figure "framework", [P:187-196]).
//
// symbolic:  stage 1 + stage 2 (GPU) → one small D2H of the per-class counts (the host-side
//            bin counters of [P:264]: kernels are issued only for non-empty classes) →
//            allocate C~ (hybrid) → stage 3 per class → long rows with the progressive
//            growth loop ([P:297]) → scan of nnz(c_i*) → D2H of nnz(C) ([P:301]).
// numeric:   stage 4 copy C~ → C (hybrid), or stage 3 again straight into C (PRECISE).
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

using namespace sg;

namespace {

thread_local std::string t_last_error;
// Host-side per-thread resources reused across handles (creating them per handle put
// cudaMallocHost / cudaFreeHost and ~40 event creations inside every multiply).
thread_local int64_t* t_pinned = nullptr;  // small pinned scratch for the counter read-backs
struct EventSet {
  int device;
  cudaEvent_t ev[6];
  cudaEvent_t tev[NUM_TIERS][2];   // stage-3 classes of the last numeric (precise) / symbolic (hybrid)
  cudaEvent_t tsym[NUM_TIERS][2];  // stage-3 classes of the last symbolic
};
thread_local std::vector<EventSet*> t_event_pool;
int g_force_tier = -1;
int64_t g_long_cap0 = 16384;
int64_t g_long_threshold = 0;
int64_t g_bk_min_w = kBkDefaultMinW;  // long rows: bucket path above this window (precise numeric)

__global__ void k_tier_to_i32(const uint8_t* t, int32_t* o, int64_t m) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) o[i] = t[i];
}

// max of nnz_row over the rows perm[first, first + count) (the window class's exact row length)
__global__ void k_rows_max(const int32_t* __restrict__ perm, int64_t first, int64_t count,
                           const int64_t* __restrict__ nnz_row, unsigned long long* out) {
  unsigned long long m = 0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < count; r += int64_t(gridDim.x) * blockDim.x)
    m = max(m, (unsigned long long)nnz_row[perm[first + r]]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(out, m);
}

__global__ void k_iota(int32_t* p, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int32_t)i;
}

__global__ void k_class_sums(int64_t m, const uint8_t* __restrict__ tier, const int64_t* __restrict__ U,
                             const int64_t* __restrict__ arp, const int64_t* __restrict__ nnz_row,
                             unsigned long long* out) {
  __shared__ unsigned long long s[3 * NUM_TIERS];
  for (int i = threadIdx.x; i < 3 * NUM_TIERS; i += blockDim.x) s[i] = 0;
  __syncthreads();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    const int t = tier[i];
    atomicAdd(&s[t], (unsigned long long)(arp[i + 1] - arp[i]));
    atomicAdd(&s[NUM_TIERS + t], (unsigned long long)U[i]);
    atomicAdd(&s[2 * NUM_TIERS + t], (unsigned long long)nnz_row[i]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * NUM_TIERS; i += blockDim.x)
    if (s[i]) atomicAdd(&out[i], s[i]);
}

std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};

cudaMemPool_t library_pool(int dev) {
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    g_pools[dev] = p;
  }
  return g_pools[dev];
}

}  // namespace

namespace sg {
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool = library_pool(dev);
  if (!pool) return cudaMallocAsync(p, bytes, s);
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}
}  // namespace sg

spgemm_status_t sg_dist_destroy(spgemm_handle_t h);
bool sg_is_dist(spgemm_handle_t h);
const char* sg_dist_error(spgemm_handle_t h);
spgemm_status_t sg_dist_stats(spgemm_handle_t h, spgemm_stats_t* out);

struct spgemm_handle_s {
  uint64_t magic = 0x53494e474c45ull;  // "SINGLE"; dist handles carry another tag here
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t flags = 0;
  int64_t m = 0, k = 0, n = 0, a_nnz = 0, b_nnz = 0;
  CsrView A{}, B{};
  std::vector<std::pair<void*, size_t>> allocs;  // symbolic workspace
  size_t bytes = 0;
  Stage12Ws ws{};
  int64_t* nnz_row = nullptr;
  int64_t* c_rp = nullptr;
  int64_t* scan_tmp = nullptr;
  int32_t* ctil_col = nullptr;
  double* ctil_val = nullptr;
  int32_t* bw_nw = nullptr;   // precise: words per window row's structure (-1: columns)
  int64_t* pinned = nullptr;  // host pinned scratch [kSumLen + 8]
  // long rows
  int64_t nlong = 0, long_first = 0;
  const int32_t* long_perm = nullptr;  // progressive long rows are long_perm[long_first, +nlong)
  LongState* lst = nullptr;
  int32_t* lact = nullptr;       // active long rows of a round
  int32_t* lovf = nullptr;       // rows that checkpointed (overflowed) in a round
  int32_t* lovf_cnt = nullptr;
  int64_t* lsizes = nullptr;     // per listed row: entries to add
  int64_t* loff = nullptr;       // their exclusive scan
  int64_t* ltable = nullptr;     // chunk tables [nlong][kMaxChunks]
  int log2c0 = 14;
  VmmArena arena_col, arena_val;  // long-row arena (hybrid), grown in place
  int64_t long_entries = 0;
  int32_t growth_rounds = 0;
  int64_t tier_count[NUM_TIERS] = {};
  int64_t tier_off[NUM_TIERS + 1] = {};
  int64_t sum_u = 0, max_u = 0, sum_cap = 0;
  int64_t bw_wmax = 0, bw_vmax = 0, bw_bmax = 0;  // T_BW class: largest window, row length, blocks
  int* work_ctr = nullptr;  // long-row dynamic scheduling counter (symbolic workspace)
  bool sym_ok = false;
  int64_t nnz_c = 0;
  std::string err;
  EventSet* evs = nullptr;
  cudaEvent_t* ev = nullptr;
  cudaEvent_t (*tev)[2] = nullptr;
  cudaEvent_t (*tsym)[2] = nullptr;
  bool tev_used[NUM_TIERS] = {};
  bool tsym_used[NUM_TIERS] = {};
  int32_t launches_sym = 0, launches_num = 0;
  int64_t bk_min_w = kBkDefaultMinW;  // precise long rows: bucket-path window threshold (at symbolic)
  int64_t bk_u = 0, bk_rows = 0;      // sum u and number of the long rows on the bucket path
  bool ev_ok = false;
  bool numeric_recorded = false;
};

namespace {

spgemm_status_t fail(spgemm_handle_t h, spgemm_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  t_last_error = buf;
  return s;
}

spgemm_status_t cuda_fail(spgemm_handle_t h, cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(h, SPGEMM_ERROR_OUT_OF_MEMORY, "%s: out of device memory", where);
  }
  return fail(h, SPGEMM_ERROR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(h, call)                                   \
  do {                                                \
    cudaError_t _e = (call);                          \
    if (_e != cudaSuccess) return cuda_fail(h, _e, #call); \
  } while (0)

template <typename T>
spgemm_status_t dalloc(spgemm_handle_t h, T** p, int64_t count) {
  const size_t bytes = sizeof(T) * size_t(count > 0 ? count : 1);
  void* q = nullptr;
  cudaError_t e = pool_malloc(&q, bytes, h->stream);
  if (e == cudaErrorMemoryAllocation) {  // cached long-row arenas hold pages: release, retry
    cudaGetLastError();
    cudaStreamSynchronize(h->stream);
    vmm_trim();
    e = pool_malloc(&q, bytes, h->stream);
  }
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMallocFromPoolAsync");
  h->allocs.emplace_back(q, bytes);
  h->bytes += bytes;
  *p = static_cast<T*>(q);
  return SPGEMM_SUCCESS;
}

#define AL(h, p, n)                                   \
  do {                                                \
    spgemm_status_t _s = dalloc(h, p, n);             \
    if (_s != SPGEMM_SUCCESS) return _s;              \
  } while (0)

void free_symbolic(spgemm_handle_t h) {
  for (auto& a : h->allocs) cudaFreeAsync(a.first, h->stream);
  h->allocs.clear();
  h->bytes = 0;
  h->ws = Stage12Ws{};
  h->nnz_row = h->c_rp = h->scan_tmp = nullptr;
  h->ctil_col = nullptr;
  h->ctil_val = nullptr;
  h->bw_nw = nullptr;
  h->work_ctr = nullptr;
  h->lst = nullptr;
  h->lact = h->lovf = h->lovf_cnt = nullptr;
  h->lsizes = h->loff = h->ltable = nullptr;
  h->long_perm = nullptr;
  if (h->arena_col.base || h->arena_val.base) {
    cudaStreamSynchronize(h->stream);  // unmapping is immediate, not stream-ordered
    vmm_release(&h->arena_col);
    vmm_release(&h->arena_val);
  }
  h->nlong = 0;
  h->long_entries = 0;
  h->growth_rounds = 0;
  h->sym_ok = false;
  h->numeric_recorded = false;
}

size_t vbytes(spgemm_handle_t h) { return (h->flags & SPGEMM_FLAG_FP32) ? sizeof(float) : sizeof(double); }

spgemm_status_t sync(spgemm_handle_t h) {
  CK(h, cudaStreamSynchronize(h->stream));
  return SPGEMM_SUCCESS;
}

int env_int(const char* name, int def) {
  const char* v = getenv(name);
  return v ? atoi(v) : def;
}

// SPGEMM_TRACE=1: synchronise after each phase and print host wall times (debug only)
struct Trace {
  bool on;
  cudaStream_t s;
  const char* who;
  std::chrono::steady_clock::time_point t0, last;
  Trace(cudaStream_t st, const char* w) : on(getenv("SPGEMM_TRACE") != nullptr), s(st), who(w) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void operator()(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[spgemm %s] %-28s +%8.3f ms  (at %8.3f)\n", who, what,
            std::chrono::duration<double, std::milli>(t - last).count(),
            std::chrono::duration<double, std::milli>(t - t0).count());
    last = t;
  }
};

// Long-row arena: positions [bump, bump + Σ sizes) for the rows in `list` (NULL: all long
// rows), mapped on demand in the VMM arenas, and their chunk tables.
spgemm_status_t long_grow_arena(spgemm_handle_t h, const int32_t* list, int64_t nlist) {
  CK(h, launch_exclusive_scan(h->lsizes, h->loff, nlist, h->scan_tmp, h->stream));
  CK(h, cudaMemcpyAsync(h->pinned, h->loff + nlist, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  spgemm_status_t s = sync(h);
  if (s != SPGEMM_SUCCESS) return s;
  const int64_t total = h->pinned[0];
  const int64_t end = h->long_entries + total;
  CK(h, vmm_ensure(&h->arena_col, size_t(end) * sizeof(int32_t)));
  CK(h, vmm_ensure(&h->arena_val, size_t(end) * vbytes(h)));
  CK(h, launch_long_assign(h->lst, list, nlist, h->loff, h->long_entries, h->ltable, h->log2c0, h->stream));
  h->long_entries = end;
  return SPGEMM_SUCCESS;
}

// Long rows with wide windows on the bucket path (longbk.cu), output rows at out_off (C: precise
// numeric; C~ slices: hybrid symbolic).  Staging and bucket tables live for this call only
// (stream-ordered pool).  Rows the path does not take are listed in fb (its count goes to
// pinned[1] as int32, for the hybrid's progressive path) or, with rank_fallback, computed by
// the rank kernel right away (precise).
spgemm_status_t run_long_buckets(spgemm_handle_t h, const int64_t* out_off, int32_t* out_col, double* out_val,
                                 int64_t* nnz_row, int32_t* fb, bool rank_fallback) {
  Stage3Args a{};
  a.f32 = (h->flags & SPGEMM_FLAG_FP32) != 0;
  a.A = h->A;
  a.B = h->B;
  a.b_nnz = h->b_nnz;
  a.n = h->n;
  a.perm = h->ws.perm;
  a.first = h->long_first;
  a.count = h->nlong;
  a.out_off = out_off;
  a.out_col = out_col;
  a.out_val = out_val;
  a.nnz_row = nnz_row;
  a.mode = MODE_FILL;
  a.bwin = h->ws.bwin;
  a.rlo = h->ws.rlo;
  a.rhi = h->ws.rhi;
  a.U = h->ws.U;
  if (!h->work_ctr) AL(h, &h->work_ctr, 1);
  a.work_ctr = h->work_ctr;
  const int64_t ndesc = h->bk_u / 1024 + h->bk_rows;
  const size_t vb = vbytes(h);
  const size_t sz[7] = {sizeof(int32_t) * size_t(h->bk_u), vb * size_t(h->bk_u), sizeof(BkDesc) * size_t(ndesc),
                        sizeof(BkRow) * size_t(h->bk_rows), 2 * sizeof(unsigned long long), 2 * sizeof(int32_t),
                        sizeof(int32_t) * size_t(h->nlong)};
  void* p[7] = {};
  for (int q = 0; q < 7; ++q)
    if (q != 6 || !fb) CK(h, pool_malloc(&p[q], sz[q], h->stream));
  BkWork bw{static_cast<int32_t*>(p[0]), static_cast<double*>(p[1]), static_cast<BkDesc*>(p[2]),
            static_cast<BkRow*>(p[3]), static_cast<unsigned long long*>(p[4]), static_cast<int32_t*>(p[5]),
            fb ? fb : static_cast<int32_t*>(p[6]), h->bk_min_w};
  cudaError_t e = launch_long_buckets(a, bw, h->bk_rows, rank_fallback, h->stream);
  if (e == cudaSuccess && !rank_fallback)
    e = cudaMemcpyAsync(h->pinned + 1, bw.cur32 + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream);
  for (int q = 0; q < 7; ++q)
    if (p[q]) cudaFreeAsync(p[q], h->stream);
  CK(h, e);
  return SPGEMM_SUCCESS;
}

// Long rows of the hybrid strategy: the paper's group 5 with progressive allocation
// ([P:297]).  Every long row starts with C0 entries (16 Ki; SPGEMM_FLAG_UPPER_BOUND: min(u_i,
// n)) in the long-row arena and runs the bitmap rank kernel tile by tile; a tile that does not
// fit is the checkpoint.  The host then grows each checkpointed row 2x (as many doublings as
// the tile needs, never above min(u_i, n): reading Q8), maps the new chunks at the arena's
// end (VMM: nothing written moves, no dump / reload copy) and relaunches only those rows,
// which resume at their checkpointed tile.
spgemm_status_t run_long(spgemm_handle_t h) {
  const int64_t nl = h->nlong;
  if (nl == 0) return SPGEMM_SUCCESS;
  AL(h, &h->lst, nl);
  AL(h, &h->lact, nl);
  AL(h, &h->lovf, nl);
  AL(h, &h->lovf_cnt, 1);
  AL(h, &h->lsizes, nl);
  AL(h, &h->loff, nl + 1);
  AL(h, &h->ltable, nl * kMaxChunks);
  CK(h, cudaMemsetAsync(h->ltable, 0, sizeof(int64_t) * nl * kMaxChunks, h->stream));  // (read whole, used by prefix)
  AL(h, &h->work_ctr, 1);
  int64_t c0 = 1;
  h->log2c0 = 0;
  while (c0 < g_long_cap0) {
    c0 <<= 1;
    ++h->log2c0;
  }
  const int64_t cap0 = (h->flags & SPGEMM_FLAG_UPPER_BOUND) ? INT64_MAX / 4 : c0;
  // virtual ranges for the arena: the device's memory size (physical pages come on demand)
  size_t freeb = 0, totalb = 0;
  CK(h, cudaMemGetInfo(&freeb, &totalb));
  CK(h, vmm_reserve(&h->arena_col, totalb / 2));
  CK(h, vmm_reserve(&h->arena_val, totalb));
  h->long_entries = 0;
  CK(h, launch_long_init(h->lst, h->long_perm, h->long_first, nl, h->ws.U, h->n, cap0, h->lsizes, h->stream));
  spgemm_status_t s = long_grow_arena(h, nullptr, nl);
  if (s != SPGEMM_SUCCESS) return s;
  const unsigned g = (unsigned)((nl + 255) / 256);
  k_iota<<<g, 256, 0, h->stream>>>(h->lact, nl);
  int64_t nactive = nl;
  for (;;) {
    CK(h, cudaMemsetAsync(h->lovf_cnt, 0, sizeof(int32_t), h->stream));
    Stage3Args a{};
    a.f32 = (h->flags & SPGEMM_FLAG_FP32) != 0;
    a.A = h->A;
    a.B = h->B;
    a.b_nnz = h->b_nnz;
    a.n = h->n;
    a.perm = h->long_perm;
    a.first = h->long_first;
    a.count = nactive;
    a.nnz_row = h->nnz_row;
    a.mode = MODE_FILL;
    a.bwin = h->ws.bwin;
    a.work_ctr = h->work_ctr;
    a.lst = h->lst;
    a.active = h->lact;
    a.chunk_table = h->ltable;
    a.arena_col = static_cast<int32_t*>(h->arena_col.base);
    a.arena_val = static_cast<double*>(h->arena_val.base);
    a.log2c0 = h->log2c0;
    a.ovf_list = h->lovf;
    a.ovf_cnt = h->lovf_cnt;
    CK(h, launch_long_bitmap(a, h->stream));
    CK(h, cudaMemcpyAsync(h->pinned + 1, h->lovf_cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
    s = sync(h);
    if (s != SPGEMM_SUCCESS) return s;
    const int64_t novf = *reinterpret_cast<int32_t*>(h->pinned + 1);
    if (novf == 0) break;
    ++h->growth_rounds;  // host grows the checkpointed rows and relaunches them ([P:297])
    CK(h, launch_long_grow(h->lst, h->lovf, novf, h->lsizes, h->stream));
    s = long_grow_arena(h, h->lovf, novf);
    if (s != SPGEMM_SUCCESS) return s;
    std::swap(h->lact, h->lovf);
    nactive = novf;
  }
  return SPGEMM_SUCCESS;
}

}  // namespace

static spgemm_status_t spgemm_numeric_any(spgemm_handle_t h, int64_t* c_row_ptr, int32_t* c_col_idx,
                                          double* c_val);

extern "C" {

const char* spgemm_status_string(spgemm_status_t s) {
  switch (s) {
    case SPGEMM_SUCCESS: return "SPGEMM_SUCCESS";
    case SPGEMM_ERROR_INVALID_VALUE: return "SPGEMM_ERROR_INVALID_VALUE";
    case SPGEMM_ERROR_INVALID_CSR: return "SPGEMM_ERROR_INVALID_CSR";
    case SPGEMM_ERROR_INDEX_OVERFLOW: return "SPGEMM_ERROR_INDEX_OVERFLOW";
    case SPGEMM_ERROR_OUT_OF_MEMORY: return "SPGEMM_ERROR_OUT_OF_MEMORY";
    case SPGEMM_ERROR_INVALID_STATE: return "SPGEMM_ERROR_INVALID_STATE";
    case SPGEMM_ERROR_CUDA: return "SPGEMM_ERROR_CUDA";
    case SPGEMM_ERROR_NCCL: return "SPGEMM_ERROR_NCCL";
    case SPGEMM_ERROR_INTERNAL: return "SPGEMM_ERROR_INTERNAL";
  }
  return "SPGEMM_UNKNOWN_STATUS";
}

const char* spgemm_last_error(spgemm_handle_t h) {
  if (h && sg_is_dist(h)) return sg_dist_error(h);
  if (!h) {
    const char* d = sg_dist_error(nullptr);
    if (t_last_error.empty() && d && *d) return d;
  }
  return h ? h->err.c_str() : t_last_error.c_str();
}

const char* spgemm_version(void) {
  return "libspgemm 0.1 (Liu & Vinter four-stage SpGEMM, arXiv 1504.05022) sm_100a";
}

spgemm_status_t spgemm_set_debug(int32_t force_tier, int64_t long_initial_capacity,
                                 int64_t long_threshold) {
  if (force_tier >= NUM_TIERS) return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "force_tier out of range");
  g_force_tier = force_tier;
  g_long_cap0 = long_initial_capacity > 0 ? long_initial_capacity : 16384;
  g_long_threshold = long_threshold > 0 ? long_threshold : 0;
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_set_debug_long_bucket(int64_t min_window) {
  g_bk_min_w = min_window == 0 ? kBkDefaultMinW : (min_window < 0 ? INT64_MAX : min_window);
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_set_debug_long_tile(int64_t tile_columns) {
  if (tile_columns < 0) return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "negative tile width");
  g_long_tile_words = (tile_columns + 31) / 32;
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_create(spgemm_handle_t* handle, int64_t m, int64_t k, int64_t n,
                              const int64_t* a_row_ptr, const int32_t* a_col_idx,
                              const double* a_val, int64_t a_nnz, const int64_t* b_row_ptr,
                              const int32_t* b_col_idx, const double* b_val, int64_t b_nnz,
                              spgemm_stream_t stream, uint32_t flags) {
  if (!handle) return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "handle out-pointer is NULL");
  *handle = nullptr;
  if (m < 0 || k < 0 || n < 0 || a_nnz < 0 || b_nnz < 0)
    return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "negative size");
  if (m > INT32_MAX || k > INT32_MAX || n > INT32_MAX)
    return fail(nullptr, SPGEMM_ERROR_INDEX_OVERFLOW, "m, k or n exceeds INT32_MAX");
  const uint32_t known = SPGEMM_FLAG_VALIDATE | SPGEMM_FLAG_INPUTS_REPLICATED | SPGEMM_FLAG_PRECISE | SPGEMM_FLAG_FP32 |
                         SPGEMM_FLAG_UPPER_BOUND;
  if (flags & ~known) return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "unknown flag bits 0x%x", flags & ~known);
  if (!a_row_ptr || !b_row_ptr) return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "NULL row_ptr");
  if ((a_nnz > 0 && (!a_col_idx || !a_val)) || (b_nnz > 0 && (!b_col_idx || !b_val)))
    return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "NULL col_idx/val with nnz > 0");
  spgemm_handle_t h = new (std::nothrow) spgemm_handle_s();
  if (!h) return fail(nullptr, SPGEMM_ERROR_OUT_OF_MEMORY, "host allocation failed");
  cudaGetDevice(&h->device);
  h->stream = static_cast<cudaStream_t>(stream);
  h->flags = flags;
  h->m = m;
  h->k = k;
  h->n = n;
  h->a_nnz = a_nnz;
  h->b_nnz = b_nnz;
  h->A = CsrView{a_row_ptr, a_col_idx, a_val};
  h->B = CsrView{b_row_ptr, b_col_idx, b_val};
  cudaError_t e = cudaSuccess;
  if (!t_pinned) {
    e = cudaMallocHost(&t_pinned, sizeof(int64_t) * (kSumLen + 8));
    if (e != cudaSuccess) {
      t_pinned = nullptr;
      spgemm_status_t s = cuda_fail(nullptr, e, "cudaMallocHost");
      delete h;
      return s;
    }
  }
  h->pinned = t_pinned;
  for (size_t i = 0; i < t_event_pool.size(); ++i)
    if (t_event_pool[i]->device == h->device) {
      h->evs = t_event_pool[i];
      t_event_pool.erase(t_event_pool.begin() + i);
      break;
    }
  if (!h->evs) {
    h->evs = new EventSet();
    h->evs->device = h->device;
    for (int i = 0; i < 6; ++i) cudaEventCreate(&h->evs->ev[i]);
    for (int t = 0; t < NUM_TIERS; ++t)
      for (int i = 0; i < 2; ++i) {
        cudaEventCreate(&h->evs->tev[t][i]);
        cudaEventCreate(&h->evs->tsym[t][i]);
      }
  }
  h->ev = h->evs->ev;
  h->tev = h->evs->tev;
  h->tsym = h->evs->tsym;
  h->ev_ok = true;
  if (flags & SPGEMM_FLAG_VALIDATE) {
    int32_t* err = nullptr;
    e = pool_malloc(reinterpret_cast<void**>(&err), sizeof(int32_t) * 2, h->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(err, 0, sizeof(int32_t) * 2, h->stream);
    if (e == cudaSuccess) e = launch_validate(m, k, a_row_ptr, a_col_idx, a_nnz, err, h->stream);
    if (e == cudaSuccess) e = launch_validate(k, n, b_row_ptr, b_col_idx, b_nnz, err + 1, h->stream);
    int32_t herr[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(herr, err, sizeof(herr), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (err) cudaFreeAsync(err, h->stream);
    if (e != cudaSuccess) {
      spgemm_status_t s = cuda_fail(nullptr, e, "validate");
      spgemm_destroy(h);
      return s;
    }
    if (herr[0] || herr[1]) {
      fail(nullptr, SPGEMM_ERROR_INVALID_CSR, "invalid CSR input: A code %d, B code %d", herr[0], herr[1]);
      spgemm_destroy(h);
      return SPGEMM_ERROR_INVALID_CSR;
    }
  }
  *handle = h;
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_symbolic(spgemm_handle_t h, int64_t* c_nnz) {
  if (!h || !c_nnz) return fail(h, SPGEMM_ERROR_INVALID_VALUE, "NULL handle or c_nnz");
  cudaSetDevice(h->device);
  free_symbolic(h);
  const int64_t m = h->m;
  const bool precise = (h->flags & SPGEMM_FLAG_PRECISE) != 0;
  const bool hybrid = !precise;
  Trace tr(h->stream, "symbolic");
  cudaEventRecord(h->ev[0], h->stream);
  AL(h, &h->c_rp, m + 1);
  if (m == 0) {
    CK(h, cudaMemsetAsync(h->c_rp, 0, sizeof(int64_t), h->stream));
    h->nnz_c = 0;
    h->sum_u = h->max_u = h->sum_cap = 0;
    for (int t = 0; t < NUM_TIERS; ++t) h->tier_count[t] = 0;
    spgemm_status_t s = sync(h);
    if (s != SPGEMM_SUCCESS) return s;
    h->sym_ok = true;
    *c_nnz = 0;
    return SPGEMM_SUCCESS;
  }
  Stage12Ws& ws = h->ws;
  ws.nblk = (m + kS12RowsPerBlock - 1) / kS12RowsPerBlock;
  AL(h, &ws.U, m);
  AL(h, &ws.tier, m);
  AL(h, &ws.perm, m);
  AL(h, &ws.ctil_off, m + 1);
  AL(h, &ws.blk_tier, ws.nblk * NUM_TIERS);
  AL(h, &ws.blk_cap, ws.nblk);
  AL(h, &ws.blk_usum, ws.nblk);
  AL(h, &ws.blk_umax, ws.nblk);
  AL(h, &ws.summary, kSumLen);
  AL(h, &ws.bwin, h->k > 0 ? h->k : 1);
  AL(h, &ws.rlo, m);
  AL(h, &ws.rhi, m);
  AL(h, &h->nnz_row, m);
  AL(h, &h->scan_tmp, scan_tmp_elems(m > (1 << 20) ? m : (1 << 20)));
  // nnz(c_i*) = 0 for rows that never reach a stage-3 kernel (u_i = 0: bin group 1 [P:216])
  CK(h, cudaMemsetAsync(h->nnz_row, 0, sizeof(int64_t) * m, h->stream));
  // window class by the relaxed bound in both strategies: precise re-bins rows longer than
  // kBwMaxV after the count; hybrid rows that outgrow k_bw_one's granules take the two walks
  // (g3d27 hierarchy hybrid 59 -> 17.6 ms, g3d7 12.3 -> 6.8; g2d9 5.4 -> 5.9, (PᵀA)P 43 -> 52)
  TierParams tp{g_force_tier, g_long_threshold, g_bk_min_w, env_int("SPGEMM_BW_STRICT", 0) ? 0 : 1};
  h->bk_min_w = g_bk_min_w;
  tp.force_tier = env_int("SPGEMM_FORCE_TIER", tp.force_tier);
  for (int t = 0; t < NUM_TIERS; ++t) h->tev_used[t] = h->tsym_used[t] = false;
  // C~ offsets in both strategies: hybrid keeps whole rows there, precise only the sorted
  // column sets of the window-bitmap rows (4 B/entry) for its numeric pass
  const int cap_mode = precise ? CAP_PRECISE : CAP_HYBRID;
  CK(h, launch_stage1(m, h->k, h->n, h->A, h->B, tp, cap_mode, ws, h->stream));
  CK(h, launch_stage2(m, ws, cap_mode, h->n, tp.bk_min_w, h->stream));
  h->launches_sym = 3;
  tr("alloc + stage 1-2");
  CK(h, cudaMemcpyAsync(h->pinned, ws.summary, sizeof(int64_t) * kSumLen, cudaMemcpyDeviceToHost, h->stream));
  spgemm_status_t s = sync(h);
  if (s != SPGEMM_SUCCESS) return s;
  tr("class counters D2H");
  for (int t = 0; t < NUM_TIERS; ++t) {
    h->tier_count[t] = h->pinned[kSumCount + t];
    h->tier_off[t] = h->pinned[kSumOff + t];
  }
  h->tier_off[NUM_TIERS] = h->pinned[kSumOff + NUM_TIERS];
  h->sum_u = h->pinned[kSumU];
  h->sum_cap = h->pinned[kSumCap];
  h->max_u = h->pinned[kSumUMax];
  h->bw_wmax = h->pinned[kSumWmax];
  h->bw_vmax = h->pinned[kSumVmax];
  h->bk_u = h->pinned[kSumBkU];  // hybrid: long rows on the bucket path (precise: after re-binning)
  h->bk_rows = h->pinned[kSumBkRows];
  // precise: C~ holds only the window-bitmap rows' sorted column sets (STRUCT); sum_cap counts
  // only those rows (ctil_capacity, CAP_PRECISE)
  AL(h, &h->ctil_col, h->sum_cap > 0 ? h->sum_cap : 1);
  if (hybrid) AL(h, &h->ctil_val, (h->sum_cap * vbytes(h) + 7) / 8);  // values of C~ (fp64 or fp32)
  tr("C~ allocation");
  cudaEventRecord(h->ev[1], h->stream);
  // stage 3: one launch per non-empty class ([P:264] "only issue kernels for non-empty bins")
  for (int t = T_G1; t < T_LONG; ++t) {
    if (h->tier_count[t] == 0) continue;
    Stage3Args a{};
    a.f32 = (h->flags & SPGEMM_FLAG_FP32) != 0;
    a.A = h->A;
    a.B = h->B;
    a.b_nnz = h->b_nnz;
    a.n = h->n;
    a.perm = ws.perm;
    a.first = h->tier_off[t];
    a.count = h->tier_count[t];
    a.out_off = ws.ctil_off;
    a.out_col = h->ctil_col;
    a.out_val = h->ctil_val;
    a.nnz_row = h->nnz_row;
    a.mode = hybrid ? MODE_FILL : (t == T_BW) ? MODE_STRUCT : MODE_COUNT;
    a.rlo = ws.rlo;
    a.bwin = ws.bwin;
    a.bw_wmax = h->bw_wmax;
    a.bw_vmax = h->bw_vmax;
    a.bw_bmax_out = ws.summary + kSumBmax;
    if (t == T_BW) {
      AL(h, &a.bw_ovf_list, h->tier_count[T_BW]);
      AL(h, &a.bw_ovf_cnt, 1);
      if (precise) {  // rows left at -1 (the full-window fallback) keep the column format
        AL(h, &h->bw_nw, m);
        CK(h, cudaMemsetAsync(h->bw_nw, 0xff, sizeof(int32_t) * m, h->stream));
        a.bw_nw = h->bw_nw;
      }
    }
    cudaEventRecord(h->tsym[t][0], h->stream);
    if (hybrid && t == T_BW) {
      // window rows in the hybrid strategy: one walk (k_bw_one: insert and accumulate per
      // product, rows written to their C~ slices in column order); rows with more blocks or
      // granules than it holds take the two walks — the structure pass (sorted column sets
      // into the slices), the exact row-length maximum, then the values by rank (DENSE)
      Stage3Args b = a;
      int64_t rest = a.count;
      if (a.b_nnz < (int64_t(1) << 31) && !env_int("SPGEMM_BW_TWO_WALK", 0)) {
        Stage3Args o1 = a;
        o1.mode = MODE_FILL;
        AL(h, &o1.bw_ovf_list, a.count);
        AL(h, &o1.bw_ovf_cnt, 1);
        CK(h, launch_bw_one(o1, h->stream));
        CK(h, cudaMemcpyAsync(h->pinned + kSumLen + 1, o1.bw_ovf_cnt, sizeof(int32_t), cudaMemcpyDeviceToHost,
                              h->stream));
        s = sync(h);
        if (s != SPGEMM_SUCCESS) return s;
        rest = *reinterpret_cast<int32_t*>(h->pinned + kSumLen + 1);
        b.perm = o1.bw_ovf_list;
        b.first = 0;
        b.count = rest;
        h->launches_sym += 1;
      }
      if (rest > 0) {
        b.mode = MODE_STRUCT;
        CK(h, launch_stage3_tier(t, b, h->stream));
        CK(h, cudaMemsetAsync(ws.summary + kSumVmax, 0, sizeof(int64_t), h->stream));
        k_rows_max<<<256, 256, 0, h->stream>>>(b.perm, b.first, b.count, h->nnz_row,
                                                reinterpret_cast<unsigned long long*>(ws.summary + kSumVmax));
        CK(h, cudaGetLastError());
        CK(h, cudaMemcpyAsync(h->pinned + kSumVmax, ws.summary + kSumVmax, 2 * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, h->stream));  // kSumVmax, kSumBmax
        s = sync(h);
        if (s != SPGEMM_SUCCESS) return s;
        b.mode = MODE_DENSE;
        b.struct_col = h->ctil_col;
        b.struct_off = ws.ctil_off;
        b.row_len = h->nnz_row;  // C~ offsets are capacities here
        b.nnz_row = nullptr;
        b.bw_vmax = h->pinned[kSumVmax];
        b.bw_bmax = h->pinned[kSumBmax];
        CK(h, launch_stage3_tier(t, b, h->stream));
        h->launches_sym += 2;
      } else {
        --h->launches_sym;
      }
    } else {
      CK(h, launch_stage3_tier(t, a, h->stream));
    }
    cudaEventRecord(h->tsym[t][1], h->stream);
    h->tsym_used[t] = true;
    ++h->launches_sym;
  }
  tr("stage 3 classes");
  h->nlong = h->tier_count[T_LONG];
  h->long_first = h->tier_off[T_LONG];
  h->long_perm = ws.perm;
  const bool any_long = h->nlong > 0;
  if (any_long) cudaEventRecord(h->tsym[T_LONG][0], h->stream);
  if (hybrid && h->nlong > 0 && h->bk_rows > 0) {
    // long rows with wide windows: bucket path into their C~ slices (upper-bound capacity);
    // the others continue on the progressive path below, listed in long_perm
    int32_t* fb = nullptr;
    AL(h, &fb, h->nlong);
    s = run_long_buckets(h, h->ws.ctil_off, h->ctil_col, h->ctil_val, h->nnz_row, fb, false);
    if (s != SPGEMM_SUCCESS) return s;
    h->launches_sym += 4;
    s = sync(h);
    if (s != SPGEMM_SUCCESS) return s;
    h->long_perm = fb;
    h->long_first = 0;
    h->nlong = *reinterpret_cast<int32_t*>(h->pinned + 1);
  }
  if (hybrid) {
    // the paper's group 5: progressive allocation with checkpoint / 2x growth [P:297]; the
    // rows' sorted results (values in the oracle's order) are their C~ slices in the long-row
    // arena, copied by stage 4
    s = run_long(h);
    if (s != SPGEMM_SUCCESS) return s;
    if (h->nlong > 0) h->launches_sym += 8 + 7 * h->growth_rounds;
  } else if (h->nlong > 0) {
    // precise: structure of long rows from a bitmap over the column window
    Stage3Args a{};
    a.f32 = (h->flags & SPGEMM_FLAG_FP32) != 0;
    a.A = h->A;
    a.B = h->B;
    a.b_nnz = h->b_nnz;
    a.n = h->n;
    a.perm = ws.perm;
    a.first = h->long_first;
    a.count = h->nlong;
    a.nnz_row = h->nnz_row;
    a.mode = MODE_COUNT;
    a.bwin = ws.bwin;
    AL(h, &h->work_ctr, 1);
    a.work_ctr = h->work_ctr;
    CK(h, launch_long_bitmap(a, h->stream));
    h->launches_sym += 1;
  }
  if (any_long) {
    cudaEventRecord(h->tsym[T_LONG][1], h->stream);
    h->tsym_used[T_LONG] = true;
  }
  cudaEventRecord(h->ev[2], h->stream);
  // stage 4 (first half): sum the numbers of nonzero entries of all rows [P:301]
  CK(h, launch_exclusive_scan(h->nnz_row, h->c_rp, m, h->scan_tmp, h->stream));
  h->launches_sym += 3;
  if (precise && h->nlong > 0) h->launches_sym += 4;
  cudaEventRecord(h->ev[3], h->stream);
  if (precise) {
    // numeric classes from the exact row lengths (tables sized by nnz(c_i*), not the bound);
    // launched before reading nnz(C) so one synchronisation returns both
    CK(h, launch_rebin(m, h->n, h->nnz_row, tp, ws, h->stream));
    h->launches_sym += 3;
    CK(h, cudaMemcpyAsync(h->pinned, ws.summary, sizeof(int64_t) * kSumLen, cudaMemcpyDeviceToHost, h->stream));
  }
  CK(h, cudaMemcpyAsync(h->pinned + kSumLen, h->c_rp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  s = sync(h);
  if (s != SPGEMM_SUCCESS) return s;
  h->nnz_c = h->pinned[kSumLen];
  tr("long rows + scan + re-binning + nnz D2H");
  if (precise) {
    for (int t = 0; t < NUM_TIERS; ++t) {
      h->tier_count[t] = h->pinned[kSumCount + t];
      h->tier_off[t] = h->pinned[kSumOff + t];
    }
    h->tier_off[NUM_TIERS] = h->pinned[kSumOff + NUM_TIERS];
    h->nlong = h->tier_count[T_LONG];
    h->long_first = h->tier_off[T_LONG];
    h->bw_vmax = h->pinned[kSumVmax];  // exact: max nnz(c_i*) over the window rows
    h->bw_bmax = h->pinned[kSumBmax];
    h->bk_u = h->pinned[kSumBkU];
    h->bk_rows = h->pinned[kSumBkRows];
  }
  h->sym_ok = true;
  *c_nnz = h->nnz_c;
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_numeric(spgemm_handle_t h, int64_t* c_row_ptr, int32_t* c_col_idx,
                               double* c_val) {
  if (!h) return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "NULL handle");
  if (h->flags & SPGEMM_FLAG_FP32)
    return fail(h, SPGEMM_ERROR_INVALID_VALUE, "fp32 handle: use spgemm_numeric_f32");
  return spgemm_numeric_any(h, c_row_ptr, c_col_idx, c_val);
}

}  // extern "C"

static spgemm_status_t spgemm_numeric_any(spgemm_handle_t h, int64_t* c_row_ptr, int32_t* c_col_idx,
                                          double* c_val) {
  if (!h->sym_ok) return fail(h, SPGEMM_ERROR_INVALID_STATE, "numeric before a successful symbolic");
  if (!c_row_ptr || (h->nnz_c > 0 && (!c_col_idx || !c_val)))
    return fail(h, SPGEMM_ERROR_INVALID_VALUE, "NULL output pointer");
  cudaSetDevice(h->device);
  cudaEventRecord(h->ev[4], h->stream);
  h->launches_num = 0;
  CK(h, cudaMemcpyAsync(c_row_ptr, h->c_rp, sizeof(int64_t) * (h->m + 1), cudaMemcpyDeviceToDevice, h->stream));
  if (h->m > 0 && h->nnz_c > 0) {
    const bool precise = (h->flags & SPGEMM_FLAG_PRECISE) != 0;
    CopyArgs ca{};
    ca.f32 = (h->flags & SPGEMM_FLAG_FP32) != 0;
    ca.m = h->m;
    ca.perm = h->long_perm;
    ca.long_first = h->long_first;
    ca.nlong = h->nlong;
    ca.c_rp = h->c_rp;
    ca.ctil_off = h->ws.ctil_off;
    ca.ctil_total = h->sum_cap;
    ca.tier = h->ws.tier;
    ca.ctil_col = h->ctil_col;
    ca.ctil_val = h->ctil_val;
    ca.chunk_table = h->ltable;
    ca.arena_col = static_cast<const int32_t*>(h->arena_col.base);
    ca.arena_val = static_cast<const double*>(h->arena_val.base);
    ca.log2c0 = h->log2c0;
    ca.c_col = c_col_idx;
    ca.c_val = c_val;
    if (precise) {
      // stage 3 again, values on, straight into C at its final offsets
      for (int t = T_G1; t < T_LONG; ++t) {
        if (h->tier_count[t] == 0) continue;
        Stage3Args a{};
        a.f32 = (h->flags & SPGEMM_FLAG_FP32) != 0;
        a.A = h->A;
        a.B = h->B;
        a.b_nnz = h->b_nnz;
        a.n = h->n;
        a.perm = h->ws.perm;
        a.first = h->tier_off[t];
        a.count = h->tier_count[t];
        a.out_off = h->c_rp;
        a.out_col = c_col_idx;
        a.out_val = c_val;
        a.nnz_row = nullptr;
        const bool dense = t == T_BW;
        a.mode = dense ? MODE_DENSE : MODE_FILL;
        a.struct_col = h->ctil_col;
        a.struct_off = h->ws.ctil_off;
        a.bw_nw = h->bw_nw;
        a.rlo = h->ws.rlo;
        a.bwin = h->ws.bwin;
        a.bw_wmax = h->bw_wmax;
        a.bw_vmax = h->bw_vmax;
        a.bw_bmax = h->bw_bmax;
        cudaEventRecord(h->tev[t][0], h->stream);
        CK(h, launch_stage3_tier(t, a, h->stream));
        cudaEventRecord(h->tev[t][1], h->stream);
        h->tev_used[t] = true;
        ++h->launches_num;
      }
      if (h->nlong > 0) {
        Stage3Args a{};
        a.f32 = (h->flags & SPGEMM_FLAG_FP32) != 0;
        a.A = h->A;
        a.B = h->B;
        a.b_nnz = h->b_nnz;
        a.n = h->n;
        a.perm = h->ws.perm;
        a.first = h->long_first;
        a.count = h->nlong;
        a.out_off = h->c_rp;
        a.out_col = c_col_idx;
        a.out_val = c_val;
        a.mode = MODE_FILL;
        a.bwin = h->ws.bwin;
        a.rlo = h->ws.rlo;
        a.rhi = h->ws.rhi;
        a.U = h->ws.U;
        a.work_ctr = h->work_ctr;
        cudaEventRecord(h->tev[T_LONG][0], h->stream);
        if (h->bk_rows > 0) {
          // wide windows: bucket partition + per-bucket sort (longbk.cu); the rest: rank kernel
          spgemm_status_t s2 = run_long_buckets(h, h->c_rp, c_col_idx, c_val, nullptr, nullptr, true);
          if (s2 != SPGEMM_SUCCESS) return s2;
          h->launches_num += 4;
        } else {
          CK(h, launch_long_bitmap(a, h->stream));
        }
        cudaEventRecord(h->tev[T_LONG][1], h->stream);
        h->tev_used[T_LONG] = true;
        ++h->launches_num;
      }
      ca.m = 0;     // nothing to copy: every row was written straight into C
      ca.nlong = 0;
    }
    CK(h, launch_copy(ca, h->stream));
    h->launches_num += (ca.m > 0 ? 1 : 0) + (ca.nlong > 0 ? 1 : 0);
  }
  cudaEventRecord(h->ev[5], h->stream);
  h->numeric_recorded = true;
  return SPGEMM_SUCCESS;
}

extern "C" {

spgemm_status_t spgemm_create_f32(spgemm_handle_t* handle, int64_t m, int64_t k, int64_t n,
                                  const int64_t* a_row_ptr, const int32_t* a_col_idx, const float* a_val,
                                  int64_t a_nnz, const int64_t* b_row_ptr, const int32_t* b_col_idx,
                                  const float* b_val, int64_t b_nnz, spgemm_stream_t stream, uint32_t flags) {
  if (flags & SPGEMM_FLAG_INPUTS_REPLICATED)
    return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "INPUTS_REPLICATED is a dist_* flag");
  return spgemm_create(handle, m, k, n, a_row_ptr, a_col_idx, reinterpret_cast<const double*>(a_val), a_nnz,
                       b_row_ptr, b_col_idx, reinterpret_cast<const double*>(b_val), b_nnz, stream,
                       flags | SPGEMM_FLAG_FP32);
}

spgemm_status_t spgemm_numeric_f32(spgemm_handle_t h, int64_t* c_row_ptr, int32_t* c_col_idx, float* c_val) {
  if (!h) return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "NULL handle");
  if (sg_is_dist(h) || !(h->flags & SPGEMM_FLAG_FP32))
    return fail(h, SPGEMM_ERROR_INVALID_VALUE, "spgemm_numeric_f32 on an fp64 handle");
  return spgemm_numeric_any(h, c_row_ptr, c_col_idx, reinterpret_cast<double*>(c_val));
}

spgemm_status_t spgemm_destroy(spgemm_handle_t h) {
  if (!h) return SPGEMM_SUCCESS;
  if (sg_is_dist(h)) return sg_dist_destroy(h);
  cudaSetDevice(h->device);
  free_symbolic(h);
  cudaStreamSynchronize(h->stream);
  if (h->evs) t_event_pool.push_back(h->evs);  // reused by the next handle of this thread
  delete h;
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_get_stats(spgemm_handle_t h, spgemm_stats_t* out) {
  if (!h || !out) return fail(h, SPGEMM_ERROR_INVALID_VALUE, "NULL handle or out");
  if (sg_is_dist(h)) return sg_dist_stats(h, out);
  memset(out, 0, sizeof(*out));
  out->m = h->m;
  out->k = h->k;
  out->n = h->n;
  out->nnz_a = h->a_nnz;
  out->nnz_b = h->b_nnz;
  out->sum_u = h->sum_u;
  out->nnz_c = h->nnz_c;
  out->max_u = h->max_u;
  for (int t = 0; t < NUM_TIERS; ++t) out->tier_rows[t] = h->tier_count[t];
  out->ctil_entries = (h->flags & SPGEMM_FLAG_PRECISE) ? 0 : h->sum_cap;
  out->long_rows = h->nlong;
  out->long_entries = h->long_entries;
  out->growth_rounds = h->growth_rounds;
  out->flags = (int32_t)h->flags;
  out->workspace_bytes = (int64_t)(h->bytes + h->arena_col.mapped + h->arena_val.mapped);
  if (h->sym_ok && h->ev_ok) {
    cudaEventSynchronize(h->ev[3]);
    cudaEventElapsedTime(&out->stage_ms[0], h->ev[0], h->ev[1]);
    cudaEventElapsedTime(&out->stage_ms[1], h->ev[1], h->ev[2]);
    cudaEventElapsedTime(&out->stage_ms[2], h->ev[2], h->ev[3]);
    if (h->numeric_recorded) {
      cudaEventSynchronize(h->ev[5]);
      cudaEventElapsedTime(&out->stage_ms[3], h->ev[4], h->ev[5]);
    }
    const bool precise = (h->flags & SPGEMM_FLAG_PRECISE) != 0;
    for (int t = 0; t < NUM_TIERS; ++t) {
      if (h->tsym_used[t]) {
        cudaEventSynchronize(h->tsym[t][1]);
        cudaEventElapsedTime(&out->tier_ms_symbolic[t], h->tsym[t][0], h->tsym[t][1]);
        if (!precise) out->tier_ms[t] = out->tier_ms_symbolic[t];
      }
      if (precise && h->tev_used[t]) {
        cudaEventSynchronize(h->tev[t][1]);
        cudaEventElapsedTime(&out->tier_ms[t], h->tev[t][0], h->tev[t][1]);
      }
    }
    out->launches_symbolic = h->launches_sym;
    out->launches_numeric = h->launches_num;
    if (h->m > 0) {
      unsigned long long* d = nullptr;
      std::vector<unsigned long long> hs(3 * NUM_TIERS);
      CK(h, pool_malloc(reinterpret_cast<void**>(&d), sizeof(unsigned long long) * 3 * NUM_TIERS, h->stream));
      CK(h, cudaMemsetAsync(d, 0, sizeof(unsigned long long) * 3 * NUM_TIERS, h->stream));
      k_class_sums<<<256, 256, 0, h->stream>>>(h->m, h->ws.tier, h->ws.U, h->A.rp, h->nnz_row, d);
      CK(h, cudaGetLastError());
      CK(h, cudaMemcpyAsync(hs.data(), d, sizeof(unsigned long long) * 3 * NUM_TIERS, cudaMemcpyDeviceToHost,
                            h->stream));
      CK(h, cudaFreeAsync(d, h->stream));
      CK(h, cudaStreamSynchronize(h->stream));
      for (int t = 0; t < NUM_TIERS; ++t) {
        out->tier_a_entries[t] = (int64_t)hs[t];
        out->tier_products[t] = (int64_t)hs[NUM_TIERS + t];
        out->tier_c_entries[t] = (int64_t)hs[2 * NUM_TIERS + t];
      }
    }
  }
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_debug_get_u(spgemm_handle_t h, int64_t* u, int32_t* tier) {
  if (!h || !u) return fail(h, SPGEMM_ERROR_INVALID_VALUE, "NULL handle or u");
  if (!h->sym_ok) return fail(h, SPGEMM_ERROR_INVALID_STATE, "no symbolic yet");
  if (h->m == 0) return SPGEMM_SUCCESS;
  CK(h, cudaMemcpyAsync(u, h->ws.U, sizeof(int64_t) * h->m, cudaMemcpyDeviceToDevice, h->stream));
  if (tier) {
    k_tier_to_i32<<<(unsigned)((h->m + 255) / 256), 256, 0, h->stream>>>(h->ws.tier, tier, h->m);
    CK(h, cudaGetLastError());
  }
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_trim_workspace_cache(int64_t keep_bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool = library_pool(dev);
  if (!pool) return fail(nullptr, SPGEMM_ERROR_CUDA, "no library memory pool");
  cudaDeviceSynchronize();
  vmm_trim();  // the cached long-row arenas (vmm.cu)
  cudaError_t e = cudaMemPoolTrimTo(pool, keep_bytes > 0 ? (size_t)keep_bytes : 0);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaMemPoolTrimTo");
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_partition_rows(const int64_t* scan, int64_t m, int nranks, int64_t* splits) {
  if (!splits || nranks < 1 || m < 0 || (m > 0 && !scan))
    return fail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "bad partition arguments");
  const int64_t total = m > 0 ? scan[m - 1] : 0;
  splits[0] = 0;
  for (int r = 1; r < nranks; ++r) {
    // s_r = min{ i : scan[i] >= ceil(r·total/P) }, as a row count (rows [0, s_r] go left)
    const __int128 num = (__int128)r * total;
    const int64_t target = (int64_t)((num + nranks - 1) / nranks);
    int64_t lo = 0, hi = m;  // first index with scan[idx] >= target
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (scan[mid] >= target) hi = mid;
      else lo = mid + 1;
    }
    int64_t s = lo < m ? lo + 1 : m;
    if (target == 0) s = 0;
    if (s < splits[r - 1]) s = splits[r - 1];
    splits[r] = s;
  }
  splits[nranks] = m;
  return SPGEMM_SUCCESS;
}

}  // extern "C"
