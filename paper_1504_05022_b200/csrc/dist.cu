// dist.cu — multi-GPU row-block SpGEMM (include/spgemm.h, "multi-GPU").  One process per
// GPU; NCCL over NVLink/NVSwitch inside the library; the id travels through torch.distributed
// (or any bootstrap) as 128 bytes.
//
// The paper is single-device; rows of C are independent (outer loop of Algorithm 1 [P:121],
// stage 1 per row [P:198], stage 3 per row [P:218-222]) and the only cross-row step is stage
// 4's sum of nnz(c_i*) [P:301].  Three input modes:
//   root (dist_create):       A and B on rank 0.  B's structure (row_ptr, col_idx) is
//                             broadcast; the partition s_r = min{ i : scan(u)[i] >= ceil(r·Σu/P) }
//                             ([P:25] "the number of necessary arithmetic operations") is
//                             computed on the root and broadcast; A's row blocks go out with
//                             grouped send / recv and are rebased.
//   replicated (flag):        every rank holds A and B; each computes the partition itself.
//   sharded (create_sharded): the caller's row partition of A; B arrives as per-rank row
//                             slices and is all-gathered (grouped broadcasts, placed at each
//                             slice's entry offset, row pointers rebased).
// Overlap: only B's and A's VALUES are needed by numeric (the precise strategy's symbolic pass
// is structure-only), so they travel on a second stream while the local symbolic pass runs;
// numeric (and the hybrid symbolic, which computes values) waits for them with an event.
// Stitching: ncclAllGather of the per-rank nnz, then each rank adds its global offset to its
// row pointers — concatenating the rank blocks gives the single-GPU CSR byte for byte.
// The host arithmetic of the protocol (partition, entry ranges, slice placement, offsets) is in
// exported functions (spgemm_partition_rows, spgemm_dist_*), which the CPU tests drive too.
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

using namespace sg;

namespace {

thread_local std::string t_dist_err;

__global__ void k_u_only(int64_t m, const int64_t* __restrict__ arp, const int32_t* __restrict__ aci,
                         const int64_t* __restrict__ brp, int64_t* __restrict__ u) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int64_t s = 0;
  for (int64_t p = arp[i]; p < arp[i + 1]; ++p) {
    const int j = aci[p];
    s += brp[j + 1] - brp[j];
  }
  u[i] = s;
}

// splits[r] for r in 0..P from the inclusive scan: the rule of spgemm_partition_rows (host)
__global__ void k_splits(const int64_t* __restrict__ scan, int64_t m, int P, int64_t* splits) {
  if (threadIdx.x != 0) return;
  const int64_t total = m > 0 ? scan[m - 1] : 0;
  splits[0] = 0;
  for (int r = 1; r < P; ++r) {
    const __int128 num = (__int128)r * total;
    const int64_t target = (int64_t)((num + P - 1) / P);
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
  splits[P] = m;
}

__global__ void k_gather_at(const int64_t* __restrict__ src, const int64_t* __restrict__ idx, int n,
                            int64_t* __restrict__ dst) {
  const int i = threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_add_offset(int64_t* p, int64_t n, int64_t off) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] += off;
}

__global__ void k_copy_add(const int64_t* __restrict__ src, int64_t* __restrict__ dst, int64_t n, int64_t off) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i] + off;
}

enum Mode : int { MODE_ROOT = 0, MODE_REPLICATED = 1, MODE_SHARDED = 2 };

}  // namespace

struct spgemm_dist_s {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int mode = MODE_ROOT;
  cudaStream_t stream = nullptr;   // caller's stream: local stages + structure traffic
  cudaStream_t vstream = nullptr;  // values (overlapped with the symbolic pass)
  cudaEvent_t ev_ready = nullptr, ev_vals = nullptr;
  uint32_t flags = 0;
  int64_t m = 0, k = 0, n = 0, a_nnz = 0, b_nnz = 0;
  CsrView A{}, B{};          // caller's
  int64_t a_row_begin = 0, a_row_end = 0, b_row_begin = 0, b_row_end = 0;  // sharded mode
  CsrView Bl{}, Al{};        // local views
  std::vector<void*> mem;    // owned device buffers
  int64_t row_begin = 0, row_end = 0, local_nnz = 0, global_nnz = 0, offset = 0;
  spgemm_handle_t local = nullptr;
  bool vals_pending = false;
  std::string err;
};

// The dist handle is carried through the public spgemm_handle_t type: its first bytes are
// never dereferenced by the single-GPU API because dist handles are tagged.
struct dist_tag {
  uint64_t magic;
  spgemm_dist_s* d;
};
static const uint64_t kDistMagic = 0x44495354535047ull;  // "DISTSPG"

namespace {

spgemm_status_t dfail(spgemm_dist_s* d, spgemm_status_t s, const std::string& msg) {
  if (d) d->err = msg;
  t_dist_err = msg;
  return s;
}

#define NCK(d, call)                                                                  \
  do {                                                                                \
    ncclResult_t _r = (call);                                                         \
    if (_r != ncclSuccess) return dfail(d, SPGEMM_ERROR_NCCL, std::string(#call ": ") + ncclGetErrorString(_r)); \
  } while (0)
#define DCK(d, call)                                                                  \
  do {                                                                                \
    cudaError_t _e = (call);                                                          \
    if (_e != cudaSuccess)                                                            \
      return dfail(d, _e == cudaErrorMemoryAllocation ? SPGEMM_ERROR_OUT_OF_MEMORY : SPGEMM_ERROR_CUDA, \
                   std::string(#call ": ") + cudaGetErrorString(_e));                 \
  } while (0)
#define SCK(call)                                                                     \
  do {                                                                                \
    spgemm_status_t _s = (call);                                                      \
    if (_s != SPGEMM_SUCCESS) return _s;                                              \
  } while (0)

template <typename T>
spgemm_status_t dmalloc(spgemm_dist_s* d, T** p, int64_t count) {
  void* q = nullptr;
  DCK(d, pool_malloc(&q, sizeof(T) * size_t(count > 0 ? count : 1), d->stream));
  d->mem.push_back(q);
  *p = static_cast<T*>(q);
  return SPGEMM_SUCCESS;
}
#define DAL(d, p, n) SCK(dmalloc(d, p, n))

spgemm_dist_s* as_dist(spgemm_handle_t h) {
  if (!h) return nullptr;
  dist_tag* t = reinterpret_cast<dist_tag*>(h);
  return t->magic == kDistMagic ? t->d : nullptr;
}

void launch_add(int64_t* p, int64_t n, int64_t off, cudaStream_t s) {
  if (n > 0 && off != 0) k_add_offset<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n, off);
}

spgemm_status_t begin(spgemm_dist_s* d) {
  for (void* p : d->mem) cudaFreeAsync(p, d->stream);
  d->mem.clear();
  if (d->local) {
    spgemm_destroy(d->local);
    d->local = nullptr;
  }
  d->vals_pending = false;
  return SPGEMM_SUCCESS;
}

// the value stream starts after everything enqueued so far on the main stream (allocations)
// splits of A's rows by the inclusive prefix sum of u (stage 1 without the classes), on the
// device; splits (device, P+1) out
spgemm_status_t device_partition(spgemm_dist_s* d, CsrView A, const int64_t* brp, int64_t* splits) {
  cudaStream_t s = d->stream;
  int64_t *u, *scan, *tmp;
  DAL(d, &u, d->m);
  DAL(d, &scan, d->m + 1);
  DAL(d, &tmp, scan_tmp_elems(d->m + 1) + 4);
  if (d->m > 0) {
    k_u_only<<<(unsigned)((d->m + 255) / 256), 256, 0, s>>>(d->m, A.rp, A.ci, brp, u);
    DCK(d, cudaGetLastError());
    DCK(d, launch_exclusive_scan(u, scan, d->m, tmp, s));  // scan[i+1] = inclusive prefix of row i
  }
  k_splits<<<1, 32, 0, s>>>(scan + 1, d->m, d->nranks, splits);
  DCK(d, cudaGetLastError());
  return SPGEMM_SUCCESS;
}

spgemm_status_t fork_values(spgemm_dist_s* d) {
  DCK(d, cudaEventRecord(d->ev_ready, d->stream));
  DCK(d, cudaStreamWaitEvent(d->vstream, d->ev_ready, 0));
  return SPGEMM_SUCCESS;
}

spgemm_status_t join_values(spgemm_dist_s* d) {
  if (!d->vals_pending) return SPGEMM_SUCCESS;
  DCK(d, cudaStreamWaitEvent(d->stream, d->ev_vals, 0));
  return SPGEMM_SUCCESS;
}

// ---- root mode: replicate B, partition, scatter A ----------------------------------------
spgemm_status_t root_inputs(spgemm_dist_s* d, int64_t* hs) {
  const int P = d->nranks, R = d->rank;
  cudaStream_t s = d->stream;
  int64_t* hdr = nullptr;  // [a_nnz, b_nnz] + splits[P+1] + bounds[2P]
  DAL(d, &hdr, 2 + (P + 1) + 2 * P);
  int64_t* splits = hdr + 2;
  int64_t* bounds = splits + P + 1;
  std::vector<int64_t> h(2);
  if (R == 0) {
    h[0] = d->a_nnz;
    h[1] = d->b_nnz;
    DCK(d, cudaMemcpyAsync(hdr, h.data(), 2 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  }
  NCK(d, ncclBroadcast(hdr, hdr, 2, ncclInt64, 0, d->comm, s));
  DCK(d, cudaMemcpyAsync(h.data(), hdr, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DCK(d, cudaStreamSynchronize(s));
  d->a_nnz = h[0];
  d->b_nnz = h[1];
  // 1. B: structure on the main stream (stages 1-3 need it), values on the value stream
  if (R == 0) {
    d->Bl = d->B;
  } else {
    int64_t* rp;
    int32_t* ci;
    double* v;
    DAL(d, &rp, d->k + 1);
    DAL(d, &ci, d->b_nnz);
    DAL(d, &v, d->b_nnz);
    d->Bl = CsrView{rp, ci, v};
  }
  SCK(fork_values(d));
  NCK(d, ncclGroupStart());
  NCK(d, ncclBroadcast(d->Bl.rp, const_cast<int64_t*>(d->Bl.rp), d->k + 1, ncclInt64, 0, d->comm, s));
  if (d->b_nnz > 0) NCK(d, ncclBroadcast(d->Bl.ci, const_cast<int32_t*>(d->Bl.ci), d->b_nnz, ncclInt32, 0, d->comm, s));
  NCK(d, ncclGroupEnd());
  // 2. partition by the prefix sum of u, on the root (device scan, device split search)
  if (R == 0) {
    SCK(device_partition(d, d->A, d->Bl.rp, splits));
    std::vector<int64_t> rps(P + 1), hb(2 * P);
    int64_t* rpd = splits + (P + 1);  // scratch for rp at the splits (overwritten below)
    k_gather_at<<<1, 1024, 0, s>>>(d->A.rp, splits, P + 1, rpd);
    DCK(d, cudaGetLastError());
    std::vector<int64_t> h2(2 * (P + 1));
    DCK(d, cudaMemcpyAsync(h2.data(), splits, 2 * (P + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DCK(d, cudaStreamSynchronize(s));
    SCK(spgemm_dist_block_entries(h2.data() + P + 1, P, hb.data()));
    std::vector<int64_t> pack(h2.begin(), h2.begin() + P + 1);
    pack.insert(pack.end(), hb.begin(), hb.end());
    DCK(d, cudaMemcpyAsync(splits, pack.data(), pack.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  }
  NCK(d, ncclBroadcast(splits, splits, (P + 1) + 2 * P, ncclInt64, 0, d->comm, s));
  std::vector<int64_t> pack((P + 1) + 2 * P);
  DCK(d, cudaMemcpyAsync(pack.data(), splits, pack.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DCK(d, cudaStreamSynchronize(s));
  for (int r = 0; r <= P; ++r) hs[r] = pack[r];
  const int64_t* hb = pack.data() + P + 1;
  d->row_begin = hs[R];
  d->row_end = hs[R + 1];
  const int64_t ml = d->row_end - d->row_begin;
  // 3. A row blocks: row pointers and columns on the main stream, values on the value stream
  if (P == 1) {
    d->Al = CsrView{d->A.rp + d->row_begin, d->A.ci, d->A.val};
  } else if (R == 0) {
    d->Al = CsrView{d->A.rp + d->row_begin, d->A.ci, d->A.val};
    NCK(d, ncclGroupStart());
    for (int r = 1; r < P; ++r) {
      const int64_t nr = hs[r + 1] - hs[r], e0 = hb[2 * r], e1 = hb[2 * r + 1];
      NCK(d, ncclSend(d->A.rp + hs[r], nr + 1, ncclInt64, r, d->comm, s));
      if (e1 > e0) NCK(d, ncclSend(d->A.ci + e0, e1 - e0, ncclInt32, r, d->comm, s));
    }
    NCK(d, ncclGroupEnd());
  } else {
    const int64_t e0 = hb[2 * R], e1 = hb[2 * R + 1];
    int64_t* rp;
    int32_t* ci;
    double* v;
    DAL(d, &rp, ml + 1);
    DAL(d, &ci, e1 - e0);
    DAL(d, &v, e1 - e0);
    NCK(d, ncclGroupStart());
    NCK(d, ncclRecv(rp, ml + 1, ncclInt64, 0, d->comm, s));
    if (e1 > e0) NCK(d, ncclRecv(ci, e1 - e0, ncclInt32, 0, d->comm, s));
    NCK(d, ncclGroupEnd());
    launch_add(rp, ml + 1, -e0, s);  // rebase: the block's entries start at 0 here
    DCK(d, cudaGetLastError());
    d->Al = CsrView{rp, ci, v};
  }
  // values: B's, then A's blocks, on the value stream (NCCL calls in the same order on all ranks)
  SCK(fork_values(d));
  NCK(d, ncclGroupStart());
  if (d->b_nnz > 0)
    NCK(d, ncclBroadcast(d->Bl.val, const_cast<double*>(d->Bl.val), d->b_nnz, ncclFloat64, 0, d->comm, d->vstream));
  if (P > 1) {
    if (R == 0) {
      for (int r = 1; r < P; ++r) {
        const int64_t e0 = hb[2 * r], e1 = hb[2 * r + 1];
        if (e1 > e0) NCK(d, ncclSend(d->A.val + e0, e1 - e0, ncclFloat64, r, d->comm, d->vstream));
      }
    } else {
      const int64_t e0 = hb[2 * R], e1 = hb[2 * R + 1];
      if (e1 > e0) NCK(d, ncclRecv(const_cast<double*>(d->Al.val), e1 - e0, ncclFloat64, 0, d->comm, d->vstream));
    }
  }
  NCK(d, ncclGroupEnd());
  DCK(d, cudaEventRecord(d->ev_vals, d->vstream));
  d->vals_pending = true;
  return SPGEMM_SUCCESS;
}

// ---- sharded mode: all-gather B's row slices ----------------------------------------------
spgemm_status_t sharded_inputs(spgemm_dist_s* d) {
  const int P = d->nranks, R = d->rank;
  cudaStream_t s = d->stream;
  // every rank's slice: (row begin, row end, nnz, row_ptr[0])
  int64_t* meta = nullptr;
  DAL(d, &meta, 4 * P);
  int64_t mine[4] = {d->b_row_begin, d->b_row_end, d->b_nnz, 0};
  if (d->b_row_end > d->b_row_begin)
    DCK(d, cudaMemcpyAsync(&mine[3], d->B.rp, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DCK(d, cudaStreamSynchronize(s));
  DCK(d, cudaMemcpyAsync(meta + 4 * R, mine, sizeof(mine), cudaMemcpyHostToDevice, s));
  NCK(d, ncclAllGather(meta + 4 * R, meta, 4, ncclInt64, d->comm, s));
  std::vector<int64_t> hm(4 * P);
  DCK(d, cudaMemcpyAsync(hm.data(), meta, hm.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DCK(d, cudaStreamSynchronize(s));
  std::vector<int64_t> rb(P), re(P), nz(P), base(P + 1);
  for (int r = 0; r < P; ++r) {
    rb[r] = hm[4 * r];
    re[r] = hm[4 * r + 1];
    nz[r] = hm[4 * r + 2];
  }
  SCK(spgemm_dist_slice_layout(rb.data(), re.data(), nz.data(), P, d->k, base.data()));
  d->b_nnz = base[P];
  int64_t* rp;
  int32_t* ci;
  double* v;
  DAL(d, &rp, d->k + 1);
  DAL(d, &ci, d->b_nnz);
  DAL(d, &v, d->b_nnz);
  d->Bl = CsrView{rp, ci, v};
  // this rank's slice in place (row pointers rebased to the slice's global entry offset), then
  // grouped broadcasts from every rank = an all-gather-v of the slices
  if (re[R] > rb[R]) {
    k_copy_add<<<(unsigned)((re[R] - rb[R] + 255) / 256), 256, 0, s>>>(d->B.rp, rp + rb[R], re[R] - rb[R],
                                                                       base[R] - hm[4 * R + 3]);
    DCK(d, cudaGetLastError());
  }
  if (nz[R] > 0) {
    DCK(d, cudaMemcpyAsync(ci + base[R], d->B.ci, nz[R] * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    DCK(d, cudaMemcpyAsync(v + base[R], d->B.val, nz[R] * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  const int64_t total = base[P];
  DCK(d, cudaMemcpyAsync(rp + d->k, &total, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  SCK(fork_values(d));
  NCK(d, ncclGroupStart());
  for (int r = 0; r < P; ++r) {
    if (re[r] > rb[r]) NCK(d, ncclBroadcast(rp + rb[r], rp + rb[r], re[r] - rb[r], ncclInt64, r, d->comm, s));
    if (nz[r] > 0) NCK(d, ncclBroadcast(ci + base[r], ci + base[r], nz[r], ncclInt32, r, d->comm, s));
  }
  NCK(d, ncclGroupEnd());
  NCK(d, ncclGroupStart());
  for (int r = 0; r < P; ++r)
    if (nz[r] > 0) NCK(d, ncclBroadcast(v + base[r], v + base[r], nz[r], ncclFloat64, r, d->comm, d->vstream));
  NCK(d, ncclGroupEnd());
  DCK(d, cudaEventRecord(d->ev_vals, d->vstream));
  d->vals_pending = true;
  // A: the caller's block, row pointers rebased to its own arrays
  d->row_begin = d->a_row_begin;
  d->row_end = d->a_row_end;
  const int64_t ml = d->row_end - d->row_begin;
  int64_t* arp;
  DAL(d, &arp, ml + 1);
  int64_t a0 = 0;
  DCK(d, cudaMemcpyAsync(&a0, d->A.rp, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DCK(d, cudaStreamSynchronize(s));
  k_copy_add<<<(unsigned)((ml + 1 + 255) / 256), 256, 0, s>>>(d->A.rp, arp, ml + 1, -a0);
  DCK(d, cudaGetLastError());
  d->Al = CsrView{arp, d->A.ci, d->A.val};
  return SPGEMM_SUCCESS;
}

spgemm_status_t make_dist(spgemm_handle_t* handle, int rank, int nranks, const uint8_t id[128],
                          spgemm_stream_t stream, uint32_t flags, spgemm_dist_s** out) {
  spgemm_dist_s* d = new spgemm_dist_s();
  d->rank = rank;
  d->nranks = nranks;
  d->stream = static_cast<cudaStream_t>(stream);
  d->flags = flags;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclResult_t r = ncclCommInitRank(&d->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    spgemm_status_t s = dfail(nullptr, SPGEMM_ERROR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    delete d;
    return s;
  }
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (cudaStreamCreateWithPriority(&d->vstream, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->ev_vals, cudaEventDisableTiming) != cudaSuccess) {
    ncclCommDestroy(d->comm);
    delete d;
    return dfail(nullptr, SPGEMM_ERROR_CUDA, "stream / event creation failed");
  }
  dist_tag* t = new dist_tag{kDistMagic, d};
  *handle = reinterpret_cast<spgemm_handle_t>(t);
  *out = d;
  return SPGEMM_SUCCESS;
}

}  // namespace

extern "C" {

spgemm_status_t spgemm_nccl_get_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!id) return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "NULL id");
  ncclUniqueId u;
  NCK((spgemm_dist_s*)nullptr, ncclGetUniqueId(&u));
  memcpy(id, &u, 128);
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_dist_create(spgemm_handle_t* handle, int rank, int nranks,
                                   const uint8_t id[128], int64_t m, int64_t k, int64_t n,
                                   const int64_t* a_row_ptr, const int32_t* a_col_idx,
                                   const double* a_val, int64_t a_nnz, const int64_t* b_row_ptr,
                                   const int32_t* b_col_idx, const double* b_val, int64_t b_nnz,
                                   spgemm_stream_t stream, uint32_t flags) {
  if (!handle || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "bad dist_create arguments");
  *handle = nullptr;
  if (m < 0 || k < 0 || n < 0) return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "negative size");
  if (m > INT32_MAX || k > INT32_MAX || n > INT32_MAX)
    return dfail(nullptr, SPGEMM_ERROR_INDEX_OVERFLOW, "m, k or n exceeds INT32_MAX");
  const bool repl = (flags & SPGEMM_FLAG_INPUTS_REPLICATED) != 0;
  if ((rank == 0 || repl) && (!a_row_ptr || !b_row_ptr))
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "NULL input on a rank that must hold it");
  spgemm_dist_s* d = nullptr;
  SCK(make_dist(handle, rank, nranks, id, stream, flags, &d));
  d->mode = repl ? MODE_REPLICATED : MODE_ROOT;
  d->m = m;
  d->k = k;
  d->n = n;
  d->a_nnz = a_nnz;
  d->b_nnz = b_nnz;
  d->A = CsrView{a_row_ptr, a_col_idx, a_val};
  d->B = CsrView{b_row_ptr, b_col_idx, b_val};
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_dist_create_sharded(spgemm_handle_t* handle, int rank, int nranks, const uint8_t id[128],
                                           int64_t m, int64_t k, int64_t n, int64_t a_row_begin, int64_t a_row_end,
                                           const int64_t* a_row_ptr, const int32_t* a_col_idx, const double* a_val,
                                           int64_t a_nnz, int64_t b_row_begin, int64_t b_row_end,
                                           const int64_t* b_row_ptr, const int32_t* b_col_idx, const double* b_val,
                                           int64_t b_nnz, spgemm_stream_t stream, uint32_t flags) {
  if (!handle || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "bad dist_create_sharded arguments");
  *handle = nullptr;
  if (m < 0 || k < 0 || n < 0 || a_nnz < 0 || b_nnz < 0)
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "negative size");
  if (m > INT32_MAX || k > INT32_MAX || n > INT32_MAX)
    return dfail(nullptr, SPGEMM_ERROR_INDEX_OVERFLOW, "m, k or n exceeds INT32_MAX");
  if (a_row_begin < 0 || a_row_end < a_row_begin || a_row_end > m || b_row_begin < 0 || b_row_end < b_row_begin ||
      b_row_end > k)
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "row range outside the matrix");
  if (!a_row_ptr || !b_row_ptr || (a_nnz > 0 && (!a_col_idx || !a_val)) || (b_nnz > 0 && (!b_col_idx || !b_val)))
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "NULL input pointer");
  if (flags & SPGEMM_FLAG_INPUTS_REPLICATED)
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "INPUTS_REPLICATED does not apply to sharded inputs");
  spgemm_dist_s* d = nullptr;
  SCK(make_dist(handle, rank, nranks, id, stream, flags, &d));
  d->mode = MODE_SHARDED;
  d->m = m;
  d->k = k;
  d->n = n;
  d->a_nnz = a_nnz;
  d->b_nnz = b_nnz;
  d->a_row_begin = a_row_begin;
  d->a_row_end = a_row_end;
  d->b_row_begin = b_row_begin;
  d->b_row_end = b_row_end;
  d->A = CsrView{a_row_ptr, a_col_idx, a_val};
  d->B = CsrView{b_row_ptr, b_col_idx, b_val};
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_dist_symbolic(spgemm_handle_t handle, int64_t* row_begin, int64_t* row_end,
                                     int64_t* local_nnz, int64_t* global_nnz) {
  spgemm_dist_s* d = as_dist(handle);
  if (!d) return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "not a dist handle");
  const int P = d->nranks, R = d->rank;
  cudaStream_t s = d->stream;
  SCK(begin(d));
  if (d->mode == MODE_ROOT) {
    std::vector<int64_t> hs(P + 1);
    SCK(root_inputs(d, hs.data()));
  } else if (d->mode == MODE_SHARDED) {
    SCK(sharded_inputs(d));
  } else {
    // replicated: every rank computes the partition itself (identical on all ranks)
    d->Bl = d->B;
    int64_t* splits = nullptr;
    DAL(d, &splits, P + 1);
    SCK(device_partition(d, d->A, d->Bl.rp, splits));
    std::vector<int64_t> hs(P + 1);
    DCK(d, cudaMemcpyAsync(hs.data(), splits, (P + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DCK(d, cudaStreamSynchronize(s));
    d->row_begin = hs[R];
    d->row_end = hs[R + 1];
    // row i of the block has entries [rp[row_begin+i], rp[row_begin+i+1]) of the full arrays
    d->Al = CsrView{d->A.rp + d->row_begin, d->A.ci, d->A.val};
  }
  const int64_t ml = d->row_end - d->row_begin;
  // --- local four-stage SpGEMM (structure-only symbolic pass overlaps the value traffic) ---
  const bool precise = (d->flags & SPGEMM_FLAG_PRECISE) != 0;
  if (!precise) SCK(join_values(d));  // the hybrid symbolic pass computes values
  spgemm_status_t st = spgemm_create(&d->local, ml, d->k, d->n, d->Al.rp, d->Al.ci, d->Al.val,
                                     0 /* unused by the kernels */, d->Bl.rp, d->Bl.ci, d->Bl.val,
                                     d->b_nnz, s, d->flags & (SPGEMM_FLAG_PRECISE | SPGEMM_FLAG_UPPER_BOUND));
  if (st != SPGEMM_SUCCESS) return dfail(d, st, std::string("local create: ") + spgemm_last_error(nullptr));
  int64_t lnnz = 0;
  st = spgemm_symbolic(d->local, &lnnz);
  if (st != SPGEMM_SUCCESS) return dfail(d, st, std::string("local symbolic: ") + spgemm_last_error(d->local));
  // --- stitch: allgather per-rank nnz (stage 4's sum across ranks [P:301]) ---------------
  int64_t* nnzs = nullptr;
  DAL(d, &nnzs, P);
  DCK(d, cudaMemcpyAsync(nnzs + R, &lnnz, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  NCK(d, ncclAllGather(nnzs + R, nnzs, 1, ncclInt64, d->comm, s));
  std::vector<int64_t> hn(P);
  DCK(d, cudaMemcpyAsync(hn.data(), nnzs, P * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DCK(d, cudaStreamSynchronize(s));
  int64_t off = 0, tot = 0;
  SCK(spgemm_dist_offsets(hn.data(), P, R, &off, &tot));
  d->local_nnz = lnnz;
  d->global_nnz = tot;
  d->offset = off;
  if (row_begin) *row_begin = d->row_begin;
  if (row_end) *row_end = d->row_end;
  if (local_nnz) *local_nnz = lnnz;
  if (global_nnz) *global_nnz = tot;
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_dist_numeric(spgemm_handle_t handle, int64_t* c_row_ptr, int32_t* c_col_idx,
                                    double* c_val) {
  spgemm_dist_s* d = as_dist(handle);
  if (!d) return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "not a dist handle");
  if (!d->local) return dfail(d, SPGEMM_ERROR_INVALID_STATE, "dist_numeric before dist_symbolic");
  SCK(join_values(d));  // A's and B's values have arrived
  spgemm_status_t st = spgemm_numeric(d->local, c_row_ptr, c_col_idx, c_val);
  if (st != SPGEMM_SUCCESS) return dfail(d, st, std::string("local numeric: ") + spgemm_last_error(d->local));
  const int64_t ml = d->row_end - d->row_begin;
  launch_add(c_row_ptr, ml + 1, d->offset, d->stream);  // global row offsets
  DCK(d, cudaGetLastError());
  return SPGEMM_SUCCESS;
}

// The device partition of the dist entry points on a caller's inclusive scan (device, m
// entries) -> splits (host, P+1): lets the GPU tests hold it against spgemm_partition_rows.
spgemm_status_t spgemm_debug_partition(const int64_t* u_inclusive_scan, int64_t m, int nranks, int64_t* splits) {
  if (!splits || nranks < 1 || nranks > 1 << 20 || m < 0 || (m > 0 && !u_inclusive_scan))
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "bad partition arguments");
  int64_t* ds = nullptr;
  cudaError_t e = cudaMalloc(&ds, sizeof(int64_t) * (nranks + 1));
  if (e == cudaSuccess) {
    k_splits<<<1, 32>>>(u_inclusive_scan, m, nranks, ds);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(splits, ds, sizeof(int64_t) * (nranks + 1), cudaMemcpyDeviceToHost);
  if (ds) cudaFree(ds);
  if (e != cudaSuccess) return dfail(nullptr, SPGEMM_ERROR_CUDA, std::string("debug_partition: ") + cudaGetErrorString(e));
  return SPGEMM_SUCCESS;
}

// ---- host arithmetic of the protocol (exported; the CPU tests drive the same functions) ----
spgemm_status_t spgemm_dist_block_entries(const int64_t* rp_at_splits, int nranks, int64_t* entry_bounds) {
  if (!rp_at_splits || !entry_bounds || nranks < 1)
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "bad block-entry arguments");
  for (int r = 0; r < nranks; ++r) {
    entry_bounds[2 * r] = rp_at_splits[r];
    entry_bounds[2 * r + 1] = rp_at_splits[r + 1];
    if (rp_at_splits[r + 1] < rp_at_splits[r])
      return dfail(nullptr, SPGEMM_ERROR_INVALID_CSR, "row pointers decrease across a split");
  }
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_dist_slice_layout(const int64_t* row_begin, const int64_t* row_end, const int64_t* nnz,
                                         int nranks, int64_t k, int64_t* entry_base) {
  if (!row_begin || !row_end || !nnz || !entry_base || nranks < 1)
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "bad slice-layout arguments");
  int64_t next_row = 0, base = 0;
  for (int r = 0; r < nranks; ++r) {
    // slices tile [0, k) in rank order (empty slices allowed)
    if (row_begin[r] != next_row || row_end[r] < row_begin[r] || nnz[r] < 0)
      return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "B slices do not tile the rows of B in rank order");
    entry_base[r] = base;
    base += nnz[r];
    next_row = row_end[r];
  }
  if (next_row != k) return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "B slices do not cover all k rows");
  entry_base[nranks] = base;
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_dist_offsets(const int64_t* local_nnz, int nranks, int rank, int64_t* offset,
                                    int64_t* total) {
  if (!local_nnz || !offset || !total || nranks < 1 || rank < 0 || rank >= nranks)
    return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "bad offset arguments");
  int64_t off = 0, tot = 0;
  for (int r = 0; r < nranks; ++r) {
    if (r < rank) off += local_nnz[r];
    tot += local_nnz[r];
  }
  *offset = off;
  *total = tot;
  return SPGEMM_SUCCESS;
}

}  // extern "C"

// Called from spgemm_destroy/get_stats/last_error when handed a dist handle.
spgemm_status_t sg_dist_destroy(spgemm_handle_t h) {
  spgemm_dist_s* d = as_dist(h);
  if (!d) return SPGEMM_ERROR_INVALID_VALUE;
  if (d->vstream) cudaStreamSynchronize(d->vstream);
  if (d->local) spgemm_destroy(d->local);
  for (void* p : d->mem) cudaFreeAsync(p, d->stream);
  cudaStreamSynchronize(d->stream);
  if (d->comm) ncclCommDestroy(d->comm);
  if (d->vstream) cudaStreamDestroy(d->vstream);
  if (d->ev_ready) cudaEventDestroy(d->ev_ready);
  if (d->ev_vals) cudaEventDestroy(d->ev_vals);
  reinterpret_cast<dist_tag*>(h)->magic = 0;
  delete reinterpret_cast<dist_tag*>(h);
  delete d;
  return SPGEMM_SUCCESS;
}

bool sg_is_dist(spgemm_handle_t h) { return as_dist(h) != nullptr; }

const char* sg_dist_error(spgemm_handle_t h) {
  spgemm_dist_s* d = as_dist(h);
  return d ? d->err.c_str() : t_dist_err.c_str();
}

spgemm_status_t sg_dist_stats(spgemm_handle_t h, spgemm_stats_t* out) {
  spgemm_dist_s* d = as_dist(h);
  if (!d || !d->local) return SPGEMM_ERROR_INVALID_STATE;
  return spgemm_get_stats(d->local, out);
}
