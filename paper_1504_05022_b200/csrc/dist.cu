// dist.cu — multi-GPU row-block SpGEMM (include/spgemm.h, "multi-GPU").  One process per
// GPU; NCCL over NVLink/NVSwitch inside the library; the id travels through
// torch.distributed (or any bootstrap) as 128 bytes.
//
// The paper is single-device; rows of C are independent (outer loop of Algorithm 1
// [P:121], stage 1 per row [P:198], stage 3 per row [P:218-222]) and the only cross-row
// step is stage 4's sum of nnz(c_i*) [P:301].  So:
//   1. B replicated: ncclBroadcast of (row_ptr, col_idx, val) from rank 0.
//   2. Partition: stage-1 bound on the root, inclusive scan, split points
//      s_r = min{ i : scan(u)[i] >= ceil(r·Σu/P) } (the paper's load-balance quantity, "the
//      number of necessary arithmetic operations" [P:25]); ncclBroadcast of the splits.
//   3. A row blocks: grouped ncclSend/ncclRecv from the root; receivers rebase row_ptr.
//   4. Local four-stage SpGEMM on rows [s_r, s_r+1).
//   5. ncclAllGather of the per-rank nnz → each rank adds its global offset to its row_ptr.
// With SPGEMM_FLAG_INPUTS_REPLICATED every rank holds A and B: steps 1-3 are local and
// only the allgather crosses NVLink.
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

// splits[r] for r in 1..P-1 from the inclusive scan (same rule as spgemm_partition_rows)
__global__ void k_splits(const int64_t* __restrict__ scan, int64_t m, int P, int64_t* splits) {
  const int r = threadIdx.x;
  if (r > P) return;
  if (r == 0) {
    splits[0] = 0;
    return;
  }
  if (r == P) {
    splits[P] = m;
    return;
  }
  const int64_t total = m > 0 ? scan[m - 1] : 0;
  const __int128 num = (__int128)r * total;
  const int64_t target = (int64_t)((num + P - 1) / P);
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (scan[mid] >= target) hi = mid;
    else lo = mid + 1;
  }
  int64_t s = lo < m ? lo + 1 : m;
  if (target == 0) s = 0;
  splits[r] = s;
}

__global__ void k_monotone(int64_t* splits, int P) {
  if (threadIdx.x == 0)
    for (int r = 1; r <= P; ++r)
      if (splits[r] < splits[r - 1]) splits[r] = splits[r - 1];
}

__global__ void k_add_offset(int64_t* p, int64_t n, int64_t off) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] += off;
}

}  // namespace

struct spgemm_dist_s {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  cudaStream_t stream = nullptr;
  uint32_t flags = 0;
  int64_t m = 0, k = 0, n = 0, a_nnz = 0, b_nnz = 0;
  CsrView A{}, B{};          // caller's (root, or all ranks if replicated)
  CsrView Bl{}, Al{};        // local views
  std::vector<void*> mem;    // owned device buffers
  int64_t row_begin = 0, row_end = 0, local_nnz = 0, global_nnz = 0, offset = 0;
  spgemm_handle_t local = nullptr;
  std::string err;
};

// The dist handle is carried through the public spgemm_handle_t type: its first bytes
// are never dereferenced by the single-GPU API because dist handles are tagged.
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

template <typename T>
spgemm_status_t dmalloc(spgemm_dist_s* d, T** p, int64_t count) {
  void* q = nullptr;
  DCK(d, pool_malloc(&q, sizeof(T) * size_t(count > 0 ? count : 1), d->stream));
  d->mem.push_back(q);
  *p = static_cast<T*>(q);
  return SPGEMM_SUCCESS;
}
#define DAL(d, p, n)                                  \
  do {                                                \
    spgemm_status_t _s = dmalloc(d, p, n);            \
    if (_s != SPGEMM_SUCCESS) return _s;              \
  } while (0)

spgemm_dist_s* as_dist(spgemm_handle_t h) {
  if (!h) return nullptr;
  dist_tag* t = reinterpret_cast<dist_tag*>(h);
  return t->magic == kDistMagic ? t->d : nullptr;
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
  spgemm_dist_s* d = new spgemm_dist_s();
  d->rank = rank;
  d->nranks = nranks;
  d->stream = static_cast<cudaStream_t>(stream);
  d->flags = flags;
  d->m = m;
  d->k = k;
  d->n = n;
  d->a_nnz = a_nnz;
  d->b_nnz = b_nnz;
  d->A = CsrView{a_row_ptr, a_col_idx, a_val};
  d->B = CsrView{b_row_ptr, b_col_idx, b_val};
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclResult_t r = ncclCommInitRank(&d->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    spgemm_status_t s = dfail(nullptr, SPGEMM_ERROR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    delete d;
    return s;
  }
  dist_tag* t = new dist_tag{kDistMagic, d};
  *handle = reinterpret_cast<spgemm_handle_t>(t);
  return SPGEMM_SUCCESS;
}

spgemm_status_t spgemm_dist_symbolic(spgemm_handle_t handle, int64_t* row_begin, int64_t* row_end,
                                     int64_t* local_nnz, int64_t* global_nnz) {
  spgemm_dist_s* d = as_dist(handle);
  if (!d) return dfail(nullptr, SPGEMM_ERROR_INVALID_VALUE, "not a dist handle");
  const bool repl = (d->flags & SPGEMM_FLAG_INPUTS_REPLICATED) != 0;
  const int P = d->nranks, R = d->rank;
  cudaStream_t s = d->stream;
  for (void* p : d->mem) cudaFreeAsync(p, s);
  d->mem.clear();
  if (d->local) {
    spgemm_destroy(d->local);
    d->local = nullptr;
  }
  int64_t* hdr = nullptr;  // [a_nnz, b_nnz] + splits[P+1] + nnz[P] + rp bounds
  DAL(d, &hdr, 2 + (P + 1) + P + 2 * P + 2);
  int64_t* splits = hdr + 2;
  int64_t* nnzs = splits + P + 1;
  std::vector<int64_t> h(2 + (P + 1));
  // --- 1. replicate B (row_ptr first: the only part stages 1-2 need) ---------------------
  if (!repl) {
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
    NCK(d, ncclGroupStart());
    NCK(d, ncclBroadcast(d->Bl.rp, const_cast<int64_t*>(d->Bl.rp), d->k + 1, ncclInt64, 0, d->comm, s));
    if (d->b_nnz > 0) {
      NCK(d, ncclBroadcast(d->Bl.ci, const_cast<int32_t*>(d->Bl.ci), d->b_nnz, ncclInt32, 0, d->comm, s));
      NCK(d, ncclBroadcast(d->Bl.val, const_cast<double*>(d->Bl.val), d->b_nnz, ncclFloat64, 0, d->comm, s));
    }
    NCK(d, ncclGroupEnd());
  } else {
    d->Bl = d->B;
  }
  // --- 2. partition by the prefix sum of u ----------------------------------------------
  if (repl || R == 0) {
    int64_t *u, *scan, *tmp;
    DAL(d, &u, d->m);
    DAL(d, &scan, d->m + 1);
    DAL(d, &tmp, scan_tmp_elems(d->m + 1) + 4);
    if (d->m > 0) {
      k_u_only<<<(unsigned)((d->m + 255) / 256), 256, 0, s>>>(d->m, d->A.rp, d->A.ci, d->Bl.rp, u);
      DCK(d, cudaGetLastError());
      DCK(d, launch_exclusive_scan(u, scan, d->m, tmp, s));  // scan[i+1] = inclusive prefix of row i
    }
    k_splits<<<1, 64 * ((P + 64) / 64), 0, s>>>(scan + 1, d->m, P, splits);
    k_monotone<<<1, 32, 0, s>>>(splits, P);
    DCK(d, cudaGetLastError());
  }
  if (!repl) NCK(d, ncclBroadcast(splits, splits, P + 1, ncclInt64, 0, d->comm, s));
  std::vector<int64_t> hs(P + 1);
  DCK(d, cudaMemcpyAsync(hs.data(), splits, (P + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DCK(d, cudaStreamSynchronize(s));
  d->row_begin = hs[R];
  d->row_end = hs[R + 1];
  const int64_t ml = d->row_end - d->row_begin;
  // --- 3. A row blocks -----------------------------------------------------------------
  if (repl || P == 1) {
    // row i of the block has entries [rp[row_begin+i], rp[row_begin+i+1]) of the full arrays
    d->Al = CsrView{d->A.rp + d->row_begin, d->A.ci, d->A.val};
  } else {
    // root tells each rank its entry range (rp at the split points), then sends the slices
    int64_t* bounds = nnzs + P;  // [2P]
    if (R == 0) {
      std::vector<int64_t> hb(2 * P);
      for (int r = 0; r < P; ++r) {
        DCK(d, cudaMemcpyAsync(&hb[2 * r], d->A.rp + hs[r], sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        DCK(d, cudaMemcpyAsync(&hb[2 * r + 1], d->A.rp + hs[r + 1], sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      }
      DCK(d, cudaStreamSynchronize(s));
      DCK(d, cudaMemcpyAsync(bounds, hb.data(), 2 * P * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    }
    NCK(d, ncclBroadcast(bounds, bounds, 2 * P, ncclInt64, 0, d->comm, s));
    std::vector<int64_t> hb(2 * P);
    DCK(d, cudaMemcpyAsync(hb.data(), bounds, 2 * P * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DCK(d, cudaStreamSynchronize(s));
    if (R == 0) {
      d->Al = CsrView{d->A.rp + d->row_begin, d->A.ci, d->A.val};
      NCK(d, ncclGroupStart());
      for (int r = 1; r < P; ++r) {
        const int64_t nr = hs[r + 1] - hs[r];
        const int64_t e0 = hb[2 * r], e1 = hb[2 * r + 1];
        NCK(d, ncclSend(d->A.rp + hs[r], nr + 1, ncclInt64, r, d->comm, s));
        if (e1 > e0) {
          NCK(d, ncclSend(d->A.ci + e0, e1 - e0, ncclInt32, r, d->comm, s));
          NCK(d, ncclSend(d->A.val + e0, e1 - e0, ncclFloat64, r, d->comm, s));
        }
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
      if (e1 > e0) {
        NCK(d, ncclRecv(ci, e1 - e0, ncclInt32, 0, d->comm, s));
        NCK(d, ncclRecv(v, e1 - e0, ncclFloat64, 0, d->comm, s));
      }
      NCK(d, ncclGroupEnd());
      k_add_offset<<<(unsigned)((ml + 1 + 255) / 256), 256, 0, s>>>(rp, ml + 1, -e0);
      DCK(d, cudaGetLastError());
      d->Al = CsrView{rp, ci, v};
    }
  }
  // --- 4. local four-stage SpGEMM ---------------------------------------------------------
  spgemm_status_t st = spgemm_create(&d->local, ml, d->k, d->n, d->Al.rp, d->Al.ci, d->Al.val,
                                     0 /* unused by the kernels */, d->Bl.rp, d->Bl.ci, d->Bl.val,
                                     d->b_nnz, s, d->flags & (SPGEMM_FLAG_PRECISE | SPGEMM_FLAG_UPPER_BOUND));
  if (st != SPGEMM_SUCCESS) return dfail(d, st, std::string("local create: ") + spgemm_last_error(nullptr));
  int64_t lnnz = 0;
  st = spgemm_symbolic(d->local, &lnnz);
  if (st != SPGEMM_SUCCESS) return dfail(d, st, std::string("local symbolic: ") + spgemm_last_error(d->local));
  // --- 5. stitch: allgather per-rank nnz ------------------------------------------------
  DCK(d, cudaMemcpyAsync(nnzs + R, &lnnz, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  NCK(d, ncclAllGather(nnzs + R, nnzs, 1, ncclInt64, d->comm, s));
  std::vector<int64_t> hn(P);
  DCK(d, cudaMemcpyAsync(hn.data(), nnzs, P * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DCK(d, cudaStreamSynchronize(s));
  int64_t off = 0, tot = 0;
  for (int r = 0; r < P; ++r) {
    if (r < R) off += hn[r];
    tot += hn[r];
  }
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
  spgemm_status_t st = spgemm_numeric(d->local, c_row_ptr, c_col_idx, c_val);
  if (st != SPGEMM_SUCCESS) return dfail(d, st, std::string("local numeric: ") + spgemm_last_error(d->local));
  const int64_t ml = d->row_end - d->row_begin;
  if (d->offset != 0) {
    k_add_offset<<<(unsigned)((ml + 1 + 255) / 256), 256, 0, d->stream>>>(c_row_ptr, ml + 1, d->offset);
    DCK(d, cudaGetLastError());
  }
  return SPGEMM_SUCCESS;
}

}  // extern "C"

// Called from spgemm_destroy/get_stats/last_error when handed a dist handle.
spgemm_status_t sg_dist_destroy(spgemm_handle_t h) {
  spgemm_dist_s* d = as_dist(h);
  if (!d) return SPGEMM_ERROR_INVALID_VALUE;
  if (d->local) spgemm_destroy(d->local);
  for (void* p : d->mem) cudaFreeAsync(p, d->stream);
  cudaStreamSynchronize(d->stream);
  if (d->comm) ncclCommDestroy(d->comm);
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
