// long.cu — stage 3 for rows too long for one shared-memory table: the paper's bin group 5
// with its progressive allocation ([P:222], [P:286-297]).
//
// Paper: each group-5 row starts with a fixed C~ capacity (256, [P:224]); when the
// partial result plus the next input sequence would exceed the allocation, "our method
// records current computation position as a checkpoint and dumps the resulting sequence
// ... Then the host allocates more global memory (we use 2x each time) and re-launches
// kernel ... The relaunched kernels obtain checkpoint information, and load existing
// results ... and continue the computation" [P:297].
//
// Here (a4/a5): one CTA per long row accumulates into an order-preserving
// hash table in global memory with nominal capacity `cap` (2·cap slots).  A batch of a_ij is
// taken only if its products fit the free slots (so it always completes); after a batch
// whose distinct count passed `cap` — or if not even one a_ij fits — the CTA records the
// checkpoint (index of the next a_ij, [P:297]) and exits.
// The host grows cap to min(2·cap, min(u_i, n)) (never above the upper bound, reading Q8),
// allocates the new tables and relaunches only the overflowed rows; the relaunched CTA
// reloads the old table and resumes at the checkpoint.  At cap = min(u_i, n) no check is
// needed (nnz(c_i*) <= min(u_i, n)).  A finished row is cluster-sorted and compacted in
// place, so its table's front holds the sorted row for stage 4.
#include <climits>

#include "common.cuh"

namespace sg {

namespace {

constexpr int kLongNT = 512;

__global__ void k_long_init(LongState* st, const int32_t* __restrict__ perm, int64_t first,
                            int64_t nlong, const int64_t* __restrict__ U, int64_t n, int64_t cap0,
                            CsrView A, CsrView B) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;  // warp per row
  if (k >= nlong) return;
  const int row = perm[first + k];
  const int64_t a0 = A.rp[row], a1 = A.rp[row + 1];
  int lo = INT_MAX, hi = -1;
  for (int64_t e = a0 + lane; e < a1; e += 32) {
    const int j = A.ci[e];
    const int64_t bs = B.rp[j], be = B.rp[j + 1];
    if (be > bs) {
      lo = min(lo, B.ci[bs]);
      hi = max(hi, B.ci[be - 1]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) {
    const int64_t u = U[row];
    const int64_t capmax = u < n ? u : n;
    LongState s;
    s.next_a = a0;
    s.capmax = capmax;
    s.cap = cap0 < capmax ? cap0 : capmax;
    if (s.cap < 1) s.cap = 1;
    s.count = 0;
    s.lo = lo;
    s.hi = hi;
    s.done = 0;
    s.pad = 0;
    st[k] = s;
  }
}

__global__ void k_long_grow(LongState* st, const int32_t* __restrict__ list, int64_t nlist,
                            int64_t* __restrict__ slots_out, int64_t* __restrict__ old_slots) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nlist) return;
  const int k = list[i];
  old_slots[k] = long_table_slots(st[k].cap);
  int64_t c = st[k].cap * 2;                  // "we use 2x each time" [P:297]
  if (c > st[k].capmax) c = st[k].capmax;     // never above min(u_i, n) (reading Q8)
  st[k].cap = c;
  slots_out[i] = long_table_slots(c);
}

__global__ void k_long_assign(const int32_t* __restrict__ list, int64_t nlist,
                              const int64_t* __restrict__ slot_off, int32_t* keys_base,
                              double* vals_base, int32_t** keys, double** vals,
                              int32_t** old_keys, double** old_vals, int64_t* old_slots,
                              const LongState* st) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nlist) return;
  const int k = list[i];
  if (old_keys) {
    old_keys[k] = keys[k];
    old_vals[k] = vals[k];
  }
  (void)old_slots;
  (void)st;
  keys[k] = keys_base + slot_off[i];
  vals[k] = vals_base ? vals_base + slot_off[i] : nullptr;
}

template <int NT>
__device__ __forceinline__ int64_t block_incl_scan64(int64_t v, int64_t* s_w, int64_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int64_t x = lane < NT / 32 ? s_w[lane] : 0;
    int64_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < NT / 32) s_w[lane] = xi - x;
    if (lane == 31) s_w[NT / 32] = xi;
  }
  __syncthreads();
  const int64_t r = inc + s_w[w];
  *total = s_w[NT / 32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ int64_t home_of(int c, int lo, double scale, int64_t spread) {
  int64_t h = (int64_t)__dmul_rz((double)(c - lo), scale);  // monotone in c
  return h < spread - 1 ? h : spread - 1;
}

// Insert key c into the global order-preserving table of S slots; returns its slot.  A probe
// run past the end wraps to slot 0 and flags the row (ordering then takes the robust path).
__device__ __forceinline__ int64_t gt_insert(int32_t* keys, int c, int64_t h, int64_t S, int& isnew,
                                             int& wrapped) {
  while (true) {
    const int k = __ldcg(keys + h);
    if (k == c) {
      isnew = 0;
      return h;
    }
    if (k == kEmptyKey) {
      const int old = atomicCAS(keys + h, kEmptyKey, c);
      if (old == kEmptyKey) {
        isnew = 1;
        return h;
      }
      if (old == c) {
        isnew = 0;
        return h;
      }
    }
    if (++h == S) {
      h = 0;
      wrapped = 1;
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_long(LongArgs a) {
  constexpr int NW = NT / 32;
  __shared__ int64_t s_w[NW + 1];
  __shared__ int64_t s_bs[NT];
  __shared__ int32_t s_len[NT];
  __shared__ double s_av[NT];
  __shared__ int s_take;
  __shared__ unsigned long long s_ins;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool fill = a.mode == MODE_FILL;
  const int k = a.active[blockIdx.x];
  const int row = a.perm[a.first + k];
  LongState st = a.st[k];
  int32_t* keys = a.keys[k];
  double* vals = fill ? a.vals[k] : nullptr;
  const int64_t S = long_table_slots(st.cap);
  const int64_t W = int64_t(st.hi) - st.lo + 1;
  // homes spread over the table (load <= 1/2 keeps clusters short for scattered columns)
  const int64_t spread = S - 64 > S / 2 ? S - 64 : S / 2;
  const double scale = W <= spread ? 1.0 : (double)spread / (double)W;
  __shared__ int s_slow;
  if (threadIdx.x == 0) s_slow = 0;
  int wrapped = 0;

  for (int64_t s = threadIdx.x; s < S; s += NT) {
    __stcg(keys + s, kEmptyKey);
    if (fill) __stcg(vals + s, 0.0);
  }
  __syncthreads();
  // reload the previous (smaller) table after a re-allocation ([P:297] "load existing results")
  if (a.old_keys && a.old_keys[k]) {
    const int32_t* ok = a.old_keys[k];
    const double* ov = fill ? a.old_vals[k] : nullptr;
    const int64_t os = a.old_slots[k];
    for (int64_t s = threadIdx.x; s < os; s += NT) {
      const int c = __ldcg(ok + s);
      if (c == kEmptyKey) continue;
      int isnew;
      const int64_t h = gt_insert(keys, c, home_of(c, st.lo, scale, spread), S, isnew, wrapped);
      if (fill) __stcg(vals + h, __ldcg(ov + s));
    }
    __syncthreads();
  }
  int64_t count = st.count;
  int64_t e = st.next_a;
  const int64_t a1 = a.A.rp[row + 1];
  const bool unbounded = st.cap >= st.capmax;
  bool overflow = false;
  while (e < a1) {
    // stage a batch of up to NT a_ij whose products fit the remaining capacity
    const int64_t ee = e + threadIdx.x;
    int32_t len = 0;
    if (ee < a1) {
      const int j = a.A.ci[ee];
      const int64_t bs = a.B.rp[j];
      len = (int32_t)(a.B.rp[j + 1] - bs);
      s_bs[threadIdx.x] = bs;
      s_len[threadIdx.x] = len;
      s_av[threadIdx.x] = fill ? a.A.val[ee] : 0.0;
    }
    int64_t tot;
    const int64_t inc = block_incl_scan64<NT>(len, s_w, &tot);
    // physical safety: the table has 2·cap slots, so a batch whose products cannot exceed
    // the free slots always completes; the nominal capacity (load 1/2) is checked after it
    const int64_t budget = unbounded ? INT64_MAX : 2 * st.cap - count - 1;
    const int fits = (ee < a1) && inc <= budget;
    const int take = __syncthreads_count(fits);
    if (take == 0) {
      overflow = true;  // checkpoint: next a_ij = e, partial result stays in the table
      break;
    }
    if (threadIdx.x == 0) s_ins = 0;
    __syncthreads();
    unsigned ins = 0;
    for (int t = w; t < take; t += NW) {
      const int64_t jb = s_bs[t];
      const int32_t jl = s_len[t];
      const double at = s_av[t];
      for (int q = lane; q < jl; q += 32) {
        const int c = __ldg(a.B.ci + jb + q);
        int isnew;
        const int64_t h = gt_insert(keys, c, home_of(c, st.lo, scale, spread), S, isnew, wrapped);
        ins += isnew;
        if (fill) atomicAdd(vals + h, __dmul_rn(at, __ldg(a.B.val + jb + q)));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ins += __shfl_xor_sync(0xffffffffu, ins, o);
    if (lane == 0) atomicAdd(&s_ins, (unsigned long long)ins);
    __syncthreads();
    count += (int64_t)s_ins;
    e += take;
    __syncthreads();
    if (!unbounded && count > st.cap && e < a1) {
      overflow = true;  // over the nominal capacity: checkpoint here, grow 2x, resume ([P:297])
      break;
    }
  }
  if (overflow) {
    if (threadIdx.x == 0) {
      a.st[k].next_a = e;
      a.st[k].count = count;
      const int pos = atomicAdd(a.overflow_cnt, 1);
      a.overflow_list[pos] = k;
    }
    return;
  }
  if (threadIdx.x == 0) {
    a.st[k].next_a = e;
    a.st[k].count = count;
    a.st[k].done = 1;
    if (a.nnz_row) a.nnz_row[row] = count;
  }
  if (!fill) return;
  if (wrapped) s_slow = 1;
  __threadfence_block();
  __syncthreads();
  if (!s_slow) {
    // order clusters (maximal runs of occupied slots) by insertion sort; a wrapped table or a
    // long cluster (clustered columns) sends the row to the robust path
    const int64_t chunk = (S + NT - 1) / NT;
    const int64_t s0 = int64_t(threadIdx.x) * chunk;
    const int64_t s1 = s0 + chunk < S ? s0 + chunk : S;
    for (int64_t s = s0; s < s1; ++s) {
      if (__ldcg(keys + s) == kEmptyKey || (s > 0 && __ldcg(keys + s - 1) != kEmptyKey)) continue;
      int64_t end = s + 1;
      while (end < S && __ldcg(keys + end) != kEmptyKey && end - s <= 128) ++end;
      if (end - s > 128) {
        s_slow = 1;
        break;
      }
      for (int64_t x = s + 1; x < end; ++x) {
        const int kx = __ldcg(keys + x);
        const double vx = __ldcg(vals + x);
        int64_t y = x - 1;
        while (y >= s && __ldcg(keys + y) > kx) {
          __stcg(keys + y + 1, __ldcg(keys + y));
          __stcg(vals + y + 1, __ldcg(vals + y));
          --y;
        }
        __stcg(keys + y + 1, kx);
        __stcg(vals + y + 1, vx);
      }
    }
    __threadfence_block();
    __syncthreads();
  }
  // in-place ordered compaction to the front of the table
  int64_t base = 0;
  for (int64_t r0 = 0; r0 < S; r0 += NT) {
    const int64_t s = r0 + threadIdx.x;
    int c = kEmptyKey;
    double v = 0.0;
    if (s < S) {
      c = __ldcg(keys + s);
      v = __ldcg(vals + s);
    }
    const bool occ = c != kEmptyKey;
    int64_t tot;
    const int64_t pos = block_incl_scan64<NT>(occ ? 1 : 0, s_w, &tot) - (occ ? 1 : 0);
    if (occ) {
      __stcg(keys + base + pos, c);
      __stcg(vals + base + pos, v);
    }
    base += tot;
    __threadfence_block();
    __syncthreads();
  }
  if (s_slow) {
    // robust path: bitonic sort of the compacted (key, value) pairs in place
    int64_t N = 1;
    while (N < count) N <<= 1;
    for (int64_t t = count + threadIdx.x; t < N && t < S; t += NT) __stcg(keys + t, INT_MAX);
    __threadfence_block();
    __syncthreads();
    for (int64_t kk = 2; kk <= N; kk <<= 1) {
      for (int64_t j = kk >> 1; j > 0; j >>= 1) {
        for (int64_t i = threadIdx.x; i < (N >> 1); i += NT) {
          const int64_t l0 = ((i & ~(j - 1)) << 1) | (i & (j - 1));
          const int64_t l1 = l0 + j;
          const bool asc = (l0 & kk) == 0;
          const int k0 = __ldcg(keys + l0), k1 = __ldcg(keys + l1);
          if ((k0 > k1) == asc) {
            __stcg(keys + l0, k1);
            __stcg(keys + l1, k0);
            const double t0 = __ldcg(vals + l0);
            __stcg(vals + l0, __ldcg(vals + l1));
            __stcg(vals + l1, t0);
          }
        }
        __threadfence_block();
        __syncthreads();
      }
    }
  }
}

}  // namespace

cudaError_t launch_long_init(LongState* st, const int32_t* perm, int64_t first, int64_t nlong,
                             const int64_t* U, int64_t n, int64_t cap0, CsrView A, CsrView B,
                             cudaStream_t s) {
  if (nlong == 0) return cudaSuccess;
  const int64_t threads = nlong * 32;
  k_long_init<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(st, perm, first, nlong, U, n, cap0, A, B);
  return cudaGetLastError();
}

cudaError_t launch_long(const LongArgs& a, cudaStream_t s) {
  if (a.nactive == 0) return cudaSuccess;
  k_long<kLongNT><<<(unsigned)a.nactive, kLongNT, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_long_grow(LongState* st, const int32_t* list, int64_t nlist, int64_t* slots_out,
                             int64_t* old_slots, cudaStream_t s) {
  if (nlist == 0) return cudaSuccess;
  k_long_grow<<<(unsigned)((nlist + 255) / 256), 256, 0, s>>>(st, list, nlist, slots_out, old_slots);
  return cudaGetLastError();
}

cudaError_t launch_long_assign(const int32_t* list, int64_t nlist, const int64_t* slot_off,
                               int32_t* keys_base, double* vals_base, int32_t** keys,
                               double** vals, int32_t** old_keys, double** old_vals,
                               int64_t* old_slots, const LongState* st, cudaStream_t s) {
  if (nlist == 0) return cudaSuccess;
  k_long_assign<<<(unsigned)((nlist + 255) / 256), 256, 0, s>>>(list, nlist, slot_off, keys_base,
                                                                vals_base, keys, vals, old_keys,
                                                                old_vals, old_slots, st);
  return cudaGetLastError();
}

}  // namespace sg
