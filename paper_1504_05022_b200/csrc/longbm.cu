// longbm.cu — PRECISE strategy, long rows: a bitmap over the row's column window.
//
// The precise method ([P:165]) first computes the structure, then the values.  For rows too
// long for a shared-memory hash (the paper's group 5, [P:222]) the structure of row i is
// the set of columns hit by its products: one bit per column of the window [lo, hi] in
// shared memory, processed in tiles of kTileBits columns.
//   k_long_bm_count : per tile, set the bits of all products' columns (atomicOr), count them.
//                     nnz(c_i*) = total popcount.  No hashing, no probing, no ordering.
//   k_long_bm_fill  : per tile, rebuild the bits, exclusive prefix popcount per 32-bit word
//                     → rank(c) = prefix[w] + popc(bits[w] & below(c)) is c's position in the
//                     sorted row; write C's columns in order, zero the values, then add every
//                     product into C.val[row_start + rank] (global fp64 atomics, order not
//                     fixed: checked with the 1e-12·Σ|a||b| tolerance, R1).
#include <climits>

#include "common.cuh"

namespace sg {

namespace {

constexpr int kBmNT = 512;
constexpr int kTileWords = 32768;                 // 1 Mi columns per tile (192 KB with prefix)
constexpr int kChunk = 256;                       // products per work item (load balance)
constexpr int64_t kTileBits = int64_t(kTileWords) * 32;

template <int NT>
__device__ __forceinline__ int block_excl_scan_i(int v, int* total, int* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int x = lane < NT / 32 ? s_w[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < NT / 32) s_w[lane] = xi - x;
    if (lane == 31) s_w[NT / 32] = xi;
  }
  __syncthreads();
  const int ex = inc - v + s_w[w];
  *total = s_w[NT / 32];
  __syncthreads();
  return ex;
}

// the row's column window: first / last column of every b_j*
__device__ __forceinline__ void row_window(const Stage3Args& a, int64_t a0, int64_t a1, int* s_red,
                                           int& lo, int& hi) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int l = INT_MAX, h = -1;
  for (int64_t e = a0 + threadIdx.x; e < a1; e += blockDim.x) {
    const int j = __ldg(a.A.ci + e);
    const int64_t bs = __ldg(a.B.rp + j), be = __ldg(a.B.rp + j + 1);
    if (be > bs) {
      l = min(l, __ldg(a.B.ci + bs));
      h = max(h, __ldg(a.B.ci + be - 1));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l = min(l, __shfl_xor_sync(0xffffffffu, l, o));
    h = max(h, __shfl_xor_sync(0xffffffffu, h, o));
  }
  if (lane == 0) {
    s_red[2 * w] = l;
    s_red[2 * w + 1] = h;
  }
  __syncthreads();
  lo = INT_MAX;
  hi = -1;
  for (int k = 0; k < (int)(blockDim.x / 32); ++k) {
    lo = min(lo, s_red[2 * k]);
    hi = max(hi, s_red[2 * k + 1]);
  }
  __syncthreads();
}

// Visit every product of row [a0, a1) with a balanced schedule: a_ij are taken NT at a time,
// each b_j* is cut into kChunk-product work items, and warps take work items round-robin
// (hub rows of B no longer leave the other warps of the CTA waiting at the barrier).
struct BmBatch {
  long long bs[kBmNT];
  int len[kBmNT];
  int cinc[kBmNT];  // inclusive scan of work items per a_ij
  double av[kBmNT];
};

template <bool VALS, typename F>
__device__ __forceinline__ void for_each_product(const Stage3Args& a, int64_t a0, int64_t a1, BmBatch& sb,
                                                 int* s_w, F&& f) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = kBmNT / 32;
  for (int64_t e0 = a0; e0 < a1; e0 += kBmNT) {
    const int64_t e = e0 + threadIdx.x;
    int len = 0;
    if (e < a1) {
      const int j = __ldg(a.A.ci + e);
      const int64_t bs = __ldg(a.B.rp + j);
      len = (int)(__ldg(a.B.rp + j + 1) - bs);
      sb.bs[threadIdx.x] = bs;
      sb.len[threadIdx.x] = len;
      if (VALS) sb.av[threadIdx.x] = __ldg(a.A.val + e);
    }
    const int nch = (len + kChunk - 1) / kChunk;
    int tot;
    const int ex = block_excl_scan_i<kBmNT>(nch, &tot, s_w);
    sb.cinc[threadIdx.x] = ex + nch;
    __syncthreads();
    for (int item = w; item < tot; item += NW) {
      int lo = 0, hi = kBmNT - 1;  // first t with cinc[t] > item
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sb.cinc[mid] > item) hi = mid;
        else lo = mid + 1;
      }
      const int t = lo;
      const int first_item = sb.cinc[t] - (sb.len[t] + kChunk - 1) / kChunk;
      const int64_t q0 = sb.bs[t] + int64_t(item - first_item) * kChunk;
      const int64_t qe = min(q0 + kChunk, (int64_t)sb.bs[t] + sb.len[t]);
      const double at = VALS ? sb.av[t] : 0.0;
      for (int64_t q = q0 + lane; q < qe; q += 32) f(q, at);
    }
    __syncthreads();
  }
}

// Long rows differ by orders of magnitude in work (c3b: 8 Ki to 2.5 Mi products): CTAs take
// their next row from a global counter instead of a fixed stride.
__device__ __forceinline__ int64_t next_row(const Stage3Args& a, int64_t r, int64_t* s_next) {
  if (!a.work_ctr) return r + gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) *s_next = int64_t(gridDim.x) + atomicAdd(a.work_ctr, 1);
  __syncthreads();
  return *s_next;
}

__global__ void __launch_bounds__(kBmNT) k_long_bm_count(Stage3Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* bm = reinterpret_cast<unsigned*>(smem);
  __shared__ int s_red[2 * (kBmNT / 32)];
  __shared__ int s_w[kBmNT / 32 + 1];
  __shared__ BmBatch sb;
  __shared__ unsigned long long s_cnt;
  __shared__ int64_t s_next;
  for (int64_t r = blockIdx.x; r < a.count; r = next_row(a, r, &s_next)) {
    const int row = __ldg(a.perm + a.first + r);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    int lo, hi;
    row_window(a, a0, a1, s_red, lo, hi);
    if (threadIdx.x == 0) s_cnt = 0;
    // tile: the row's window, at most kTileBits columns, in multiples of kBmNT words
    const int64_t wwords = (int64_t(hi) - lo) / 32 + 1;
    const int64_t tmax = (((a.n + 31) / 32 + 1 + kBmNT - 1) / kBmNT * kBmNT) < kTileWords
                             ? (((a.n + 31) / 32 + 1 + kBmNT - 1) / kBmNT * kBmNT) : kTileWords;
    const int tw = (int)((wwords < tmax ? wwords : tmax) + kBmNT - 1) / kBmNT * kBmNT;
    const int64_t tbits = int64_t(tw) * 32;
    for (int64_t base = lo; base <= hi; base += tbits) {
      for (int k = threadIdx.x; k < tw; k += kBmNT) bm[k] = 0u;
      __syncthreads();
      for_each_product<false>(a, a0, a1, sb, s_w, [&](int64_t q, double) {
        const int64_t d = int64_t(__ldg(a.B.ci + q)) - base;
        if (d >= 0 && d < tbits) atomicOr(&bm[d >> 5], 1u << (d & 31));  // line 8: insert
      });
      unsigned c = 0;
      for (int k = threadIdx.x; k < tw; k += kBmNT) c += __popc(bm[k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt, (unsigned long long)c);
      __syncthreads();
    }
    if (threadIdx.x == 0 && a.nnz_row) a.nnz_row[row] = (int64_t)s_cnt;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBmNT) k_long_bm_fill(Stage3Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* bm = reinterpret_cast<unsigned*>(smem);
  const int64_t tmax0 = (((a.n + 31) / 32 + 1 + kBmNT - 1) / kBmNT * kBmNT) < kTileWords
                            ? (((a.n + 31) / 32 + 1 + kBmNT - 1) / kBmNT * kBmNT) : kTileWords;
  int* pre = reinterpret_cast<int*>(smem + size_t(tmax0) * sizeof(unsigned));
  __shared__ int s_red[2 * (kBmNT / 32)];
  __shared__ int s_w[kBmNT / 32 + 1];
  __shared__ BmBatch sb;
  __shared__ int64_t s_next;
  for (int64_t r = blockIdx.x; r < a.count; r = next_row(a, r, &s_next)) {
    const int row = __ldg(a.perm + a.first + r);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    const int64_t o = __ldg(a.out_off + row);
    int lo, hi;
    row_window(a, a0, a1, s_red, lo, hi);
    const int64_t wwords = (int64_t(hi) - lo) / 32 + 1;
    const int64_t tmax = (((a.n + 31) / 32 + 1 + kBmNT - 1) / kBmNT * kBmNT) < kTileWords
                             ? (((a.n + 31) / 32 + 1 + kBmNT - 1) / kBmNT * kBmNT) : kTileWords;
    const int tw = (int)((wwords < tmax ? wwords : tmax) + kBmNT - 1) / kBmNT * kBmNT;
    const int64_t tbits = int64_t(tw) * 32;
    const int WPT = tw / kBmNT;  // words per thread in the prefix scan
    int64_t done = 0;  // entries of the row already placed by earlier tiles
    for (int64_t base = lo; base <= hi; base += tbits) {
      for (int k = threadIdx.x; k < tw; k += kBmNT) bm[k] = 0u;
      __syncthreads();
      for_each_product<false>(a, a0, a1, sb, s_w, [&](int64_t q, double) {
        const int64_t d = int64_t(__ldg(a.B.ci + q)) - base;
        if (d >= 0 && d < tbits) atomicOr(&bm[d >> 5], 1u << (d & 31));  // line 8: insert
      });
      // exclusive prefix popcount over the tile's words (thread t owns words [t·WPT, +WPT))
      int loc = 0;
      for (int k = 0; k < WPT; ++k) loc += __popc(bm[threadIdx.x * WPT + k]);
      int tot;
      int run = block_excl_scan_i<kBmNT>(loc, &tot, s_w);
      for (int k = 0; k < WPT; ++k) {
        const int wi = threadIdx.x * WPT + k;
        const unsigned bits = bm[wi];
        if ((wi & 1) == 0) pre[wi >> 1] = run;
        // C's columns of this tile, in order, and zeroed values
        unsigned b = bits;
        int p = run;
        while (b) {
          const int bit = __ffs(b) - 1;
          b &= b - 1;
          a.out_col[o + done + p] = (int)(base + int64_t(wi) * 32 + bit);
          a.out_val[o + done + p] = 0.0;
          ++p;
        }
        run += __popc(bits);
      }
      __threadfence();
      __syncthreads();
      // values: every product of a column in this tile adds into its rank (line 11)
      for_each_product<true>(a, a0, a1, sb, s_w, [&](int64_t q, double at) {
        const int64_t d = int64_t(__ldg(a.B.ci + q)) - base;
        if (d >= 0 && d < tbits) {
          const int wi = (int)(d >> 5);
          const unsigned below = (1u << (d & 31)) - 1u;
          const int rank = pre[wi >> 1] + ((wi & 1) ? __popc(bm[wi - 1]) : 0) + __popc(bm[wi] & below);
          atomicAdd(a.out_val + o + done + rank, __dmul_rn(at, __ldg(a.B.val + q)));
        }
      });
      done += tot;
      __syncthreads();
    }
    __syncthreads();
  }
}

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace

cudaError_t launch_long_bitmap(const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  const bool fill = a.mode == MODE_FILL;
  if (a.work_ctr) {
    cudaError_t e0 = cudaMemsetAsync(a.work_ctr, 0, sizeof(int), s);
    if (e0 != cudaSuccess) return e0;
  }
  // tiles never exceed the column range [0, n): size shared memory by it (c3b: 8 Ki words)
  const int64_t nwords = ((a.n + 31) / 32 + 1 + kBmNT - 1) / kBmNT * kBmNT;
  const int64_t tw = nwords < kTileWords ? nwords : kTileWords;
  const size_t sm = size_t(tw) * (fill ? 6 : 4);
  auto kern = fill ? k_long_bm_fill : k_long_bm_count;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBmNT, sm);
  if (per_sm < 1) per_sm = 1;
  // fill: at most two CTAs per SM keep the rows being accumulated (fp64 atomics into C) plus
  // B resident in L2; more concurrent rows thrash it (c3b: 1 CTA 88 ms, 2 CTAs 76, 3 CTAs 81)
  if (fill && per_sm > 2) per_sm = 2;
  int64_t grid = int64_t(sm_count()) * per_sm;
  if (grid > a.count) grid = a.count;
  kern<<<(unsigned)grid, kBmNT, sm, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sg
