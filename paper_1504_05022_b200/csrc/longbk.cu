// longbk.cu — values of long rows whose column window is wider than one bitmap tile
// (precise numeric; the paper's group 5 [P:222], [P:286-297]).
//
// The rank kernel (longbm.cu) walks every a_ij of the row once per tile of the window and
// splits each b_j* over eight warp-owned rank ranges: on a window of 4 Mi columns (R-MAT
// scale 22) that is 16 tiles x 8 owners, about one product per owner per a_ij.  Here the row's
// products are instead partitioned once, in Algorithm-1 order, by column range ("bucket"), and
// each bucket is sorted on its own — the ESC of the paper's group 4 ([P:277-284]: expand,
// sort, compress) applied to column ranges of one row:
//
//   k_bk_part  CTA per row (rows taken from a global counter).  Buckets: (c - lo) >> sh, with
//              about kBkTarget products each (bk_shape).  Warp w owns a contiguous range of
//              the row's a_ij.  Pass 1 counts the products per (bucket, warp); their scan gives
//              every (bucket, warp) its first slot, so pass 2 writes each product
//              (c, a_ij·b_jk) (line 6 of Algorithm 1) to the row's staging area with the items
//              of every bucket in product order (j ascending, then k): a stable partition.
//              Within one warp step the lanes hold one b_j*'s sorted columns, so the lanes of
//              a bucket form one run: rank = lane - run start, no atomics.
//   k_bk_sort  CTA per bucket: the bucket's products sorted by (column, p) (esc_sort.cuh:
//              counting pass into ~32-product sub-buckets, warp bitonic sorts), runs of equal
//              columns summed left to right (lines 9, 11: the oracle's order, bit for bit,
//              DESIGN.md R1); the distinct entries overwrite the bucket's items.
//   k_bk_copy  CTA per row: scan of its buckets' distinct counts, copy into C at row_ptr.
// Rows that do not qualify (bk_eligible) or whose largest bucket exceeds kBkCap go to the
// rank kernel (fallback list).
#include "common.cuh"
#include "walk.cuh"
#include "esc_sort.cuh"

namespace sg {

namespace {

using walk::kFull;
using walk::walk_row;

constexpr int kPNT = 256;            // k_bk_part
constexpr int kPNW = kPNT / 32;
constexpr int kSNT = 256;            // k_bk_sort (kBkCap items per bucket)
constexpr int kCNT = 256;            // k_bk_copy

__device__ __forceinline__ unsigned lanemask_le_() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

template <int NT>
__device__ __forceinline__ int bk_block_excl_scan(int v, int* total, int* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int x = lane < NT / 32 ? s_w[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, xi, o);
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

// ------------------------------------------------------------------------------- partition
template <typename IT, typename V>
__global__ void __launch_bounds__(kPNT) k_bk_part(Stage3Args a, BkWork bw) {
  __shared__ int s_cur[kBkMaxBuckets][kPNW];  // counts, then the (bucket, warp) write cursors
  __shared__ int s_w[kPNW + 1];
  __shared__ int s_ovf;
  __shared__ long long s_P, s_D;
  __shared__ int64_t s_next;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned le = lanemask_le_();
  V* sval = vcast<V>(bw.stg_val);

  for (int64_t r = blockIdx.x; r < a.count;) {
    const int row = __ldg(a.perm + a.first + r);
    const int lo = __ldg(a.rlo + row);
    const int64_t W = int64_t(__ldg(a.rhi + row)) - lo + 1;
    const int64_t u = __ldg(a.U + row);
    if (!bk_eligible(u, W, bw.min_w)) {
      if (tid == 0) bw.fb_list[atomicAdd(bw.cur32 + 1, 1)] = row;
    } else {
      int sh, nbk;
      bk_shape(u, W, sh, nbk);
      const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
      const int64_t na = a1 - a0;
      const int64_t e0 = a0 + na * wid / kPNW, e1 = a0 + na * (wid + 1) / kPNW;  // this warp's a_ij
      for (int b = tid; b < nbk; b += kPNT)
#pragma unroll
        for (int w = 0; w < kPNW; ++w) s_cur[b][w] = 0;
      if (tid == 0) s_ovf = 0;
      __syncthreads();
      // pass 1: products per (bucket, warp)
      walk_row<false, IT, V>(a, e0, e1, lane, [&](int c, V, V, bool act) {
        if (act) atomicAdd(&s_cur[(unsigned)(c - lo) >> sh][wid], 1);
      });
      __syncthreads();
      // bucket sizes and starts (thread t: buckets 2t, 2t+1); cursor of (b, w) = start_b +
      // the products of warps < w in bucket b
      int sz[2] = {0, 0};
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int b = 2 * tid + q;
        if (b < nbk)
#pragma unroll
          for (int w = 0; w < kPNW; ++w) sz[q] += s_cur[b][w];
      }
      int tot;
      const int st0 = bk_block_excl_scan<kPNT>(sz[0] + sz[1], &tot, s_w);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int b = 2 * tid + q;
        if (b < nbk) {
          int cur = st0 + (q ? sz[0] : 0);
#pragma unroll
          for (int w = 0; w < kPNW; ++w) {
            const int x = s_cur[b][w];
            s_cur[b][w] = cur;
            cur += x;
          }
          if (sz[q] > kBkCap) s_ovf = 1;
        }
      }
      __syncthreads();
      if (s_ovf) {
        if (tid == 0) bw.fb_list[atomicAdd(bw.cur32 + 1, 1)] = row;
      } else {
        if (tid == 0) {
          s_P = (long long)atomicAdd(bw.cur64 + 0, (unsigned long long)u);
          s_D = (long long)atomicAdd(bw.cur64 + 1, (unsigned long long)nbk);
          bw.rows[atomicAdd(bw.cur32 + 0, 1)] = BkRow{row, nbk, (int64_t)s_D};  // buckets [D, D + nbk)
        }
        __syncthreads();
        const int64_t P = s_P, D = s_D;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int b = 2 * tid + q;
          if (b < nbk) {
            BkDesc d;
            d.off = P + st0 + (q ? sz[0] : 0);
            d.size = sz[q];
            d.blo = lo + (b << sh);
            d.sh = sh;
            d.uniq = 0;
            bw.desc[D + b] = d;
          }
        }
        // pass 2: write every product at its slot (stable within each bucket)
        walk_row<true, IT, V>(a, e0, e1, lane, [&](int c, V v, V at, bool act) {
          const unsigned b = act ? (unsigned)(c - lo) >> sh : 0xffffffe0u + lane;  // idle: unique
          const unsigned bp = __shfl_up_sync(kFull, b, 1);
          const unsigned S = __ballot_sync(kFull, lane == 0 || bp != b);  // run starts
          const int rs = 31 - __clz(S & le);
          const int pos = act ? s_cur[b][wid] + (lane - rs) : 0;
          __syncwarp();
          if (act && lane == rs) {
            const unsigned nx = S & ~le;
            s_cur[b][wid] += (nx ? __ffs(nx) - 1 : 32) - lane;
          }
          __syncwarp();
          if (act) {
            bw.stg_col[P + pos] = c;
            sval[P + pos] = Arith<V>::mul(at, v);  // line 6
          }
        });
      }
    }
    // next row: dynamic (long rows differ by orders of magnitude in work)
    __syncthreads();
    if (tid == 0) s_next = int64_t(gridDim.x) + atomicAdd(a.work_ctr, 1);
    __syncthreads();
    r = s_next;
  }
}

// ------------------------------------------------------------------------------- bucket sort
template <typename V>
__global__ void __launch_bounds__(kSNT) k_bk_sort(BkWork bw) {
  using SM = escs::Smem<kBkCap, V>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x;
  V* sv = vcast<V>(bw.stg_val);
  const int64_t nd = (int64_t)bw.cur64[1];
  for (int64_t d = blockIdx.x; d < nd; d += gridDim.x) {
    const BkDesc D = bw.desc[d];
    const int n = D.size;
    for (int i = tid; i < n; i += kSNT) {  // the bucket's products, in product order
      sm.key[i] = (unsigned)(bw.stg_col[D.off + i] - D.blo);
      sm.pval[i] = sv[D.off + i];
    }
    __syncthreads();
    // sort by (column, p), runs summed left to right; the distinct entries overwrite the items
    const int pb = escs::sort_products<kSNT, kBkCap, V>(sm, n, D.sh);
    const int uniq = escs::compress_write<kSNT, kBkCap, V>(sm, n, pb, D.blo, bw.stg_col + D.off, sv + D.off);
    if (tid == 0) bw.desc[d].uniq = uniq;
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------- copy to C
template <typename V>
__global__ void __launch_bounds__(kCNT) k_bk_copy(BkWork bw, const int64_t* __restrict__ c_rp,
                                                  int32_t* __restrict__ out_col, double* out_val,
                                                  int64_t* __restrict__ nnz_row) {
  __shared__ int s_off[kBkMaxBuckets + 1];
  __shared__ int s_w[kCNT / 32 + 1];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const V* sv = vcast<V>(bw.stg_val);
  V* ov = vcast<V>(out_val);
  const int nr = *bw.cur32;
  for (int rr = blockIdx.x; rr < nr; rr += gridDim.x) {
    const BkRow R = bw.rows[rr];
    const int64_t base = c_rp[R.row];
    int x[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int b = 2 * tid + q;
      if (b < R.nbk) x[q] = bw.desc[R.desc0 + b].uniq;
    }
    int tot;
    const int ex = bk_block_excl_scan<kCNT>(x[0] + x[1], &tot, s_w);
    if (tid == 0 && nnz_row) nnz_row[R.row] = tot;  // hybrid: the row's length
    if (2 * tid < R.nbk) s_off[2 * tid] = ex;
    if (2 * tid + 1 < R.nbk) s_off[2 * tid + 1] = ex + x[0];
    __syncthreads();
    for (int b = wid; b < R.nbk; b += kCNT / 32) {
      const BkDesc D = bw.desc[R.desc0 + b];
      const int64_t o = base + s_off[b];
      for (int i = lane; i < D.uniq; i += 32) {
        out_col[o + i] = bw.stg_col[D.off + i];
        ov[o + i] = sv[D.off + i];
      }
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_long_buckets(const Stage3Args& a, const BkWork& bw, int64_t max_rows, bool rank_fallback,
                                cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  const int sms = num_sms();
  cudaError_t e = cudaMemsetAsync(bw.cur64, 0, 2 * sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(bw.cur32, 0, 2 * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.work_ctr, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  const bool i32 = a.b_nnz < (int64_t(1) << 31);
  {
    auto kern = a.f32 ? (i32 ? k_bk_part<int, float> : k_bk_part<int64_t, float>)
                      : (i32 ? k_bk_part<int, double> : k_bk_part<int64_t, double>);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPNT, 0);
    int64_t grid = int64_t(sms) * (per_sm > 0 ? per_sm : 1);
    if (grid > a.count) grid = a.count;
    kern<<<(unsigned)grid, kPNT, 0, s>>>(a, bw);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (max_rows > 0) {
    auto kern = a.f32 ? k_bk_sort<float> : k_bk_sort<double>;
    const size_t bytes = a.f32 ? sizeof(escs::Smem<kBkCap, float>) : sizeof(escs::Smem<kBkCap, double>);
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)) != cudaSuccess)
      return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSNT, bytes);
    kern<<<(unsigned)(int64_t(sms) * (per_sm > 0 ? per_sm : 1)), kSNT, bytes, s>>>(bw);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    auto kc = a.f32 ? k_bk_copy<float> : k_bk_copy<double>;
    const int64_t g = max_rows < int64_t(sms) * 8 ? max_rows : int64_t(sms) * 8;
    kc<<<(unsigned)g, kCNT, 0, s>>>(bw, a.out_off, a.out_col, a.out_val, a.nnz_row);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (!rank_fallback) return cudaSuccess;
  // rows that stay on the rank kernel
  Stage3Args b = a;
  b.perm = bw.fb_list;
  b.first = 0;
  b.count_dev = bw.cur32 + 1;
  return launch_long_bitmap(b, s);
}

}  // namespace sg
