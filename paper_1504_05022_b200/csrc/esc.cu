// esc.cu — stage 3 values of the warp classes (w64..w2048) and the ESC classes (e2048..e8192):
// rows whose u_i products fit one CTA's shared memory.  The method is the ESC of the paper's
// bitonic-ESC group ([P:277-284]: "expand" the candidates, "sort" them, "compress"
// duplicates), re-derived for B200:
//
//   1. expand: every product (c - lo, a_ij·b_jk) lands at its position p in the row's product
//      order (j ascending, then k ascending: Algorithm 1 [P:121-135]); the batch's products are
//      cut into equal warp ranges walked 32 at a time (product -> a_ij by a forward scan of the
//      batch's offsets), with four steps of gathers in flight;
//   2. sort by (column, p): one counting pass into ~32-product buckets and a warp bitonic
//      network per bucket (esc_sort.cuh) — measured faster than a block radix sort over all
//      window bits and than a pairwise run merge (c3a numeric 106.9 -> 72.6 ms);
//   3. compress: runs of equal columns summed left to right (the oracle's order, so values are
//      bit-identical to it, R1) and written in column order.
// Counting (precise symbolic) is done by the warp hash (warp.cu) and the CTA hash (stage3.cu).
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "esc_sort.cuh"

namespace sg {

namespace {

// ----------------------------------------------------------------------------------------
// Bucket ESC (esc_sort.cuh): expand the row's products in product order, sort them by
// (column, p) with one counting pass into ~32-product buckets plus warp bitonic sorts, sum the
// runs left to right.  Replaces the block radix sort (4 passes over 22-bit keys on c3a) and the
// run merge (log2(runs) rounds) for the warp and ESC classes.
template <int NT, int CAP, typename IT, typename V>
__global__ void __launch_bounds__(NT) k_esc_bk(Stage3Args a) {
  constexpr int NW = NT / 32;
  constexpr int UNR = 4;  // products per lane whose loads are in flight together
  using SM = escs::Smem<CAP, V>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  __shared__ IT s_bs[NT];
  __shared__ int s_pex[NT + 1];
  __shared__ V s_av[NT];
  __shared__ int s_w[NW + 1];
  __shared__ unsigned s_max[NW];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  const int64_t count = a.count_dev ? (int64_t)*a.count_dev : a.count;
  const int64_t rper = (count + gridDim.x - 1) / gridDim.x;  // contiguous rows per CTA
  const int64_t rend = min(int64_t(blockIdx.x) * rper + rper, count);
  for (int64_t r = int64_t(blockIdx.x) * rper; r < rend; ++r) {
    const int row = __ldg(a.perm + a.first + r);
    const int lo = __ldg(a.rlo + row);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    // 1. expand (lines 3-6 of Algorithm 1): product p of the row at key/pval[p].  Per batch of
    //    NT a_ij: the batch's products are cut into NW equal ranges, warp w walks its range 32
    //    products per step (product -> its a_ij by a forward scan of the batch's offsets), with
    //    the loads of UNR steps issued before their stores.
    int u = 0;
    unsigned kmax = 0;
    for (int64_t e0 = a0; e0 < a1; e0 += NT) {
      const int64_t e = e0 + tid;
      int len = 0;
      if (e < a1) {
        const int j = __ldg(a.A.ci + e);
        const int64_t b0 = __ldg(a.B.rp + j);
        len = (int)(__ldg(a.B.rp + j + 1) - b0);
        s_bs[tid] = (IT)b0;
        s_av[tid] = __ldg(vcast<V>(a.A.val) + e);
      }
      int tot;
      const int ex = escs::block_excl_scan<NT>(len, &tot, s_w);
      s_pex[tid] = ex;
      if (tid == NT - 1) s_pex[NT] = tot;
      __syncthreads();
      const int na = (int)((a1 - e0) < NT ? (a1 - e0) : NT);
      const int pw0 = (int)((int64_t(tot) * w) / NW), pw1 = (int)((int64_t(tot) * (w + 1)) / NW);
      int p = pw0 + lane;
      // t: the a_ij of product p (largest t with s_pex[t] <= p), by binary search once
      int t = 0;
      {
        int lo2 = 0, hi2 = na - 1;
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2 + 1) >> 1;
          if (s_pex[mid] <= p) lo2 = mid;
          else hi2 = mid - 1;
        }
        t = lo2;
      }
      for (; p - lane < pw1; p += 32 * UNR) {
        unsigned kk[UNR];
        V vv[UNR];
        int pp[UNR];
#pragma unroll
        for (int x = 0; x < UNR; ++x) {
          const int q = p + 32 * x;
          pp[x] = q;
          if (q < pw1) {
            while (s_pex[t + 1] <= q) ++t;
            const IT g = s_bs[t] + (IT)(q - s_pex[t]);
            kk[x] = (unsigned)(__ldg(a.B.ci + g) - lo);
            vv[x] = Arith<V>::mul(s_av[t], __ldg(vcast<V>(a.B.val) + g));  // line 6
          }
        }
#pragma unroll
        for (int x = 0; x < UNR; ++x)
          if (pp[x] < pw1) {
            sm.key[u + pp[x]] = kk[x];
            sm.pval[u + pp[x]] = vv[x];
            kmax = kk[x] > kmax ? kk[x] : kmax;
          }
      }
      u += tot;
      __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    if (lane == 0) s_max[w] = kmax;
    __syncthreads();
    unsigned km = 0;
#pragma unroll
    for (int x = 0; x < NW; ++x) km = s_max[x] > km ? s_max[x] : km;
    const int kb = km ? 32 - __clz(km) : 0;
    // 2. sort by (column, p); 3. compress into the row's output
    const int pb = escs::sort_products<NT, CAP, V>(sm, u, kb);
    const int64_t o = __ldg(a.out_off + row);
    const int nnz = escs::compress_write<NT, CAP, V>(sm, u, pb, lo, a.out_col + o, vcast<V>(a.out_val) + o);
    if (tid == 0 && a.nnz_row) a.nnz_row[row] = nnz;
    __syncthreads();
  }
}

template <int NT, int CAP, typename IT, typename V>
cudaError_t launch_bk_k(const Stage3Args& a, cudaStream_t s) {
  const size_t bytes = sizeof(escs::Smem<CAP, V>);
  auto kern = k_esc_bk<NT, CAP, IT, V>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = int64_t(num_sms()) * per_sm;
  if (grid > a.count) grid = a.count;
  kern<<<(unsigned)grid, NT, bytes, s>>>(a);
  return cudaGetLastError();
}

template <int NT, int CAP>
cudaError_t launch_bk_t(const Stage3Args& a, cudaStream_t s) {
  const bool i32 = a.b_nnz < (int64_t(1) << 31);
  if (a.f32) return i32 ? launch_bk_k<NT, CAP, int, float>(a, s) : launch_bk_k<NT, CAP, int64_t, float>(a, s);
  return i32 ? launch_bk_k<NT, CAP, int, double>(a, s) : launch_bk_k<NT, CAP, int64_t, double>(a, s);
}


}  // namespace

// Rows of the warp classes (u <= 0.8·S): the bucket ESC in one CTA of S items.
cudaError_t launch_esc_items(int S, const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  switch (S) {
    case 64: return launch_bk_t<32, 64>(a, s);
    case 128: return launch_bk_t<32, 128>(a, s);
    case 256: return launch_bk_t<64, 256>(a, s);
    case 512: return launch_bk_t<64, 512>(a, s);
    case 1024: return launch_bk_t<128, 1024>(a, s);
#ifndef SG_W2048_NT
#define SG_W2048_NT 256
#endif
    case 2048: return launch_bk_t<SG_W2048_NT, 2048>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

// ESC classes: the bucket ESC with 2048 / 4096 / 8192 items per CTA.
cudaError_t launch_esc(int tier, const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  switch (tier) {
    case T_E2048: return launch_bk_t<256, 2048>(a, s);
#ifndef SG_E4096_NT
#define SG_E4096_NT 512  // 512 threads: c5 e4096 121.8 -> 106.4 ms per wave (256 for w2048: 14.0 vs 17.3 ms on c3a)
#endif
    case T_E4096: return launch_bk_t<SG_E4096_NT, 4096>(a, s);
    case T_E8192: return launch_bk_t<512, 8192>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sg
