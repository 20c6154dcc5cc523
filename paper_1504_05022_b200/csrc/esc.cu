// esc.cu — stage 3, classes e2048/e4096/e8192: rows whose u_i products fit one CTA's shared
// memory but whose bound min(u_i, n) is too large for a warp table.  These are the paper's
// group-4/5 sizes; the method is the ESC of its bitonic-ESC group ([P:277-284]: "expand" the
// candidates, "sort" them, "compress" duplicates), with a stable LSD radix sort of the whole
// row in one CTA instead of the paper's bitonic sort:
//
//   1. expand: every product (c - lo, a_ij·b_jk) lands at its position p in the row's
//      product order (j ascending, then k ascending: Algorithm 1 [P:121-135]); p comes from a
//      block scan of nnz(b_j*) — no atomics, one warp per a_ij, coalesced b_j* loads;
//   2. sort: cub::BlockRadixSort (stable) over the bits of the row's column window, items in
//      blocked p order, so equal columns stay in p order;
//   3. compress: each run of equal columns is summed left to right (the oracle's order, so
//      values are bit-identical to it, R1) and the row is written in order.
// COUNT (precise symbolic) uses the CTA hash of the same size (stage3.cu): counting needs no order.
// The warp classes' rows (u <= 2048) are sorted by a run merge instead (k_esc_merge below):
// every b_j* is already sorted, so ⌈log2 runs⌉ stable pairwise merges sort the row.
#include <climits>
#include <cstdlib>
#include <type_traits>

#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"
#include "esc_sort.cuh"

namespace sg {

namespace {

template <int NT>
__device__ __forceinline__ int esc_block_excl_scan(int v, int* total, int* s_w) {
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

constexpr int kEscRadixBits = 6;  // digit width of the block radix sort (4 passes for 23-bit windows)

template <int NT, int IPT, bool VALS, typename V>
struct EscSmem {
  static constexpr int U = NT * IPT;
  // the sort carries the 16-bit product index p; values stay in place (pval) and are
  // gathered once after the sort (6 B per item per pass instead of 12)
  using Sort = cub::BlockRadixSort<unsigned, NT, IPT, typename std::conditional<VALS, unsigned short, cub::NullType>::type,
                                   kEscRadixBits>;
  struct Rows {
    unsigned key[U];
    V val[VALS ? U : 1];
  };
  union {
    typename Sort::TempStorage sort;
    Rows rows;
  };
  V pval[VALS ? U : 1];
};

template <int NT, int IPT, int MODE, typename IT, typename V>
__global__ void __launch_bounds__(NT) k_esc_sort(Stage3Args a) {
  constexpr bool VALS = MODE == MODE_FILL;
  constexpr int U = NT * IPT;
  constexpr int NW = NT / 32;
  using SM = EscSmem<NT, IPT, VALS, V>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  __shared__ IT s_bs[NT];
  __shared__ int s_len[NT], s_pex[NT];
  __shared__ V s_av[VALS ? NT : 1];
  __shared__ int s_w[NW + 1];
  __shared__ unsigned s_max[NW];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  const int64_t rper = (a.count + gridDim.x - 1) / gridDim.x;  // contiguous rows per CTA
  const int64_t rend = min(int64_t(blockIdx.x) * rper + rper, a.count);
  for (int64_t r = int64_t(blockIdx.x) * rper; r < rend; ++r) {
    const int row = __ldg(a.perm + a.first + r);
    const int lo = __ldg(a.rlo + row);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    // 1. expand (lines 3-6 of Algorithm 1): product p of the row at rows.key/val[p]
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
        if (VALS) s_av[tid] = __ldg(vcast<V>(a.A.val) + e);
      }
      int tot;
      const int ex = esc_block_excl_scan<NT>(len, &tot, s_w);  // syncs
      s_len[tid] = len;
      s_pex[tid] = u + ex;
      __syncthreads();
      const int na = (int)((a1 - e0) < NT ? (a1 - e0) : NT);
      for (int t = w; t < na; t += NW) {
        const IT bs = s_bs[t];
        const int lt = s_len[t], pe = s_pex[t];
        const V at = VALS ? s_av[t] : V(0);
        for (int q = lane; q < lt; q += 32) {
          const unsigned k = (unsigned)(__ldg(a.B.ci + bs + q) - lo);
          sm.rows.key[pe + q] = k;
          kmax = k > kmax ? k : kmax;
          if (VALS) sm.pval[pe + q] = Arith<V>::mul(at, __ldg(vcast<V>(a.B.val) + bs + q));  // line 6
        }
      }
      u += tot;
      __syncthreads();
    }
    // window bits of the row (the radix sort's end bit)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned x = __shfl_xor_sync(0xffffffffu, kmax, o);
      kmax = x > kmax ? x : kmax;
    }
    if (lane == 0) s_max[w] = kmax;
    // 2. sort: blocked items in p order; padding sorts last (stable: after equal keys)
    unsigned k[IPT];
    typename std::conditional<VALS, unsigned short, cub::NullType>::type pi[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int p = tid * IPT + i;
      k[i] = p < u ? sm.rows.key[p] : 0xffffffffu;
      if constexpr (VALS) pi[i] = (unsigned short)p;
    }
    __syncthreads();
    unsigned km = 0;
#pragma unroll
    for (int x = 0; x < NW; ++x) km = s_max[x] > km ? s_max[x] : km;
    const int end_bit = km ? 32 - __clz(km) : 1;
    if constexpr (VALS) {
      typename SM::Sort(sm.sort).Sort(k, pi, 0, end_bit);
    } else {
      typename SM::Sort(sm.sort).Sort(k, 0, end_bit);
    }
    __syncthreads();
    const unsigned pad = end_bit >= 32 ? 0xffffffffu : ((1u << end_bit) - 1u);
    (void)pad;
    V v[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      sm.rows.key[tid * IPT + i] = k[i];
      if constexpr (VALS) {
        v[i] = tid * IPT + i < u ? sm.pval[pi[i]] : V(0);
        sm.rows.val[tid * IPT + i] = v[i];
      }
    }
    __syncthreads();
    // 3. compress: heads of runs of equal columns; run sums left to right (lines 9, 11)
    int heads = 0;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int p = tid * IPT + i;
      const bool head = p < u && (p == 0 || sm.rows.key[p - 1] != k[i]);
      if (head) {
        ++heads;
        if constexpr (VALS) {
          V acc = v[i];
          for (int x = p + 1; x < u && sm.rows.key[x] == k[i]; ++x) acc = Arith<V>::add(acc, sm.rows.val[x]);
          v[i] = acc;
        }
      } else {
        k[i] = 0xffffffffu;  // not a head
      }
    }
    int nnz;
    int pos = esc_block_excl_scan<NT>(heads, &nnz, s_w);  // syncs: all reads above are done
    if (MODE == MODE_FILL) {
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        if (tid * IPT + i < u && k[i] != 0xffffffffu) {
          sm.rows.key[pos] = k[i];
          if constexpr (VALS) sm.rows.val[pos] = v[i];
          ++pos;
        }
      }
      __syncthreads();
      const int64_t o = __ldg(a.out_off + row);
      for (int i = tid; i < nnz; i += NT) {
        a.out_col[o + i] = (int)sm.rows.key[i] + lo;
        if constexpr (VALS) vcast<V>(a.out_val)[o + i] = sm.rows.val[i];
      }
    }
    if (tid == 0 && a.nnz_row) a.nnz_row[row] = nnz;
    __syncthreads();
  }
}

template <int NT, int IPT, int MODE, typename IT, typename V>
cudaError_t launch_esc_k(const Stage3Args& a, cudaStream_t s) {
  using SM = EscSmem<NT, IPT, MODE == MODE_FILL, V>;
  const size_t bytes = sizeof(SM);
  auto kern = k_esc_sort<NT, IPT, MODE, IT, V>;
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

// the bucket ESC needs key + product-index bits within 32: windows up to 2^29 columns
bool esc_old(const Stage3Args& a) {
  static const bool v = getenv("SPGEMM_ESC_OLD") != nullptr;  // A/B switch (development)
  return v || a.n > (int64_t(1) << escs::max_key_bits<8192>());
}

// ----------------------------------------------------------------------------------------
// Run-merge ESC.  Every b_j* is sorted (Q3), so the expanded row is already a sequence of
// sorted runs (one per nonempty b_j*, in j order).  Merging runs pairwise, left run first on
// ties (stable: product order p is kept among equal columns), sorts the row in ⌈log2 runs⌉
// rounds instead of one radix pass per digit.  Each round: thread t produces output positions
// [t·IPT, (t+1)·IPT): binary search for its pair of runs and its merge-path split, then a
// sequential merge; keys and values ping-pong between two shared buffers.
template <int NT, int IPT, typename V>
struct MergeSmem {
  static constexpr int U = NT * IPT;
  unsigned key[2][U];
  unsigned short idx[2][U];  // product position p: values stay in pval until the compression
  V pval[U];
  unsigned short rb[U + 2];  // run boundaries (nonempty runs)
};

template <int NT, int IPT, typename IT, typename V>
__global__ void __launch_bounds__(NT) k_esc_merge(Stage3Args a) {
  constexpr int U = NT * IPT;
  constexpr int NW = NT / 32;
  using SM = MergeSmem<NT, IPT, V>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  __shared__ IT s_bs[NT];
  __shared__ int s_len[NT], s_pex[NT];
  __shared__ V s_av[NT];
  __shared__ int s_w[NW + 1];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  const int64_t rper = (a.count + gridDim.x - 1) / gridDim.x;  // contiguous rows per CTA
  const int64_t rend = min(int64_t(blockIdx.x) * rper + rper, a.count);
  for (int64_t r = int64_t(blockIdx.x) * rper; r < rend; ++r) {
    const int row = __ldg(a.perm + a.first + r);
    const int lo = __ldg(a.rlo + row);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    // 1. expand (lines 3-6 of Algorithm 1) into buffer 0; run starts of the nonempty b_j*
    int u = 0, nr = 0;
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
      int tot, rtot;
      const int ex = esc_block_excl_scan<NT>(len, &tot, s_w);
      const int rex = esc_block_excl_scan<NT>(len > 0 ? 1 : 0, &rtot, s_w);
      s_len[tid] = len;
      s_pex[tid] = u + ex;
      if (len > 0) sm.rb[nr + rex] = (unsigned short)(u + ex);
      __syncthreads();
      const int na = (int)((a1 - e0) < NT ? (a1 - e0) : NT);
      for (int t = w; t < na; t += NW) {
        const IT bs = s_bs[t];
        const int lt = s_len[t], pe = s_pex[t];
        const V at = s_av[t];
        for (int q = lane; q < lt; q += 32) {
          sm.key[0][pe + q] = (unsigned)(__ldg(a.B.ci + bs + q) - lo);
          sm.idx[0][pe + q] = (unsigned short)(pe + q);
          sm.pval[pe + q] = Arith<V>::mul(at, __ldg(vcast<V>(a.B.val) + bs + q));  // line 6
        }
      }
      u += tot;
      nr += rtot;
      __syncthreads();
    }
    if (tid == 0) sm.rb[nr] = (unsigned short)u;
    __syncthreads();
    // 2. merge rounds (src buffer b, runs [rb[k], rb[k+1]), k < nr)
    int b = 0;
    while (nr > 1) {
      const int nr2 = (nr + 1) >> 1;
      int x = tid * IPT;
      const int xe = min(x + IPT, u);
      if (x < xe) {
        // the pair holding x: largest k with rb[2k] <= x
        int lo2 = 0, hi2 = nr2 - 1;
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2 + 1) >> 1;
          if (sm.rb[2 * mid] <= x) lo2 = mid;
          else hi2 = mid - 1;
        }
        int k = lo2;
        while (x < xe) {
          const int l0 = sm.rb[2 * k];
          const int l1 = 2 * k + 1 < nr ? sm.rb[2 * k + 1] : u;
          const int r1 = 2 * k + 2 <= nr ? sm.rb[min(2 * k + 2, nr)] : u;
          const int nl = l1 - l0, nrr = r1 - l1;
          const int d = x - l0;
          // merge path: i elements from the left run precede output d (left first on ties)
          int ilo = d > nrr ? d - nrr : 0, ihi = d < nl ? d : nl;
          while (ilo < ihi) {
            const int mid = (ilo + ihi) >> 1;
            if (sm.key[b][l0 + mid] <= sm.key[b][l1 + d - mid - 1]) ilo = mid + 1;
            else ihi = mid;
          }
          int i = ilo, j = d - ilo;
          const int xend = min(xe, r1);
          for (; x < xend; ++x) {
            const bool takel = i < nl && (j >= nrr || sm.key[b][l0 + i] <= sm.key[b][l1 + j]);
            const int src = takel ? l0 + i : l1 + j;
            sm.key[b ^ 1][x] = sm.key[b][src];
            sm.idx[b ^ 1][x] = sm.idx[b][src];
            i += takel ? 1 : 0;
            j += takel ? 0 : 1;
          }
          ++k;
        }
      }
      __syncthreads();
      // new run starts: rb[k] = rb[2k]
      unsigned short nb[(U + 2 + NT - 1) / NT];
#pragma unroll
      for (int q = 0; q < (U + 2 + NT - 1) / NT; ++q) {
        const int k = tid + q * NT;
        nb[q] = (k <= nr2 && 2 * k <= nr) ? sm.rb[min(2 * k, nr)] : 0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < (U + 2 + NT - 1) / NT; ++q) {
        const int k = tid + q * NT;
        if (k < nr2) sm.rb[k] = nb[q];
      }
      if (tid == 0) sm.rb[nr2] = (unsigned short)u;
      nr = nr2;
      b ^= 1;
      __syncthreads();
    }
    // 3. compress: runs of equal columns summed left to right (lines 9, 11), written in order
    const unsigned* key = sm.key[b];
    const unsigned short* idx = sm.idx[b];
    int heads = 0;
    for (int i = 0; i < IPT; ++i) {
      const int p = tid * IPT + i;
      heads += (p < u && (p == 0 || key[p - 1] != key[p])) ? 1 : 0;
    }
    int nnz;
    int pos = esc_block_excl_scan<NT>(heads, &nnz, s_w);
    const int64_t o = __ldg(a.out_off + row);
    V vh[IPT];
    for (int i = 0; i < IPT; ++i) {
      const int p = tid * IPT + i;
      if (p < u && (p == 0 || key[p - 1] != key[p])) {
        V acc = sm.pval[idx[p]];
        for (int x = p + 1; x < u && key[x] == key[p]; ++x) acc = Arith<V>::add(acc, sm.pval[idx[x]]);
        vh[i] = acc;
      }
    }
    __syncthreads();  // all reads of the sorted buffer done: compact in place of the other one
    for (int i = 0; i < IPT; ++i) {
      const int p = tid * IPT + i;
      if (p < u && (p == 0 || key[p - 1] != key[p])) {
        sm.key[b ^ 1][pos] = key[p];
        sm.pval[pos] = vh[i];
        ++pos;
      }
    }
    __syncthreads();
    for (int i = tid; i < nnz; i += NT) {
      a.out_col[o + i] = (int)sm.key[b ^ 1][i] + lo;
      vcast<V>(a.out_val)[o + i] = sm.pval[i];
    }
    if (tid == 0 && a.nnz_row) a.nnz_row[row] = nnz;
    __syncthreads();
  }
}

template <int NT, int IPT, typename IT, typename V>
cudaError_t launch_merge_k(const Stage3Args& a, cudaStream_t s) {
  const size_t bytes = sizeof(MergeSmem<NT, IPT, V>);
  auto kern = k_esc_merge<NT, IPT, IT, V>;
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

template <int NT, int IPT>
cudaError_t launch_esc_t(const Stage3Args& a, cudaStream_t s) {
  const bool i32 = a.b_nnz < (int64_t(1) << 31);
  if (a.f32)
    return i32 ? launch_esc_k<NT, IPT, MODE_FILL, int, float>(a, s) : launch_esc_k<NT, IPT, MODE_FILL, int64_t, float>(a, s);
  return i32 ? launch_esc_k<NT, IPT, MODE_FILL, int, double>(a, s) : launch_esc_k<NT, IPT, MODE_FILL, int64_t, double>(a, s);
}

// Merge kernels use an odd number of items per thread: each thread reads and writes its own
// consecutive positions, so an odd stride keeps the 32 lanes on 32 different banks.
template <int NT, int IPT>
cudaError_t launch_merge_t(const Stage3Args& a, cudaStream_t s) {
  const bool i32 = a.b_nnz < (int64_t(1) << 31);
  if (a.f32) return i32 ? launch_merge_k<NT, IPT, int, float>(a, s) : launch_merge_k<NT, IPT, int64_t, float>(a, s);
  return i32 ? launch_merge_k<NT, IPT, int, double>(a, s) : launch_merge_k<NT, IPT, int64_t, double>(a, s);
}

}  // namespace

// Rows of the warp classes (u <= 0.8·S) sorted in one CTA of at least S items by the run
// merge (measured faster than the radix sort at these sizes; slower at 4096+, c3a / c5).
cudaError_t launch_esc_items(int S, const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  if (!esc_old(a)) switch (S) {
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
  switch (S) {
    case 64: return launch_merge_t<32, 3>(a, s);
    case 128: return launch_merge_t<32, 5>(a, s);
    case 256: return launch_merge_t<64, 5>(a, s);
    case 512: return launch_merge_t<64, 9>(a, s);
    case 1024: return launch_merge_t<128, 9>(a, s);
    case 2048: return launch_merge_t<256, 9>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

// e2048: run merge (5.9 vs 6.3 ms on c3a); e4096 / e8192: radix (merge 25.0 vs 21.1 ms)
cudaError_t launch_esc(int tier, const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  if (!esc_old(a)) switch (tier) {
    case T_E2048: return launch_bk_t<256, 2048>(a, s);
#ifndef SG_E4096_NT
#define SG_E4096_NT 512  // 512 threads: c5 e4096 121.8 -> 106.4 ms per wave (256 for w2048: 14.0 vs 17.3 ms on c3a)
#endif
    case T_E4096: return launch_bk_t<SG_E4096_NT, 4096>(a, s);
    case T_E8192: return launch_bk_t<512, 8192>(a, s);
    default: return cudaErrorInvalidValue;
  }
  switch (tier) {
    case T_E2048: return launch_merge_t<256, 9>(a, s);
    case T_E4096: return launch_esc_t<256, 16>(a, s);
    case T_E8192: return launch_esc_t<512, 16>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sg
