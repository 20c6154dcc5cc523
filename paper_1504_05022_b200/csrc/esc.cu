// esc.cu — stage 3, classes e2048/e4096/e8192: rows whose u_i products fit one CTA's shared
// memory but whose bound min(u_i, n) is too large for a warp table.  These are the paper's
// group-4/5 sizes; the method here is the ESC idea of its bitonic-ESC group ([P:277-284]:
// expand the candidates, sort, compress duplicates) with a counting sort instead of bitonic:
//
//   1. expand: every product (c, a_ij·b_jk, p) with p its position in the row's product order
//      (j ascending, then k ascending: the order of Algorithm 1 [P:121-135]);
//   2. counting sort into NB ≈ u buckets by the monotone bucket b(c) = ⌊(c-lo)·NB/W⌋
//      (count, exclusive scan, scatter — shared-memory integer atomics only);
//   3. each bucket (a few entries) sorted by (c, p) with an insertion sort;
//   4. compress: equal columns fused in p order — the oracle's accumulation order, so values
//      are bit-identical to it (R1) — then an ordered write of the buckets.
// No hash probing, no value atomics; cost O(u) plus the small per-bucket sorts.
#include <climits>

#include "common.cuh"

namespace sg {

namespace {

constexpr int kEscChunk = 128;  // products per work item

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

template <int NT>
struct EscBatch {
  long long bs[NT];
  int len[NT];
  int pex[NT];   // exclusive product prefix within the batch
  int cinc[NT];  // inclusive prefix of work items
  double av[NT];
};

// Visit every product of row [a0, a1) as f(q, a_ij, p): balanced work items of kEscChunk
// products, p = the product's index in the row's (j, k) order.
template <int NT, bool VALS, typename F>
__device__ __forceinline__ void esc_products(const Stage3Args& a, int64_t a0, int64_t a1, EscBatch<NT>& sb,
                                             int* s_w, F&& f) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = NT / 32;
  int pbase = 0;
  for (int64_t e0 = a0; e0 < a1; e0 += NT) {
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
    int ptot;
    const int pex = esc_block_excl_scan<NT>(len, &ptot, s_w);
    const int nch = (len + kEscChunk - 1) / kEscChunk;
    int ctot;
    const int cex = esc_block_excl_scan<NT>(nch, &ctot, s_w);
    sb.pex[threadIdx.x] = pex;
    sb.cinc[threadIdx.x] = cex + nch;
    __syncthreads();
    for (int item = w; item < ctot; item += NW) {
      int lo = 0, hi = NT - 1;  // first t with cinc[t] > item
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sb.cinc[mid] > item) hi = mid;
        else lo = mid + 1;
      }
      const int t = lo;
      const int first = sb.cinc[t] - (sb.len[t] + kEscChunk - 1) / kEscChunk;
      const int off0 = (item - first) * kEscChunk;
      const int off1 = min(off0 + kEscChunk, sb.len[t]);
      const double at = VALS ? sb.av[t] : 0.0;
      const int pt = pbase + sb.pex[t];
      for (int off = off0 + lane; off < off1; off += 32) f((int64_t)sb.bs[t] + off, at, pt + off);
    }
    pbase += ptot;
    __syncthreads();
  }
}

template <int LOG2U, int NT>
__global__ void __launch_bounds__(NT, 1) k_cta_esc(Stage3Args a) {
  constexpr int UMAX = 1 << LOG2U;
  constexpr int NBMAX = UMAX;  // ~1 product per bucket: the per-bucket sorts are trivial
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  const bool fill = a.mode == MODE_FILL;
  // layout: vals double[UMAX] (fill) | keys int[UMAX] | pidx int[UMAX] (fill) | bstart int[NBMAX+1] | bcur int[NBMAX]
  double* vals = reinterpret_cast<double*>(smem);
  int* keys = reinterpret_cast<int*>(smem + (fill ? size_t(UMAX) * sizeof(double) : 0));
  int* pidx = keys + UMAX;
  int* bstart = keys + (fill ? 2 * UMAX : UMAX);
  int* bcur = bstart + NBMAX + 1;
  __shared__ EscBatch<NT> sb;
  __shared__ int s_w[NW + 1];
  __shared__ int s_red[3 * NW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

  for (int64_t r = blockIdx.x; r < a.count; r += gridDim.x) {
    const int row = __ldg(a.perm + a.first + r);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    // window [lo, hi] and u of the row
    int lo = INT_MAX, hi = -1, u = 0;
    for (int64_t e = a0 + threadIdx.x; e < a1; e += NT) {
      const int j = __ldg(a.A.ci + e);
      const int64_t bs = __ldg(a.B.rp + j), be = __ldg(a.B.rp + j + 1);
      if (be > bs) {
        lo = min(lo, __ldg(a.B.ci + bs));
        hi = max(hi, __ldg(a.B.ci + be - 1));
        u += (int)(be - bs);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      u += __shfl_xor_sync(0xffffffffu, u, o);
    }
    if (lane == 0) {
      s_red[w] = lo;
      s_red[NW + w] = hi;
      s_red[2 * NW + w] = u;
    }
    __syncthreads();
    lo = INT_MAX;
    hi = -1;
    u = 0;
    for (int k = 0; k < NW; ++k) {
      lo = min(lo, s_red[k]);
      hi = max(hi, s_red[NW + k]);
      u += s_red[2 * NW + k];
    }
    int NB = 32;
    while (NB < NBMAX && NB < u) NB <<= 1;
    const float scale = (float)NB / (float)(int64_t(hi) - lo + 1);
    for (int b = threadIdx.x; b <= NB; b += NT) bstart[b] = 0;
    __syncthreads();
    // 1-2. expand + count per bucket
    esc_products<NT, false>(a, a0, a1, sb, s_w, [&](int64_t q, double, int) {
      const int c = __ldg(a.B.ci + q);
      const int b = min((int)__fmul_rz((float)(c - lo), scale), NB - 1);  // monotone in c
      atomicAdd(&bstart[b], 1);
    });
    // exclusive scan of the bucket counts (each thread owns NB/NT or 1 buckets)
    {
      constexpr int PER = NBMAX / NT > 0 ? NBMAX / NT : 1;
      const int b0 = threadIdx.x * PER;
      int v[PER];
      int loc = 0;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        v[k] = (b0 + k < NB) ? bstart[b0 + k] : 0;
        loc += v[k];
      }
      int tot;
      int run = esc_block_excl_scan<NT>(loc, &tot, s_w);
#pragma unroll
      for (int k = 0; k < PER; ++k)
        if (b0 + k < NB) {
          bstart[b0 + k] = run;
          bcur[b0 + k] = run;
          run += v[k];
        }
      if (threadIdx.x == 0) bstart[NB] = tot;
      __syncthreads();
    }
    // 2. scatter (column, product index, value) into the buckets
    esc_products<NT, true>(a, a0, a1, sb, s_w, [&](int64_t q, double at, int p) {
      const int c = __ldg(a.B.ci + q);
      const int b = min((int)__fmul_rz((float)(c - lo), scale), NB - 1);
      const int slot = atomicAdd(&bcur[b], 1);
      keys[slot] = c;
      if (fill) {
        pidx[slot] = p;
        vals[slot] = __dmul_rn(at, __ldg(a.B.val + q));  // line 6: value <- a_ij b_jk
      }
    });
    // 3-4. sort each bucket by (column, p), fuse equal columns in p order
    for (int b = threadIdx.x; b < NB; b += NT) {
      const int s0 = bstart[b], s1 = bstart[b + 1];
      for (int x = s0 + 1; x < s1; ++x) {
        const int kx = keys[x];
        const int px = fill ? pidx[x] : 0;
        const double vx = fill ? vals[x] : 0.0;
        int y = x - 1;
        while (y >= s0 && (keys[y] > kx || (fill && keys[y] == kx && pidx[y] > px))) {
          keys[y + 1] = keys[y];
          if (fill) {
            pidx[y + 1] = pidx[y];
            vals[y + 1] = vals[y];
          }
          --y;
        }
        keys[y + 1] = kx;
        if (fill) {
          pidx[y + 1] = px;
          vals[y + 1] = vx;
        }
      }
      int d = s0;  // fused entries are written to the front of the bucket
      for (int x = s0; x < s1; ++x) {
        if (x > s0 && keys[x] == keys[d - 1]) {
          if (fill) vals[d - 1] = __dadd_rn(vals[d - 1], vals[x]);  // line 11: accumulate
        } else {
          keys[d] = keys[x];
          if (fill) vals[d] = vals[x];  // line 9: c_ik <- value
          ++d;
        }
      }
      bcur[b] = d - s0;  // distinct columns of the bucket
    }
    __syncthreads();
    // 5. ordered write: exclusive scan of the distinct counts
    {
      constexpr int PER = NBMAX / NT > 0 ? NBMAX / NT : 1;
      const int b0 = threadIdx.x * PER;
      int loc = 0;
#pragma unroll
      for (int k = 0; k < PER; ++k)
        if (b0 + k < NB) loc += bcur[b0 + k];
      int tot;
      int pos = esc_block_excl_scan<NT>(loc, &tot, s_w);
      if (fill) {
        const int64_t o = __ldg(a.out_off + row);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int b = b0 + k;
          if (b >= NB) break;
          const int s0 = bstart[b];
          for (int t = 0; t < bcur[b]; ++t) {
            a.out_col[o + pos + t] = keys[s0 + t];
            a.out_val[o + pos + t] = vals[s0 + t];
          }
          pos += bcur[b];
        }
      }
      if (threadIdx.x == 0 && a.nnz_row) a.nnz_row[row] = tot;
      __syncthreads();
    }
  }
}

int esc_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

template <int LOG2U, int NT>
cudaError_t launch_esc_t(const Stage3Args& a, cudaStream_t s) {
  constexpr int UMAX = 1 << LOG2U;
  const bool fill = a.mode == MODE_FILL;
  const size_t sm = size_t(UMAX) * (fill ? 16 : 4) + size_t(UMAX) * 8 + 8;
  auto kern = k_cta_esc<LOG2U, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, sm);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = int64_t(esc_sms()) * per_sm * 4;
  if (grid > a.count) grid = a.count;
  kern<<<(unsigned)grid, NT, sm, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_esc(int tier, const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  switch (tier) {
    case T_E2048: return launch_esc_t<11, 256>(a, s);
    case T_E4096: return launch_esc_t<12, 256>(a, s);
    case T_E8192: return launch_esc_t<13, 512>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sg
