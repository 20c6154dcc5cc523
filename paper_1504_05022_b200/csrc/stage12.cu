// stage12.cu — stage 1 (upper bound, [P:198-212]) and stage 2 (binning + hybrid C~
// offsets, [P:214-260]) on the GPU, plus a generic int64 exclusive scan (stage 4's sum of
// nnz(c_i*), [P:301]) and the CSR validation kernel.
//
// The paper runs stage 2 on one CPU core ("a few simple linear time traverses" [P:224]);
// here it is three kernels so U never crosses PCIe (reading R11):
//   k_stage1   u_i, class t_i, per-block class histogram, per-block sums of C~ capacity
//   k_stage2_scan     one CTA: class offsets (class-major, block order) + capacity offsets
//   k_stage2_scatter  stable scatter of row ids into perm (ascending row id within a
//                     class: deterministic) + exclusive scan of capacities → C~ offsets
#include <climits>

#include "common.cuh"

namespace sg {

namespace {

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_sum(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T x = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += x;
  }
  return v;
}

// Block-wide exclusive scan of one int64 per thread; returns exclusive prefix, *total.
template <int NT>
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total, int64_t* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t inc = warp_incl_sum(v);
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    int64_t x = lane < NT / 32 ? s_w[lane] : 0;
    int64_t xi = warp_incl_sum(x);
    if (lane < NT / 32) s_w[lane] = xi - x;
    if (lane == 31) s_w[NT / 32] = xi;
  }
  __syncthreads();
  int64_t ex = inc - v + s_w[w];
  *total = s_w[NT / 32];
  __syncthreads();
  return ex;
}

// ---------------------------------------------------------------------------- stage 1
// Per row j of B one 16-byte record: first and last column ((INT_MAX, -1) when empty; rows
// are sorted, Q3) and nnz(b_j*) — stage 1 then gathers one record per a_ij instead of two row
// pointers and a window pair.
__global__ void k_bwin(int64_t k, const int64_t* __restrict__ brp, const int32_t* __restrict__ bci,
                       int4* __restrict__ bwin) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const int64_t b0 = __ldg(brp + j), b1 = __ldg(brp + j + 1);
  bwin[j] = b1 > b0 ? make_int4(__ldg(bci + b0), __ldg(bci + b1 - 1), (int)(b1 - b0), 0)
                    : make_int4(INT_MAX, -1, 0, 0);
}

__device__ __forceinline__ void acc_row(int64_t& u, int& lo, int& hi, const int4* bwin, int j) {
  const int4 w = __ldg(bwin + j);
  u += w.z;  // line 4: u_i += nnz(b_j*)
  lo = min(lo, w.x);
  hi = max(hi, w.y);
}

// Algorithm "first stage" [P:198-212]: one thread per entry of U, u_i = sum nnz(b_j*); with it
// the row's column window [lo, hi] (for the window-bitmap class) and the class of the row.
template <int NT, int RPT>
__global__ void __launch_bounds__(NT) k_stage1(int64_t m, int64_t n, CsrView A,
                                               const int64_t* __restrict__ brp,
                                               const int4* __restrict__ bwin, TierParams tp,
                                               int cap_mode, int64_t* __restrict__ U,
                                               uint8_t* __restrict__ tier, int32_t* __restrict__ rlo,
                                               int32_t* __restrict__ rhi,
                                               int32_t* __restrict__ blk_tier,
                                               int64_t* __restrict__ blk_cap,
                                               int64_t* __restrict__ blk_usum,
                                               int64_t* __restrict__ blk_umax,
                                               int64_t* __restrict__ summary) {
  __shared__ int s_hist[NUM_TIERS];
  __shared__ int64_t s_red[3][NT / 32];
  if (threadIdx.x < NUM_TIERS) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * NT * RPT;
  int64_t capsum = 0, usum = 0, umax = 0, wmax = 0, vmax = 0;
  unsigned long long bku = 0, bkr = 0;
#pragma unroll 1
  for (int r = 0; r < RPT; ++r) {
    const int64_t i = base + int64_t(r) * NT + threadIdx.x;
    if (i < m) {
      const int64_t a0 = __ldg(A.rp + i), a1 = __ldg(A.rp + i + 1);
      int64_t u = 0;                                     // line 2: u_i <- 0
      int lo = INT_MAX, hi = -1;
      int64_t p = a0;
      for (; p + 4 <= a1; p += 4) {                      // line 3: each a_ij in a_i*
        const int j0 = __ldg(A.ci + p), j1 = __ldg(A.ci + p + 1);
        const int j2 = __ldg(A.ci + p + 2), j3 = __ldg(A.ci + p + 3);
        acc_row(u, lo, hi, bwin, j0);
        acc_row(u, lo, hi, bwin, j1);
        acc_row(u, lo, hi, bwin, j2);
        acc_row(u, lo, hi, bwin, j3);
      }
      for (; p < a1; ++p) acc_row(u, lo, hi, bwin, __ldg(A.ci + p));
      const int64_t W = hi >= lo ? int64_t(hi) - lo + 1 : 0;
      const int t = classify(u, n, tp, W);
      U[i] = u;
      tier[i] = (uint8_t)t;
      rlo[i] = lo;
      rhi[i] = hi;
      atomicAdd(&s_hist[t], 1);
      capsum += ctil_capacity(cap_mode, t, u, n, W, tp.bk_min_w);
      if (cap_mode == CAP_HYBRID && t == T_LONG && bk_eligible(u, W, tp.bk_min_w)) {
        bku += (unsigned long long)u;  // hybrid long rows on the bucket path
        ++bkr;
      }
      usum += u;
      umax = u > umax ? u : umax;
      if (t == T_BW) {
        wmax = W > wmax ? W : wmax;
        const int64_t v = u < W ? u : W;
        vmax = v > vmax ? v : vmax;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bku += __shfl_xor_sync(0xffffffffu, bku, o);
    bkr += __shfl_xor_sync(0xffffffffu, bkr, o);
  }
  if ((threadIdx.x & 31) == 0 && bkr > 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(summary + kSumBkU), bku);
    atomicAdd(reinterpret_cast<unsigned long long*>(summary + kSumBkRows), bkr);
  }
  // window maxima of the bw rows: one global atomic per block (the same two addresses for
  // every block: per-row or per-warp atomics serialise at L2)
  {
    __shared__ unsigned long long s_wv[2];
    if (threadIdx.x == 0) s_wv[0] = s_wv[1] = 0ull;
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      wmax = max(wmax, (int64_t)__shfl_xor_sync(0xffffffffu, wmax, o));
      vmax = max(vmax, (int64_t)__shfl_xor_sync(0xffffffffu, vmax, o));
    }
    if ((threadIdx.x & 31) == 0 && wmax > 0) {
      atomicMax(&s_wv[0], (unsigned long long)wmax);
      atomicMax(&s_wv[1], (unsigned long long)vmax);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_wv[0] > 0) {
      atomicMax(reinterpret_cast<unsigned long long*>(summary + kSumWmax), s_wv[0]);
      atomicMax(reinterpret_cast<unsigned long long*>(summary + kSumVmax), s_wv[1]);
    }
  }
  // block reductions
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    capsum += __shfl_xor_sync(0xffffffffu, capsum, o);
    usum += __shfl_xor_sync(0xffffffffu, usum, o);
    const int64_t x = __shfl_xor_sync(0xffffffffu, umax, o);
    umax = x > umax ? x : umax;
  }
  if (lane == 0) {
    s_red[0][w] = capsum;
    s_red[1][w] = usum;
    s_red[2][w] = umax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t c = 0, us = 0, um = 0;
    for (int k = 0; k < NT / 32; ++k) {
      c += s_red[0][k];
      us += s_red[1][k];
      um = s_red[2][k] > um ? s_red[2][k] : um;
    }
    blk_cap[blockIdx.x] = c;
    blk_usum[blockIdx.x] = us;
    blk_umax[blockIdx.x] = um;
  }
  if (threadIdx.x < NUM_TIERS) blk_tier[int64_t(blockIdx.x) * NUM_TIERS + threadIdx.x] = s_hist[threadIdx.x];
}

// PRECISE: classes for the numeric pass from the exact row lengths of the symbolic pass.
template <int NT, int RPT>
__global__ void __launch_bounds__(NT) k_rebin(int64_t m, int64_t n, const int64_t* __restrict__ U,
                                              const int64_t* __restrict__ nnz_row, TierParams tp,
                                              const int32_t* __restrict__ rlo, const int32_t* __restrict__ rhi,
                                              uint8_t* __restrict__ tier, int32_t* __restrict__ blk_tier,
                                              int64_t* __restrict__ blk_cap, int64_t* __restrict__ blk_usum,
                                              int64_t* __restrict__ blk_umax, int64_t* __restrict__ summary) {
  __shared__ int s_hist[NUM_TIERS];
  __shared__ unsigned long long s_vmax;
  if (threadIdx.x < NUM_TIERS) s_hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_vmax = 0ull;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * NT * RPT;
  int64_t vmax = 0;
  unsigned long long bku = 0, bkr = 0;  // long rows on the bucket path (longbk.cu)
  for (int r = 0; r < RPT; ++r) {
    const int64_t i = base + int64_t(r) * NT + threadIdx.x;
    if (i < m) {
      const int t = classify_exact(U[i], nnz_row[i], (int)tier[i], tp);
      tier[i] = (uint8_t)t;
      atomicAdd(&s_hist[t], 1);
      if (t == T_BW) vmax = nnz_row[i] > vmax ? nnz_row[i] : vmax;
      if (t == T_LONG && bk_eligible(U[i], int64_t(rhi[i]) - rlo[i] + 1, tp.bk_min_w)) {
        bku += (unsigned long long)U[i];
        ++bkr;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bku += __shfl_xor_sync(0xffffffffu, bku, o);
    bkr += __shfl_xor_sync(0xffffffffu, bkr, o);
  }
  if ((threadIdx.x & 31) == 0 && bkr > 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(summary + kSumBkU), bku);
    atomicAdd(reinterpret_cast<unsigned long long*>(summary + kSumBkRows), bkr);
  }
  // max nnz(c_i*) of the bw rows: one global atomic per block
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vmax = max(vmax, (int64_t)__shfl_xor_sync(0xffffffffu, vmax, o));
  if ((threadIdx.x & 31) == 0 && vmax > 0) atomicMax(&s_vmax, (unsigned long long)vmax);
  __syncthreads();
  if (threadIdx.x == 0 && s_vmax > 0)
    atomicMax(reinterpret_cast<unsigned long long*>(summary + kSumVmax), s_vmax);
  if (threadIdx.x == 0) {
    blk_cap[blockIdx.x] = 0;
    blk_usum[blockIdx.x] = 0;
    blk_umax[blockIdx.x] = 0;
  }
  if (threadIdx.x < NUM_TIERS) blk_tier[int64_t(blockIdx.x) * NUM_TIERS + threadIdx.x] = s_hist[threadIdx.x];
  (void)n;
}

// ---------------------------------------------------------------------------- stage 2
// One CTA: per class, exclusive scan of per-block counts (class-major order, so perm holds
// class 0 rows, then class 1 rows, ...); exclusive scan of per-block C~ capacities.
template <int NT>
__global__ void __launch_bounds__(NT) k_stage2_scan(int64_t nblk, int32_t* blk_tier,
                                                    int64_t* blk_cap, const int64_t* blk_usum,
                                                    const int64_t* blk_umax, int64_t* summary) {
  __shared__ int64_t s_w[NT / 32 + 1];
  int64_t running = 0;
  for (int t = 0; t < NUM_TIERS; ++t) {
    if (threadIdx.x == 0) summary[kSumOff + t] = running;
    int64_t carry = running;
    for (int64_t b0 = 0; b0 < nblk; b0 += NT) {
      const int64_t b = b0 + threadIdx.x;
      const int64_t v = b < nblk ? blk_tier[b * NUM_TIERS + t] : 0;
      int64_t tot;
      const int64_t ex = block_excl_scan<NT>(v, &tot, s_w);
      if (b < nblk) blk_tier[b * NUM_TIERS + t] = (int32_t)(carry + ex);
      carry += tot;
    }
    if (threadIdx.x == 0) summary[kSumCount + t] = carry - running;
    running = carry;
  }
  if (threadIdx.x == 0) summary[kSumOff + NUM_TIERS] = running;
  int64_t carry = 0, us = 0, um = 0;
  for (int64_t b0 = 0; b0 < nblk; b0 += NT) {
    const int64_t b = b0 + threadIdx.x;
    const int64_t v = b < nblk ? blk_cap[b] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan<NT>(v, &tot, s_w);
    if (b < nblk) blk_cap[b] = carry + ex;
    carry += tot;
    if (b < nblk) {
      us += blk_usum[b];
      um = blk_umax[b] > um ? blk_umax[b] : um;
    }
  }
  // reduce us / um
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    us += __shfl_xor_sync(0xffffffffu, us, o);
    const int64_t x = __shfl_xor_sync(0xffffffffu, um, o);
    um = x > um ? x : um;
  }
  __shared__ int64_t s_u[NT / 32], s_m[NT / 32];
  if ((threadIdx.x & 31) == 0) {
    s_u[threadIdx.x >> 5] = us;
    s_m[threadIdx.x >> 5] = um;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t a = 0, b = 0;
    for (int k = 0; k < NT / 32; ++k) {
      a += s_u[k];
      b = s_m[k] > b ? s_m[k] : b;
    }
    summary[kSumU] = a;
    summary[kSumUMax] = b;
    summary[kSumCap] = carry;
  }
}

template <int NT, int RPT>
__global__ void __launch_bounds__(NT) k_stage2_scatter(int64_t m, int64_t n, int cap_mode, int64_t bk_min_w,
                                                       const uint8_t* __restrict__ tier,
                                                       const int64_t* __restrict__ U,
                                                       const int32_t* __restrict__ rlo,
                                                       const int32_t* __restrict__ rhi,
                                                       const int32_t* __restrict__ blk_tier_off,
                                                       const int64_t* __restrict__ blk_cap_off,
                                                       int32_t* __restrict__ perm,
                                                       int64_t* __restrict__ ctil_off) {
  constexpr int NW = NT / 32;
  __shared__ int s_run[NUM_TIERS];
  __shared__ int s_wcnt[NW][NUM_TIERS + 1];
  __shared__ int64_t s_w[NW + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x < NUM_TIERS) s_run[threadIdx.x] = blk_tier_off[int64_t(blockIdx.x) * NUM_TIERS + threadIdx.x];
  for (int k = threadIdx.x; k < NW * (NUM_TIERS + 1); k += NT) (&s_wcnt[0][0])[k] = 0;
  int64_t cap_carry = blk_cap_off[blockIdx.x];
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * NT * RPT;
#pragma unroll 1
  for (int r = 0; r < RPT; ++r) {
    const int64_t i = base + int64_t(r) * NT + threadIdx.x;
    const bool valid = i < m;
    const int t = valid ? (int)tier[i] : NUM_TIERS;
    const int64_t cap = valid && cap_mode != CAP_NONE
                            ? ctil_capacity(cap_mode, t, U[i], n, int64_t(rhi[i]) - rlo[i] + 1, bk_min_w) : 0;
    const unsigned peers = __match_any_sync(0xffffffffu, t);
    const int wrank = __popc(peers & lanemask_lt());
    if (wrank == 0) s_wcnt[w][t] = __popc(peers);
    int64_t tot;
    const int64_t ex = block_excl_scan<NT>(cap, &tot, s_w);  // contains __syncthreads
    if (valid) {
      int pos = s_run[t] + wrank;
      for (int k = 0; k < w; ++k) pos += s_wcnt[k][t];
      perm[pos] = (int32_t)i;
      if (cap_mode != CAP_NONE) ctil_off[i] = cap_carry + ex;
    }
    cap_carry += tot;
    __syncthreads();
    if (threadIdx.x < NUM_TIERS) {
      int s = 0;
      for (int k = 0; k < NW; ++k) {
        s += s_wcnt[k][threadIdx.x];
        s_wcnt[k][threadIdx.x] = 0;
      }
      s_run[threadIdx.x] += s;
    }
    __syncthreads();
  }
  (void)lane;
}

// ------------------------------------------------------------------- generic scan
constexpr int kScanNT = 512;
constexpr int kScanIPT = 8;
constexpr int64_t kScanTile = int64_t(kScanNT) * kScanIPT;

__global__ void __launch_bounds__(kScanNT) k_scan_reduce(const int64_t* __restrict__ x, int64_t len,
                                                         int64_t* __restrict__ part) {
  __shared__ int64_t s_w[kScanNT / 32];
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    const int64_t i = base + int64_t(k) * kScanNT + threadIdx.x;
    if (i < len) s += x[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int k = 0; k < kScanNT / 32; ++k) t += s_w[k];
    part[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_top(int64_t* part, int64_t nb) {
  __shared__ int64_t s_w[1024 / 32 + 1];
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
    const int64_t b = b0 + threadIdx.x;
    const int64_t v = b < nb ? part[b] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan<1024>(v, &tot, s_w);
    if (b < nb) part[b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) part[nb] = carry;
}

__global__ void __launch_bounds__(kScanNT) k_scan_down(const int64_t* __restrict__ x, int64_t len,
                                                       const int64_t* __restrict__ part,
                                                       int64_t nb, int64_t* __restrict__ y) {
  __shared__ int64_t s_w[kScanNT / 32 + 1];
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  // each thread owns kScanIPT consecutive elements
  int64_t v[kScanIPT];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    const int64_t i = base + int64_t(threadIdx.x) * kScanIPT + k;
    v[k] = i < len ? x[i] : 0;
    s += v[k];
  }
  int64_t tot;
  int64_t ex = block_excl_scan<kScanNT>(s, &tot, s_w) + part[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanIPT; ++k) {
    const int64_t i = base + int64_t(threadIdx.x) * kScanIPT + k;
    if (i < len) y[i] = ex;
    ex += v[k];
  }
  if (blockIdx.x == nb - 1 && threadIdx.x == 0) y[len] = part[nb];
}

// ------------------------------------------------------------------ CSR validation
__global__ void k_validate(int64_t rows, int64_t cols, const int64_t* __restrict__ rp,
                           const int32_t* __restrict__ ci, int64_t nnz, int32_t* err) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) {
    if (rp[0] != 0) atomicOr(err, 1);
    if (rp[rows] != nnz) atomicOr(err, 4);
  }
  if (i >= rows) return;
  const int64_t a = rp[i], b = rp[i + 1];
  if (b < a) {
    atomicOr(err, 2);
    return;
  }
  if (a < 0 || b > nnz) {
    atomicOr(err, 4);
    return;
  }
  int prev = -1;
  for (int64_t p = a; p < b; ++p) {
    const int c = ci[p];
    if (c < 0 || int64_t(c) >= cols) atomicOr(err, 8);
    if (c <= prev) atomicOr(err, 16);
    prev = c;
  }
}

}  // namespace

cudaError_t launch_stage1(int64_t m, int64_t k, int64_t n, CsrView A, CsrView B, TierParams tp,
                          int cap_mode, Stage12Ws& ws, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(ws.summary + kSumWmax, 0, 5 * sizeof(int64_t), s);  // .. kSumBkRows
  if (e != cudaSuccess) return e;
  if (k > 0) k_bwin<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(k, B.rp, B.ci, ws.bwin);
  k_stage1<kS12Threads, kS12RowsPerThread><<<(unsigned)ws.nblk, kS12Threads, 0, s>>>(
      m, n, A, B.rp, ws.bwin, tp, cap_mode, ws.U, ws.tier, ws.rlo, ws.rhi, ws.blk_tier, ws.blk_cap,
      ws.blk_usum, ws.blk_umax, ws.summary);
  return cudaGetLastError();
}

cudaError_t launch_stage2(int64_t m, Stage12Ws& ws, int cap_mode, int64_t n, int64_t bk_min_w, cudaStream_t s) {
  k_stage2_scan<1024><<<1, 1024, 0, s>>>(ws.nblk, ws.blk_tier, ws.blk_cap, ws.blk_usum, ws.blk_umax,
                                         ws.summary);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || m == 0) return e;
  k_stage2_scatter<kS12Threads, kS12RowsPerThread><<<(unsigned)ws.nblk, kS12Threads, 0, s>>>(
      m, n, cap_mode, bk_min_w, ws.tier, ws.U, ws.rlo, ws.rhi, ws.blk_tier, ws.blk_cap, ws.perm, ws.ctil_off);
  return cudaGetLastError();
}

cudaError_t launch_rebin(int64_t m, int64_t n, const int64_t* nnz_row, TierParams tp, Stage12Ws& ws,
                         cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(ws.summary + kSumVmax, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ws.summary + kSumBkU, 0, 2 * sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  k_rebin<kS12Threads, kS12RowsPerThread><<<(unsigned)ws.nblk, kS12Threads, 0, s>>>(
      m, n, ws.U, nnz_row, tp, ws.rlo, ws.rhi, ws.tier, ws.blk_tier, ws.blk_cap, ws.blk_usum, ws.blk_umax, ws.summary);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_stage2(m, ws, CAP_NONE, n, tp.bk_min_w, s);
}

int64_t scan_tmp_elems(int64_t len) { return (len + kScanTile - 1) / kScanTile + 2; }

cudaError_t launch_exclusive_scan(const int64_t* x, int64_t* y, int64_t len, int64_t* tmp,
                                  cudaStream_t s) {
  if (len == 0) return cudaMemsetAsync(y, 0, sizeof(int64_t), s);
  const int64_t nb = (len + kScanTile - 1) / kScanTile;
  k_scan_reduce<<<(unsigned)nb, kScanNT, 0, s>>>(x, len, tmp);
  k_scan_top<<<1, 1024, 0, s>>>(tmp, nb);
  k_scan_down<<<(unsigned)nb, kScanNT, 0, s>>>(x, len, tmp, nb, y);
  return cudaGetLastError();
}

cudaError_t launch_validate(int64_t rows, int64_t cols, const int64_t* rp, const int32_t* ci,
                            int64_t nnz, int32_t* err, cudaStream_t s) {
  const int64_t nb = rows / 256 + 1;
  k_validate<<<(unsigned)nb, 256, 0, s>>>(rows, cols, rp, ci, nnz, err);
  return cudaGetLastError();
}

}  // namespace sg
