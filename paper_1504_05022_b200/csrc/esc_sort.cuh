// esc_sort.cuh — the "sort" and "compress" steps of the ESC ([P:277-284]) for one row (or one
// bucket of a long row) whose products sit in shared memory in product order p (Algorithm 1:
// j ascending, then k): key[p] = column - base (< 2^kb), pval[p] = a_ij·b_jk.
//
// Sort by (key, p) — so equal columns keep product order and each sum runs in the oracle's
// order — in one counting pass plus small sorts instead of a radix sort over all key bits:
//   1. bucket b = key >> s, with about 32 products per bucket (2^lnb buckets, lnb from u);
//   2. histogram, scan, scatter of the composite ((key & (2^s - 1)) << pb) | p into its bucket
//      (order inside a bucket does not matter: the composite is unique and carries p);
//   3. each bucket sorted by one warp: a register bitonic network for <= 32 or <= 64 items,
//      a shared-memory bitonic network (virtual +inf padding) above that.
// Buckets are in key order and composites order (low key bits, p), so the whole sequence is
// ordered by (key, p).  Compress: runs of equal columns summed left to right (lines 9, 11),
// heads counted by a block scan, the row written in column order.
#pragma once
#include "common.cuh"

namespace sg {
namespace escs {

constexpr unsigned kFull = 0xffffffffu;

// NBMAX buckets at most: enough for ~32 products per bucket, and for key + product bits within
// 32 while the window has at most kMaxKeyBits(CAP) bits (launchers check n against it)
template <int CAP, typename V>
struct Smem {
  static constexpr int NBMAX = CAP / 8;
  unsigned key[CAP];
  V pval[CAP];
  unsigned arr[CAP];
  int bst[NBMAX + 1];
  int bcur[NBMAX];
};

__device__ __forceinline__ int ceil_log2(unsigned x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c((x + 1) / 2); }
// widest key (window) the composite (key low bits, p) fits 32 bits for with NBMAX buckets
template <int CAP>
__host__ __device__ constexpr int max_key_bits() { return 32 - ilog2c(CAP) + ilog2c(CAP / 8); }

template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* total, int* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += x;
  }
  if (NT == 32) {
    *total = __shfl_sync(kFull, inc, 31);
    return inc - v;
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

// ascending bitonic network over element e = h·32 + lane, H registers per lane (H = 1, 2);
// the first comparator of each merge of size k pairs e with e ^ (k - 1) (the "flip"), so every
// comparator puts the minimum at the lower index
template <int H>
__device__ __forceinline__ void warp_bitonic(unsigned (&v)[H], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * H; k <<= 1) {
#pragma unroll
    for (int m = k - 1; m > 0; m = (m == k - 1) ? (k >> 2) : (m >> 1)) {
      const int hb = (m == k - 1) ? (k >> 1) : m;  // the bit that tells the lower index
      if (m & 32) {  // H == 2: pairs (lane, h=0) <-> (lane ^ (m & 31), h=1)
        const unsigned t1 = __shfl_xor_sync(kFull, v[H - 1], m & 31);
        const unsigned t0 = __shfl_xor_sync(kFull, v[0], m & 31);
        v[0] = min(v[0], t1);
        v[H - 1] = max(v[H - 1], t0);
      } else {
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const unsigned t = __shfl_xor_sync(kFull, v[h], m);
          v[h] = (lane & hb) ? max(v[h], t) : min(v[h], t);
        }
      }
      if (m == 1) break;
    }
  }
}

// one warp sorts a[0, n) in shared memory (n > 64): ascending bitonic network over the next
// power of two, indices >= n are +inf and never move
__device__ __forceinline__ void warp_bitonic_smem(unsigned* a, int n, int lane) {
  const int P = 1 << ceil_log2((unsigned)n);
  for (int k = 2; k <= P; k <<= 1) {
    for (int m = k - 1; m > 0; m = (m == k - 1) ? (k >> 2) : (m >> 1)) {
      for (int q = lane; q < P / 2; q += 32) {
        int i, j;
        if (m == k - 1) {
          const int half = k >> 1;
          const int blk = q / half, r = q % half;
          i = blk * k + r;
          j = blk * k + k - 1 - r;
        } else {
          i = ((q & ~(m - 1)) << 1) | (q & (m - 1));
          j = i | m;
        }
        if (j < n) {
          const unsigned x = a[i], y = a[j];
          if (y < x) {
            a[i] = y;
            a[j] = x;
          }
        }
      }
      __syncwarp();
      if (m == 1) break;
    }
  }
}

// Sort the u <= CAP products (key[], pval[] in product order; keys < 2^kb) by (key, p) into
// sm.arr (composites).  Returns pb (sm.arr[x] & (2^pb - 1) is the product index at x).
template <int NT, int CAP, typename V>
__device__ __forceinline__ int sort_products(Smem<CAP, V>& sm, int u, int kb) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int pb = ceil_log2((unsigned)u) > 0 ? ceil_log2((unsigned)u) : 1;
#ifndef SG_ESC_BKT
#define SG_ESC_BKT 32
#endif
  int lnb = ceil_log2((unsigned)((u + SG_ESC_BKT - 1) / SG_ESC_BKT));  // ~SG_ESC_BKT products per bucket
  lnb = max(lnb, kb + pb - 32);
  lnb = min(lnb, ceil_log2(Smem<CAP, V>::NBMAX));
  lnb = min(lnb, kb);
  const int s = kb - lnb;
  const int NB = 1 << lnb;
  const unsigned smask = (s >= 32) ? 0xffffffffu : ((1u << s) - 1u);
  for (int b = tid; b < NB; b += NT) sm.bcur[b] = 0;
  __syncthreads();
  for (int p = tid; p < u; p += NT) atomicAdd(&sm.bcur[sm.key[p] >> s], 1);
  __syncthreads();
  {
    constexpr int PER = (Smem<CAP, V>::NBMAX + NT - 1) / NT;
    const int b0 = tid * ((NB + NT - 1) / NT);
    const int nb = min((NB + NT - 1) / NT, max(0, NB - b0));
    int c[PER];
    int loc = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      c[q] = q < nb ? sm.bcur[b0 + q] : 0;
      loc += c[q];
    }
    __shared__ int s_w[NW + 1];
    int tot;
    int run = block_excl_scan<NT>(loc, &tot, s_w);
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (q < nb) {
        sm.bst[b0 + q] = run;
        sm.bcur[b0 + q] = run;
        run += c[q];
      }
    if (tid == 0) sm.bst[NB] = tot;
  }
  __syncthreads();
  for (int p = tid; p < u; p += NT) {
    const unsigned k = sm.key[p];
    const int pos = atomicAdd(&sm.bcur[k >> s], 1);
    sm.arr[pos] = ((k & smask) << pb) | (unsigned)p;
  }
  __syncthreads();
  for (int b = w; b < NB; b += NW) {
    const int st = sm.bst[b], n = sm.bst[b + 1] - st;
    if (n <= 1) continue;
    if (n <= 32) {
      unsigned v[1] = {lane < n ? sm.arr[st + lane] : 0xffffffffu};
      warp_bitonic<1>(v, lane);
      if (lane < n) sm.arr[st + lane] = v[0];
    } else if (n <= 64) {
      unsigned v[2] = {sm.arr[st + lane], 32 + lane < n ? sm.arr[st + 32 + lane] : 0xffffffffu};
      warp_bitonic<2>(v, lane);
      sm.arr[st + lane] = v[0];
      if (32 + lane < n) sm.arr[st + 32 + lane] = v[1];
    } else {
      warp_bitonic_smem(sm.arr + st, n, lane);
    }
  }
  __syncthreads();
  return pb;
}

// Compress the sorted products: the row's distinct columns (base + key) in order with their
// sums (left to right in product order: lines 9, 11), written to out_col / out_val from
// position 0.  Returns the number of distinct columns.
template <int NT, int CAP, typename V>
__device__ __forceinline__ int compress_write(Smem<CAP, V>& sm, int u, int pb, int base, int32_t* out_col,
                                              V* out_val) {
  constexpr int IPT = CAP / NT;
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x;
  const unsigned pm = (1u << pb) - 1u;
  unsigned kk[IPT];
  V acc[IPT];
  int heads = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int x = tid * IPT + i;
    kk[i] = 0xffffffffu;
    if (x < u) {
      const unsigned p = sm.arr[x] & pm;
      const unsigned k = sm.key[p];
      const bool head = x == 0 || sm.key[sm.arr[x - 1] & pm] != k;
      if (head) {
        V a = sm.pval[p];
        for (int y = x + 1; y < u; ++y) {
          const unsigned q = sm.arr[y] & pm;
          if (sm.key[q] != k) break;
          a = Arith<V>::add(a, sm.pval[q]);
        }
        acc[i] = a;
        kk[i] = k;
        ++heads;
      }
    }
  }
  __shared__ int s_w[NW + 1];
  int nnz;
  int pos = block_excl_scan<NT>(heads, &nnz, s_w);
#pragma unroll
  for (int i = 0; i < IPT; ++i)
    if (kk[i] != 0xffffffffu) {
      out_col[pos] = (int)kk[i] + base;
      out_val[pos] = acc[i];
      ++pos;
    }
  return nnz;
}

}  // namespace escs
}  // namespace sg
