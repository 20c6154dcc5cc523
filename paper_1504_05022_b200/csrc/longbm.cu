// longbm.cu — rows too long for one shared-memory class (the paper's group 5, [P:222],
// [P:286-297]) and, for values, the CTA-hash classes: a bitmap over the row's column window.
//
// The precise method ([P:165]) first computes the structure, then the values.  The structure
// of row i is the set of columns hit by its products: one bit per column of the window
// [lo, hi] in shared memory, processed in tiles of at most `tile words` x 32 columns.
//   k_long_bm_count : per tile, set the bits of all products' columns (red.shared.or), count
//                     them.  nnz(c_i*) = total popcount.  No hashing, no probing, no ordering.
//   k_long_rank     : per tile, rebuild the bits, exclusive prefix popcount per 32-bit word
//                     -> rank(c) = prefix[w] + popc(bits[w] & below(c)) is c's position in
//                     the sorted row; write the row's columns in order.  Values (lines 6, 9,
//                     11 of Algorithm 1): the tile's ranks are split into NW equal ranges, one
//                     per warp; every warp walks the row's a_ij in j-ascending order and, of
//                     each b_j*, only the segment whose columns fall in its range (found by
//                     binary search: b_j* is sorted), adding a_ij*b_jk into its own ranks of
//                     the output in place.  Each column is therefore accumulated by one warp,
//                     in j-ascending order, starting from -0.0 (the identity of +): the
//                     oracle's order, bit for bit, with no atomics (R1, reading Q1).
// Tiles exist only because shared memory is finite (c3a: n = 4 Mi columns); a row whose
// window spans several tiles restricts every b_j* to the tile's columns by binary search
// too, so each tile visits only its own products (plus one search per a_ij).
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace sg {

namespace {

constexpr int kBmNT = 512;                        // count kernel
constexpr int kRkNT = 256;                        // rank kernel
constexpr int kRkNW = kRkNT / 32;
constexpr int kDefaultCountTileWords = 32768;     // 1 Mi columns (128 KB)
constexpr int kDefaultRankTileWords = 8192;       // 256 Ki columns (64 KB bits + 32 KB ranks)
constexpr int kChunk = 256;                       // products per work item (load balance)

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

// the row's column window: first / last column of every b_j* (the (first, last) record of
// stage 1, a.bwin)
template <int NT>
__device__ __forceinline__ void row_window(const Stage3Args& a, int64_t a0, int64_t a1, int* s_red,
                                           int& lo, int& hi) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int l = INT_MAX, h = -1;
  for (int64_t e = a0 + threadIdx.x; e < a1; e += NT) {
    const int4 bw = __ldg(a.bwin + __ldg(a.A.ci + e));
    l = min(l, bw.x);
    h = max(h, bw.y);
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
  for (int k = 0; k < NT / 32; ++k) {
    lo = min(lo, s_red[2 * k]);
    hi = max(hi, s_red[2 * k + 1]);
  }
  __syncthreads();
}

// first position q in b_j* = B.ci[bs, bs+len) with B.ci[q] >= c (first/last: b_j*'s range)
__device__ __forceinline__ int lower_bound_row(const int32_t* __restrict__ bci, int64_t bs, int len, int first,
                                               int last, int64_t c) {
  if (c <= first) return 0;
  if (c > last) return len;
  int lo = 0, hi = len;  // bci[bs+lo-1] < c <= bci[bs+hi]
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(bci + bs + mid) < c) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// A batch of up to NT a_ij of the row, staged in shared memory, with each b_j*'s segment
// [s0, s1) restricted to the current tile and its cut into kChunk-product work items.
template <int NT>
struct Batch {
  long long bs[NT];
  int len[NT];
  int s0[NT];
  int cinc[NT];  // inclusive scan of work items per a_ij
  double av[NT];
};

// Stage the batch [e0, e0+NT) (thread t <-> a_ij t) restricted to columns [cbeg, cend).
template <int NT, bool VALS>
__device__ __forceinline__ int stage_batch(const Stage3Args& a, int64_t e0, int64_t a1, int64_t cbeg, int64_t cend,
                                           bool restrict_cols, Batch<NT>& sb, int* s_w) {
  const int64_t e = e0 + threadIdx.x;
  int s0 = 0, s1 = 0;
  if (e < a1) {
    const int j = __ldg(a.A.ci + e);
    const int4 bw = __ldg(a.bwin + j);
    const int64_t bs = __ldg(a.B.rp + j);
    const int len = bw.z;
    s1 = len;
    if (restrict_cols && len > 0) {
      s0 = lower_bound_row(a.B.ci, bs, len, bw.x, bw.y, cbeg);
      s1 = lower_bound_row(a.B.ci, bs, len, bw.x, bw.y, cend);
    }
    sb.bs[threadIdx.x] = bs;
    sb.len[threadIdx.x] = s1;
    sb.s0[threadIdx.x] = s0;
    if (VALS) sb.av[threadIdx.x] = __ldg(a.A.val + e);
  }
  const int nch = (s1 - s0 + kChunk - 1) / kChunk;
  int tot;
  const int ex = block_excl_scan_i<NT>(nch, &tot, s_w);
  sb.cinc[threadIdx.x] = ex + nch;
  __syncthreads();
  return tot;
}

// Work item -> (a_ij slot t, product range [q0, qe) of b_j*), balanced over warps.
template <int NT>
__device__ __forceinline__ void work_item(const Batch<NT>& sb, int item, int& t, int64_t& q0, int64_t& qe) {
  int lo = 0, hi = NT - 1;  // first t with cinc[t] > item
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sb.cinc[mid] > item) hi = mid;
    else lo = mid + 1;
  }
  t = lo;
  const int first_item = sb.cinc[t] - (sb.len[t] - sb.s0[t] + kChunk - 1) / kChunk;
  q0 = sb.bs[t] + sb.s0[t] + int64_t(item - first_item) * kChunk;
  qe = min(q0 + kChunk, (int64_t)sb.bs[t] + sb.len[t]);
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

__device__ __forceinline__ void sh_red_or(unsigned* p, unsigned v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

// Bits of the products [q0, qe) (at most kChunk) of one b_j* (columns already restricted to
// the tile at base): the column loads of the whole work item are issued before the shared-
// memory ORs, so the gathers overlap instead of one round trip per 32 products.
__device__ __forceinline__ void set_bits(const int32_t* __restrict__ bci, int64_t q0, int64_t qe, int lane,
                                         int64_t base, unsigned* bm) {
  constexpr int K = kChunk / 32;
  unsigned d[K];
#pragma unroll
  for (int u = 0; u < K; ++u) {
    const int64_t q = q0 + 32 * u + lane;
    d[u] = q < qe ? (unsigned)(__ldg(bci + q) - base) : 0xffffffffu;
  }
#pragma unroll
  for (int u = 0; u < K; ++u)
    if (d[u] != 0xffffffffu) sh_red_or(&bm[d[u] >> 5], 1u << (d[u] & 31));
}

// Words of a tile: the row's window in multiples of NT words, at most tmax.
template <int NT>
__device__ __forceinline__ int tile_words(int lo, int hi, int64_t tmax) {
  const int64_t wwords = (int64_t(hi) - lo) / 32 + 1;
  const int64_t t = wwords < tmax ? wwords : tmax;
  return (int)((t + NT - 1) / NT * NT);
}

// ------------------------------------------------------------------------- count (symbolic)
__global__ void __launch_bounds__(kBmNT) k_long_bm_count(Stage3Args a, int tmax) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* bm = reinterpret_cast<unsigned*>(smem);
  __shared__ int s_red[2 * (kBmNT / 32)];
  __shared__ int s_w[kBmNT / 32 + 1];
  __shared__ Batch<kBmNT> sb;
  __shared__ unsigned long long s_cnt;
  __shared__ int64_t s_next;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t r = blockIdx.x; r < a.count; r = next_row(a, r, &s_next)) {
    const int row = __ldg(a.perm + a.first + r);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    int lo, hi;
    row_window<kBmNT>(a, a0, a1, s_red, lo, hi);
    if (threadIdx.x == 0) s_cnt = 0;
    const int tw = tile_words<kBmNT>(lo, hi, tmax);
    const int64_t tbits = int64_t(tw) * 32;
    const bool multi = int64_t(hi) - lo + 1 > tbits;
    for (int64_t base = lo; base <= hi; base += tbits) {
      for (int k = threadIdx.x; k < tw; k += kBmNT) bm[k] = 0u;
      __syncthreads();
      for (int64_t e0 = a0; e0 < a1; e0 += kBmNT) {
        const int items = stage_batch<kBmNT, false>(a, e0, a1, base, base + tbits, multi, sb, s_w);
        for (int item = w; item < items; item += kBmNT / 32) {
          int t;
          int64_t q0, qe;
          work_item<kBmNT>(sb, item, t, q0, qe);
          set_bits(a.B.ci, q0, qe, lane, base, bm);  // line 8: insert
        }
        __syncthreads();
      }
      unsigned c = 0;
      for (int k = threadIdx.x; k < tw; k += kBmNT) c += __popc(bm[k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0) atomicAdd(&s_cnt, (unsigned long long)c);
      __syncthreads();
    }
    if (threadIdx.x == 0 && a.nnz_row) a.nnz_row[row] = (int64_t)s_cnt;
    __syncthreads();
  }
}

// --------------------------------------------------------------------- rank fill (values)
// Output of work index r (position in the class): C's row at out_off[row] (precise, C~
// classes); PROG (hybrid long rows, the paper's progressive allocation [P:297]): long row
// k = active[r], written through its chunk table into the long-row arena; a tile whose
// entries do not fit the row's current capacity is the checkpoint — the row stops there
// (earlier tiles stay written), reports how much it needs, and resumes at that tile after the
// host has grown its allocation.
template <int NT, bool PROG, typename VT>
__global__ void __launch_bounds__(NT) k_long_rank(Stage3Args a, int tmax) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* bm = reinterpret_cast<unsigned*>(smem);
  int* pre = reinterpret_cast<int*>(smem + size_t(tmax) * sizeof(unsigned));
  __shared__ int s_red[2 * NW];
  __shared__ int s_w[NW + 1];
  __shared__ Batch<NT> sb;
  __shared__ int s_split[NT][NW + 1];
  __shared__ int s_cb[NW + 1];
  __shared__ int64_t s_next;
  __shared__ int64_t s_tab[PROG ? kMaxChunks : 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t count = a.count_dev ? (int64_t)*a.count_dev : a.count;  // fallback lists: on the device
  for (int64_t r = blockIdx.x; r < count; r = next_row(a, r, &s_next)) {
    const int k_long = PROG ? __ldg(a.active + r) : 0;
    const int row = __ldg(a.perm + a.first + (PROG ? int64_t(k_long) : r));
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    int32_t* oc;
    VT* ov;
    int64_t done = 0;  // entries of the row placed by earlier tiles
    int64_t cap = 0, start = INT64_MIN;
    if (PROG) {
      oc = a.arena_col;
      ov = vcast<VT>(a.arena_val);
      const LongState st = a.lst[k_long];
      done = st.count;
      cap = st.cap;
      start = st.next_col;
      if (threadIdx.x < kMaxChunks) s_tab[threadIdx.x] = a.chunk_table[int64_t(k_long) * kMaxChunks + threadIdx.x];
    } else {
      const int64_t o = __ldg(a.out_off + row);
      oc = a.out_col + o;
      ov = vcast<VT>(a.out_val) + o;
    }
    // row position p -> element of oc / ov
    auto at_pos = [&](int64_t p) -> int64_t { return PROG ? s_tab[chunk_of(p, a.log2c0)] + p : p; };
    int lo, hi;
    row_window<NT>(a, a0, a1, s_red, lo, hi);
    const int tw = tile_words<NT>(lo, hi, tmax);
    const int64_t tbits = int64_t(tw) * 32;
    const bool multi = int64_t(hi) - lo + 1 > tbits;
    const int WPT = tw / NT;  // words per thread in the prefix scan
    bool overflow = false;
    for (int64_t base = start == INT64_MIN ? lo : start; base <= hi; base += tbits) {
      const int64_t tend = min(base + tbits, int64_t(hi) + 1);
      for (int k = threadIdx.x; k < tw; k += NT) bm[k] = 0u;
      __syncthreads();
      // 1. the tile's bits (line 8 of Algorithm 1 for every product of the tile)
      for (int64_t e0 = a0; e0 < a1; e0 += NT) {
        const int items = stage_batch<NT, false>(a, e0, a1, base, tend, multi, sb, s_w);
        for (int item = w; item < items; item += NW) {
          int t;
          int64_t q0, qe;
          work_item<NT>(sb, item, t, q0, qe);
          set_bits(a.B.ci, q0, qe, lane, base, bm);  // line 8: insert
        }
        __syncthreads();
      }
      // 2. exclusive prefix popcount per word (thread t owns words [t*WPT, (t+1)*WPT)); the
      //    tile's columns in order; values start at -0.0 (the identity of +: the first add
      //    is line 9's assignment)
      int loc = 0;
      for (int k = 0; k < WPT; ++k) loc += __popc(bm[threadIdx.x * WPT + k]);
      int T;
      int run = block_excl_scan_i<NT>(loc, &T, s_w);
      if (PROG && done + T > cap) {
        // checkpoint ([P:297] "records current computation position"): this tile and the rest
        // of the row wait for a larger allocation
        if (threadIdx.x == 0) {
          a.lst[k_long].next_col = base;
          a.lst[k_long].count = done;
          a.lst[k_long].need = done + T;
          a.ovf_list[atomicAdd(a.ovf_cnt, 1)] = k_long;
        }
        overflow = true;
        break;
      }
      const int run0 = run;
      for (int k = 0; k < WPT; ++k) {
        const int wi = threadIdx.x * WPT + k;
        unsigned b = bm[wi];
        pre[wi] = run;
        int p = run;
        const int cb = (int)(base + int64_t(wi) * 32);
        while (b) {
          oc[at_pos(done + p)] = cb + __ffs(b) - 1;
          b &= b - 1;
          ++p;
        }
        run = p;
      }
      // 3. values.  The tile's ranks are split into NW equal ranges: warp k owns the ranks
      //    [floor(k*T/NW), floor((k+1)*T/NW)), i.e. the columns [cb[k], cb[k+1]); every warp
      //    walks the a_ij in j-ascending order and adds, of each b_j*, only the products of its
      //    own columns.  The values accumulate in place in the output (L2).
      {
        const int w0 = 0, wn = T;
        for (int k = 0; k <= NW; ++k) {
          const int rk = w0 + (k < NW ? (int)((int64_t(k) * wn) / NW) : wn);
          if (rk >= T) {
            if (threadIdx.x == 0) s_cb[k] = (int)tend;
          } else if (rk >= run0 && rk < run) {  // the word holding rank rk is one of mine
            int q = run0;
            for (int kk = 0; kk < WPT; ++kk) {
              const int wi = threadIdx.x * WPT + kk;
              unsigned b = bm[wi];
              const int pc = __popc(b);
              if (rk < q + pc) {
                for (int z = rk - q; z > 0; --z) b &= b - 1;  // drop the lower set bits
                s_cb[k] = (int)(base + int64_t(wi) * 32 + __ffs(b) - 1);
                break;
              }
              q += pc;
            }
          }
        }
        for (int i = threadIdx.x; i < wn; i += NT) ov[at_pos(done + i)] = VT(-0.0);  // identity of + (line 9)
        __syncthreads();
        for (int64_t e0 = a0; e0 < a1; e0 += NT) {
          const int64_t e = e0 + threadIdx.x;
          if (e < a1) {
            const int j = __ldg(a.A.ci + e);
            const int4 bw = __ldg(a.bwin + j);
            const int64_t bs = __ldg(a.B.rp + j);
            sb.bs[threadIdx.x] = bs;
            sb.av[threadIdx.x] = (double)__ldg(vcast<VT>(a.A.val) + e);  // exact for float too
            // lower bounds of the warps' column boundaries in b_j* (binary searches advanced
            // in lockstep, their loads in flight together): first the window's own segment
            // [s0, s1) (pruned by b_j*'s first / last column), then the NW-1 interior
            // boundaries inside that segment only
            int lo_k[NW + 1], hi_k[NW + 1];
#pragma unroll
            for (int k = 0; k <= NW; k += NW) {
              const int c = s_cb[k];
              lo_k[k] = (bw.z == 0 || c <= bw.x) ? 0 : (c > bw.y ? bw.z : 1);
              hi_k[k] = (bw.z == 0 || c <= bw.x) ? 0 : (c > bw.y ? bw.z : bw.z - 1);
            }
            // invariant: bci[bs + lo - 1] < c <= bci[bs + hi]
            for (bool more = true; more;) {
              more = false;
#pragma unroll
              for (int k = 0; k <= NW; k += NW) {
                if (lo_k[k] < hi_k[k]) {
                  const int mid = (lo_k[k] + hi_k[k]) >> 1;
                  if (__ldg(a.B.ci + bs + mid) < s_cb[k]) lo_k[k] = mid + 1;
                  else hi_k[k] = mid;
                  more = more || lo_k[k] < hi_k[k];
                }
              }
            }
#pragma unroll
            for (int k = 1; k < NW; ++k) {
              lo_k[k] = lo_k[0];
              hi_k[k] = lo_k[NW];
            }
            for (bool more = lo_k[0] < lo_k[NW]; more;) {
              more = false;
#pragma unroll
              for (int k = 1; k < NW; ++k) {
                if (lo_k[k] < hi_k[k]) {
                  const int mid = (lo_k[k] + hi_k[k]) >> 1;
                  if (__ldg(a.B.ci + bs + mid) < s_cb[k]) lo_k[k] = mid + 1;
                  else hi_k[k] = mid;
                  more = more || lo_k[k] < hi_k[k];
                }
              }
            }
#pragma unroll
            for (int k = 0; k <= NW; ++k) s_split[threadIdx.x][k] = lo_k[k];
          }
          __syncthreads();
          const int na = (int)min(int64_t(NT), a1 - e0);
          for (int t = 0; t < na; ++t) {
            const int s0 = s_split[t][w], en = s_split[t][w + 1];
            if (s0 >= en) continue;
            const int32_t* __restrict__ sc = a.B.ci + sb.bs[t];
            const VT* __restrict__ sv = vcast<VT>(a.B.val) + sb.bs[t];
            const VT at = (VT)sb.av[t];
            // columns inside one b_j* are distinct: the chunks of a segment touch distinct
            // outputs, so four of them are gathered, ranked and updated together
            for (int q0 = s0; q0 < en; q0 += 128) {
              int x[4];
              VT v[4], old[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int q = q0 + 32 * u + lane;
                x[u] = -1;
                if (q < en) {
                  const unsigned d = (unsigned)(__ldg(sc + q) - base);
                  v[u] = __ldg(sv + q);
                  const unsigned wd = d >> 5;
                  x[u] = pre[wd] + __popc(bm[wd] & ((1u << (d & 31)) - 1u)) - w0;
                }
              }
              VT* p[4];
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (x[u] >= 0) {
                  p[u] = ov + at_pos(done + x[u]);
                  old[u] = *p[u];
                }
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (x[u] >= 0) *p[u] = Arith<VT>::add(old[u], Arith<VT>::mul(at, v[u]));  // lines 6, 9, 11
            }
            __syncwarp();  // the next segment may add into a column this one just wrote
          }
          __syncthreads();
        }
        __syncthreads();
      }
      done += T;
      __syncthreads();
    }
    if (threadIdx.x == 0 && !overflow) {
      if (a.nnz_row) a.nnz_row[row] = done;
      if (PROG) {
        a.lst[k_long].count = done;
        a.lst[k_long].next_col = INT64_MAX;
      }
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

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace

int64_t g_long_tile_words = 0;  // debug knob (spgemm_set_debug_long_tile): 0 = by shared memory

// ------------------------------------------------------------- progressive bookkeeping
namespace {

__global__ void k_long_init(LongState* st, const int32_t* __restrict__ perm, int64_t first, int64_t nlong,
                            const int64_t* __restrict__ U, int64_t n, int64_t cap0, int64_t* sizes) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nlong) return;
  const int64_t u = U[perm[first + k]];
  LongState s;
  s.capmax = u < n ? u : n;
  s.cap = cap0 < s.capmax ? cap0 : s.capmax;
  s.count = 0;
  s.next_col = INT64_MIN;
  s.need = s.cap;
  st[k] = s;
  sizes[k] = s.cap;
}

__global__ void k_long_grow(LongState* st, const int32_t* __restrict__ list, int64_t nlist, int64_t* sizes) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nlist) return;
  LongState& s = st[list[i]];
  int64_t c = s.cap;
  while (c < s.need) c = c * 2 < s.capmax ? c * 2 : s.capmax;  // "we use 2x each time" [P:297]
  sizes[i] = c - s.cap;
  s.need = c;  // the new capacity, applied by the assignment
}

__global__ void k_long_assign(LongState* st, const int32_t* __restrict__ list, int64_t nlist,
                              const int64_t* __restrict__ off, int64_t base, int64_t* table, int log2c0) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nlist) return;
  const int k = list ? list[i] : (int)i;
  LongState& s = st[k];
  const int64_t old = list ? s.cap : 0;
  const int64_t cap = s.need;
  // positions [old, cap) are one contiguous block at base + off[i]: every new chunk maps
  // position p to (base + off[i]) + (p - old)
  for (int g = chunks_for(old, log2c0); g < chunks_for(cap, log2c0); ++g)
    table[int64_t(k) * kMaxChunks + g] = base + off[i] - old;
  s.cap = cap;
}

}  // namespace

cudaError_t launch_long_init(LongState* st, const int32_t* perm, int64_t first, int64_t nlong, const int64_t* U,
                             int64_t n, int64_t cap0, int64_t* sizes, cudaStream_t s) {
  if (nlong == 0) return cudaSuccess;
  k_long_init<<<(unsigned)((nlong + 255) / 256), 256, 0, s>>>(st, perm, first, nlong, U, n, cap0, sizes);
  return cudaGetLastError();
}

cudaError_t launch_long_grow(LongState* st, const int32_t* list, int64_t nlist, int64_t* sizes, cudaStream_t s) {
  if (nlist == 0) return cudaSuccess;
  k_long_grow<<<(unsigned)((nlist + 255) / 256), 256, 0, s>>>(st, list, nlist, sizes);
  return cudaGetLastError();
}

cudaError_t launch_long_assign(LongState* st, const int32_t* list, int64_t nlist, const int64_t* off, int64_t base,
                               int64_t* table, int log2c0, cudaStream_t s) {
  if (nlist == 0) return cudaSuccess;
  k_long_assign<<<(unsigned)((nlist + 255) / 256), 256, 0, s>>>(st, list, nlist, off, base, table, log2c0);
  return cudaGetLastError();
}

cudaError_t launch_long_bitmap(const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  if (a.work_ctr) {
    cudaError_t e0 = cudaMemsetAsync(a.work_ctr, 0, sizeof(int), s);
    if (e0 != cudaSuccess) return e0;
  }
  const bool fill = a.mode == MODE_FILL;
  const int nt = fill ? kRkNT : kBmNT;
  // tiles never exceed the column range [0, n)
  const int64_t nwords = round_up((a.n + 31) / 32 + 1, nt);
  int64_t tmax = fill ? kDefaultRankTileWords : kDefaultCountTileWords;
  if (g_long_tile_words > 0) tmax = g_long_tile_words;
  tmax = round_up(tmax, nt);
  if (tmax > nwords) tmax = nwords;
  const size_t sm = size_t(tmax) * (fill ? 8 : 4);
  int per_sm = 1;
  cudaError_t e;
  if (fill) {
    auto kern = a.f32 ? (a.lst ? k_long_rank<kRkNT, true, float> : k_long_rank<kRkNT, false, float>)
                      : (a.lst ? k_long_rank<kRkNT, true, double> : k_long_rank<kRkNT, false, double>);
    const size_t smv = sm;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smv);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smv);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = int64_t(sm_count()) * per_sm;
    if (grid > a.count) grid = a.count;
    kern<<<(unsigned)grid, nt, smv, s>>>(a, (int)tmax);
  } else {
    e = cudaFuncSetAttribute(k_long_bm_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_long_bm_count, nt, sm);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = int64_t(sm_count()) * per_sm;
    if (grid > a.count) grid = a.count;
    k_long_bm_count<<<(unsigned)grid, nt, sm, s>>>(a, (int)tmax);
  }
  return cudaGetLastError();
}

}  // namespace sg
