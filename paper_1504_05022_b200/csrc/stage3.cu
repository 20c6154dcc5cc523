// stage3.cu — stage 3 ("computing the resulting matrix", [P:262-284]) for rows whose
// products fit on chip.  Each kernel computes, for a row i, the sorted duplicate-free set
// {k : exists j, a_ij and b_jk stored} and c_ik = sum_j a_ij·b_jk — Algorithm "Pseudocode
// for the SpGEMM" lines 3-11 [P:121-135]: per product an "insert" (new column) or an
// "accumulate" (existing column).
//
// The paper's group-3 heap [P:266-275] and group-4 bitonic ESC [P:277-284] were sized for
// 48-96 KB scratchpads and 32-wide thread bunches; on B200 they become:
//   k_group<G>   u_i <= G <= 32: G lanes per row, lane = one product; the products are
//                sorted by (column, product index) with a register bitonic network and
//                fused left to right — the ESC idea with the whole row in registers.
//   (warp.cu)    one warp per row, S-slot shared-memory hash (classes w64..w2048).
//   k_cta_hash   one CTA per row, a 2H-slot shared-memory hash that counts the row's
//                distinct columns (symbolic); the values of these rows come from the ESC
//                (esc.cu) or the bitmap rank kernel (longbm.cu).
// Values: products are rounded separately (__dmul_rn, no FMA) and summed with __dadd_rn.
// k_group and the warp classes add in j-ascending order starting from the first product (the
// warp hash starts from -0.0, the identity of +), i.e. the oracle's order [P:129-131].
#include <climits>

#include "common.cuh"

namespace sg {

namespace {

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// --------------------------------------------------------------- G-lane sort groups
template <int G, int NT, bool KEY32, typename V>
__global__ void __launch_bounds__(NT) k_group(Stage3Args a) {
  static_assert(G >= 1 && G <= 32 && (G & (G - 1)) == 0, "G must be a power of two <= 32");
  __shared__ int s_col[NT];
  __shared__ V s_val[NT];
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gfirst = threadIdx.x & ~(G - 1);
  const int gshift = lane & ~(G - 1);
  const unsigned gbits = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gshift);
  const int warp = threadIdx.x >> 5;
  constexpr int WPB = NT / 32;
  constexpr int GPW = 32 / G;
  const bool fill = a.mode == MODE_FILL;

  // each CTA takes a contiguous range of tiles (neighbouring rows share b_j*: L1 reuse)
  const int64_t ntiles = (a.count + GPW - 1) / GPW;
  const int64_t tper = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t tend = min(int64_t(blockIdx.x) * tper + tper, ntiles);
  for (int64_t wt = int64_t(blockIdx.x) * tper + warp; wt < tend; wt += WPB) {
    const int64_t gi = wt * GPW + lane / G;
    const bool has = gi < a.count;
    const int row = has ? __ldg(a.perm + a.first + gi) : 0;
    const int64_t a0 = has ? __ldg(a.A.rp + row) : 0;
    const int64_t a1 = has ? __ldg(a.A.rp + row + 1) : 0;
    int64_t maxlen = a1 - a0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t x = __shfl_xor_sync(0xffffffffu, maxlen, o);
      maxlen = x > maxlen ? x : maxlen;
    }
    int cnt = 0;  // products gathered so far in this group
    unsigned long long key = ~0ull;
    V myv = V(0);
    for (int64_t e0 = 0; e0 < maxlen; e0 += G) {
      const int64_t e = a0 + e0 + gl;
      int len = 0;
      int64_t bs = 0;
      V av = V(0);
      if (e < a1) {
        const int j = __ldg(a.A.ci + e);
        if (fill) av = __ldg(vcast<V>(a.A.val) + e);
        bs = __ldg(a.B.rp + j);
        len = (int)(__ldg(a.B.rp + j + 1) - bs);
      }
      int inc = len;
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, inc, o, G);
        if (gl >= o) inc += x;
      }
      const int tot = __shfl_sync(0xffffffffu, inc, G - 1, G);
      const int q = gl - cnt;  // product index (within this chunk) this lane receives
      int lo = 0;
#pragma unroll
      for (int step = G / 2; step >= 1; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, inc, lo + step - 1, G);
        if (v <= q) lo += step;
      }
      const int64_t obs = __shfl_sync(0xffffffffu, bs, lo, G);
      const V oa = __shfl_sync(0xffffffffu, av, lo, G);
      const int oex = __shfl_sync(0xffffffffu, inc - len, lo, G);
      if (q >= 0 && q < tot) {
        const int64_t qq = obs + (q - oex);
        const int c = __ldg(a.B.ci + qq);
        key = ((unsigned long long)(unsigned)c << 32) | (unsigned)gl;
        if (fill) myv = Arith<V>::mul(oa, __ldg(vcast<V>(a.B.val) + qq));  // line 6: value <- a_ij b_jk
      }
      cnt += tot;
    }
    if (!fill) {
      // count only: distinct columns of the group = leaders of equal-key lane sets
      const unsigned long long gk = key == ~0ull ? ~0ull - lane : ((unsigned long long)(lane / G) << 32) | (key >> 32);
      const unsigned same = __match_any_sync(0xffffffffu, gk);
      const bool lead = key != ~0ull && (__ffs(same) - 1) == lane;
      const int nnz = __popc(__ballot_sync(0xffffffffu, lead) & gbits);
      if (has && gl == 0 && a.nnz_row) a.nnz_row[row] = nnz;
      continue;
    }
    // bitonic sort of (column, product index) across the G lanes of the group; columns below
    // 2^27 pack with the 5-bit product index into one 32-bit key
    int col, src;
    bool valid;
    if (KEY32) {
      unsigned k32 = key == ~0ull ? 0xffffffffu : ((unsigned)(key >> 32) << 5) | (unsigned)gl;
#pragma unroll
      for (int k = 2; k <= G; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const unsigned p = __shfl_xor_sync(0xffffffffu, k32, j);
          const bool up = (gl & k) == 0, lower = (gl & j) == 0;
          k32 = (lower == up) ? min(k32, p) : max(k32, p);
        }
      }
      valid = k32 != 0xffffffffu;
      col = valid ? (int)(k32 >> 5) : -1;
      src = (int)(k32 & 31u);
    } else {
#pragma unroll
      for (int k = 2; k <= G; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const unsigned long long p = __shfl_xor_sync(0xffffffffu, key, j);
          const bool up = (gl & k) == 0, lower = (gl & j) == 0;
          key = (lower == up) ? (key < p ? key : p) : (key > p ? key : p);
        }
      }
      valid = key != ~0ull;
      col = valid ? (int)(key >> 32) : -1;
      src = (int)(key & 31u);
    }
    const V v = __shfl_sync(0xffffffffu, myv, valid ? src : gl, G);
    const int prev = __shfl_up_sync(0xffffffffu, col, 1, G);
    const bool head = valid && (gl == 0 || prev != col);
    const unsigned hb = __ballot_sync(0xffffffffu, head) & gbits;
    const int nnz = __popc(hb);
    if (has && gl == 0 && a.nnz_row) a.nnz_row[row] = nnz;
    if (fill) {
      s_col[threadIdx.x] = col;
      s_val[threadIdx.x] = v;
      __syncwarp();
      if (has && head) {
        V acc = v;                                          // line 9: c_ik <- value
        for (int t = gl + 1; t < G && s_col[gfirst + t] == col; ++t)
          acc = Arith<V>::add(acc, s_val[gfirst + t]);      // line 11: c_ik += value
        const int pos = __popc(hb & lanemask_lt());
        const int64_t o = __ldg(a.out_off + row) + pos;
        a.out_col[o] = col;
        vcast<V>(a.out_val)[o] = acc;
      }
      __syncwarp();
    }
  }
}

// --------------------------------------------------------------- CTA hash (counting)
// COUNT only (precise symbolic and the e / c classes): nnz(c_i*) = the number of distinct
// columns the row's products insert ([P:121-135] lines 7-8 / 10 without values).  The values
// of these rows come from the ESC (e classes) or the bitmap rank kernel (c classes).
template <int LOG2H, int NT>
__global__ void __launch_bounds__(NT) k_cta_hash(Stage3Args a) {
  constexpr int H = 1 << LOG2H;
  constexpr int S = 2 * H;  // physical slots (nnz <= H: load <= 1/2)
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  int* keys = reinterpret_cast<int*>(smem);
  __shared__ int s_cnt;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

  const int64_t rper = (a.count + gridDim.x - 1) / gridDim.x;  // contiguous rows per CTA
  const int64_t rend = min(int64_t(blockIdx.x) * rper + rper, a.count);
  for (int64_t r = int64_t(blockIdx.x) * rper; r < rend; ++r) {
    const int row = __ldg(a.perm + a.first + r);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    for (int s = threadIdx.x; s < S; s += NT) keys[s] = kEmptyKey;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int inserted = 0;
    for (int64_t e = a0 + w; e < a1; e += NW) {
      const int j = __ldg(a.A.ci + e);
      const int64_t jb = __ldg(a.B.rp + j), je = __ldg(a.B.rp + j + 1);
      for (int64_t q = jb + lane; q < je; q += 32) {
        const int c = __ldg(a.B.ci + q);
        int h = (int)(((unsigned)c * 0x9E3779B1u) >> (32 - LOG2H - 1));
        volatile int* vk = keys;
        while (true) {
          const int k = vk[h];
          if (k == c) break;
          if (k == kEmptyKey) {
            const int old = atomicCAS(&keys[h], kEmptyKey, c);
            if (old == kEmptyKey) {
              ++inserted;
              break;
            }
            if (old == c) break;
          }
          h = (h + 1) & (S - 1);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) inserted += __shfl_xor_sync(0xffffffffu, inserted, o);
    if (lane == 0) atomicAdd(&s_cnt, inserted);
    __syncthreads();
    if (threadIdx.x == 0 && a.nnz_row) a.nnz_row[row] = s_cnt;
    __syncthreads();
  }
}

// --------------------------------------------------------------- launch helpers
int g_num_sms = 0;

}  // namespace

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

namespace {

template <typename K>
cudaError_t launch_persistent(K kernel, int nt, size_t dsmem, int64_t work_units, int units_per_block,
                              const Stage3Args& a, cudaStream_t s) {
  if (dsmem > 0) {  // opt in whenever static + dynamic may exceed the 48 KB default
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, dsmem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t need = (work_units + units_per_block - 1) / units_per_block;
  int64_t cap = int64_t(num_sms()) * per_sm * 8;
  int64_t grid = need < cap ? need : cap;
  if (grid < 1) grid = 1;
  kernel<<<(unsigned)grid, nt, dsmem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_stage3_tier(int tier, const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  constexpr size_t per_slot = 4;  // k_cta_hash counts only
  switch (tier) {
#define SG_GROUP(G, UPB)                                                                              \
  if (a.f32 && a.mode == MODE_FILL)                                                                     \
    return a.n < (int64_t(1) << 27) ? launch_persistent(k_group<G, 256, true, float>, 256, 0, a.count, UPB, a, s) \
                                     : launch_persistent(k_group<G, 256, false, float>, 256, 0, a.count, UPB, a, s); \
  return a.n < (int64_t(1) << 27) ? launch_persistent(k_group<G, 256, true, double>, 256, 0, a.count, UPB, a, s) \
                                   : launch_persistent(k_group<G, 256, false, double>, 256, 0, a.count, UPB, a, s)
    case T_G1: SG_GROUP(1, 256);
    case T_G2: SG_GROUP(2, 128);
    case T_G4: SG_GROUP(4, 64);
    case T_G8: SG_GROUP(8, 32);
    case T_G16: SG_GROUP(16, 16);
    case T_G32: SG_GROUP(32, 8);
#undef SG_GROUP
    case T_W64:
    case T_W128:
    case T_W256:
    case T_W512:
    case T_W1024:
    case T_W2048:
      // values: the row's products sorted in one CTA (ESC, esc.cu) — cheaper than hash + sort;
      // counting / structure / dense lookup: the warp hash (warp.cu)
      if (a.mode == MODE_FILL) return launch_esc_items(64 << (tier - T_W64), a, s);
      return launch_warp_tier(tier, a, s);
    case T_BW:
      return launch_bw_tier(a, s);
    // ESC (sorted) for values; counting only needs distinct keys: the CTA hash of the same size
    // (e4096: twice the size, load <= 1/4 — c5 count 33 -> 23 ms at 2^20; larger tables for
    // e2048 / e8192 measured slower on c3a / c3b: clearing and occupancy)
    case T_E2048:
      if (a.mode == MODE_COUNT) return launch_persistent(k_cta_hash<11, 256>, 256, 4096 * 4, a.count, 1, a, s);
      return launch_esc(tier, a, s);
    case T_E4096:
      if (a.mode == MODE_COUNT) return launch_persistent(k_cta_hash<13, 512>, 512, 16384 * 4, a.count, 1, a, s);
      return launch_esc(tier, a, s);
    case T_E8192:
      if (a.mode == MODE_COUNT) return launch_persistent(k_cta_hash<13, 512>, 512, 16384 * 4, a.count, 1, a, s);
      return launch_esc(tier, a, s);
    // values of the CTA-hash classes: the bitmap rank kernel (longbm.cu) — ordered, no atomics
    case T_C2048:
    case T_C4096:
    case T_C8192:
      if (a.mode == MODE_FILL) return launch_long_bitmap(a, s);
      break;
    default: return cudaErrorInvalidValue;
  }
  switch (tier) {
    case T_C2048: return launch_persistent(k_cta_hash<11, 256>, 256, 4096 * per_slot, a.count, 1, a, s);
    case T_C4096: return launch_persistent(k_cta_hash<12, 512>, 512, 8192 * per_slot, a.count, 1, a, s);
    case T_C8192: return launch_persistent(k_cta_hash<13, 512>, 512, 16384 * per_slot, a.count, 1, a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sg
