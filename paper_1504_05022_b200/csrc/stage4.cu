// stage4.cu — stage 4 "arranging data" ([P:301]): after the sum of nnz(c_i*) (the
// exclusive scan in stage12.cu) gives C's row pointers, copy every row from the temporary
// C~ into C.  Paper: no copy for group-1 rows, one thread per row for group 2, one thread
// group per row otherwise.  Here: one warp per 32 consecutive rows, whose outputs form one
// contiguous span of C (k_copy_flat); long rows copy from their slices of the long-row arena.
#include "common.cuh"

namespace sg {

namespace {

// Flat copy: warp w owns rows [32w, 32w+32); their outputs form one contiguous span of C.
// Lane p-th output finds its row by a shuffle binary search over the 33 row pointers, so
// every store instruction writes 32 consecutive entries.
template <typename V>
__global__ void __launch_bounds__(256) k_copy_flat(CopyArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (a.m + 31) / 32;
  for (int64_t wi = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; wi < nwarps;
       wi += int64_t(gridDim.x) * blockDim.x / 32) {
    const int64_t i0 = wi * 32;
    const int64_t i = i0 + lane;
    const bool has = i < a.m;
    const int64_t rp = has ? __ldg(a.c_rp + i) : __ldg(a.c_rp + a.m);
    const int64_t end = __shfl_sync(0xffffffffu, has ? __ldg(a.c_rp + i + 1) : rp, 31);
    const int64_t beg = __shfl_sync(0xffffffffu, rp, 0);
    const int64_t src = has ? __ldg(a.ctil_off + i) : 0;
    // long rows without a C~ slice live in the arena (progressive path); long rows of the
    // bucket path have an upper-bound slice like every other class
    const bool lng = has && a.tier[i] == T_LONG &&
                     (i + 1 < a.m ? __ldg(a.ctil_off + i + 1) : a.ctil_total) == src;
    // four 32-entry chunks per iteration: their loads are in flight together
    constexpr int U = 4;
    for (int64_t p0 = beg; p0 < end; p0 += 32 * U) {
      int64_t q[U];
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int64_t p = p0 + 32 * x + lane;
        // last lane k with rp_k <= p (rows are ascending; empty rows share rp values)
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int64_t v = __shfl_sync(0xffffffffu, rp, lo + step);
          if (lo + step < 32 && v <= p) lo += step;
        }
        const int64_t rbeg = __shfl_sync(0xffffffffu, rp, lo);
        const int64_t rsrc = __shfl_sync(0xffffffffu, src, lo);
        const bool rl = __shfl_sync(0xffffffffu, lng, lo);
        q[x] = (p < end && !rl) ? rsrc + (p - rbeg) : -1;
      }
      int cv[U];
      V vv[U];
#pragma unroll
      for (int x = 0; x < U; ++x)
        if (q[x] >= 0) {
          cv[x] = __ldcs(a.ctil_col + q[x]);
          vv[x] = __ldcs(vcast<V>(a.ctil_val) + q[x]);
        }
#pragma unroll
      for (int x = 0; x < U; ++x)
        if (q[x] >= 0) {
          const int64_t p = p0 + 32 * x + lane;
          a.c_col[p] = cv[x];
          vcast<V>(a.c_val)[p] = vv[x];
        }
    }
  }
}

// long rows: their C~ slice lives in the long-row arena behind the row's chunk table
template <typename V>
__global__ void __launch_bounds__(512) k_copy_long(CopyArgs a) {
  const int64_t k = blockIdx.x;
  const int row = a.perm[a.long_first + k];
  const int64_t d = a.c_rp[row];
  const int64_t len = a.c_rp[row + 1] - d;
  const int64_t* tab = a.chunk_table + k * kMaxChunks;
  for (int64_t t = threadIdx.x; t < len; t += blockDim.x) {
    const int64_t x = __ldg(tab + chunk_of(t, a.log2c0)) + t;
    a.c_col[d + t] = __ldcs(a.arena_col + x);
    vcast<V>(a.c_val)[d + t] = __ldcs(vcast<V>(a.arena_val) + x);
  }
}

int sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace

cudaError_t launch_copy(const CopyArgs& a, cudaStream_t s) {
  if (a.m > 0) {
    const int64_t cap = int64_t(sms()) * 16;
    const int64_t g2 = ((a.m + 31) / 32 + 7) / 8;
    if (a.f32) k_copy_flat<float><<<(unsigned)(g2 < cap ? g2 : cap), 256, 0, s>>>(a);
    else k_copy_flat<double><<<(unsigned)(g2 < cap ? g2 : cap), 256, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (a.nlong > 0) {
    if (a.f32) k_copy_long<float><<<(unsigned)a.nlong, 512, 0, s>>>(a);
    else k_copy_long<double><<<(unsigned)a.nlong, 512, 0, s>>>(a);
    return cudaGetLastError();
  }
  return cudaSuccess;
}

}  // namespace sg
