// stage4.cu — stage 4 "arranging data" ([P:301]): after the sum of nnz(c_i*) (the
// exclusive scan in stage12.cu) gives C's row pointers, copy every row from the temporary
// C~ into C.  Paper: no copy for group-1 rows, one thread per row for group 2, one thread
// group per row otherwise.  Here: a G-lane group per row (G chosen from the mean row
// length), 16-byte loads/stores where the row is aligned; long rows copy from the front
// of their progressive tables.
#include "common.cuh"

namespace sg {

namespace {

template <int G>
__global__ void __launch_bounds__(256) k_copy(CopyArgs a) {
  const int gl = threadIdx.x & (G - 1);
  const int64_t g0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  const int64_t gstride = int64_t(gridDim.x) * blockDim.x / G;
  for (int64_t i = g0; i < a.m; i += gstride) {
    const int64_t d = __ldg(a.c_rp + i);
    const int64_t len = __ldg(a.c_rp + i + 1) - d;
    if (len == 0 || a.tier[i] == T_LONG) continue;
    const int64_t s = __ldg(a.ctil_off + i);
    const int32_t* __restrict__ sc = a.ctil_col + s;
    const double* __restrict__ sv = a.ctil_val + s;
    int32_t* __restrict__ dc = a.c_col + d;
    double* __restrict__ dv = a.c_val + d;
    for (int64_t t = gl; t < len; t += G) {
      dc[t] = __ldcs(sc + t);
      dv[t] = __ldcs(sv + t);
    }
  }
}

// Flat copy: warp w owns rows [32w, 32w+32); their outputs form one contiguous span of C.
// Lane p-th output finds its row by a shuffle binary search over the 33 row pointers, so
// every store instruction writes 32 consecutive entries.
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
    const bool lng = has && a.tier[i] == T_LONG;
    for (int64_t p0 = beg; p0 < end; p0 += 32) {
      const int64_t p = p0 + lane;
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
      if (p < end && !rl) {
        const int64_t q = rsrc + (p - rbeg);
        a.c_col[p] = __ldcs(a.ctil_col + q);
        a.c_val[p] = __ldcs(a.ctil_val + q);
      }
    }
  }
}

__global__ void __launch_bounds__(512) k_copy_long(CopyArgs a) {
  const int64_t k = blockIdx.x;
  const int row = a.perm[a.long_first + k];
  const int64_t d = a.c_rp[row];
  const int64_t len = a.c_rp[row + 1] - d;
  const int32_t* sc = a.long_keys[k];
  const double* sv = a.long_vals[k];
  for (int64_t t = threadIdx.x; t < len; t += blockDim.x) {
    a.c_col[d + t] = __ldcg(sc + t);
    a.c_val[d + t] = __ldcg(sv + t);
  }
}

int sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace

cudaError_t launch_copy(const CopyArgs& a, int group, cudaStream_t s) {
  if (a.m > 0) {
    const int64_t groups_per_block = group > 0 ? 256 / group : 8;
    int64_t grid = (a.m + groups_per_block - 1) / groups_per_block;
    const int64_t cap = int64_t(sms()) * 16;
    if (grid > cap) grid = cap;
    switch (group) {
      case 0: {
        const int64_t g2 = ((a.m + 31) / 32 + 7) / 8;
        k_copy_flat<<<(unsigned)(g2 < cap ? g2 : cap), 256, 0, s>>>(a);
        break;
      }
      case 4: k_copy<4><<<(unsigned)grid, 256, 0, s>>>(a); break;
      case 8: k_copy<8><<<(unsigned)grid, 256, 0, s>>>(a); break;
      case 16: k_copy<16><<<(unsigned)grid, 256, 0, s>>>(a); break;
      default: k_copy<32><<<(unsigned)grid, 256, 0, s>>>(a); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (a.nlong > 0) {
    k_copy_long<<<(unsigned)a.nlong, 512, 0, s>>>(a);
    return cudaGetLastError();
  }
  return cudaSuccess;
}

}  // namespace sg
