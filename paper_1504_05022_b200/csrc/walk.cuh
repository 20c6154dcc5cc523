// walk.cuh — the warp walk over the products of one row of A in Algorithm-1 order
// ([P:121-135]: for each a_ij in j order, for each b_jk in k order), shared by the warp classes
// (warp.cu) and the long-row bucket partition (longbk.cu).  Internal; not part of the ABI.
#pragma once
#include "common.cuh"

namespace sg {
namespace walk {

constexpr unsigned kFull = 0xffffffffu;

// One a_ij chunk (up to 32 entries of row i of A): lane e holds b_j*'s start and length and a_ij.
// IT: index type of B's entries (int32_t when nnz(B) < 2^31: one shuffle and one IMAD.WIDE per
// address instead of 64-bit arithmetic).
template <typename IT, typename V>
struct AChunk {
  IT bs;
  int len;
  V av;
};

template <bool VALS, typename IT, typename V>
__device__ __forceinline__ AChunk<IT, V> load_achunk(const Stage3Args& a, int64_t e, int64_t a1) {
  AChunk<IT, V> ch{0, 0, V(0)};
  if (e < a1) {
    const int j = __ldg(a.A.ci + e);
    if (VALS) ch.av = __ldg(vcast<V>(a.A.val) + e);
    const int64_t b0 = __ldg(a.B.rp + j);
    ch.bs = (IT)b0;
    ch.len = (int)(__ldg(a.B.rp + j + 1) - b0);
  }
  return ch;
}

constexpr int kGroup = 4;  // b_j* whose loads are in flight together

// Walk all products of row i in Algorithm-1 order, calling op(c, v, at, act) once per b_j*
// segment of up to 32 entries (c: this lane's column, v: b_jk, at: a_ij; V the value type).
template <bool VALS, typename IT, typename V, typename Op>
__device__ __forceinline__ void walk_row(const Stage3Args& a, int64_t a0, int64_t a1, int lane, Op&& op) {
  const V* __restrict__ bval = vcast<V>(a.B.val);
  for (int64_t e0 = a0; e0 < a1; e0 += 32) {
    const AChunk<IT, V> ch = load_achunk<VALS, IT, V>(a, e0 + lane, a1);
    const int nE = (int)((a1 - e0) < 32 ? (a1 - e0) : 32);
    if (!__any_sync(kFull, ch.len > 32)) {
      for (int t0 = 0; t0 < nE; t0 += kGroup) {
        int c[kGroup];
        V v[kGroup], at[kGroup];
        bool act[kGroup];
#pragma unroll
        for (int u = 0; u < kGroup; ++u) {
          const int t = t0 + u;  // <= 31; lanes past the chunk have len 0
          const IT q = __shfl_sync(kFull, ch.bs, t) + (IT)lane;
          const int len = __shfl_sync(kFull, ch.len, t);
          act[u] = lane < len;
          c[u] = act[u] ? __ldg(a.B.ci + q) : kEmptyKey;
          if (VALS) {
            at[u] = __shfl_sync(kFull, ch.av, t);
            v[u] = act[u] ? __ldg(bval + q) : V(0);
          }
        }
#pragma unroll
        for (int u = 0; u < kGroup; ++u)
          if (t0 + u < nE) op(c[u], VALS ? v[u] : V(0), VALS ? at[u] : V(0), act[u]);
      }
    } else {
      for (int t = 0; t < nE; ++t) {
        const IT bs = __shfl_sync(kFull, ch.bs, t);
        const int len = __shfl_sync(kFull, ch.len, t);
        const V at = VALS ? __shfl_sync(kFull, ch.av, t) : V(0);
        for (int q0 = 0; q0 < len; q0 += 32) {
          const bool act = q0 + lane < len;
          const IT q = bs + (IT)(q0 + lane);
          const int c = act ? __ldg(a.B.ci + q) : kEmptyKey;
          const V v = (VALS && act) ? __ldg(bval + q) : V(0);
          op(c, v, at, act);
        }
      }
    }
  }
}

}  // namespace walk
}  // namespace sg
