// warp.cu — stage 3 warp-per-row classes ("computing the resulting matrix", [P:262-284];
// Algorithm 1 lines 3-11 [P:121-135]).
//
// Lanes walk the rows b_j* of the row's a_ij in j-ascending order, one b_j* (up to 32 of its
// entries) per instruction (walk_row); the loads of four consecutive b_j* are issued before
// their inserts.  Columns inside one b_j* are distinct, so no two lanes of one instruction
// insert or accumulate into one slot: values of a column are added in j-ascending order from
// the identity -0.0, i.e. the oracle's rounding (R1), without value atomics.
//
//   k_wrow          w64..w2048 counting: S-slot linear-probing hash (precise symbolic)
//   k_bw_struct2    bw rows, block directory: STRUCT (precise symbolic) and FILL (hybrid)
//   k_bwrow         bw rows over the full window: DENSE (precise numeric, from the STRUCT
//                   set), and the STRUCT / FILL fallback for rows with too many blocks
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "walk.cuh"

namespace sg {

namespace {

using walk::kFull;
using walk::kGroup;
using walk::walk_row;

__device__ __forceinline__ unsigned lanemask_lt_() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <int LOG2S>
__device__ __forceinline__ unsigned whash(int c) {
  return ((unsigned)c * 0x9E3779B1u) >> (32 - LOG2S);
}

// Insert c (if act) into keys; a lane that claims a new slot appends c to list.  Returns the
// slot.  Warp-uniform probing rounds; the common case (found at home) is one LDS + one vote.
template <int LOG2S, bool LIST>
__device__ __forceinline__ unsigned winsert(int* keys, int* list, int& cnt, int c, bool act) {
  constexpr unsigned MASK = (1u << LOG2S) - 1;
  volatile int* vk = keys;
  unsigned h = whash<LOG2S>(c);
  int k = vk[h];
  bool pend = act && k != c;
  while (true) {
    bool claimed = false;
    if (pend) {
      if (k == kEmptyKey) {
        const int old = atomicCAS(&keys[h], kEmptyKey, c);
        if (old == kEmptyKey) {
          claimed = true;
          pend = false;
        } else if (old == c) {
          pend = false;
        } else {
          h = (h + 1) & MASK;
          k = vk[h];
          pend = k != c;
        }
      } else {
        h = (h + 1) & MASK;
        k = vk[h];
        pend = k != c;
      }
    }
    const unsigned cb = __ballot_sync(kFull, claimed);
    if (cb) {
      if (LIST && claimed) list[cnt + __popc(cb & lanemask_lt_())] = c;
      cnt += __popc(cb);
    }
    if (!__any_sync(kFull, pend)) break;
  }
  return h;
}

// The same walk for 32-bit B offsets with the a_ij chunk staged in shared memory: lane e of a
// chunk writes one 16-byte record {b_j* start, nnz(b_j*), a_ij} to the warp's stage buffer
// (32 records, 512 B) and every step reads its record with one broadcast LDS.128 — instead of
// two or three shuffles per b_j* — and the steps of four b_j* are issued back to back (their
// gathers in flight together).  Records of lanes past the row's end have nnz 0, so the
// four-step groups need no bounds check: those steps run with every lane idle (act false).
template <typename V>
__device__ __forceinline__ V rec_val(const int4& r);
template <>
__device__ __forceinline__ double rec_val<double>(const int4& r) { return __hiloint2double(r.w, r.z); }
template <>
__device__ __forceinline__ float rec_val<float>(const int4& r) { return __int_as_float(r.z); }

template <bool VALS, typename V, typename Op>
__device__ __forceinline__ void walk_row_staged(const int32_t* __restrict__ aci, const V* __restrict__ aval,
                                                const int64_t* __restrict__ brp, const int32_t* __restrict__ bci,
                                                const V* __restrict__ bval, int64_t a0, int64_t a1,
                                                int lane, unsigned stage, Op&& op) {
  for (int64_t e0 = a0; e0 < a1; e0 += 32) {
    const int64_t e = e0 + lane;
    int bs = 0, len = 0;
    V av = V(0);
    if (e < a1) {
      const int j = __ldg(aci + e);
      const int64_t b0 = __ldg(brp + j);
      bs = (int)b0;
      len = (int)(__ldg(brp + j + 1) - b0);
      if (VALS) av = __ldg(aval + e);
    }
    const double avd = (double)av;  // record bits: the double, or the float in the low word
    const int lo_w = sizeof(V) == 8 ? __double2loint(avd) : __float_as_int((float)av);
    const int hi_w = sizeof(V) == 8 ? __double2hiint(avd) : 0;
    __syncwarp();
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stage + 16u * lane), "r"(bs), "r"(len),
                 "r"(lo_w), "r"(hi_w) : "memory");
    __syncwarp();
    const int nE = (int)((a1 - e0) < 32 ? (a1 - e0) : 32);
    if (!__any_sync(kFull, len > 32)) {
      for (int t0 = 0; t0 < nE; t0 += kGroup) {
        int c[kGroup];
        V v[kGroup], at[kGroup];
        bool act[kGroup];
#pragma unroll
        for (int u = 0; u < kGroup; ++u) {
          int4 r;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(stage + 16u * (t0 + u)) : "memory");
          act[u] = lane < r.y;
#ifndef SG_NO_CLAMP
          // idle lanes load b_j*'s last entry (or entry 0 of B for an empty step): no
          // predication, no default values; their result goes to a scratch slot (act)
          const int q = r.x + min(lane, max(r.y - 1, 0));
          c[u] = __ldg(bci + q);
          if (VALS) {
            at[u] = rec_val<V>(r);
            v[u] = __ldg(bval + q);
          }
#else
          const int q = r.x + lane;
          c[u] = act[u] ? __ldg(bci + q) : kEmptyKey;
          if (VALS) {
            at[u] = rec_val<V>(r);
            v[u] = act[u] ? __ldg(bval + q) : V(0);
          }
#endif
        }
#pragma unroll
        for (int u = 0; u < kGroup; ++u) op(c[u], VALS ? v[u] : V(0), VALS ? at[u] : V(0), act[u]);
      }
    } else {
      for (int t = 0; t < nE; ++t) {
        int4 r;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(stage + 16u * t) : "memory");
        const V at = VALS ? rec_val<V>(r) : V(0);  // fp64: both words; fp32: the low word
        for (int q0 = 0; q0 < r.y; q0 += 32) {
          const bool act = q0 + lane < r.y;
          const int q = r.x + q0 + lane;
          const int c = act ? __ldg(bci + q) : kEmptyKey;
          const V v = (VALS && act) ? __ldg(bval + q) : V(0);
          op(c, v, at, act);
        }
      }
    }
  }
}

// walk_row_staged when B's offsets fit 32 bits and the kernel has a stage buffer, else walk_row.
template <bool VALS, typename IT, typename V, typename Op>
__device__ __forceinline__ void walk_any(const Stage3Args& a, int64_t a0, int64_t a1, int lane, unsigned stage,
                                         Op&& op) {
  if constexpr (std::is_same<IT, int>::value) {
    walk_row_staged<VALS, V>(a.A.ci, vcast<V>(a.A.val), a.B.rp, a.B.ci, vcast<V>(a.B.val), a0, a1, lane, stage, op);
  } else {
    walk_row<VALS, IT, V>(a, a0, a1, lane, op);
  }
}

// Counting (precise symbolic, rows with W > 2^17): an S-slot table per warp, nnz = the
// number of claimed slots.  Values of these rows are computed by the ESC (esc.cu).
template <int LOG2S, int NW, typename IT>
__global__ void __launch_bounds__(NW * 32) k_wrow(Stage3Args a) {
  constexpr int S = 1 << LOG2S;
  __shared__ __align__(16) int s_keys[NW][S];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int* keys = s_keys[w];

  const int64_t rper = (a.count + gridDim.x - 1) / gridDim.x;  // contiguous rows per CTA
  const int64_t rend = min(int64_t(blockIdx.x) * rper + rper, a.count);
  for (int64_t r = int64_t(blockIdx.x) * rper + w; r < rend; r += NW) {
    const int row = __ldg(a.perm + a.first + r);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    int4* k4 = reinterpret_cast<int4*>(keys);
#pragma unroll
    for (int s = lane; s < S / 4; s += 32) k4[s] = make_int4(kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey);
    __syncwarp();
    int cnt = 0;
    walk_row<false, IT, double>(a, a0, a1, lane, [=, &cnt](int c, double, double, bool act) {
      winsert<LOG2S, false>(keys, nullptr, cnt, c, act);  // lines 7-8 / 10
    });
    __syncwarp();
    if (lane == 0 && a.nnz_row) a.nnz_row[row] = cnt;
    __syncwarp();
  }
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += x;
  }
  return v;
}

// ----------------------------------------------------------------------------------------
// T_BW: the sparse accumulator of Gilbert et al. ([P:142], the dense vector of Algorithm 1's
// "insert/accumulate") restricted to the row's column window [lo, lo + W): bit d of the
// warp's bitmap stands for column lo + d, one summary bit per bitmap word.  Inserting is one
// shared-memory OR per product (no probing, no votes); the row comes out ordered by scanning
// only the nonzero words; a column's position in the row is the popcount rank of its bit.
//
// Per-warp dynamic shared memory (32-bit words): bm[nwd] | sm[nsw] | FILL: pre[nwd/2] (uint16
// rank of each nonzero word's first bit) | lst[nvp] (nonzero words, ascending) | vals[nv].
//   COUNT  one pass over the products, popcounts of the nonzero words (precise symbolic)
//   FILL   pass 1 sets the bits; ranks and columns from the nonzero words; pass 2 adds each
//          product into vals[rank] (j-ascending per column: the oracle's order) and the row
//          is written in order with no sort (precise numeric into C, hybrid into C~)
// The bitmap is zero between rows: every row clears the words it set.
// 32-bit shared-window addressing (the per-warp regions are carved from dynamic shared memory;
// explicit ld/st/atom.shared keep every access a direct LDS/STS/ATOMS).  The helpers are volatile
// asm WITHOUT a memory clobber: their order among themselves is kept (volatile), while the
// read-only global gathers of B (__ldg) may be scheduled across them — the next steps' loads
// are in flight while the current step's shared-memory work runs.  Lane-to-lane hand-offs
// through shared memory are fenced by __syncwarp().
__device__ __forceinline__ unsigned sh_atom_or(unsigned addr, unsigned v) {
  unsigned r;
  asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(r) : "r"(addr), "r"(v));
  return r;
}
__device__ __forceinline__ void sh_red_or(unsigned addr, unsigned v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ unsigned sh_ld(unsigned addr) {
  unsigned r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sh_st(unsigned addr, unsigned v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ unsigned sh_ld_u16(unsigned addr) {
  unsigned short r;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sh_st_u16(unsigned addr, unsigned v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
}
__device__ __forceinline__ double sh_ld_f64(unsigned addr) {
  double r;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sh_st_f64(unsigned addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v));
}
template <typename V>
__device__ __forceinline__ V sh_ldv(unsigned addr);
template <>
__device__ __forceinline__ double sh_ldv<double>(unsigned addr) { return sh_ld_f64(addr); }
template <>
__device__ __forceinline__ float sh_ldv<float>(unsigned addr) {
  float r;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sh_stv(unsigned addr, double v) { sh_st_f64(addr, v); }
__device__ __forceinline__ void sh_stv(unsigned addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v));
}
__device__ __forceinline__ int4 sh_ld_v4(unsigned addr) {
  int4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint2 sh_ld_v2(unsigned addr) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sh_st_v4_zero(unsigned addr) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(0u));
}

// Per-warp shared-memory layout of the window class (byte offsets from the warp's base).
// Products -> bits (COUNT, STRUCT, FILL): a bitmap over the whole window
//   bm   uint32[nwd]   window bitmap, bit d <-> column lo + d
//   sm   uint32[nsw]   summary, bit w <-> bm[w] != 0 (one summary word per 1024-column block)
//   pre  uint16[nwd]   rank of each nonzero word's first bit    (FILL)
//   lst  int32[nvp]    nonzero words, ascending                 (FILL)
//   vals double[nv]    the row's values in column order         (FILL)
// Sorted set -> ranks (DENSE): only the row's nonzero 1024-column blocks are materialised
//   dir  uint16[nsw]   block -> slot + 1 (0: block empty)
//   bits uint32[ns·32] the bitmap of each slot's block
//   pre  uint16[ns·32] rank of each nonzero word's first bit
//   vals double[nv]
struct BwLayout {
  int nwd, nsw, nvp, nv, ns;
  unsigned o_sm, o_pre, o_lst, o_vals, o_stage, bytes;  // per warp, bytes is a multiple of 16
};

constexpr unsigned kRecSlot = 264u;  // DENSE: bytes per slot of 8-byte word records (33 records)

__host__ __device__ inline BwLayout bw_layout(int mode, int64_t wmax, int64_t vmax, int64_t bmax) {
  BwLayout L;
  L.nwd = (int)(((wmax > 0 ? wmax : 1) + 1023) / 1024 * 32);
  L.nsw = (L.nwd / 32 + 31) / 32 * 32;
  L.nv = (int)(vmax > 0 ? vmax : 1);
  L.nvp = (L.nv + 3) & ~3;
  L.ns = (int)(bmax > 0 ? (bmax < L.nsw ? bmax : L.nsw) : L.nsw);
  unsigned off;
  if (mode == MODE_DENSE) {
    L.o_sm = 0;                                  // dir
    off = (2u * L.nsw + 15u) & ~15u;             // records {bits, rank} per slot word (8 B),
    L.o_lst = off;                               // 33 per slot: a stencil's z-neighbour planes
    off += kRecSlot * L.ns;                      // (same word, other slot) in other banks
    off = (off + 15u) & ~15u;
    L.o_pre = off;                               // (end of the zeroed region)
    L.o_vals = off;
    off += 8u * (L.nv + 1);  // + scratch
    off = (off + 15u) & ~15u;
    L.o_stage = off;         // a_ij chunk records of walk_row_staged
    off += 512u;
  } else {  // STRUCT: bitmap + summary
    L.o_stage = 0;
    off = 4u * L.nwd;
    L.o_sm = off;
    off += 4u * L.nsw;
    L.o_pre = L.o_lst = L.o_vals = off;
  }
  L.bytes = (off + 15u) & ~15u;
  return L;
}

template <int MODE, typename IT, typename V>
#ifndef SG_BW_MINB
#define SG_BW_MINB 4  // 64 registers: c2 DENSE 6.1 -> 5.8 ms (vs 40 + spills)
#endif
__global__ void __launch_bounds__(256, SG_BW_MINB) k_bwrow(Stage3Args a, BwLayout L) {
  static_assert(MODE == MODE_STRUCT || MODE == MODE_DENSE, "window class: STRUCT or DENSE");
  extern __shared__ __align__(16) uint32_t s_bw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nwd = L.nwd, nsw = L.nsw;
  // byte addresses in the shared window
  const unsigned bm = (unsigned)__cvta_generic_to_shared(s_bw) + unsigned(w) * L.bytes;
  const unsigned sm = bm + L.o_sm, pre = bm + L.o_pre, lst = bm + L.o_lst, vals = bm + L.o_vals;
  const unsigned zero_end = MODE == MODE_DENSE ? L.o_pre : L.o_pre;  // bm (+ sm) / dir + bits
  for (unsigned i = lane; i < (zero_end + 15u) / 16u; i += 32) sh_st_v4_zero(bm + 16u * i);
  __syncwarp();
  int bmax = 0;  // STRUCT: most nonzero 1024-column blocks in one row (sizes DENSE's slots)

  const int64_t count = a.count_dev ? (int64_t)*a.count_dev : a.count;
  // each CTA takes a contiguous range of the class's rows (ascending row ids): neighbouring
  // rows share b_j*, reused from L1 (DENSE: 4.85 -> 4.64 ms on c2 against a strided order)
  const bool contig = true;
  const int64_t per = contig ? (count + gridDim.x - 1) / gridDim.x : count;
  const int64_t rend = contig ? min(int64_t(blockIdx.x) * per + per, count) : count;
  const int64_t rstep = contig ? nw : int64_t(gridDim.x) * nw;
  for (int64_t r = contig ? int64_t(blockIdx.x) * per + w : int64_t(blockIdx.x) * nw + w; r < rend; r += rstep) {
    const int row = __ldg(a.perm + a.first + r);
    const int lo = __ldg(a.rlo + row);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    const int64_t o = __ldg(a.out_off + row);
    int nnz = 0;
    if (MODE != MODE_DENSE) {
      // lines 7-8 / 10 of Algorithm 1 for every product: set the column's bit.  With the
      // summary: only the lane that finds a word empty sets its summary bit, so summary
      // atomics are rare and seldom share an address.
      // Branch-free: an idle lane (act false) re-sets the bit of column lo, a column of the row.
      walk_row<false, IT, V>(a, a0, a1, lane, [=](int c, V, V, bool act) {
        const unsigned d = act ? (unsigned)(c - lo) : 0u;
        const unsigned wa = bm + ((d >> 5) << 2);
        if (sh_atom_or(wa, 1u << (d & 31)) == 0u) sh_red_or(sm + ((d >> 10) << 2), 1u << ((d >> 5) & 31));
      });
      __syncwarp();
    }
    if (MODE == MODE_STRUCT) {
      // the sorted column set, block by nonzero block (clears bitmap and summary)
      int32_t* oc = a.out_col + o;
      int nb = 0;
      for (int s0 = 0; s0 < nsw; s0 += 32) {
        const unsigned swl = sh_ld(sm + 4u * (s0 + lane));
        unsigned nzb = __ballot_sync(kFull, swl != 0u);
        nb += __popc(nzb);
        if (swl) sh_st(sm + 4u * (s0 + lane), 0u);
        while (nzb) {
          const int b = __ffs(nzb) - 1;
          nzb &= nzb - 1;
          const unsigned sw = __shfl_sync(kFull, swl, b);
          const unsigned wa = bm + 4u * ((s0 + b) * 32 + lane);
          unsigned word = (sw >> lane) & 1u ? sh_ld(wa) : 0u;
          if (word) sh_st(wa, 0u);
          const int pc = __popc(word);
          const int inc = warp_incl_scan(pc, lane);
          int p = nnz + inc - pc;
          const int cb = lo + ((s0 + b) * 32 + lane) * 32;
          while (word) {
            oc[p++] = cb + __ffs(word) - 1;
            word &= word - 1;
          }
          nnz += __shfl_sync(kFull, inc, 31);
        }
      }
      bmax = max(bmax, nb);
      if (lane == 0 && a.nnz_row) a.nnz_row[row] = nnz;
      __syncwarp();
      continue;
    }
    const unsigned dir = sm, bits = lst;  // DENSE names
    int nslot = 0, nwr = -1;
    if (MODE == MODE_DENSE) {
      // the sorted column set from the symbolic pass: slots of the nonzero blocks in column
      // order, bits, ranks, and C's columns directly
      nnz = (int)(a.row_len ? __ldg(a.row_len + row) : __ldg(a.out_off + row + 1) - o);
      const int32_t* sc = a.struct_col + __ldg(a.struct_off + row);
      nwr = a.bw_nw ? __ldg(a.bw_nw + row) : -1;
      if (nwr >= 0) {
        // the row as its nonzero words (first column, bits), ascending: a word's record is
        // {bits, rank of its first bit} with the rank from one scan of the popcounts; the
        // word's columns go to C at their ranks
        const uint2* sw = reinterpret_cast<const uint2*>(sc);
        int prevb = -1, rank0 = 0;
        for (int p0 = 0; p0 < nwr; p0 += 32) {
          const int p = p0 + lane;
          const bool in = p < nwr;
          const uint2 ent = in ? __ldg(sw + p) : make_uint2(0u, 0u);
          const int d = (int)ent.x - lo;  // a multiple of 32
          const int blk = in ? d >> 10 : -1;
          int bp = __shfl_up_sync(kFull, blk, 1);
          if (lane == 0) bp = prevb;
          const bool newblk = in && bp != blk;
          const unsigned nm = __ballot_sync(kFull, newblk);
          const int slot = nslot + __popc(nm & (lanemask_lt_() | (1u << lane))) - 1;
          const int pc = __popc(ent.y);
          const int inc = warp_incl_scan(pc, lane);
          if (in) {
            const int rank = rank0 + inc - pc;
            if (newblk) sh_st_u16(dir + 2u * unsigned(blk), (unsigned)(slot + 1));
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(bits + unsigned(slot) * kRecSlot + 8u * ((d >> 5) & 31)),
                         "r"(ent.y), "r"((unsigned)rank));
            unsigned wd = ent.y;
            const int cb = (int)ent.x - 1;
            int32_t* q = a.out_col + o + rank;  // C's columns of the word, at their ranks
            while (wd) {
              *q++ = cb + __ffs(wd);
              wd &= wd - 1;
            }
          }
          nslot += __popc(nm);
          prevb = __shfl_sync(kFull, blk, 31);
          rank0 += __shfl_sync(kFull, inc, 31);
        }
      }
      int prevd = -1;  // d of the previous chunk's last column
      for (int p0 = 0; nwr < 0 && p0 < nnz; p0 += 32) {
        const int p = p0 + lane;
        const bool in = p < nnz;
        const int c = in ? __ldg(sc + p) : 0;
        const int d = c - lo;
        int dp = __shfl_up_sync(kFull, d, 1);
        if (lane == 0) dp = prevd;
        const bool newblk = in && (dp < 0 || (dp >> 10) != (d >> 10));
        const unsigned nm = __ballot_sync(kFull, newblk);
        const int slot = nslot + __popc(nm & (lanemask_lt_() | (1u << lane))) - 1;
        // the bits of a word's lanes (contiguous: the set is sorted) are ORed together first,
        // so each word takes one RED (same-address REDs serialise: 7.6x the ideal wavefronts)
        const int wkey = in ? (d >> 5) : -1 - lane;
        unsigned wbits = in ? 1u << (d & 31) : 0u;
#pragma unroll 1
        for (int sh = 1; sh < 32; sh <<= 1) {  // (not unrolled: keeps the kernel at 48 registers)
          const unsigned vo = __shfl_down_sync(kFull, wbits, sh);
          const int ko = __shfl_down_sync(kFull, wkey, sh);
          if (lane + sh < 32 && ko == wkey) wbits |= vo;
        }
        const bool wfirst = dp < 0 || (dp >> 5) != (d >> 5);  // first entry of its word overall
        const int kprev = __shfl_up_sync(kFull, wkey, 1);
        if (in) {
          a.out_col[o + p] = c;
          if (newblk) sh_st_u16(dir + 2u * (d >> 10), (unsigned)(slot + 1));
          const unsigned ra = bits + unsigned(slot) * kRecSlot + 8u * ((d >> 5) & 31);
          if (lane == 0 || kprev != wkey) sh_red_or(ra, wbits);  // first lane of its run here
          if (wfirst) sh_st(ra + 4u, (unsigned)p);
        }
        nslot += __popc(nm);
        prevd = __shfl_sync(kFull, d, 31);
      }
    }
    for (int p = lane; p < nnz; p += 32) sh_stv(vals + 8u * p, V(-0.0));  // identity of +: first add == line 9
    __syncwarp();
    // lines 6, 9, 11: c_ik += a_ij b_jk at the column's rank
    // Branch-free: an idle lane looks up column lo (present) and adds into a scratch slot.
    // Lanes of one b_j* hold distinct columns, so no two lanes of an instruction share a slot;
    // successive b_j* are ordered by the warp's in-order shared-memory accesses.
    const unsigned scratch = vals + 8u * unsigned(L.nv);
    auto accumulate = [=](int c, V v, V at, bool act) {
      const unsigned d = act ? (unsigned)(c - lo) : 0u;
      // one 8-byte record: the word's bits and its first rank;
      // record (d>>5)%32 of slot dir-1: bits + (dir-1)*kRecSlot + ((d >> 2) & 0xf8)
      const uint2 rec = sh_ld_v2(bits - kRecSlot + sh_ld_u16(dir + 2u * (d >> 10)) * kRecSlot + ((d >> 2) & 0xf8u));
      const unsigned rank = rec.y + __popc(rec.x & ((1u << (d & 31)) - 1u));
      const unsigned va = act ? vals + 8u * rank : scratch;
      sh_stv(va, Arith<V>::add(sh_ldv<V>(va), Arith<V>::mul(at, v)));
      __syncwarp();  // the next step's lanes may read this slot (memory-model order, not just lockstep)
    };
    walk_any<true, IT, V>(a, a0, a1, lane, bm + L.o_stage, accumulate);
    __syncwarp();
    V* ov = vcast<V>(a.out_val) + o;
    for (int p = lane; p < nnz; p += 32) ov[p] = sh_ldv<V>(vals + 8u * p);
    for (int s = 0; s < nslot; ++s) sh_st(bits + unsigned(s) * kRecSlot + 8u * lane, 0u);
    for (int q = lane; q < (2 * nsw) / 16; q += 32) sh_st_v4_zero(dir + 16u * q);
    if (lane == 0 && a.nnz_row) a.nnz_row[row] = nnz;
    __syncwarp();
  }
  if (MODE == MODE_STRUCT && lane == 0 && bmax > 0 && a.bw_bmax_out)
    atomicMax(reinterpret_cast<unsigned long long*>(a.bw_bmax_out), (unsigned long long)bmax);
}


// ----------------------------------------------------------------------------------------
// T_BW STRUCT with a block directory: only the row's nonzero 1024-column blocks get a
// bitmap slot (allocated on first touch, warp-synchronously: the lanes of one b_j* hold
// ascending columns, so each newly touched block is claimed by the first lane of its run).
// Per warp: dir uint16[nsw] (block -> slot + 1) | bits uint32[ns·32].  ~2.3 KB per warp
// instead of W/8: 2x the resident warps on c2.  Inserting is a fire-and-forget shared OR.
// A row touching more than ns blocks is appended to an overflow list and redone by the
// full-window kernel.  (64-bit B offsets; k_bw_sym below is the 32-bit version.)
struct Bs2Layout {
  int nsw, ns;
  unsigned o_bits, o_pre, o_stage, bytes;
};

__host__ __device__ inline Bs2Layout bs2_layout(int64_t wmax, int ns) {
  Bs2Layout L;
  const int nwd = (int)(((wmax > 0 ? wmax : 1) + 1023) / 1024 * 32);
  L.nsw = (nwd / 32 + 31) / 32 * 32;
  L.ns = ns;
  L.o_bits = (2u * L.nsw + 15u) & ~15u;
  L.o_pre = L.o_bits + 128u * ns;
  L.o_stage = L.o_pre;         // o_pre is 16-aligned
  L.bytes = L.o_stage + 512u;  // a_ij chunk records of walk_row_staged
  return L;
}

template <typename IT, typename V>
__global__ void __launch_bounds__(256) k_bw_struct2(Stage3Args a, Bs2Layout L) {
  extern __shared__ __align__(16) uint32_t s_bw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned dir = (unsigned)__cvta_generic_to_shared(s_bw) + unsigned(w) * L.bytes;
  const unsigned bits = dir + L.o_bits;
  const unsigned stage = dir + L.o_stage, bitsm = bits - 128u;
  const int ns = L.ns, nsw = L.nsw;
  for (unsigned i = lane; i < L.o_pre / 16u; i += 32) sh_st_v4_zero(dir + 16u * i);
  __syncwarp();
  const unsigned lt = lanemask_lt_();
  int bmax = 0;

  const int64_t per = (a.count + gridDim.x - 1) / gridDim.x;  // contiguous rows per CTA (L1 reuse)
  const int64_t rend = min(int64_t(blockIdx.x) * per + per, a.count);
  for (int64_t r = int64_t(blockIdx.x) * per + w; r < rend; r += nw) {
    const int row = __ldg(a.perm + a.first + r);
    const int lo = __ldg(a.rlo + row);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    int nslot = 0;  // warp-uniform
    walk_any<false, IT, V>(a, a0, a1, lane, stage, [=, &nslot](int c, V, V, bool act) {
      const unsigned d = act ? (unsigned)(c - lo) : 0u;
      const unsigned blk = d >> 10;
      unsigned s = act ? sh_ld_u16(dir + 2u * blk) : 1u;
      const bool need = s == 0u;
      const unsigned nm = __ballot_sync(kFull, need);
      if (nm) {  // first touch of some blocks: the first lane of each block's run claims a slot
        const unsigned bp = __shfl_up_sync(kFull, blk, 1);
        const bool lead = need && (lane == 0 || !((nm >> (lane - 1)) & 1u) || bp != blk);
        const unsigned lm = __ballot_sync(kFull, lead);
        const int id = nslot + __popc(lm & lt) + 1;
        if (lead && id <= ns) sh_st_u16(dir + 2u * blk, (unsigned)id);
        nslot += __popc(lm);
        __syncwarp();
        if (need) s = sh_ld_u16(dir + 2u * blk);
      }
      // word (s-1)*32 + (d>>5)%32 of the slots: bits - 128 + 128 s + ((d >> 3) & 0x7c)
      if (act && s != 0u) sh_red_or(bitsm + (s << 7) + ((d >> 3) & 0x7cu), 1u << (d & 31));
    });
    __syncwarp();
    if (nslot > ns) {
      // too many blocks: clear and hand the row to the full-window kernel
      for (int s = 0; s < ns; ++s) sh_st(bits + 4u * (unsigned(s) * 32u + lane), 0u);
      for (int q = lane; q < nsw / 8; q += 32) sh_st_v4_zero(dir + 16u * q);
      if (lane == 0) a.bw_ovf_list[atomicAdd(a.bw_ovf_cnt, 1)] = row;
      __syncwarp();
      continue;
    }
    // the sorted column set: blocks in ascending order, words by their wmask bits
    const int64_t o = __ldg(a.out_off + row);
    int32_t* oc = a.out_col + o;
    int nnz = 0;
    for (int s0 = 0; s0 < nsw; s0 += 32) {
      const unsigned dl = sh_ld_u16(dir + 2u * (s0 + lane));
      unsigned nzb = __ballot_sync(kFull, dl != 0u);
      if (dl) sh_st_u16(dir + 2u * (s0 + lane), 0u);
      while (nzb) {
        const int b = __ffs(nzb) - 1;
        nzb &= nzb - 1;
        const unsigned slot = __shfl_sync(kFull, dl, b) - 1u;
        const unsigned wa = bits + 4u * (slot * 32u + lane);
        unsigned word = sh_ld(wa);
        if (word) sh_st(wa, 0u);
        const int pc = __popc(word);
        const int inc = warp_incl_scan(pc, lane);
        int p = nnz + inc - pc;
        const int cb = lo + ((s0 + b) * 32 + lane) * 32 - 1;
        int32_t* q = oc + p;
        while (word) {
          *q++ = cb + __ffs(word);
          word &= word - 1;
        }
        nnz += __shfl_sync(kFull, inc, 31);
      }
    }
    bmax = max(bmax, nslot);
    if (lane == 0 && a.nnz_row) a.nnz_row[row] = nnz;
    __syncwarp();
  }
  if (lane == 0 && bmax > 0 && a.bw_bmax_out)
    atomicMax(reinterpret_cast<unsigned long long*>(a.bw_bmax_out), (unsigned long long)bmax);
}

// ----------------------------------------------------------------------------------------
// T_BW STRUCT (precise symbolic), 32-bit B offsets: the block-directory bitmap of
// k_bw_struct2 with the per-step work cut down.
//  * walk: the a_ij chunk is staged as 16-byte records (one LDS.64 per b_j*); the four steps
//    of a group load their columns and directory slots first and take ONE vote for first
//    touches of a block (rare) instead of one per step; slot 0 is a dummy, so idle lanes and
//    rows past the slot limit OR into it without a branch.
//  * emission: the row's nonzero words are first compacted, in column order, into a list of
//    (first column, bits) pairs in the warp's stage buffer; each full list of 32 words costs
//    one scan, so the per-block scans of k_bw_struct2 (36 % of its instructions on c2) go.
// Per warp: dir uint16[nsw] | bits uint32[(ns+1)·32] | stage 64 x 8 B.
struct SymLayout {
  int nsw, ns;
  unsigned o_bits, o_stage, bytes;
};
// slots of 33 words: the same word of different slots (a stencil's z-neighbour planes) lands in
// different banks
constexpr unsigned kSlotBytes = 132u;

__host__ __device__ inline SymLayout sym_layout(int64_t wmax, int ns) {
  SymLayout L;
  const int nwd = (int)(((wmax > 0 ? wmax : 1) + 1023) / 1024 * 32);
  L.nsw = (nwd / 32 + 31) / 32 * 32;
  L.ns = ns;
  L.o_bits = (2u * L.nsw + 15u) & ~15u;
  L.o_stage = (L.o_bits + kSlotBytes * (ns + 1) + 15u) & ~15u;
  L.bytes = L.o_stage + 512u;
  return L;
}

#ifndef SG_SYM_MINB
#define SG_SYM_MINB 6
#endif
__global__ void __launch_bounds__(256, SG_SYM_MINB) k_bw_sym(Stage3Args a, SymLayout L) {
  extern __shared__ __align__(16) uint32_t s_bw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned dir = (unsigned)__cvta_generic_to_shared(s_bw) + unsigned(w) * L.bytes;
  const unsigned bits = dir + L.o_bits, stage = dir + L.o_stage;
  const int ns = L.ns, nsw = L.nsw;
  const int32_t* __restrict__ aci = a.A.ci;
  const int64_t* __restrict__ brp = a.B.rp;
  const int32_t* __restrict__ bci = a.B.ci;
  for (unsigned i = lane; i < L.o_stage / 16u; i += 32) sh_st_v4_zero(dir + 16u * i);
  __syncwarp();
  const unsigned lt = lanemask_lt_(), le = lt | (1u << lane);
  int bmax = 0;

  const int64_t per = (a.count + gridDim.x - 1) / gridDim.x;  // contiguous rows per CTA (L1 reuse)
  const int64_t rend = min(int64_t(blockIdx.x) * per + per, a.count);
  for (int64_t r = int64_t(blockIdx.x) * per + w; r < rend; r += nw) {
    const int row = __ldg(a.perm + a.first + r);
    const int lo = __ldg(a.rlo + row);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    int nslot = 0;  // warp-uniform
    for (int64_t e0 = a0; e0 < a1; e0 += 32) {
      const int64_t e = e0 + lane;
      int bs = 0, len = 0;
      if (e < a1) {
        const int j = __ldg(aci + e);
        const int64_t b0 = __ldg(brp + j);
        bs = (int)b0;
        len = (int)(__ldg(brp + j + 1) - b0);
      }
      __syncwarp();
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(stage + 8u * lane), "r"(bs), "r"(len) : "memory");
      __syncwarp();
      const int nE = (int)min(int64_t(32), a1 - e0);
      const bool chunk_long = __any_sync(kFull, len > 32);  // one vote per 32 a_ij
      for (int t0 = 0; t0 < nE; t0 += kGroup) {
        if (chunk_long) {
          // a b_j* longer than 32 in this chunk: the general path for its groups
          for (int u = 0; u < kGroup && t0 + u < nE; ++u) {
            const uint2 rec = sh_ld_v2(stage + 8u * (t0 + u));
            for (int q0 = 0; q0 < (int)rec.y; q0 += 32) {
              const bool act = q0 + lane < (int)rec.y;
              const unsigned dd = act ? (unsigned)(__ldg(bci + (int)rec.x + q0 + lane) - lo) : 0u;
              unsigned s1 = act ? sh_ld_u16(dir + 2u * (dd >> 10)) : 0u;
              const bool nd = act && s1 == 0u;
              const unsigned nm = __ballot_sync(kFull, nd);
              if (nm) {
                const unsigned blk = dd >> 10;
                const unsigned bp = __shfl_up_sync(kFull, blk, 1);
                const bool lead = nd && (lane == 0 || !((nm >> (lane - 1)) & 1u) || bp != blk);
                const unsigned lm = __ballot_sync(kFull, lead);
                const int id = nslot + __popc(lm & lt) + 1;
                if (lead && id <= ns) sh_st_u16(dir + 2u * blk, (unsigned)id);
                nslot += __popc(lm);
                __syncwarp();
                if (nd) s1 = sh_ld_u16(dir + 2u * blk);
              }
              sh_red_or(bits + s1 * kSlotBytes + ((dd >> 3) & 0x7cu), act ? 1u << (dd & 31) : 0u);
            }
          }
          continue;
        }
        unsigned d[kGroup], sl[kGroup];
        bool need[kGroup];
#pragma unroll
        for (int u = 0; u < kGroup; ++u) {
          const uint2 rec = sh_ld_v2(stage + 8u * (t0 + u));  // lanes past the row: len 0
          const bool act = lane < (int)rec.y;
          const int q = (int)rec.x + lane;  // 32-bit index: one IMAD.WIDE per gather
          d[u] = act ? (unsigned)(__ldg(bci + q) - lo) : 0u;
          sl[u] = act ? sh_ld_u16(dir + 2u * (d[u] >> 10)) : 0u;  // 0: dummy slot / no slot yet
          need[u] = act && sl[u] == 0u;
        }
        const bool any_need = need[0] || need[1] || need[2] || need[3];
        if (__any_sync(kFull, any_need)) {
          // first touch of some blocks: the first lane of each block's run claims a slot,
          // step by step (the steps' order is the walk's order)
#pragma unroll
          for (int u = 0; u < kGroup; ++u) {
            const unsigned nm = __ballot_sync(kFull, need[u]);
            if (nm) {
              const unsigned blk = d[u] >> 10;
              const unsigned bp = __shfl_up_sync(kFull, blk, 1);
              const bool lead = need[u] && (lane == 0 || !((nm >> (lane - 1)) & 1u) || bp != blk);
              const unsigned lm = __ballot_sync(kFull, lead);
              const int id = nslot + __popc(lm & lt) + 1;
              if (lead && id <= ns) sh_st_u16(dir + 2u * blk, (unsigned)id);
              nslot += __popc(lm);
              __syncwarp();
#pragma unroll
              for (int v2 = u; v2 < kGroup; ++v2)  // later steps may touch the same new blocks
                if (need[v2]) {
                  sl[v2] = sh_ld_u16(dir + 2u * (d[v2] >> 10));
                  need[v2] = sl[v2] == 0u;
                }
            }
          }
        }
        // line 8 of Algorithm 1: set the column's bit (idle lanes and slot-less rows: no RED)
#pragma unroll
        for (int u = 0; u < kGroup; ++u)  // idle lanes and slot-less rows: OR 0 into the dummy slot
          sh_red_or(bits + sl[u] * kSlotBytes + ((d[u] >> 3) & 0x7cu), sl[u] ? 1u << (d[u] & 31) : 0u);
      }
    }
    __syncwarp();
    if (nslot > ns) {
      // too many blocks: clear and hand the row to the full-window kernel
      for (int s = 1; s <= ns; ++s) sh_st(bits + kSlotBytes * s + 4u * lane, 0u);
      for (int q = lane; q < nsw / 8; q += 32) sh_st_v4_zero(dir + 16u * q);
      if (lane == 0) a.bw_ovf_list[atomicAdd(a.bw_ovf_cnt, 1)] = row;
      __syncwarp();
      continue;
    }
    // the row's structure: nonzero words in column order -> list (stage) -> the row's slice,
    // as the words themselves ((first column, bits) pairs: DENSE takes their ranks by one scan)
    // when 8 B per word fits the slice, else as the sorted column set
    const int64_t o = __ldg(a.out_off + row);
    int32_t* oc = a.out_col + o;
    bool words = false;
    if (a.bw_nw) {
      // at most 32 words per slot: count them only when that bound does not settle it
      const int64_t cap = __ldg(a.out_off + row + 1) - o;
      words = 64 * int64_t(nslot) <= cap;
      if (!words) {
        int nwt = 0;
        for (int s = 1; s <= nslot; ++s) nwt += __popc(__ballot_sync(kFull, sh_ld(bits + s * kSlotBytes + 4u * lane) != 0u));
        words = 2 * int64_t(nwt) <= cap;
      }
      if (lane == 0 && !words) a.bw_nw[row] = -1;
    }
    int nnz = 0, nl = 0;
    if (words) {
      // nonzero words straight to the slice in column order (coalesced 8-byte stores)
      int nwo = 0;
      unsigned pcs = 0;
      for (int s0 = 0; s0 < nsw; s0 += 32) {
        const unsigned dl = sh_ld_u16(dir + 2u * (s0 + lane));
        unsigned nzb = __ballot_sync(kFull, dl != 0u);
        if (dl) sh_st_u16(dir + 2u * (s0 + lane), 0u);
        while (nzb) {
          const int b = __ffs(nzb) - 1;
          nzb &= nzb - 1;
          const unsigned wa = bits + __shfl_sync(kFull, dl, b) * kSlotBytes + 4u * lane;
          const unsigned word = sh_ld(wa);
          const unsigned nzw = __ballot_sync(kFull, word != 0u);
          if (word) {
            sh_st(wa, 0u);
            reinterpret_cast<uint2*>(oc)[nwo + __popc(nzw & lt)] =
                make_uint2((unsigned)(lo + ((s0 + b) * 32 + lane) * 32), word);
            pcs += __popc(word);
          }
          nwo += __popc(nzw);
        }
      }
      nnz = (int)__reduce_add_sync(kFull, pcs);
      bmax = max(bmax, nslot);
      if (lane == 0) a.bw_nw[row] = nwo;
      if (lane == 0 && a.nnz_row) a.nnz_row[row] = nnz;
      __syncwarp();
      continue;
    }
    auto flush = [&](int cnt) {  // emit list entries [0, cnt) (cnt <= 32)
      uint2 ent = make_uint2(0u, 0u);
      if (lane < cnt) ent = sh_ld_v2(stage + 8u * lane);
      const int pc = __popc(ent.y);
      const int inc = warp_incl_scan(pc, lane);
      int32_t* q = oc + nnz + inc - pc;
      unsigned wd = ent.y;
      const int cb = (int)ent.x - 1;
      while (wd) {
        *q++ = cb + __ffs(wd);
        wd &= wd - 1;
      }
      nnz += __shfl_sync(kFull, inc, 31);
    };
    for (int s0 = 0; s0 < nsw; s0 += 32) {
      const unsigned dl = sh_ld_u16(dir + 2u * (s0 + lane));
      unsigned nzb = __ballot_sync(kFull, dl != 0u);
      if (dl) sh_st_u16(dir + 2u * (s0 + lane), 0u);
      while (nzb) {
        const int b = __ffs(nzb) - 1;
        nzb &= nzb - 1;
        const unsigned wa = bits + __shfl_sync(kFull, dl, b) * kSlotBytes + 4u * lane;
        const unsigned word = sh_ld(wa);
        const unsigned nzw = __ballot_sync(kFull, word != 0u);
        if (word) {
          sh_st(wa, 0u);
          const int pos = nl + __popc(nzw & lt);  // < 64
          asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(stage + 8u * pos),
                       "r"((unsigned)(lo + ((s0 + b) * 32 + lane) * 32)), "r"(word) : "memory");
        }
        nl += __popc(nzw);
        __syncwarp();
        if (nl >= 32) {
          flush(32);
          nl -= 32;
          __syncwarp();
          if (lane < nl) {
            const uint2 rest = sh_ld_v2(stage + 8u * (32 + lane));
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(stage + 8u * lane), "r"(rest.x), "r"(rest.y)
                         : "memory");
          }
          __syncwarp();
        }
      }
    }
    if (nl > 0) flush(nl);
    bmax = max(bmax, nslot);
    if (lane == 0 && a.nnz_row) a.nnz_row[row] = nnz;
    __syncwarp();
  }
  if (lane == 0 && bmax > 0 && a.bw_bmax_out)
    atomicMax(reinterpret_cast<unsigned long long*>(a.bw_bmax_out), (unsigned long long)bmax);
}

// ----------------------------------------------------------------------------------------
// T_BW in ONE walk (hybrid strategy, 32-bit B offsets): the dense accumulator of [P:142]
// restricted to the row's column window, with storage only where the products land.  The
// window is cut into 1024-column blocks (a directory, slots claimed on first touch, as in
// k_bw_sym) and each block into 8-column granules; a granule is claimed on first touch and
// holds 8 values and a presence mask.  Every product is inserted and accumulated in the same
// step (Algorithm 1 lines 6-11): set its column's bit, add a_ij*b_jk to its value — in
// j-ascending order per column from -0.0, the oracle's rounding (R1).  At the end
// the row's granules are sorted by column (one warp bitonic sort of their keys), their
// popcounts scanned into positions, and each lane writes its granule's entries to the row's
// C~ slice in order.  No structure pass, no ranks.  A row touching more than kOneSlots blocks
// or kOneGran granules is listed in bw_ovf_list and goes through the two-walk path
// (k_bw_sym + k_bwrow DENSE).
// Per warp: dir u16[nsw] | sblk u16[NS] (block of each slot) | gtab u8[NS*128] (granule of
// each 8 columns, +1) | gkey u32[NG] | gbits u32[NG] | vals V[8*NG] + scratch | stage 512 B.
constexpr int kOneSlots = 12;
constexpr int kOneGran = 56;

struct OneLayout {
  int nsw;
  unsigned o_sblk, o_gtab, o_gkey, o_gbits, o_vals, o_stage, o_zero, bytes;
};

__host__ __device__ inline OneLayout one_layout(int64_t wmax, int vbytes) {
  OneLayout L;
  const int nb = (int)(((wmax > 0 ? wmax : 1) + 1023) / 1024);
  L.nsw = (nb + 31) / 32 * 32;
  L.o_sblk = (2u * L.nsw + 15u) & ~15u;
  L.o_gtab = (L.o_sblk + 2u * kOneSlots + 15u) & ~15u;
  L.o_gkey = (L.o_gtab + 128u * kOneSlots + 15u) & ~15u;
  L.o_gbits = L.o_gkey + 4u * kOneGran;
  L.o_zero = (L.o_gbits + 4u * kOneGran + 15u) & ~15u;  // [0, o_zero): zero between rows
  L.o_vals = L.o_zero;
  L.o_stage = (L.o_vals + unsigned(vbytes) * (8u * kOneGran + 2u) + 15u) & ~15u;
  L.bytes = L.o_stage + 512u;
  return L;
}

__device__ __forceinline__ unsigned sh_ld_u8(unsigned addr) {
  unsigned short r;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void sh_st_u8(unsigned addr, unsigned v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
}

// ascending bitonic sort of 64 keys held two per lane (k0: element lane, k1: element 32+lane)
__device__ __forceinline__ void warp_sort64(unsigned& k0, unsigned& k1, int lane) {
#pragma unroll
  for (int size = 2; size <= 64; size <<= 1) {
    if (size == 64) {  // the merge across the halves: element i vs i+32, then within halves
      const unsigned lo = min(k0, k1), hi = max(k0, k1);
      k0 = lo;
      k1 = hi;
    }
#pragma unroll
    for (int stride = (size == 64 ? 16 : size / 2); stride > 0; stride >>= 1) {
      // within each 32-element half, element index i = lane (k0) or 32 + lane (k1)
      const bool up0 = size == 64 ? true : ((lane & size) == 0);
      const bool up1 = size == 64 ? true : (((32 + lane) & size) == 0);
      const unsigned o0 = __shfl_xor_sync(kFull, k0, stride), o1 = __shfl_xor_sync(kFull, k1, stride);
      const bool lower = (lane & stride) == 0;
      k0 = (lower == up0) ? min(k0, o0) : max(k0, o0);
      k1 = (lower == up1) ? min(k1, o1) : max(k1, o1);
    }
  }
}

template <typename V>
__global__ void __launch_bounds__(256, 4) k_bw_one(Stage3Args a, OneLayout L) {
  extern __shared__ __align__(16) uint32_t s_bw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned dir = (unsigned)__cvta_generic_to_shared(s_bw) + unsigned(w) * L.bytes;
  const unsigned sblk = dir + L.o_sblk, gtab = dir + L.o_gtab, gkey = dir + L.o_gkey, gbits = dir + L.o_gbits;
  const unsigned vals = dir + L.o_vals, stage = dir + L.o_stage;
  const unsigned scratch = vals + unsigned(sizeof(V)) * (8u * kOneGran);
  const int32_t* __restrict__ aci = a.A.ci;
  const V* __restrict__ aval = vcast<V>(a.A.val);
  const int64_t* __restrict__ brp = a.B.rp;
  const int32_t* __restrict__ bci = a.B.ci;
  const V* __restrict__ bval = vcast<V>(a.B.val);
  for (unsigned i = lane; i < L.o_zero / 16u; i += 32) sh_st_v4_zero(dir + 16u * i);
  for (unsigned i = lane; i < 8u * kOneGran + 2u; i += 32) sh_stv(vals + unsigned(sizeof(V)) * i, V(-0.0));
  __syncwarp();
  const unsigned lt = lanemask_lt_();

  const int64_t per = (a.count + gridDim.x - 1) / gridDim.x;  // contiguous rows per CTA (L1 reuse)
  const int64_t rend = min(int64_t(blockIdx.x) * per + per, a.count);
  for (int64_t r = int64_t(blockIdx.x) * per + w; r < rend; r += nw) {
    const int row = __ldg(a.perm + a.first + r);
    const int lo = __ldg(a.rlo + row);
    const int64_t a0 = __ldg(a.A.rp + row), a1 = __ldg(a.A.rp + row + 1);
    int nslot = 0, ngr = 0;  // warp-uniform

    // first touch of blocks, then of granules, for one step (lanes of a b_j* hold ascending
    // columns, so the lanes needing one new block / granule are contiguous: the first of
    // each run claims it); sl / gi stay 0 when the row runs out of slots / granules
    auto claim = [&](unsigned d, bool act, unsigned& sl, unsigned& gi) {
      const bool nsl = act && sl == 0u;
      unsigned nm = __ballot_sync(kFull, nsl);
      if (nm) {
        const unsigned blk = d >> 10;
        const unsigned bp = __shfl_up_sync(kFull, blk, 1);
        const bool lead = nsl && (lane == 0 || !((nm >> (lane - 1)) & 1u) || bp != blk);
        const unsigned lm = __ballot_sync(kFull, lead);
        const int id = nslot + __popc(lm & lt) + 1;
        if (lead && id <= kOneSlots) {
          sh_st_u16(dir + 2u * blk, (unsigned)id);
          sh_st_u16(sblk + 2u * (id - 1), blk);
        }
        nslot += __popc(lm);
        __syncwarp();
        if (nsl) {
          sl = sh_ld_u16(dir + 2u * blk);
          if (sl) gi = sh_ld_u8(gtab + (sl - 1u) * 128u + ((d >> 3) & 127u));
        }
      }
      const bool ngl = act && sl != 0u && gi == 0u;
      nm = __ballot_sync(kFull, ngl);
      if (nm) {
        const unsigned key = d >> 3;
        const unsigned kp = __shfl_up_sync(kFull, key, 1);
        const bool lead = ngl && (lane == 0 || !((nm >> (lane - 1)) & 1u) || kp != key);
        const unsigned lm = __ballot_sync(kFull, lead);
        const int id = ngr + __popc(lm & lt) + 1;
        if (lead && id <= kOneGran) {
          sh_st_u8(gtab + (sl - 1u) * 128u + (key & 127u), (unsigned)id);
          sh_st(gkey + 4u * (id - 1), key);
        }
        ngr += __popc(lm);
        __syncwarp();
        if (ngl) gi = sh_ld_u8(gtab + (sl - 1u) * 128u + (key & 127u));
      }
    };
    // line 8 (insert: the column's bit) and lines 9 / 11 (accumulate) of one product
    auto insert_add = [&](unsigned d, unsigned gi, V pr) {
      if (gi) sh_red_or(gbits + 4u * (gi - 1u), 1u << (d & 7u));
      const unsigned va = gi ? vals + unsigned(sizeof(V)) * ((gi - 1u) * 8u + (d & 7u)) : scratch;
      sh_stv(va, Arith<V>::add(sh_ldv<V>(va), pr));
      __syncwarp();  // the next step's lanes may read this slot
    };

    bool fail = false;
    for (int64_t e0 = a0; e0 < a1 && !fail; e0 += 32) {
      const int64_t e = e0 + lane;
      int bs = 0, len = 0;
      V av = V(0);
      if (e < a1) {
        const int j = __ldg(aci + e);
        const int64_t b0 = __ldg(brp + j);
        bs = (int)b0;
        len = (int)(__ldg(brp + j + 1) - b0);
        av = __ldg(aval + e);
      }
      const double avd = (double)av;
      const int lo_w = sizeof(V) == 8 ? __double2loint(avd) : __float_as_int((float)av);
      const int hi_w = sizeof(V) == 8 ? __double2hiint(avd) : 0;
      __syncwarp();
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stage + 16u * lane), "r"(bs), "r"(len),
                   "r"(lo_w), "r"(hi_w) : "memory");
      __syncwarp();
      const int nE = (int)min(int64_t(32), a1 - e0);
      if (__any_sync(kFull, len > 32)) {
        for (int t = 0; t < nE && !fail; ++t) {
          int4 rr;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(rr.x), "=r"(rr.y), "=r"(rr.z), "=r"(rr.w) : "r"(stage + 16u * t) : "memory");
          const V at = rec_val<V>(rr);
          for (int q0 = 0; q0 < rr.y; q0 += 32) {
            const bool act = q0 + lane < rr.y;
            const int q = rr.x + q0 + lane;
            const unsigned d = act ? (unsigned)(__ldg(bci + q) - lo) : 0u;
            const V pr = act ? Arith<V>::mul(at, __ldg(bval + q)) : V(0);
            unsigned sl = act ? sh_ld_u16(dir + 2u * (d >> 10)) : 0u;
            unsigned gi = sl ? sh_ld_u8(gtab + (sl - 1u) * 128u + ((d >> 3) & 127u)) : 0u;
            claim(d, act, sl, gi);
            if (nslot > kOneSlots || ngr > kOneGran) {
              fail = true;
              break;
            }
            insert_add(d, gi, pr);
          }
        }
        continue;
      }
      for (int t0 = 0; t0 < nE; t0 += kGroup) {
        unsigned d[kGroup], sl[kGroup], gi[kGroup];
        V pr[kGroup];
        bool act[kGroup];
        bool need = false;
#pragma unroll
        for (int u = 0; u < kGroup; ++u) {
          int4 rr;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(rr.x), "=r"(rr.y), "=r"(rr.z), "=r"(rr.w) : "r"(stage + 16u * (t0 + u)) : "memory");
          act[u] = lane < rr.y;
          const int q = rr.x + min(lane, max(rr.y - 1, 0));
          const int c = __ldg(bci + q);
          pr[u] = Arith<V>::mul(rec_val<V>(rr), __ldg(bval + q));
          d[u] = act[u] ? (unsigned)(c - lo) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kGroup; ++u) {
          sl[u] = act[u] ? sh_ld_u16(dir + 2u * (d[u] >> 10)) : 0u;
          gi[u] = sl[u] ? sh_ld_u8(gtab + (sl[u] - 1u) * 128u + ((d[u] >> 3) & 127u)) : 0u;
          need = need || (act[u] && gi[u] == 0u);
        }
        if (__any_sync(kFull, need)) {
          // first touches, step by step in walk order; a later step of the group may hit a
          // block / granule claimed by an earlier one, so its lookups are refreshed (once,
          // just before its own claims) when the group has claimed anything so far
          bool claimed = false;  // warp-uniform
#pragma unroll
          for (int u = 0; u < kGroup; ++u) {
            if (claimed && act[u] && gi[u] == 0u) {
              sl[u] = sh_ld_u16(dir + 2u * (d[u] >> 10));
              gi[u] = sl[u] ? sh_ld_u8(gtab + (sl[u] - 1u) * 128u + ((d[u] >> 3) & 127u)) : 0u;
            }
            const int ns0 = nslot, ng0 = ngr;
            claim(d[u], act[u], sl[u], gi[u]);
            claimed = claimed || nslot != ns0 || ngr != ng0;
          }
          if (nslot > kOneSlots || ngr > kOneGran) {
            fail = true;
            break;
          }
        }
#pragma unroll
        for (int u = 0; u < kGroup; ++u) insert_add(d[u], gi[u], pr[u]);
      }
    }
    __syncwarp();
    const int ns = min(nslot, kOneSlots), ng = min(ngr, kOneGran);
    if (!fail) {
      // the row's granules in column order: sort (key << 8 | granule), scan the popcounts
      unsigned k0 = lane < ng ? (sh_ld(gkey + 4u * lane) << 8) | unsigned(lane) : 0xffffffffu;
      unsigned k1 = 32 + lane < ng ? (sh_ld(gkey + 4u * (32 + lane)) << 8) | unsigned(32 + lane) : 0xffffffffu;
      if (ng > 32) {
        warp_sort64(k0, k1, lane);
      } else {
        // 32 keys: the first half of the network
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
          for (int stride = size / 2; stride > 0; stride >>= 1) {
            const unsigned o0 = __shfl_xor_sync(kFull, k0, stride);
            const bool up = (lane & size) == 0, lower = (lane & stride) == 0;
            k0 = (lower == up) ? min(k0, o0) : max(k0, o0);
          }
      }
      const unsigned b0 = k0 != 0xffffffffu ? sh_ld(gbits + 4u * (k0 & 0xffu)) : 0u;
      const unsigned b1 = k1 != 0xffffffffu ? sh_ld(gbits + 4u * (k1 & 0xffu)) : 0u;
      const int p0c = __popc(b0), p1c = __popc(b1);
      const int inc0 = warp_incl_scan(p0c, lane);
      const int tot0 = __shfl_sync(kFull, inc0, 31);
      const int inc1 = warp_incl_scan(p1c, lane);
      const int nnz = tot0 + __shfl_sync(kFull, inc1, 31);
      // each lane writes its granules' entries at their positions, restoring the values to
      // -0.0 and the masks to 0 behind it
      const int64_t o = __ldg(a.out_off + row);
      int32_t* oc = a.out_col + o;
      V* ov = vcast<V>(a.out_val) + o;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const unsigned kk = h ? k1 : k0;
        unsigned wd = h ? b1 : b0;
        int p = h ? tot0 + inc1 - p1c : inc0 - p0c;
        if (kk != 0xffffffffu) {
          const unsigned g = kk & 0xffu;
          const int cb = lo + (int)((kk >> 8) << 3) - 1;
          const unsigned vb = vals + unsigned(sizeof(V)) * (8u * g);
          sh_st(gbits + 4u * g, 0u);
          while (wd) {
            const int f = __ffs(wd);
            wd &= wd - 1;
            const unsigned va = vb + unsigned(sizeof(V)) * unsigned(f - 1);
            oc[p] = cb + f;
            ov[p] = sh_ldv<V>(va);
            sh_stv(va, V(-0.0));
            ++p;
          }
        }
      }
      if (lane == 0) a.nnz_row[row] = nnz;
    } else {
      // out of slots or granules: restore the cleared state, hand the row to the two-walk path
      for (int g = lane; g < ng; g += 32) {
        sh_st(gbits + 4u * g, 0u);
        for (int k = 0; k < 8; ++k) sh_stv(vals + unsigned(sizeof(V)) * (8u * g + k), V(-0.0));
      }
      if (lane == 0) a.bw_ovf_list[atomicAdd(a.bw_ovf_cnt, 1)] = row;
    }
    // directory entries of the row's blocks and their granule tables
    if (lane < ns) sh_st_u16(dir + 2u * sh_ld_u16(sblk + 2u * lane), 0u);
    for (int i = lane; i < ns * 8; i += 32) sh_st_v4_zero(gtab + 16u * i);
    __syncwarp();
  }
}

}  // namespace

template <typename K>
static cudaError_t launch_warp_kernel(K kernel, int nw, int64_t rows, const Stage3Args& a, cudaStream_t s) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nw * 32, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (rows + nw - 1) / nw;
  const int64_t cap = int64_t(num_sms()) * per_sm * 4;
  int64_t grid = need < cap ? need : cap;
  if (grid < 1) grid = 1;
  kernel<<<(unsigned)grid, nw * 32, 0, s>>>(a);
  return cudaGetLastError();
}

// Warp classes T_W64..T_W2048: S = 64 << (tier - T_W64) slots; the count uses 2S for S <= 512
// (load <= 0.4 instead of 0.8: c3a w64..w512 counts 1.6x faster; at 1024/2048 the halved
// occupancy cancels the shorter probes).  Warps per block: as many as the 48 KB static
// shared-memory limit allows, at most 8.
cudaError_t launch_warp_tier(int tier, const Stage3Args& a, cudaStream_t s) {
  const bool i32 = a.b_nnz < (int64_t(1) << 31);
#define SG_NW(BYTES) ((49152 / (BYTES)) < 8 ? (49152 / (BYTES)) : 8)
#define SG_W(LOG2S)                                                                           \
  {                                                                                           \
    constexpr int LC = LOG2S <= 9 ? LOG2S + 1 : LOG2S;                                        \
    constexpr int NC = SG_NW(4 << LC);                                                        \
    return i32 ? launch_warp_kernel(k_wrow<LC, NC, int>, NC, a.count, a, s)                  \
               : launch_warp_kernel(k_wrow<LC, NC, int64_t>, NC, a.count, a, s);             \
  }
  if (a.mode != MODE_COUNT) return cudaErrorInvalidValue;  // values: the ESC (stage3.cu)
  switch (tier) {
    case T_W64: SG_W(6)
    case T_W128: SG_W(7)
    case T_W256: SG_W(8)
    case T_W512: SG_W(9)
    case T_W1024: SG_W(10)
    case T_W2048: SG_W(11)
    default: return cudaErrorInvalidValue;
  }
#undef SG_W
#undef SG_NW
}

// T_BW launch: shared memory sized by the class's largest window and row length; warps per
// block chosen for the most resident warps per SM.
template <int MODE>
static cudaError_t launch_bw_mode(const Stage3Args& a, cudaStream_t s) {
  const BwLayout L = bw_layout(MODE, a.bw_wmax, a.bw_vmax, a.bw_bmax);
  const bool i32 = a.b_nnz < (int64_t(1) << 31);
  const bool f32 = a.f32 && MODE == MODE_DENSE;
  auto kern = f32 ? (i32 ? k_bwrow<MODE, int, float> : k_bwrow<MODE, int64_t, float>)
                  : (i32 ? k_bwrow<MODE, int, double> : k_bwrow<MODE, int64_t, double>);
  int best_nw = 1, best_warps = 0;
  for (int nw = 8; nw >= 1; nw >>= 1) {
    const size_t bytes = size_t(nw) * L.bytes;
    if (bytes > 227 * 1024) continue;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, bytes);
    if (e != cudaSuccess) return e;
    if (per_sm * nw > best_warps) {
      best_warps = per_sm * nw;
      best_nw = nw;
    }
  }
  if (best_warps == 0) return cudaErrorInvalidConfiguration;
  const size_t bytes = size_t(best_nw) * L.bytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  const int64_t need = (a.count + best_nw - 1) / best_nw;
  const int64_t cap = int64_t(num_sms()) * (best_warps / best_nw);
  const int64_t grid = need < cap ? need : cap;
  kern<<<(unsigned)grid, best_nw * 32, bytes, s>>>(a, L);
  return cudaGetLastError();
}

constexpr int kBs2Slots = 16;

template <typename IT>
static cudaError_t launch_bs2(const Stage3Args& a, cudaStream_t s) {
  const Bs2Layout L = bs2_layout(a.bw_wmax, kBs2Slots);
  auto kern = k_bw_struct2<IT, double>;
  constexpr int nw = 8;
  const size_t bytes = size_t(nw) * L.bytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (a.count + nw - 1) / nw;
  const int64_t cap = int64_t(num_sms()) * per_sm;
  kern<<<(unsigned)(need < cap ? need : cap), nw * 32, bytes, s>>>(a, L);
  return cudaGetLastError();
}

static cudaError_t launch_sym(const Stage3Args& a, cudaStream_t s) {
  const SymLayout L = sym_layout(a.bw_wmax, kBs2Slots);
  constexpr int nw = 8;
  const size_t bytes = size_t(nw) * L.bytes;
  cudaError_t e = cudaFuncSetAttribute(k_bw_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bw_sym, nw * 32, bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (a.count + nw - 1) / nw;
  const int64_t cap = int64_t(num_sms()) * per_sm;
  k_bw_sym<<<(unsigned)(need < cap ? need : cap), nw * 32, bytes, s>>>(a, L);
  return cudaGetLastError();
}

// Hybrid window rows in one walk (k_bw_one); rows out of slots or granules are listed in
// a.bw_ovf_list / a.bw_ovf_cnt (zeroed here) for the two-walk path.
cudaError_t launch_bw_one(const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  const OneLayout L = one_layout(a.bw_wmax, a.f32 ? 4 : 8);
  auto kern = a.f32 ? k_bw_one<float> : k_bw_one<double>;
  constexpr int nw = 8;
  const size_t bytes = size_t(nw) * L.bytes;
  if (bytes > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaMemsetAsync(a.bw_ovf_cnt, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (a.count + nw - 1) / nw;
  const int64_t cap = int64_t(num_sms()) * per_sm;
  kern<<<(unsigned)(need < cap ? need : cap), nw * 32, bytes, s>>>(a, L);
  return cudaGetLastError();
}

// Window class: STRUCT (the sorted column sets: block directory first, the full window for
// rows with more nonzero blocks than slots) or DENSE (values by rank from those sets).
cudaError_t launch_bw_tier(const Stage3Args& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  const int64_t blocks = (a.bw_wmax + 1023) / 1024;
  if (a.mode == MODE_DENSE) return launch_bw_mode<MODE_DENSE>(a, s);
  if (a.mode != MODE_STRUCT) return cudaErrorInvalidValue;
  if (blocks > kBs2Slots && a.bw_ovf_list && a.bw_ovf_cnt) {
    // block-directory pass, then the full-window pass over the rows that overflowed it
    cudaError_t e = cudaMemsetAsync(a.bw_ovf_cnt, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    const bool i32 = a.b_nnz < (int64_t(1) << 31);
    e = i32 ? launch_sym(a, s) : launch_bs2<int64_t>(a, s);
    if (e != cudaSuccess) return e;
    Stage3Args b = a;
    b.perm = a.bw_ovf_list;
    b.first = 0;
    b.count = a.count;  // grid bound; the kernel reads the real count from count_dev
    b.count_dev = a.bw_ovf_cnt;
    return launch_bw_mode<MODE_STRUCT>(b, s);
  }
  return launch_bw_mode<MODE_STRUCT>(a, s);
}

}  // namespace sg
