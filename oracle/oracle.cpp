/*
 * oracle.cpp — CPU reference ("oracle") for C = A·B on CSR matrices.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1504_05022_b200/) never links, imports or calls it, and it shares no code,
 * header, table or helper with the CUDA path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, line numbers are [P:n]):
 *   - oracle_upper_bound:  Algorithm "Pseudocode for the first stage on GPUs" [P:198-212]
 *                          u_i = sum over nonzeros a_ij of nnz(b_j*).
 *   - oracle_bins:         Algorithm "Pseudocode for the second stage on a CPU core"
 *                          [P:226-260]: 38 bins in 5 groups and the hybrid C~ sizes
 *                          (u_i for groups 1-4, 256 for group 5) [P:224].
 *   - oracle_spgemm_count / oracle_spgemm_fill:
 *                          the plain definition of C = A·B that the paper's method
 *                          reaches (Algorithm "Pseudocode for the SpGEMM" [P:115-138]:
 *                          row-wise Gustavson, "insert" or "accumulate" per product),
 *                          with the dense-vector sparse accumulator (SPA) of Gilbert et
 *                          al. cited at [P:142].  Rows come out sorted and duplicate-
 *                          free (CSR, [P:113]); no numeric dropping ("does not take into
 *                          consideration cancellation" [P:169]).
 *   - oracle_spgemm_fill_f32: the same fill in single precision (SpSGEMM, the paper's SP
 *                          experiments [P:403], [P:663]).
 *   - oracle_validate_csr: the CSR invariants the paper assumes (sorted columns, the
 *                          footnote at [P:178]).
 *
 * Floating point: products are rounded separately (no FMA: built with
 * -ffp-contract=off) and accumulated in the fixed order j ascending, then column
 * ascending (reading R1).  The first product of an entry initialises the
 * accumulator ("c_ik <- value", Algorithm line 9 [P:129]); later ones are added
 * ("c_ik <- c_ik + value", line 11 [P:131]).
 *
 * Pinned by tests/test_oracle.py (dense brute force, identity, permutation,
 * power-of-two scaling, size identities, stencil closed forms, Galerkin closed form,
 * associativity, SPEC worked examples under tests/golden/).
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

/* ---- CSR validation ------------------------------------------------------------- */
/* 0 = valid; 1 = row_ptr[0] != 0; 2 = row_ptr decreasing; 3 = row_ptr[rows] != nnz;
   4 = column out of range; 5 = columns not strictly ascending in a row. */
int oracle_validate_csr(int64_t rows, int64_t cols, const int64_t* rp, const int32_t* ci,
                        int64_t nnz) {
  if (rows < 0 || cols < 0 || nnz < 0) return 3;
  if (rp[0] != 0) return 1;
  for (int64_t i = 0; i < rows; ++i)
    if (rp[i + 1] < rp[i]) return 2;
  if (rp[rows] != nnz) return 3;
  for (int64_t i = 0; i < rows; ++i) {
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      if (ci[p] < 0 || (int64_t)ci[p] >= cols) return 4;
      if (p > rp[i] && ci[p] <= ci[p - 1]) return 5;
    }
  }
  return 0;
}

/* ---- Stage 1: upper bound [P:198-212] -------------------------------------------- */
/* u[i] = sum_{a_ij != 0} nnz(b_j*) for i in [r0, r1); returns sum of those u. */
int64_t oracle_upper_bound(int64_t r0, int64_t r1, const int64_t* a_rp, const int32_t* a_ci,
                           const int64_t* b_rp, int64_t* u) {
  int64_t total = 0;
#pragma omp parallel for schedule(static) reduction(+ : total)
  for (int64_t i = r0; i < r1; ++i) {
    int64_t ui = 0;                                   /* line 2: u_i <- 0          */
    for (int64_t p = a_rp[i]; p < a_rp[i + 1]; ++p) { /* line 3: each a_ij in a_i* */
      int64_t j = a_ci[p];
      ui += b_rp[j + 1] - b_rp[j];                    /* line 4: u_i += nnz(b_j*)  */
    }
    u[i - r0] = ui;
    total += ui;
  }
  return total;
}

/* ---- Stage 2: binning, Algorithm 3 [P:226-260] ---------------------------------- */
/* bin[i] in 0..37 exactly as the algorithm's ranges; ctil[i] = nnz(c~_i*) as set by
   the algorithm (u_i for bins 0..36, 256 for bin 37); returns nnz(C~) (line 35). */
int64_t oracle_bins(int64_t m, const int64_t* u, int32_t* bin, int64_t* ctil) {
  int64_t total = 0;
  for (int64_t i = 0; i < m; ++i) {
    int64_t ui = u[i];
    int32_t b;
    int64_t c;
    if (ui == 0) { b = 0; c = 0; }                          /* group 1 */
    else if (ui == 1) { b = 1; c = 1; }                     /* group 2 */
    else if (ui >= 2 && ui <= 32) { b = (int32_t)ui; c = ui; } /* group 3 */
    else if (ui >= 33 && ui <= 64) { b = 33; c = ui; }      /* group 4 */
    else if (ui >= 65 && ui <= 128) { b = 34; c = ui; }
    else if (ui >= 129 && ui <= 256) { b = 35; c = ui; }
    else if (ui >= 257 && ui <= 512) { b = 36; c = ui; }
    else { b = 37; c = 256; }                               /* group 5: u_i > 512 */
    bin[i] = b;
    ctil[i] = c;
    total += c;
  }
  return total;
}

/* ---- C = A·B: count pass (structure) --------------------------------------------- */
/* For rows [r0, r1): nnz_row[i - r0] = |{k : exists j, a_ij stored and b_jk stored}|.
   Returns sum of nnz_row.  SPA marker per thread ([P:142]). */
int64_t oracle_spgemm_count(int64_t r0, int64_t r1, int64_t n, const int64_t* a_rp,
                            const int32_t* a_ci, const int64_t* b_rp, const int32_t* b_ci,
                            int64_t* nnz_row, int threads) {
  int64_t total = 0;
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads) reduction(+ : total)
#endif
  {
    std::vector<int64_t> mark((size_t)std::max<int64_t>(n, 1), -1);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 256)
#endif
    for (int64_t i = r0; i < r1; ++i) {
      int64_t cnt = 0;
      for (int64_t p = a_rp[i]; p < a_rp[i + 1]; ++p) {
        int64_t j = a_ci[p];
        for (int64_t q = b_rp[j]; q < b_rp[j + 1]; ++q) {
          int32_t c = b_ci[q];
          if (mark[c] != i) { mark[c] = i; ++cnt; }   /* "insert c_ik to c_i*" */
        }
      }
      nnz_row[i - r0] = cnt;
      total += cnt;
    }
  }
  return total;
}

/* ---- C = A·B: fill pass (structure + values + error bound) ------------------------ */
/* c_rp has (r1 - r0 + 1) entries, relative: c_rp[0] = 0.  bound (nullable) receives
   sum_j |a_ij| |b_jk| per output entry, for the 1e-12 tolerance check. */
void oracle_spgemm_fill(int64_t r0, int64_t r1, int64_t n, const int64_t* a_rp,
                        const int32_t* a_ci, const double* a_val, const int64_t* b_rp,
                        const int32_t* b_ci, const double* b_val, const int64_t* c_rp,
                        int32_t* c_ci, double* c_val, double* bound, int threads) {
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
  {
    size_t nn = (size_t)std::max<int64_t>(n, 1);
    std::vector<double> acc(nn), absacc(bound ? nn : 1);
    std::vector<int64_t> mark(nn, -1);
    std::vector<int32_t> list;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 256)
#endif
    for (int64_t i = r0; i < r1; ++i) {
      list.clear();                                    /* line 2: c_i* <- empty     */
      for (int64_t p = a_rp[i]; p < a_rp[i + 1]; ++p) { /* line 3: each a_ij        */
        int64_t j = a_ci[p];
        double a = a_val[p];
        for (int64_t q = b_rp[j]; q < b_rp[j + 1]; ++q) { /* line 5: each b_jk     */
          int32_t c = b_ci[q];
          double prod = a * b_val[q];                  /* line 6: value <- a_ij b_jk */
          if (mark[c] != i) {                          /* line 7: c_ik not in c_i*   */
            mark[c] = i;
            list.push_back(c);                         /* line 8: insert            */
            acc[c] = prod;                             /* line 9: c_ik <- value     */
            if (bound) absacc[c] = std::fabs(a) * std::fabs(b_val[q]);
          } else {
            acc[c] = acc[c] + prod;                    /* line 11: accumulate       */
            if (bound) absacc[c] = absacc[c] + std::fabs(a) * std::fabs(b_val[q]);
          }
        }
      }
      std::sort(list.begin(), list.end());             /* CSR: ascending columns   */
      int64_t base = c_rp[i - r0];
      for (size_t t = 0; t < list.size(); ++t) {
        c_ci[base + (int64_t)t] = list[t];
        c_val[base + (int64_t)t] = acc[list[t]];
        if (bound) bound[base + (int64_t)t] = absacc[list[t]];
      }
    }
  }
}

/* ---- SpSGEMM fill (the paper's single-precision runs, [P:403], [P:663]) ------------
   The same algorithm as oracle_spgemm_fill in IEEE single precision: the product a_ij·b_jk
   is rounded to float (line 6), the first product of an entry initialises it (line 9),
   later ones are added in float (line 11), in the fixed order j ascending, then column
   ascending.  Bound (double) = sum of |a_ij|·|b_jk| for the tolerance check. */
void oracle_spgemm_fill_f32(int64_t r0, int64_t r1, int64_t n, const int64_t* a_rp,
                            const int32_t* a_ci, const float* a_val, const int64_t* b_rp,
                            const int32_t* b_ci, const float* b_val, const int64_t* c_rp,
                            int32_t* c_ci, float* c_val, double* bound, int threads) {
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
  {
    size_t nn = (size_t)std::max<int64_t>(n, 1);
    std::vector<float> acc(nn);
    std::vector<double> absacc(bound ? nn : 1);
    std::vector<int64_t> mark(nn, -1);
    std::vector<int32_t> list;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 256)
#endif
    for (int64_t i = r0; i < r1; ++i) {
      list.clear();                                    /* line 2: c_i* <- empty     */
      for (int64_t p = a_rp[i]; p < a_rp[i + 1]; ++p) { /* line 3: each a_ij        */
        int64_t j = a_ci[p];
        float a = a_val[p];
        for (int64_t q = b_rp[j]; q < b_rp[j + 1]; ++q) { /* line 5: each b_jk     */
          int32_t c = b_ci[q];
          float prod = a * b_val[q];                   /* line 6: value <- a_ij b_jk (float) */
          if (mark[c] != i) {                          /* line 7: c_ik not in c_i*   */
            mark[c] = i;
            list.push_back(c);                         /* line 8: insert            */
            acc[c] = prod;                             /* line 9: c_ik <- value     */
            if (bound) absacc[c] = std::fabs((double)a) * std::fabs((double)b_val[q]);
          } else {
            acc[c] = acc[c] + prod;                    /* line 11: accumulate (float) */
            if (bound) absacc[c] = absacc[c] + std::fabs((double)a) * std::fabs((double)b_val[q]);
          }
        }
      }
      std::sort(list.begin(), list.end());             /* CSR: ascending columns   */
      int64_t base = c_rp[i - r0];
      for (size_t t = 0; t < list.size(); ++t) {
        c_ci[base + (int64_t)t] = list[t];
        c_val[base + (int64_t)t] = acc[list[t]];
        if (bound) bound[base + (int64_t)t] = absacc[list[t]];
      }
    }
  }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  /* extern "C" */
