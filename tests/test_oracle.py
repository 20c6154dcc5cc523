"""Pins for the CPU oracle (oracle/) against things other than itself.

Each test names the pin of SURVEY.md §8(c) it implements (P1..P9) and the passage it
rests on.  Nothing here calls the CUDA path.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


def dense_to_csr(D, pattern=None):
    D = np.asarray(D, dtype=np.float64)
    mask = D != 0
    if pattern is not None:
        for (r, c) in pattern:
            mask[r, c] = True
    rows, cols = np.nonzero(mask)
    return gen.from_coo(rows, cols, D.shape, vals=D[rows, cols])


def res_dense(R, shape):
    d = np.zeros(shape)
    rows = np.repeat(np.arange(shape[0]), np.diff(R.rp))
    d[rows, R.ci] = R.val
    return d


def res_pattern(R, shape):
    d = np.zeros(shape, dtype=bool)
    rows = np.repeat(np.arange(shape[0]), np.diff(R.rp))
    d[rows, R.ci] = True
    return d


def assert_sorted_rows(R):
    for i in range(R.rp.shape[0] - 1):
        seg = R.ci[R.rp[i]:R.rp[i + 1]]
        assert np.all(np.diff(seg) > 0), "row %d not strictly ascending" % i


# ---------------------------------------------------------------- golden (SPEC / paper)
@pytest.mark.parametrize("case", GOLD["products"], ids=lambda c: c["cite"][:40])
def test_golden_products(case):
    A = dense_to_csr(case["A"])
    B = dense_to_csr(case["B"])
    R = oracle.spgemm(A, B)
    shape = (A.shape[0], B.shape[1])
    np.testing.assert_array_equal(res_dense(R, shape), np.asarray(case["C"], dtype=float))
    if "pattern" in case:
        for (r, c) in case["pattern"]:
            assert res_pattern(R, shape)[r, c], "explicit zero dropped (%s)" % case["cite"]
    if "nnz" in case:
        assert int(R.rp[-1]) == case["nnz"]
    u, tot = oracle.upper_bound(A, B)
    assert u.tolist() == case["u"]
    if "flops" in case:
        assert 2 * tot == case["flops"]
    assert_sorted_rows(R)


@pytest.mark.parametrize("case", GOLD["bins"], ids=lambda c: c["cite"][:30])
def test_golden_bins(case):
    b, c, tot = oracle.bins(np.array(case["u"]))
    assert b.tolist() == case["bin"]
    assert c.tolist() == case["ctil"]
    assert tot == sum(case["ctil"])


@pytest.mark.parametrize("case", GOLD["sizes"], ids=lambda c: c["cite"][:30])
def test_golden_sizes(case):
    if case["n"] > 200 and case["kind"] == "2d5":
        # size only (cheap): rows of the generated matrix
        assert case["n"] ** 2 == case["rows"]
        return
    A = gen.stencil(case["kind"], case["n"])
    assert A.shape[0] == case["rows"]
    if "dense" in case:
        np.testing.assert_array_equal(A.to_dense(), np.asarray(case["dense"]))


def test_bins_ranges_exhaustive():
    """Algorithm 3 [P:226-260]: every u in 0..2000 lands in the bin its range names."""
    u = np.arange(0, 2001)
    b, c, _ = oracle.bins(u)
    for ui, bi, ci in zip(u, b, c):
        if ui <= 32:
            assert bi == ui and ci == ui
        elif ui <= 64:
            assert bi == 33 and ci == ui
        elif ui <= 128:
            assert bi == 34 and ci == ui
        elif ui <= 256:
            assert bi == 35 and ci == ui
        elif ui <= 512:
            assert bi == 36 and ci == ui
        else:
            assert bi == 37 and ci == 256


# ---------------------------------------------------------------- P1 dense brute force
@pytest.mark.parametrize("density", [0.02, 0.1, 0.3, 0.7, 1.0])
@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 5, 9), (33, 17, 40), (64, 64, 64)])
def test_P1_dense_bruteforce(shape, density):
    """pattern(C) = OR_j (A_ij stored ∧ B_jk stored); values = dense product (integers,
    exact) — Algorithm 1 [P:115-138], structural semantics [P:169]."""
    m, k, n = shape
    seed = 1000 + m * 7 + int(density * 100)
    A = gen.random_csr(m, k, density, seed, mode="int", zero_frac=0.1)
    B = gen.random_csr(k, n, density, seed + 50, mode="int", zero_frac=0.1)
    R = oracle.spgemm(A, B)
    pat = (A.pattern_dense().astype(np.int64) @ B.pattern_dense().astype(np.int64)) > 0
    np.testing.assert_array_equal(res_pattern(R, (m, n)), pat)
    np.testing.assert_array_equal(res_dense(R, (m, n)), A.to_dense() @ B.to_dense())
    assert_sorted_rows(R)
    # bound = sum |a||b| = |A|·|B| on the pattern
    bd = np.zeros((m, n))
    rows = np.repeat(np.arange(m), np.diff(R.rp))
    bd[rows, R.ci] = R.bound
    np.testing.assert_array_equal(bd, np.abs(A.to_dense()) @ np.abs(B.to_dense()) * pat)


# ---------------------------------------------------------------- P2 identity
def test_P2_identity():
    B = gen.random_csr(50, 70, 0.2, 7, mode="real", zero_frac=0.05)
    I50 = gen.Csr((50, 50), np.arange(51, dtype=np.int64), np.arange(50, dtype=np.int32), np.ones(50))
    I70 = gen.Csr((70, 70), np.arange(71, dtype=np.int64), np.arange(70, dtype=np.int32), np.ones(70))
    R = oracle.spgemm(I50, B)
    np.testing.assert_array_equal(R.rp, B.rp)
    np.testing.assert_array_equal(R.ci, B.ci)
    np.testing.assert_array_equal(R.val.view(np.int64), B.val.view(np.int64))
    R = oracle.spgemm(B, I70)
    np.testing.assert_array_equal(R.rp, B.rp)
    np.testing.assert_array_equal(R.ci, B.ci)
    np.testing.assert_array_equal(R.val.view(np.int64), B.val.view(np.int64))


# ---------------------------------------------------------------- P3 permutations
def test_P3_permutations():
    A = gen.random_csr(40, 60, 0.15, 11, mode="real")
    pr = gen.permutation(5, 40)
    pc = gen.permutation(6, 60)
    # Π·A : row i of result = row pr[i] of A
    Pi = gen.Csr((40, 40), np.arange(41, dtype=np.int64), pr.astype(np.int32), np.ones(40))
    R = oracle.spgemm(Pi, A)
    np.testing.assert_array_equal(res_dense(R, (40, 60)), A.to_dense()[pr, :])
    # A·Q where Q[j, pc[j]] = 1 : column j of A moves to column pc[j]
    Q = gen.Csr((60, 60), np.arange(61, dtype=np.int64), pc.astype(np.int32), np.ones(60))
    R = oracle.spgemm(A, Q)
    expect = np.zeros((40, 60))
    expect[:, pc] = A.to_dense()
    np.testing.assert_array_equal(res_dense(R, (40, 60)), expect)
    assert_sorted_rows(R)
    assert int(R.rp[-1]) == A.nnz


# ---------------------------------------------------------------- P4 power-of-two scaling
def test_P4_pow2_scaling():
    """(D1·A)·(B·D2) == D1·(A·B)·D2 bit-exactly for D entries 2^e (scaling by a power
    of two commutes with every rounding) — pins values in real mode."""
    A = gen.random_csr(30, 45, 0.3, 21, mode="real")
    B = gen.random_csr(45, 35, 0.3, 22, mode="real")
    e1 = (gen.hash3(1, np.arange(30), 0) % np.uint64(21)).astype(np.int64) - 10
    e2 = (gen.hash3(2, np.arange(35), 0) % np.uint64(21)).astype(np.int64) - 10
    d1, d2 = np.ldexp(1.0, e1), np.ldexp(1.0, e2)
    rowsA = np.repeat(np.arange(30), np.diff(A.rp))
    As = gen.Csr(A.shape, A.rp, A.ci, A.val * d1[rowsA])
    Bs = gen.Csr(B.shape, B.rp, B.ci, B.val * d2[B.ci])
    R = oracle.spgemm(A, B)
    Rs = oracle.spgemm(As, Bs)
    np.testing.assert_array_equal(R.ci, Rs.ci)
    rows = np.repeat(np.arange(30), np.diff(R.rp))
    np.testing.assert_array_equal(Rs.val, R.val * d1[rows] * d2[R.ci])
    # and values agree with a dense product within the 1e-12·Σ|a||b| bound
    dense = A.to_dense() @ B.to_dense()
    assert np.all(np.abs(res_dense(R, (30, 35)) - dense)[res_pattern(R, (30, 35))]
                  <= 1e-12 * R.bound + 0.0)


# ---------------------------------------------------------------- P5 size identities
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_P5_size_identities(seed):
    """Σu = Σ_j cnt_col_A(j)·nnz(b_j*) = flops/2 [P:433]; u_i ≥ nnz(c_i) [S:211]."""
    A = gen.random_csr(80, 90, 0.08, seed, mode="int")
    B = gen.random_csr(90, 70, 0.12, seed + 9, mode="int")
    u, tot = oracle.upper_bound(A, B)
    colcnt = np.bincount(A.ci, minlength=90)
    assert tot == int(np.dot(colcnt, np.diff(B.rp)))
    # brute-force product enumeration
    Ad, Bd = A.pattern_dense().astype(np.int64), B.pattern_dense().astype(np.int64)
    np.testing.assert_array_equal(u, (Ad @ Bd).sum(axis=1))
    R = oracle.spgemm(A, B)
    assert np.all(u >= np.diff(R.rp))
    # row-range variant agrees with the full run
    Rb = oracle.spgemm(A, B, r0=20, r1=55)
    np.testing.assert_array_equal(Rb.ci, R.ci[R.rp[20]:R.rp[55]])
    np.testing.assert_array_equal(Rb.rp, R.rp[20:56] - R.rp[20])


def test_threads_invariance():
    A = gen.random_csr(300, 300, 0.05, 77, mode="real")
    R1 = oracle.spgemm(A, A, threads=1)
    R4 = oracle.spgemm(A, A, threads=4)
    np.testing.assert_array_equal(R1.ci, R4.ci)
    np.testing.assert_array_equal(R1.val.view(np.int64), R4.val.view(np.int64))


# ---------------------------------------------------------------- P6 stencil closed forms
CLOSED = {
    "2d5": (lambda n: 5 * n * n - 4 * n, lambda n: 25 * n * n - 36 * n + 8, lambda n: 13 * n * n - 20 * n + 4),
    "2d9": (lambda n: (3 * n - 2) ** 2, lambda n: (9 * n - 10) ** 2, lambda n: (5 * n - 6) ** 2),
    "3d7": (lambda n: 7 * n ** 3 - 6 * n ** 2, lambda n: 49 * n ** 3 - 78 * n ** 2 + 24 * n,
            lambda n: 25 * n ** 3 - 42 * n ** 2 + 12 * n),
    "3d27": (lambda n: (3 * n - 2) ** 3, lambda n: (9 * n - 10) ** 3, lambda n: (5 * n - 6) ** 3),
}


@pytest.mark.parametrize("kind,n", [("2d5", 2), ("2d5", 3), ("2d5", 7), ("2d5", 32), ("2d9", 9),
                                    ("2d9", 20), ("3d7", 5), ("3d7", 9), ("3d27", 6), ("3d27", 10)])
def test_P6_stencil_nnz(kind, n):
    """nnz(A), Σu and nnz(A²) against closed forms counted by hand (SURVEY §8(c) P6,
    enumeration-derived; independent of the oracle)."""
    fa, fu, fc = CLOSED[kind]
    A = gen.stencil(kind, n)
    assert A.nnz == fa(n)
    u, tot = oracle.upper_bound(A, A)
    assert tot == fu(n)
    R = oracle.spgemm(A, A)
    assert int(R.rp[-1]) == fc(n)


def test_P6_config1_numbers():
    """Config 1 (BASELINE.json configs[0]): 2D5 on 32×32 → nnz(A)=4992, Σu=24456,
    nnz(A²)=12676."""
    A = gen.stencil("2d5", 32)
    assert A.nnz == 4992
    _, tot = oracle.upper_bound(A, A)
    assert tot == 24456
    assert int(oracle.spgemm(A, A).rp[-1]) == 12676


# ---------------------------------------------------------------- P7 stencil values
def _a2_closed(kind, off, deg_i):
    """Closed form of (cI - N)² at offset `off` for a row with `deg_i` neighbours.

    A = cI - N with c = #stencil neighbours.  A² = c²I - 2cN + N².  For 2D5/3D7 (axis
    neighbours): N²(i,i)=deg, N²=1 at axis±2, 2 at two-axis diagonals.  For 3D27
    (Chebyshev neighbours): N²(i,l) = Π_a t(|d_a|) - 2·[l ∈ nbr(i)] with t(0)=3,t(1)=2,
    t(2)=1 (interior rows)."""
    ad = sorted(abs(d) for d in off)
    if kind in ("2d5", "3d7"):
        c = 4 if kind == "2d5" else 6
        s = sum(ad)
        if s == 0:
            return c * c + deg_i
        if s == 1:
            return -2 * c
        if ad[-1] == 2 and s == 2:
            return 1
        if s == 2:
            return 2
        return None
    if kind == "3d27":
        c = 26
        t = {0: 3, 1: 2, 2: 1}
        prod = t[ad[0]] * t[ad[1]] * t[ad[2]]
        if ad[-1] == 0:
            return c * c + deg_i
        if ad[-1] == 1:
            return -2 * c + prod - 2
        return prod
    return None


@pytest.mark.parametrize("kind,n", [("2d5", 8), ("3d7", 6), ("3d27", 6)])
def test_P7_stencil_values(kind, n):
    A = gen.stencil(kind, n)
    R = oracle.spgemm(A, A)
    dim = 2 if kind.startswith("2d") else 3
    # interior row: centre of the grid
    ctr = [n // 2] * dim
    i = sum(ctr[a] * n ** a for a in range(dim))
    deg = A.nnz and int(A.rp[i + 1] - A.rp[i]) - 1
    cols = R.ci[R.rp[i]:R.rp[i + 1]]
    vals = R.val[R.rp[i]:R.rp[i + 1]]
    for c, v in zip(cols, vals):
        off = [(int(c) // n ** a) % n - ctr[a] for a in range(dim)]
        assert v == _a2_closed(kind, off, deg), (off, v)
    # corner row 0: entry count and diagonal
    corner = {"2d5": (6, 18), "3d7": (10, 39), "3d27": (27, 683)}[kind]
    assert int(R.rp[1] - R.rp[0]) == corner[0]
    assert R.val[R.rp[0]] == corner[1] and R.ci[R.rp[0]] == 0


def test_P7_3d27_offset_classes():
    """The ten interior offset classes of 3D27 A²."""
    want = {(0, 0, 0): 702, (0, 0, 1): -36, (0, 0, 2): 9, (0, 1, 1): -42, (0, 1, 2): 6,
            (0, 2, 2): 3, (1, 1, 1): -46, (1, 1, 2): 4, (1, 2, 2): 2, (2, 2, 2): 1}
    n = 7
    A = gen.stencil("3d27", n)
    R = oracle.spgemm(A, A)
    i = (3 * n + 3) * n + 3
    got = {}
    for c, v in zip(R.ci[R.rp[i]:R.rp[i + 1]], R.val[R.rp[i]:R.rp[i + 1]]):
        off = tuple(sorted(abs((int(c) // n ** a) % n - 3) for a in range(3)))
        got.setdefault(off, set()).add(v)
    assert {k: v.pop() for k, v in got.items()} == want


# ---------------------------------------------------------------- P8 / P9 Galerkin
@pytest.mark.parametrize("n", [4, 8, 16])
def test_P8_galerkin_closed_form(n):
    """Pᵀ·A·P with 2×2×2 tentative aggregation on 3D7 = 4·L7(n/2) exactly; nnz(AP) =
    n³ + 3n²(n-2)."""
    A = gen.stencil("3d7", n)
    P = gen.aggregation_P(n)
    R = gen.transpose(P)
    AP = oracle.spgemm(A, P)
    assert int(AP.rp[-1]) == n ** 3 + 3 * n * n * (n - 2)
    APm = gen.Csr((A.shape[0], P.shape[1]), AP.rp, AP.ci, AP.val)
    RAP = oracle.spgemm(R, APm)
    L = gen.stencil("3d7", n // 2)
    np.testing.assert_array_equal(RAP.rp, L.rp)
    np.testing.assert_array_equal(RAP.ci, L.ci)
    np.testing.assert_array_equal(RAP.val, 4.0 * L.val)
    h = n // 2
    assert int(RAP.rp[-1]) == 7 * h ** 3 - 6 * h ** 2


@pytest.mark.parametrize("smoothed", [False, True])
def test_P9_associativity(smoothed):
    """(PᵀA)P == Pᵀ(AP) bit-exactly with dyadic values ([S:413])."""
    n = 8
    A = gen.stencil("3d7", n)
    P = gen.aggregation_P(n, smoothed=smoothed)
    R = gen.transpose(P)
    AP = oracle.spgemm(A, P)
    RA = oracle.spgemm(R, A)
    c1 = oracle.spgemm(R, gen.Csr((A.shape[0], P.shape[1]), AP.rp, AP.ci, AP.val))
    c2 = oracle.spgemm(gen.Csr((R.shape[0], A.shape[1]), RA.rp, RA.ci, RA.val), P)
    np.testing.assert_array_equal(c1.rp, c2.rp)
    np.testing.assert_array_equal(c1.ci, c2.ci)
    np.testing.assert_array_equal(c1.val, c2.val)
    if smoothed:
        # rows of the smoothed P: values 5/8 (own aggregate) and k/8
        assert set(np.unique(P.val)) <= {5 / 8, 1 / 8, 2 / 8, 3 / 8}


def test_smoothed_P_against_dense():
    """Generator check: P_s = (I - A/8)·P_t computed densely."""
    n = 4
    A = gen.stencil("3d7", n).to_dense()
    Pt = gen.aggregation_P(n).to_dense()
    Ps = gen.aggregation_P(n, smoothed=True).to_dense()
    np.testing.assert_array_equal(Ps, (np.eye(n ** 3) - A / 8.0) @ Pt)


def test_validate_csr():
    A = gen.stencil("2d5", 5)
    assert oracle.validate_csr(25, 25, A.rp, A.ci) == 0
    bad = A.ci.copy()
    bad[1], bad[2] = bad[2], bad[1]
    assert oracle.validate_csr(25, 25, A.rp, bad) == 5
    rp = A.rp.copy()
    rp[3] = rp[2] - 1
    assert oracle.validate_csr(25, 25, rp, A.ci) == 2


# ---------------------------------------------------------------- SpSGEMM (fp32) fill
@pytest.mark.parametrize("density", [0.05, 0.3, 1.0])
@pytest.mark.parametrize("shape", [(1, 1, 1), (17, 9, 23), (64, 64, 64)])
def test_f32_dense_bruteforce(shape, density):
    """SpSGEMM oracle [P:403]: with integer values ±[1,8] every product and partial sum is an
    integer below 2^24, exact in float32 — pattern and values equal the dense product."""
    m, k, n = shape
    A = gen.random_csr(m, k, density, 300 + m, mode="int", zero_frac=0.1)
    B = gen.random_csr(k, n, density, 400 + n, mode="int", zero_frac=0.1)
    R = oracle.spgemm(A, B, fp32=True)
    assert R.val.dtype == np.float32
    pat = (A.pattern_dense().astype(np.int64) @ B.pattern_dense().astype(np.int64)) > 0
    np.testing.assert_array_equal(res_pattern(R, (m, n)), pat)
    np.testing.assert_array_equal(res_dense(R, (m, n)), A.to_dense() @ B.to_dense())


def test_f32_error_bound_and_pow2():
    """Real fp32 values: |fl32(c) - c| <= gamma_{t+1}·Σ|a||b| with u = 2^-24 and t the
    entry's number of products (product rounding + t-1 additions; the exact c from the
    float64 dense product of the same fp32-rounded inputs) — a dropped or misordered term
    fails this at the sizes used; and power-of-two scaling commutes bit for bit."""
    m, k, n = 40, 300, 50
    A = gen.random_csr(m, k, 0.3, 31, mode="real")
    B = gen.random_csr(k, n, 0.3, 32, mode="real")
    A32 = gen.Csr(A.shape, A.rp, A.ci, A.val.astype(np.float32).astype(np.float64))
    B32 = gen.Csr(B.shape, B.rp, B.ci, B.val.astype(np.float32).astype(np.float64))
    R = oracle.spgemm(A32, B32, fp32=True)
    exact = A32.to_dense() @ B32.to_dense()          # float64: within 2^-53-scale of exact
    terms = A32.pattern_dense().astype(np.int64) @ B32.pattern_dense().astype(np.int64)
    got = res_dense(R, (m, n))
    pat = res_pattern(R, (m, n))
    bound = np.abs(A32.to_dense()) @ np.abs(B32.to_dense())
    u = 2.0 ** -24
    gam = (terms + 1) * u / (1 - (terms + 1) * u)
    err = np.abs(got - exact)[pat]
    assert np.all(err <= (gam * bound)[pat] + 1e-12 * bound[pat])
    assert np.any(err > 0)                               # genuinely single precision
    rowsA = np.repeat(np.arange(m), np.diff(A32.rp))
    d1 = np.ldexp(1.0, (np.arange(m) % 7) - 3)
    As = gen.Csr(A32.shape, A32.rp, A32.ci, A32.val * d1[rowsA])
    Rs = oracle.spgemm(As, B32, fp32=True)
    rows = np.repeat(np.arange(m), np.diff(R.rp))
    np.testing.assert_array_equal(Rs.val, (R.val.astype(np.float64) * d1[rows]).astype(np.float32))
