"""Parity of the CUDA path (through the C ABI) with the oracle — SURVEY.md §8(c).

Structure (row_ptr, col_idx) must be bit-exact; values exact in the integer / dyadic /
coefficient modes and within 1e-12·Σ|a||b| in real mode.  Sizes span several tiles and
ragged tails; every stage-2 class and the long-row growth path are exercised.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle
from util import compare, run_gpu

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


@pytest.fixture(autouse=True)
def _reset_debug():
    import paper_1504_05022_b200 as sg
    sg.set_debug(-1, 0, 0)
    sg.set_debug_long_tile(0)
    sg.set_debug_long_bucket(0)
    yield
    sg.set_debug(-1, 0, 0)
    sg.set_debug_long_tile(0)
    sg.set_debug_long_bucket(0)


def _dense_csr(D, pattern=None):
    D = np.asarray(D, dtype=np.float64)
    mask = D != 0
    for (r, c) in (pattern or []):
        mask[r, c] = True
    rows, cols = np.nonzero(mask)
    return gen.from_coo(rows, cols, D.shape, vals=D[rows, cols])


@pytest.mark.parametrize("case", GOLD["products"], ids=lambda c: c["cite"][:40])
def test_golden(case):
    A, B = _dense_csr(case["A"]), _dense_csr(case["B"])
    g = run_gpu(A, B)
    R = oracle.spgemm(A, B)
    compare(g, R, exact=True)
    assert g["u"].tolist() == case["u"]


@pytest.mark.parametrize("mode", ["int", "real"])
@pytest.mark.parametrize("shape,density", [((1, 1, 1), 1.0), ((37, 53, 41), 0.1), ((200, 150, 300), 0.05),
                                           ((300, 300, 300), 0.2), ((64, 2000, 3000), 0.02)])
def test_random(shape, density, mode):
    m, k, n = shape
    A = gen.random_csr(m, k, density, 11 + m, mode=mode, zero_frac=0.05)
    B = gen.random_csr(k, n, density, 12 + n, mode=mode, zero_frac=0.05)
    g = run_gpu(A, B)
    R = oracle.spgemm(A, B)
    compare(g, R, exact=(mode == "int"))
    u, _ = oracle.upper_bound(A, B)
    np.testing.assert_array_equal(g["u"], u)


BOUNDARY_U = [0, 1, 2, 3, 4, 5, 8, 9, 16, 17, 31, 32, 33, 51, 52, 64, 65, 102, 103, 204, 205, 409, 410, 819,
              820, 1638, 1639, 2048, 2049, 4096, 4097, 8192, 8193, 9000]


@pytest.mark.parametrize("dup", [0.0, 0.5, 0.95])
def test_tier_boundaries(dup):
    """Rows with u on both sides of every class threshold (SPEC acceptance 1 [S:482])."""
    A, B = gen.forced_u_pair(BOUNDARY_U, n=20000, seed=5, mode="int", dup=dup)
    g = run_gpu(A, B, stats=True)
    R = oracle.spgemm(A, B)
    compare(g, R, exact=True, what="dup=%s" % dup)
    np.testing.assert_array_equal(g["u"], np.array(BOUNDARY_U))
    assert np.all(np.diff(g["rp"]) <= g["u"])  # u_i >= nnz(c_i*) [S:211]


def _classify(u, n, W):
    """Python restatement of the stage-2 rule for the exact-integer check."""
    if u == 0:
        return 0
    cap = min(u, n)
    if u <= 32:
        g = 0
        while (1 << g) < u:
            g += 1
        return 1 + g
    if 0 < W <= (1 << 17) and min(cap, W) <= 8192:   # window bitmap (the relaxed bound, both strategies)
        return 19
    for t in range(7, 13):
        if 4 * (64 << (t - 7)) >= 5 * cap:
            return t
    for t in range(16, 19):          # bucket-ESC classes by the product count u
        if u <= (2048 << (t - 16)):
            return t
    for t in range(13, 16):
        if cap <= (2048 << (t - 13)):
            return t
    return 20


def _windows(A, B):
    """W_i = max_j (last column of b_j*) - min_j (first column of b_j*) + 1 over the a_ij."""
    W = np.zeros(A.shape[0], dtype=np.int64)
    for i in range(A.shape[0]):
        lo, hi = None, None
        for j in A.ci[A.rp[i]:A.rp[i + 1]]:
            if B.rp[j + 1] > B.rp[j]:
                f, l = int(B.ci[B.rp[j]]), int(B.ci[B.rp[j + 1] - 1])
                lo = f if lo is None else min(lo, f)
                hi = l if hi is None else max(hi, l)
        W[i] = 0 if lo is None else hi - lo + 1
    return W


def test_stage12_integers():
    """Stage 1 U and the stage-2 class of every row, exactly."""
    A, B = gen.forced_u_pair(BOUNDARY_U * 3, n=20000, seed=9, mode="int")
    g = run_gpu(A, B, stats=True)
    u, tot = oracle.upper_bound(A, B)
    np.testing.assert_array_equal(g["u"], u)
    assert g["stats"]["sum_u"] == tot
    W = _windows(A, B)
    want = [_classify(int(x), B.shape[1], int(w)) for x, w in zip(u, W)]
    np.testing.assert_array_equal(g["tier"], np.array(want))
    counts = np.bincount(np.array(want), minlength=21)
    from paper_1504_05022_b200 import TIER_NAMES
    assert g["stats"]["tier_rows"] == {TIER_NAMES[t]: int(c) for t, c in enumerate(counts) if c}


@pytest.mark.parametrize("tier", list(range(1, 21)))
def test_forced_tier(tier):
    """Every row that a class can hold is routed through it; results agree with the oracle
    (and so with every other class: P11 tier-forced agreement)."""
    import paper_1504_05022_b200 as sg
    us = [2, 3, 7, 16, 30, 32, 40, 100, 300, 700, 1500, 3000, 6000]
    A, B = gen.forced_u_pair(us, n=9000, seed=tier, mode="int", dup=0.5)
    sg.set_debug(tier, 0, 0)
    g = run_gpu(A, B)
    R = oracle.spgemm(A, B)
    compare(g, R, exact=True, what="tier %d" % tier)


@pytest.mark.parametrize("tier", [3, 6, 7, 9, 11, 12, 13, 15, 16, 17, 18, 19, 20])
def test_forced_tier_precise(tier):
    """PRECISE strategy: symbolic (structure) and numeric (dense / bitmap) classes agree
    with the oracle when rows are forced through each class."""
    import paper_1504_05022_b200 as sg
    us = [2, 3, 7, 16, 30, 32, 40, 100, 300, 700, 1500, 3000, 6000]
    A, B = gen.forced_u_pair(us, n=9000, seed=tier + 50, mode="int", dup=0.5)
    sg.set_debug(tier, 0, 0)
    g = run_gpu(A, B, flags=sg.FLAG_PRECISE)
    R = oracle.spgemm(A, B)
    compare(g, R, exact=True, what="precise tier %d" % tier)


@pytest.mark.parametrize("u", [600, 1500, 5000])
@pytest.mark.parametrize("dup", [0.0, 0.5, 0.95])
def test_long_growth(u, dup):
    """Progressive re-allocation [P:297]: tiny initial capacity forces 1-6 growth rounds;
    the resumed result equals the unbounded one [S:297] (SPEC acceptance 5 [S:487])."""
    import paper_1504_05022_b200 as sg
    us = [u, u // 2, 700, u]
    A, B = gen.forced_u_pair(us, n=60000, seed=u + int(dup * 10), mode="int", dup=dup)
    sg.set_debug(-1, 64, 40)  # long path for cap > 40, initial capacity 64
    g = run_gpu(A, B, stats=True)
    R = oracle.spgemm(A, B)
    compare(g, R, exact=True, what="u=%d dup=%s" % (u, dup))
    assert g["stats"]["long_rows"] == 4
    if int(np.diff(R.rp).max()) > 64:  # some row outgrew the initial capacity: re-allocation ran
        assert g["stats"]["growth_rounds"] >= 1


@pytest.mark.parametrize("flags_name", ["PRECISE", "UPPER_BOUND"])
def test_strategies_equal(flags_name):
    """Strategy invariance [S:213]: hybrid == precise == upper bound."""
    import paper_1504_05022_b200 as sg
    A = gen.rmat(11, 16, (0.57, 0.19, 0.19, 0.05), seed=3, mode="int")
    R = oracle.spgemm(A, A)
    sg.set_debug(-1, 256, 1000)
    g = run_gpu(A, A, flags=getattr(sg, "FLAG_" + flags_name))
    compare(g, R, exact=True, what=flags_name)
    g2 = run_gpu(A, A, flags=0)
    compare(g2, R, exact=True, what="hybrid")


@pytest.mark.parametrize("kind,n", [("2d5", 32), ("2d9", 20), ("3d7", 12), ("3d27", 14)])
def test_stencils(kind, n):
    A = gen.stencil(kind, n)
    g = run_gpu(A, A)
    R = oracle.spgemm(A, A)
    compare(g, R, exact=True, what=kind)


def test_config1_full():
    """BASELINE configs[0]: 2D 5-point 32×32, A² — full size, exact."""
    A = gen.stencil("2d5", 32)
    g = run_gpu(A, A, stats=True)
    R = oracle.spgemm(A, A)
    compare(g, R, exact=True)
    assert g["nnz"] == 12676 and g["stats"]["sum_u"] == 24456


@pytest.mark.parametrize("scale,abcd", [(12, (0.45, 0.15, 0.15, 0.25)), (13, (0.57, 0.19, 0.19, 0.05))])
@pytest.mark.parametrize("mode", ["int", "real"])
def test_rmat(scale, abcd, mode):
    A = gen.rmat(scale, 16, abcd, seed=gen.SEED, mode=mode)
    g = run_gpu(A, A)
    R = oracle.spgemm(A, A)
    compare(g, R, exact=(mode == "int"), what="rmat s%d" % scale)


def test_rmat_long_rows_default_path():
    """Graph500 skew at scale 14 has rows beyond every shared-memory class (T_LONG)."""
    import paper_1504_05022_b200 as sg
    A = gen.rmat(14, 16, (0.57, 0.19, 0.19, 0.05), seed=gen.SEED, mode="int")
    sg.set_debug(-1, 2048, 0)
    g = run_gpu(A, A, stats=True)
    R = oracle.spgemm(A, A)
    compare(g, R, exact=True)
    assert g["stats"]["long_rows"] > 0


@pytest.mark.parametrize("smoothed", [False, True])
def test_galerkin(smoothed):
    """Config 4 at 16³: both association orders; exact (dyadic values)."""
    n = 16
    A = gen.stencil("3d7", n)
    P = gen.aggregation_P(n, smoothed=smoothed)
    Rm = gen.transpose(P)
    gAP = run_gpu(A, P)
    oAP = oracle.spgemm(A, P)
    compare(gAP, oAP, exact=True, what="AP")
    AP = gen.Csr((A.shape[0], P.shape[1]), gAP["rp"], gAP["ci"], gAP["val"])
    gRAP = run_gpu(Rm, AP)
    oRAP = oracle.spgemm(Rm, AP)
    compare(gRAP, oRAP, exact=True, what="R(AP)")
    gRA = run_gpu(Rm, A)
    RA = gen.Csr((Rm.shape[0], A.shape[1]), gRA["rp"], gRA["ci"], gRA["val"])
    gRAP2 = run_gpu(RA, P)
    np.testing.assert_array_equal(gRAP["rp"], gRAP2["rp"])
    np.testing.assert_array_equal(gRAP["ci"], gRAP2["ci"])
    np.testing.assert_array_equal(gRAP["val"], gRAP2["val"])
    if not smoothed:
        L = gen.stencil("3d7", n // 2)
        np.testing.assert_array_equal(gRAP["ci"], L.ci)
        np.testing.assert_array_equal(gRAP["val"], 4.0 * L.val)


def test_band_uniform():
    """Config 5 shape at n = 2^14: band(64) × uniform(64)."""
    n = 1 << 14
    A = gen.band(n, mode="real")
    B = gen.uniform_rows(n, n, 64, mode="real")
    g = run_gpu(A, B)
    R = oracle.spgemm(A, B)
    compare(g, R, exact=False)


def test_edge_cases():
    # all rows empty
    A = gen.Csr((5, 7), np.zeros(6, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    B = gen.random_csr(7, 9, 0.5, 1)
    g = run_gpu(A, B)
    assert g["nnz"] == 0 and g["rp"].tolist() == [0] * 6
    # B empty (n columns but no entries)
    A = gen.random_csr(6, 4, 0.5, 2)
    B = gen.Csr((4, 3), np.zeros(5, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    g = run_gpu(A, B)
    assert g["nnz"] == 0
    # k = 0
    A = gen.Csr((3, 0), np.zeros(4, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    B = gen.Csr((0, 5), np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    g = run_gpu(A, B)
    assert g["nnz"] == 0 and g["rp"].tolist() == [0] * 4


def test_m_zero():
    import torch

    import paper_1504_05022_b200 as sg
    A = gen.Csr((0, 4), np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    B = gen.random_csr(4, 4, 0.5, 3)
    op = sg.SpGEMM(sg.DeviceCsr.from_host(A), sg.DeviceCsr.from_host(B))
    assert op.symbolic() == 0
    C = op.numeric()
    torch.cuda.synchronize()
    assert C.rp.cpu().tolist() == [0]


def test_determinism_and_cancellation():
    A = gen.random_csr(400, 400, 0.05, 21, mode="real")
    g1 = run_gpu(A, A)
    g2 = run_gpu(A, A)
    np.testing.assert_array_equal(g1["ci"], g2["ci"])
    np.testing.assert_array_equal(g1["val"].view(np.int64), g2["val"].view(np.int64))
    # explicit cancellation keeps a stored zero
    A = _dense_csr([[1.0, 1.0]])
    B = _dense_csr([[2.0], [-2.0]])
    g = run_gpu(A, B)
    assert g["nnz"] == 1 and g["val"][0] == 0.0


def test_bitexact_warp_tiers_vs_oracle_real():
    """Classes that accumulate in j-ascending order (G-lane sort, warp hash) reproduce
    the oracle's rounding bit for bit in real mode (reading R1)."""
    us = [2, 5, 9, 17, 32, 40, 100, 300, 700, 1500]
    A, B = gen.forced_u_pair(us * 20, n=5000, seed=77, mode="real", dup=0.7)
    g = run_gpu(A, B)
    R = oracle.spgemm(A, B)
    np.testing.assert_array_equal(g["ci"], R.ci)
    np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))


def test_validate_flag():
    import paper_1504_05022_b200 as sg
    A = gen.random_csr(10, 10, 0.3, 4)
    bad = gen.Csr(A.shape, A.rp, A.ci[::-1].copy(), A.val)
    with pytest.raises(sg.SpgemmError) as e:
        sg.SpGEMM(sg.DeviceCsr.from_host(bad), sg.DeviceCsr.from_host(A), sg.FLAG_VALIDATE)
    assert e.value.status == 2
    op = sg.SpGEMM(sg.DeviceCsr.from_host(A), sg.DeviceCsr.from_host(A), sg.FLAG_VALIDATE)
    op.destroy()


def test_numeric_before_symbolic():
    import paper_1504_05022_b200 as sg
    A = gen.random_csr(10, 10, 0.3, 4)
    op = sg.SpGEMM(sg.DeviceCsr.from_host(A), sg.DeviceCsr.from_host(A))
    with pytest.raises(sg.SpgemmError):
        op.numeric()
    op.destroy()


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
def test_bw_block_directory_overflow(flags_name):
    """Window-bitmap rows whose products touch more 1024-column blocks than the precise
    symbolic pass has directory slots (16) are redone over the full window: a wide window
    (n = 100 000 < 2^17) and rows of 60-200 uniform columns (≈ 50-100 nonzero blocks), mixed
    with narrow rows that fit the directory.  Exact in int mode against the oracle."""
    import paper_1504_05022_b200 as sg
    n = 100_000
    lengths = np.array([3 + (i * 7) % 5 for i in range(300)])
    A = gen.random_rows(300, 3000, lengths, seed=11, mode="int")
    wide = gen.random_rows(1500, n, np.array([60 + (j * 13) % 140 for j in range(1500)]), seed=12, mode="int")
    # narrow B rows: columns inside one 1024-column block
    narrow = gen.random_rows(1500, 1000, np.array([5 + j % 20 for j in range(1500)]), seed=13, mode="int")
    rp = np.concatenate([wide.rp, wide.rp[-1] + narrow.rp[1:]])
    B = gen.Csr((3000, n), rp, np.concatenate([wide.ci, narrow.ci]), np.concatenate([wide.val, narrow.val]))
    flags = getattr(sg, flags_name) if flags_name else 0
    g = run_gpu(A, B, flags=flags, stats=True)
    R = oracle.spgemm(A, B)
    compare(g, R, exact=True, what="bw overflow")
    assert "bw" in g["stats"]["tier_rows"]


def _wide_pair(seed, a_lens, n=400_000, k=2000, blen=64):
    """Row i of A picks a_lens[i] rows of B, each with blen uniform columns over n > 2^17
    (no window-bitmap rows): u_i = 64·a_lens[i] spans the w, e and long classes, with
    about u²/2n repeated columns per row."""
    B = gen.random_rows(k, n, np.full(k, blen), seed=seed, mode="real")
    A = gen.random_rows(len(a_lens), k, np.array(a_lens), seed=seed + 1, mode="real")
    return A, B


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
def test_determinism_real_all_classes(flags_name):
    """Run-to-run bit-identical values in real mode through the w (ESC merge) and e (ESC
    radix) classes (R1: every class is order-fixed)."""
    import paper_1504_05022_b200 as sg
    flags = getattr(sg, flags_name) if flags_name else 0
    A, B = _wide_pair(5, [1, 3, 10, 20, 40, 100] * 6)
    g1 = run_gpu(A, B, flags=flags, stats=True)
    g2 = run_gpu(A, B, flags=flags)
    R = oracle.spgemm(A, B)
    compare(g1, R, exact=False, what="real classes")
    np.testing.assert_array_equal(g1["ci"], g2["ci"])
    np.testing.assert_array_equal(g1["val"].view(np.int64), g2["val"].view(np.int64))
    classes = set(g1["stats"]["tier_rows"])
    assert any(c.startswith("w") for c in classes) and any(c.startswith("e") for c in classes), classes


def test_esc_bitexact_vs_oracle_real():
    """The ESC sorts (run merge for the warp classes' values, radix for e-classes) are stable
    and sum each column left to right: values bit-identical to the oracle in real mode."""
    import paper_1504_05022_b200 as sg
    A, B = _wide_pair(8, [2, 10, 20, 40, 100] * 8)
    g = run_gpu(A, B, flags=sg.FLAG_PRECISE, stats=True)
    R = oracle.spgemm(A, B)
    np.testing.assert_array_equal(g["ci"], R.ci)
    np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
@pytest.mark.parametrize("mode", ["int", "real"])
def test_long_multi_tile(flags_name, mode):
    """Long rows whose column window spans many bitmap tiles (a 8 Ki-column tile knob against
    windows of up to 400 000 columns): the tile loop of the count and rank kernels, with every
    b_j* cut to the tile by binary search.  Structure exact; values bit-identical to the
    oracle in both value modes (each column is summed by one warp in j order, [P:121-135]),
    and run to run."""
    import paper_1504_05022_b200 as sg
    flags = getattr(sg, flags_name) if flags_name else 0
    B = gen.random_rows(2000, 400_000, np.full(2000, 64), seed=31, mode=mode)
    A = gen.random_rows(60, 2000, np.array([1, 3, 10, 20, 40, 100, 300] * 8 + [2, 5, 7, 9]), seed=32, mode=mode)
    sg.set_debug(-1, 0, 40)          # every row with min(u, n) > 40 takes the long path
    sg.set_debug_long_tile(8192)     # tiles of 8 Ki (values) / 16 Ki (count) columns
    sg.set_debug_long_bucket(-1)     # wide windows too (the bucket path: test_long_bucket_path)
    g = run_gpu(A, B, flags=flags, stats=True)
    g2 = run_gpu(A, B, flags=flags)
    R = oracle.spgemm(A, B)
    assert g["stats"]["long_rows"] > 0
    np.testing.assert_array_equal(g["rp"], R.rp)
    np.testing.assert_array_equal(g["ci"], R.ci)
    np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))
    np.testing.assert_array_equal(g2["val"].view(np.int64), g["val"].view(np.int64))


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
@pytest.mark.parametrize("tier", [13, 14, 15, 20])
def test_long_and_chash_bitexact_real(flags_name, tier):
    """The CTA-hash classes (values by the rank kernel) and the long rows accumulate each
    column in j-ascending order without atomics: real-mode values bit-identical to the oracle
    and to a second run, including the growth path of the hybrid strategy."""
    import paper_1504_05022_b200 as sg
    flags = getattr(sg, flags_name) if flags_name else 0
    us = [40, 100, 300, 700, 1500, 3000, 6000, 9000]
    A, B = gen.forced_u_pair(us * 4, n=30000, seed=tier + 90, mode="real", dup=0.6)
    sg.set_debug(tier, 256 if tier == 20 else 0, 40 if tier == 20 else 0)
    g = run_gpu(A, B, flags=flags, stats=True)
    g2 = run_gpu(A, B, flags=flags)
    R = oracle.spgemm(A, B)
    np.testing.assert_array_equal(g["rp"], R.rp)
    np.testing.assert_array_equal(g["ci"], R.ci)
    np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))
    np.testing.assert_array_equal(g2["val"].view(np.int64), g["val"].view(np.int64))
    from paper_1504_05022_b200 import TIER_NAMES
    assert TIER_NAMES[tier] in g["stats"]["tier_rows"]


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
@pytest.mark.parametrize("mode", ["int", "real"])
def test_warp_classes_crowded_window(flags_name, mode):
    """Warp-class rows whose columns crowd one end of a wide window (a 2 000-column cluster
    plus one far column, W = 10^6) and rows with a mildly crowded window: structure exactly,
    values bit for bit against the oracle (j-ascending sums), both strategies.  (An
    order-preserving warp hash for these values was measured 2-4x slower than the run-merge
    ESC on c3a and dropped; the rows stay as a parity case for any window-keyed kernel.)"""
    import paper_1504_05022_b200 as sg
    n = 1_000_000
    rng = np.random.default_rng(5)
    rows, cols = [], []
    for j in range(40):  # B rows 0..39: 30 columns in [0, 2000) (crowded) or in [0, 60000) (mild)
        hi = 2000 if j < 20 else 60000
        c = np.sort(rng.choice(hi, 30, replace=False))
        rows += [j] * 30
        cols += list(c)
    rows.append(40)
    cols.append(n - 1)  # the far column: the window spans [0, n)
    B = gen.from_coo(np.array(rows), np.array(cols), (41, n))
    B = gen.with_values(B, mode, 11)
    arow, acol = [], []
    for i in range(64):
        js = list(range(0, 20)) if i % 2 == 0 else list(range(20, 40))
        js = sorted(set(js[: 5 + (i % 16)]) | {40})
        arow += [i] * len(js)
        acol += js
    A = gen.with_values(gen.from_coo(np.array(arow), np.array(acol), (64, 41)), mode, 12)
    g = run_gpu(A, B, flags=getattr(sg, flags_name) if flags_name else 0)
    R = oracle.spgemm(A, B)
    assert set(np.unique(g["tier"])) <= set(range(7, 13)), "rows expected in the warp classes"
    np.testing.assert_array_equal(g["rp"], R.rp)
    np.testing.assert_array_equal(g["ci"], R.ci)
    np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
@pytest.mark.parametrize("mode", ["int", "real"])
@pytest.mark.parametrize("min_window", [1, 0])
def test_long_bucket_path(mode, min_window, flags_name):
    """Long rows on the bucket path (longbk.cu): the row's products partitioned by
    column range in product order, each bucket sorted stably and its runs summed left to right.
    Rows: wide windows (2 Mi columns) with 8 Ki-60 Ki products; one row whose products crowd
    one bucket past its capacity (fallback to the rank kernel); short-window rows (rank kernel
    unless the knob sends every long row to the bucket path).  Structure exact, values bit for
    bit against the oracle and run to run.  Precise: into C after the exact count; hybrid: into
    upper-bound C~ slices, the other long rows on the progressive path, stage 4 copying both."""
    import paper_1504_05022_b200 as sg
    flags = getattr(sg, flags_name) if flags_name else 0
    n = 1 << 21
    lens = np.array([16, 64, 200, 400, 31, 5] * 500)[:3000]
    B = gen.random_rows(3000, n, lens, seed=51, mode=mode)
    # rows 3000..3039: crowded, all columns in [0, 6000)
    Bc = gen.random_rows(40, 6000, np.full(40, 300), seed=52, mode=mode)
    Bn = gen.random_rows(20, 50_000, np.full(20, 500), seed=53, mode=mode)  # short windows
    rp = np.concatenate([B.rp, B.rp[-1] + Bc.rp[1:], B.rp[-1] + Bc.rp[-1] + Bn.rp[1:]])
    Bfull = gen.Csr((3060, n), rp, np.concatenate([B.ci, Bc.ci, Bn.ci]), np.concatenate([B.val, Bc.val, Bn.val]))
    rows, cols = [], []
    for i in range(48):
        if i < 40:
            js = np.sort(np.unique((np.arange(40 + 8 * i) * 7919 + i * 31) % 3000))
        elif i < 44:
            js = np.array([0] + list(range(3000, 3040)))  # 12 000 products in [0, 6000) + a wide
            #                                            b_0*: one bucket holds > kBkCap products
        else:
            js = np.arange(3040, 3060)             # 10 000 products, window 50 000
        rows += [i] * len(js)
        cols += list(js)
    A = gen.with_values(gen.from_coo(np.array(rows), np.array(cols), (48, 3060)), mode, 54)
    sg.set_debug_long_bucket(min_window)
    g = run_gpu(A, Bfull, flags=flags, stats=True)
    g2 = run_gpu(A, Bfull, flags=flags)
    R = oracle.spgemm(A, Bfull)
    assert g["stats"]["tier_rows"].get("long", 0) >= 40
    np.testing.assert_array_equal(g["rp"], R.rp)
    np.testing.assert_array_equal(g["ci"], R.ci)
    np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))
    np.testing.assert_array_equal(g2["val"].view(np.int64), g["val"].view(np.int64))


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
def test_window_class_relaxed_bound(flags_name):
    """Precise strategy: rows with 2048 < min(u, W) <= 8192 and W <= 2^17 start in the window
    class; after the count, those longer than 2048 leave it for the ESC / CTA classes, the rest
    (columns repeated by many b_j*) keep the dense accumulator.  Hybrid takes the same bound:
    its one-walk kernel keeps the rows whose granules fit, the others take the two walks into
    their C~ slices.  Structure exact, values bit for bit against the oracle."""
    import paper_1504_05022_b200 as sg
    flags = getattr(sg, flags_name) if flags_name else 0
    n = 100_000
    Bw = gen.random_rows(300, n, np.full(300, 20), seed=61, mode="real")       # spread columns
    Bn = gen.random_rows(300, 600, np.full(300, 40), seed=62, mode="real")     # 600-column band
    off = np.zeros(300, dtype=np.int64) + 50_000
    rp = np.concatenate([Bw.rp, Bw.rp[-1] + Bn.rp[1:]])
    ci = np.concatenate([Bw.ci, Bn.ci + off[0]]).astype(np.int32)
    B = gen.Csr((600, n), rp, ci, np.concatenate([Bw.val, Bn.val]))
    rows, cols = [], []
    for i in range(40):
        js = np.arange(0, 300, 1 + i % 3) if i % 2 == 0 else np.arange(300, 600, 1 + i % 3)
        rows += [i] * len(js)
        cols += list(js)
    A = gen.with_values(gen.from_coo(np.array(rows), np.array(cols), (40, 600)), "real", 63)
    g = run_gpu(A, B, flags=flags, stats=True)
    R = oracle.spgemm(A, B)
    np.testing.assert_array_equal(g["rp"], R.rp)
    np.testing.assert_array_equal(g["ci"], R.ci)
    np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
@pytest.mark.parametrize("mode", ["int", "real"])
def test_rank_kernel_large_tiles(flags_name, mode):
    """Long rows of 28 Ki to 60 Ki entries in one bitmap tile next to short long rows: the rank
    kernel's warp-owned rank ranges over large tiles (accumulating into the row's output in
    L2; rank windows bounding that footprint measured slower on c3b: 71 vs 51 ms), both
    strategies (hybrid: the progressive path).  Bit for bit against the oracle."""
    import paper_1504_05022_b200 as sg
    flags = getattr(sg, flags_name) if flags_name else 0
    B = gen.random_rows(1200, 200_000, np.full(1200, 100), seed=71, mode=mode)
    A = gen.random_rows(12, 1200, np.array([300, 600, 40, 900] * 3), seed=72, mode=mode)
    g = run_gpu(A, B, flags=flags, stats=True)
    R = oracle.spgemm(A, B)
    assert g["stats"]["tier_rows"].get("long", 0) >= 6
    assert np.diff(R.rp).max() > 50_000
    np.testing.assert_array_equal(g["rp"], R.rp)
    np.testing.assert_array_equal(g["ci"], R.ci)
    np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))


@pytest.mark.gpu
@pytest.mark.parametrize("fp32", [False, True])
def test_window_rows_word_and_column_structure(fp32):
    """Precise strategy, window class: the structure pass stores a row as its nonzero bitmap
    words ((first column, bits) pairs) when 8 B per word fits the row's slice, else as its
    sorted columns.  Rows of clustered columns (many per word: word format) and rows whose
    products land in distinct words with no repeats (u = nnz, one column per word: column
    format) share one launch; stencil rows at the block boundaries as well.  Values bit for
    bit against the oracle (fp32: the SpSGEMM oracle)."""
    import paper_1504_05022_b200 as sg
    n = 60_000
    # B rows 0..199: 24 columns in 3 clusters of 8 consecutive columns; 200..399: 16 columns
    # 128 apart (one per word)
    rows, cols = [], []
    for r in range(200):
        base = (r * 97) % (n - 3000)
        for k in range(3):
            rows += [r] * 8
            cols += list(range(base + 1000 * k + (r % 32), base + 1000 * k + (r % 32) + 8))
    for r in range(200, 400):
        rows += [r] * 16
        cols += list(20_000 + (r - 200) + 64 * np.arange(16) * 2)
    B = gen.with_values(gen.from_coo(np.array(rows), np.array(cols), (400, n)), "real", 81)
    ar, ac = [], []
    for i in range(64):
        if i % 2 == 0:
            js = np.arange(i, i + 6) % 200                    # clustered: word format
        else:
            js = 200 + (i * 3) % 60 + np.array([0, 60, 120])   # spread b_j*: words ~ nnz = u
        ar += [i] * len(js)
        ac += list(js)
    A = gen.with_values(gen.from_coo(np.array(ar), np.array(ac), (64, 400)), "real", 82)
    g = run_gpu(A, B, flags=sg.FLAG_PRECISE, stats=True, fp32=fp32)
    assert set(g["stats"]["tier_rows"]) == {"bw"}
    R = oracle.spgemm(A, B, fp32=fp32)
    np.testing.assert_array_equal(g["rp"], R.rp)
    np.testing.assert_array_equal(g["ci"], R.ci)
    vt = np.int32 if fp32 else np.int64
    np.testing.assert_array_equal(g["val"].view(vt), R.val.view(vt))


def test_long_arena_cache_reuse():
    """The hybrid long-row VMM arenas are kept for the next multiply (mapped pages and stale
    data included): back-to-back progressive multiplies of different sizes, then again after
    trim_workspace_cache released them — every result equals the oracle bit for bit."""
    import paper_1504_05022_b200 as sg
    cases = []
    for k, (u, dup) in enumerate([(5000, 0.0), (1500, 0.5), (5000, 0.95)]):
        A, B = gen.forced_u_pair([u, u // 2, 700, u], n=60000, seed=900 + k, mode="real", dup=dup)
        cases.append((A, B, oracle.spgemm(A, B)))
    try:
        sg.set_debug(-1, 64, 40)  # long path for cap > 40, initial capacity 64: growth rounds
        for rnd in range(2):
            for A, B, R in cases:
                g = run_gpu(A, B, stats=True)
                assert g["stats"]["long_rows"] == 4
                np.testing.assert_array_equal(g["rp"], R.rp)
                np.testing.assert_array_equal(g["ci"], R.ci)
                np.testing.assert_array_equal(g["val"].view(np.int64), R.val.view(np.int64))
            sg.trim_workspace_cache(0)
    finally:
        sg.set_debug(-1, 0, 0)
