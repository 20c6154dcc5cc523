"""BASELINE.json configs through the CUDA path at FULL size, in the bench's launch
configuration, compared ELEMENT BY ELEMENT with the oracle.

Every row of C is checked: the oracle recomputes the product in row blocks of ~2e8
intermediate products (row-range oracle, all host cores), and each block is compared with the
same rows of the GPU result copied back — row_ptr and col_idx bit-exact, values exact in the
coef / int modes and within 1e-12·Σ|a||b| in real mode.  Closed forms of SURVEY §8(c)
(P6 stencil nnz and Σu, P8 Galerkin) are asserted on top.  c3a runs at scale 22 (the bench
workload), c3b at scale 18, c2 at 128³, c4 at 256³, both strategies; c5 is one rank's block
of n = 2^23 (a P = 8 share of the 8×B200 config).
"""
import numpy as np
import pytest

import gen
import oracle
from util import TOL

pytestmark = pytest.mark.gpu

STRATS = ["hybrid", "precise"]


def _flags(strategy):
    import paper_1504_05022_b200 as sg
    return sg.FLAG_PRECISE if strategy == "precise" else 0


def _run(dA, dB, flags=0):
    import torch

    import paper_1504_05022_b200 as sg
    op = sg.SpGEMM(dA, dB, flags)
    nnz = op.symbolic()
    C = op.numeric()
    torch.cuda.synchronize()
    st = op.stats()
    op.destroy()
    return C, nnz, st


def check_full(C, A, B, exact, chunk_products=200_000_000):
    """Every row of the GPU result C (device CSR) against the row-range oracle."""
    rp = C.rp.cpu().numpy()
    u, tot = oracle.upper_bound(A, B)
    assert np.all(np.diff(rp) <= u)                       # u_i >= nnz(c_i*) [S:211]
    cs = np.cumsum(u)
    m = A.shape[0]
    r0 = 0
    while r0 < m:
        start = int(cs[r0 - 1]) if r0 else 0
        r1 = int(np.searchsorted(cs, start + chunk_products, side="right"))
        r1 = min(max(r1, r0 + 1), m)
        R = oracle.spgemm(A, B, r0, r1, with_bound=not exact)
        g0, g1 = int(rp[r0]), int(rp[r1])
        np.testing.assert_array_equal(rp[r0:r1 + 1] - rp[r0], R.rp, err_msg="row_ptr rows [%d,%d)" % (r0, r1))
        ci = C.ci[g0:g1].cpu().numpy()
        np.testing.assert_array_equal(ci, R.ci, err_msg="col_idx rows [%d,%d)" % (r0, r1))
        val = C.val[g0:g1].cpu().numpy()
        if exact:
            bad = np.nonzero(val != R.val)[0]
            assert bad.size == 0, "rows [%d,%d): %d values differ" % (r0, r1, bad.size)
        else:
            bad = np.nonzero(~(np.abs(val - R.val) <= TOL * R.bound))[0]
            assert bad.size == 0, "rows [%d,%d): %d values outside 1e-12·bound" % (r0, r1, bad.size)
        r0 = r1
    assert int(rp[-1]) == int(C.ci.numel())
    return tot


def _dev(M):
    import paper_1504_05022_b200 as sg
    return sg.DeviceCsr.from_host(M)


@pytest.mark.parametrize("strategy", STRATS)
def test_c2_full(strategy):
    n = 128
    A = gen.stencil("3d27", n)
    dA = _dev(A)
    C, nnz, st = _run(dA, dA, _flags(strategy))
    assert nnz == (5 * n - 6) ** 3 == 254840104          # P6 closed form
    assert st["sum_u"] == (9 * n - 10) ** 3 == 1489355288
    check_full(C, A, A, exact=True)


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("smoothed", [False, True])
def test_c4_full(smoothed, strategy):
    """Config 4 at 256³: R·(A·P); the tentative product equals 4·L7(128) exactly (P8)."""
    n = 256
    A = gen.stencil("3d7", n)
    P = gen.aggregation_P(n, smoothed=smoothed)
    R = gen.transpose(P)
    dA, dP, dR = (_dev(x) for x in (A, P, R))
    AP, nnz_ap, _ = _run(dA, dP, _flags(strategy))
    RAP, nnz_rap, _ = _run(dR, AP, _flags(strategy))
    if not smoothed:
        assert nnz_ap == n ** 3 + 3 * n * n * (n - 2) == 66715648
        L = gen.stencil("3d7", n // 2)
        np.testing.assert_array_equal(RAP.rp.cpu().numpy(), L.rp)
        np.testing.assert_array_equal(RAP.ci.cpu().numpy(), L.ci)
        np.testing.assert_array_equal(RAP.val.cpu().numpy(), 4.0 * L.val)
    else:
        assert nnz_ap == 166202368 and nnz_rap == 68129272   # SURVEY §8(d) 4b [computed]
    check_full(AP, A, P, exact=True)
    APh = gen.Csr((A.shape[0], P.shape[1]), *AP.to_host())
    check_full(RAP, R, APh, exact=True)


@pytest.mark.parametrize("strategy", STRATS)
def test_c3b_full(strategy):
    """Graph500-skew R-MAT at scale 18 (heavy tail; long rows on the progressive path in
    hybrid, on the bitmap path in precise), real values as timed."""
    A = gen.rmat(18, 16, (0.57, 0.19, 0.19, 0.05), seed=gen.SEED, mode="real")
    dA = _dev(A)
    C, nnz, st = _run(dA, dA, _flags(strategy))
    assert st["long_rows"] > 0
    tot = check_full(C, A, A, exact=False)
    assert st["sum_u"] == tot


@pytest.mark.parametrize("strategy", STRATS)
def test_c3a_full(strategy):
    """Config 3a exactly as benched: R-MAT scale 22, edge factor 16, (0.45,0.15,0.15,0.25),
    real values; 2.5e9 products, every row checked."""
    import torch

    from gen import torchgen as tg
    t, shape = tg.rmat(22, 16, (0.45, 0.15, 0.15, 0.25), seed=gen.SEED, mode="real")
    A = tg.to_csr(t, shape)
    del t
    torch.cuda.empty_cache()
    dA = _dev(A)
    C, nnz, st = _run(dA, dA, _flags(strategy))
    assert st["tier_rows"].get("long", 0) > 0 and st["sum_u"] > 2.4e9  # (wide windows: bucket path)
    tot = check_full(C, A, A, exact=False)
    assert st["sum_u"] == tot


def test_c5_rank_block():
    """Config 5 shape at full n = 2^23: one rank's row block at P = 8 (band(64) × uniform(64)),
    every row checked (u = 4096 products per interior row)."""
    n = 1 << 23
    rows = (0, n // 8)
    from gen import torchgen as tg
    A = tg.to_csr(*tg.band(n, rows=rows))
    B = tg.to_csr(*tg.uniform_rows(n, n, 64))
    C, nnz, st = _run(_dev(A), _dev(B))
    assert st["sum_u"] == int(np.dot(np.bincount(A.ci, minlength=n), np.diff(B.rp)))
    check_full(C, A, B, exact=False)
