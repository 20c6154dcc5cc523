"""BASELINE.json configs through the CUDA path in the bench's launch configuration.

Full sizes where one GPU holds them (c1, c2, c4a/c4b, c3b, a c5 row block the size of one rank's
share at P = 8), checked on sampled rows the oracle recomputes one by one (row-range oracle),
plus properties that hold at any size: the closed forms of SURVEY §8(c) P6/P8, Σu, and
u_i >= nnz(c_i*).  Smaller instances of c3a and c5 are compared in full.
"""
import numpy as np
import pytest

import gen
import oracle
from util import TOL

pytestmark = pytest.mark.gpu


def _run(A, B=None, flags=0):
    import torch

    import paper_1504_05022_b200 as sg
    dA = sg.DeviceCsr.from_host(A)
    dB = dA if B is None else sg.DeviceCsr.from_host(B)
    op = sg.SpGEMM(dA, dB, flags)
    nnz = op.symbolic()
    C = op.numeric()
    torch.cuda.synchronize()
    st = op.stats()
    op.destroy()
    return C, nnz, st


def _check_sampled(C, A, B, rows, exact):
    """Compare sampled row blocks of the GPU result with the row-range oracle."""
    rp = C.rp.cpu().numpy()
    for (r0, r1) in rows:
        R = oracle.spgemm(A, B, r0, r1)
        g0, g1 = int(rp[r0]), int(rp[r1])
        np.testing.assert_array_equal(rp[r0:r1 + 1] - rp[r0], R.rp)
        ci = C.ci[g0:g1].cpu().numpy()
        val = C.val[g0:g1].cpu().numpy()
        np.testing.assert_array_equal(ci, R.ci)
        if exact:
            np.testing.assert_array_equal(val, R.val)
        else:
            assert np.all(np.abs(val - R.val) <= TOL * R.bound)


def _samples(m, k=6, width=64, seed=0):
    rng = np.random.default_rng(seed)
    starts = sorted(set([0, m - width] + rng.integers(0, m - width, size=k).tolist()))
    return [(s, s + width) for s in starts]


@pytest.mark.parametrize("strategy", ["hybrid", "precise"])
def test_c2_full(strategy):
    import paper_1504_05022_b200 as sg
    n = 128
    A = gen.stencil("3d27", n)
    C, nnz, st = _run(A, flags=sg.FLAG_PRECISE if strategy == "precise" else 0)
    assert nnz == (5 * n - 6) ** 3 == 254840104          # P6 closed form
    assert st["sum_u"] == (9 * n - 10) ** 3 == 1489355288
    _check_sampled(C, A, A, _samples(A.shape[0]), exact=True)


@pytest.mark.parametrize("smoothed", [False, True])
def test_c4_full(smoothed):
    """Config 4 at 256³: R·(A·P); the tentative product equals 4·L7(128) exactly (P8)."""
    import torch

    import paper_1504_05022_b200 as sg
    n = 256
    A = gen.stencil("3d7", n)
    P = gen.aggregation_P(n, smoothed=smoothed)
    R = gen.transpose(P)
    dA, dP, dR = (sg.DeviceCsr.from_host(x) for x in (A, P, R))
    AP = sg.spgemm(dA, dP)
    RAP = sg.spgemm(dR, AP)
    torch.cuda.synchronize()
    if not smoothed:
        assert AP.nnz == n ** 3 + 3 * n * n * (n - 2) == 66715648
        L = gen.stencil("3d7", n // 2)
        np.testing.assert_array_equal(RAP.rp.cpu().numpy(), L.rp)
        np.testing.assert_array_equal(RAP.ci.cpu().numpy(), L.ci)
        np.testing.assert_array_equal(RAP.val.cpu().numpy(), 4.0 * L.val)
    else:
        assert AP.nnz == 166202368 and RAP.nnz == 68129272   # SURVEY §8(d) 4b [computed]
        APh = gen.Csr((A.shape[0], P.shape[1]), *AP.to_host())
        _check_sampled(RAP, R, APh, _samples(R.shape[0], width=32), exact=True)
        _check_sampled(AP, A, P, _samples(A.shape[0], width=32), exact=True)


@pytest.mark.parametrize("strategy", ["hybrid", "precise"])
def test_c3b_full(strategy):
    """Graph500-skew R-MAT at scale 18 (heavy tail; long rows on the progressive path in
    hybrid, on the bitmap path in precise)."""
    import paper_1504_05022_b200 as sg
    A = gen.rmat(18, 16, (0.57, 0.19, 0.19, 0.05), seed=gen.SEED, mode="int")
    C, nnz, st = _run(A, flags=sg.FLAG_PRECISE if strategy == "precise" else 0)
    assert st["long_rows"] > 0
    u, tot = oracle.upper_bound(A, A)
    assert st["sum_u"] == tot
    rp = C.rp.cpu().numpy()
    assert np.all(np.diff(rp) <= u)
    # sample the longest rows and random ones
    big = np.argsort(-u)[:3]
    rows = [(int(i), int(i) + 1) for i in big] + _samples(A.shape[0], k=4, width=32)
    _check_sampled(C, A, A, rows, exact=True)


def test_c3a_scaled():
    """Config 3a's generator at scale 16 (same parameters), compared in full."""
    A = gen.rmat(16, 16, (0.45, 0.15, 0.15, 0.25), seed=gen.SEED, mode="real")
    C, nnz, st = _run(A)
    R = oracle.spgemm(A, A)
    np.testing.assert_array_equal(C.rp.cpu().numpy(), R.rp)
    np.testing.assert_array_equal(C.ci.cpu().numpy(), R.ci)
    assert np.all(np.abs(C.val.cpu().numpy() - R.val) <= TOL * R.bound)


def test_c5_rank_block():
    """Config 5 shape, one rank's share at P = 8 of n = 2^20 (band(64) × uniform(64))."""
    n = 1 << 20
    rows = (0, n // 8)
    A = gen.band(n, rows=rows)
    B = gen.uniform_rows(n, n, 64)
    C, nnz, st = _run(A, B)
    assert st["sum_u"] == int(np.dot(np.bincount(A.ci, minlength=n), np.diff(B.rp)))
    _check_sampled(C, A, B, _samples(A.shape[0], k=4, width=16), exact=False)
