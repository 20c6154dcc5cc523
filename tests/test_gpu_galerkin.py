"""The paper's Galerkin workload ([P:393-397]): AMG hierarchies of smoothed
aggregation with a Jacobi smoother for the 2D 5/9-point (1024x1024) and 3D 7/27-point (101^3)
Poisson problems, both association orders P^T(AP) and (P^T A)P, every level, fp64, every row
compared with the oracle (values within 1e-12·Σ|a||b|; the smoothed operators are not dyadic).
Level 0 runs at the paper's size; the coarse levels follow from it."""
import numpy as np
import pytest

import gen
import oracle
from util import TOL

pytestmark = pytest.mark.gpu


def _mul(A, B, flags):
    import torch

    import paper_1504_05022_b200 as sg
    dA, dB = sg.DeviceCsr.from_host(A), sg.DeviceCsr.from_host(B)
    C = sg.spgemm(dA, dB, flags)
    torch.cuda.synchronize()
    rp, ci, val = C.to_host()
    return gen.Csr((A.shape[0], B.shape[1]), rp, ci, val)


def _check(G, A, B):
    R = oracle.spgemm(A, B)
    np.testing.assert_array_equal(G.rp, R.rp)
    np.testing.assert_array_equal(G.ci, R.ci)
    assert np.all(np.abs(G.val - R.val) <= TOL * R.bound)


@pytest.mark.parametrize("kind,n", [("2d5", 1024), ("2d9", 1024), ("3d7", 101), ("3d27", 101)])
@pytest.mark.parametrize("strategy", ["precise", "hybrid"])
def test_galerkin_hierarchy(kind, n, strategy):
    import paper_1504_05022_b200 as sg
    flags = sg.FLAG_PRECISE if strategy == "precise" else 0
    for A, P, R in gen.amg_levels(kind, n, 3):
        AP = _mul(A, P, flags)
        _check(AP, A, P)
        RAP = _mul(R, AP, flags)
        _check(RAP, R, AP)
        RA = _mul(R, A, flags)
        _check(RA, R, A)
        RA_P = _mul(RA, P, flags)
        _check(RA_P, RA, P)
        # both orders give the same operator: identical pattern, values within rounding
        np.testing.assert_array_equal(RAP.rp, RA_P.rp)
        np.testing.assert_array_equal(RAP.ci, RA_P.ci)
        scale = np.abs(RAP.val).max()
        assert np.all(np.abs(RAP.val - RA_P.val) <= 1e-12 * scale * 64)
