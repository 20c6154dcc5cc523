"""Generators: closed-form counts of the input recipes, and the torch (device) generators
bit-identical to the numpy ones (checked on CPU tensors)."""
import numpy as np
import pytest
import torch

import gen
from gen import torchgen as tg


def test_hash_values_match():
    a = np.arange(5000, dtype=np.int64)
    b = (a * 7) % 913
    h_np = gen.hash3(123, a, b).view(np.int64)
    h_t = tg.hash3(123, torch.from_numpy(a), torch.from_numpy(b)).numpy()
    np.testing.assert_array_equal(h_np, h_t)
    for mode in ("int", "real", "dyadic", "one"):
        v_np = gen.values(99, a, b, mode)
        v_t = tg.values(99, torch.from_numpy(a), torch.from_numpy(b), mode).numpy()
        np.testing.assert_array_equal(v_np.view(np.int64), v_t.view(np.int64))


def test_band_match():
    n = 1000
    A = gen.band(n)
    (rp, ci, val), shape = tg.band(n, device="cpu")
    np.testing.assert_array_equal(A.rp, rp.numpy())
    np.testing.assert_array_equal(A.ci, ci.numpy())
    np.testing.assert_array_equal(A.val.view(np.int64), val.numpy().view(np.int64))
    # rows [i-32, i+31] ∩ [0, n): 64 per interior row
    assert A.nnz == 64 * n - (32 * 33 // 2 + 31 * 32 // 2)
    B = gen.band(n, rows=(100, 300))
    (rp, ci, val), _ = tg.band(n, rows=(100, 300), device="cpu")
    np.testing.assert_array_equal(B.ci, ci.numpy())


def test_uniform_rows_match():
    U = gen.uniform_rows(600, 2000, 64)  # collisions happen at this width
    (rp, ci, val), _ = tg.uniform_rows(600, 2000, 64, device="cpu", chunk=128)
    np.testing.assert_array_equal(U.rp, rp.numpy())
    np.testing.assert_array_equal(U.ci, ci.numpy())
    np.testing.assert_array_equal(U.val.view(np.int64), val.numpy().view(np.int64))
    d = np.diff(U.ci.reshape(600, 64), axis=1)
    assert np.all(d > 0)  # 64 distinct sorted columns per row


@pytest.mark.parametrize("abcd", [(0.45, 0.15, 0.15, 0.25), (0.57, 0.19, 0.19, 0.05)])
def test_rmat_match(abcd):
    A = gen.rmat(10, 16, abcd, seed=7, mode="real")
    (rp, ci, val), _ = tg.rmat(10, 16, abcd, seed=7, mode="real", device="cpu", chunk=4096)
    np.testing.assert_array_equal(A.rp, rp.numpy())
    np.testing.assert_array_equal(A.ci, ci.numpy())
    np.testing.assert_array_equal(A.val.view(np.int64), val.numpy().view(np.int64))
    assert A.nnz <= 16 * 1024  # duplicates merged


def test_stencil_and_P_shapes():
    A = gen.stencil("3d7", 6)
    P = gen.aggregation_P(6)
    assert P.nnz == 216 and np.all(np.diff(P.rp) == 1)
    R = gen.transpose(P)
    assert R.shape == (27, 216) and np.all(np.diff(R.rp) == 8)
    np.testing.assert_array_equal(gen.transpose(R).ci, P.ci)
