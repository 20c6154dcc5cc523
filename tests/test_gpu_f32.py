"""SpSGEMM: the paper's single-precision runs ([P:403], [P:663]) through
spgemm_create_f32 / spgemm_numeric_f32 — every class, both strategies, long rows with
several bitmap tiles and the growth path.  Every class accumulates in the oracle's order, so
fp32 values are bit-identical to the fp32 oracle (oracle_spgemm_fill_f32) in real mode."""
import numpy as np
import pytest

import gen
import oracle
from util import run_gpu

pytestmark = pytest.mark.gpu


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


def _exact(g, R):
    np.testing.assert_array_equal(g["rp"], R.rp)
    np.testing.assert_array_equal(g["ci"], R.ci)
    assert g["val"].dtype == np.float32
    np.testing.assert_array_equal(g["val"].view(np.int32), R.val.view(np.int32))


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
@pytest.mark.parametrize("tier", list(range(1, 21)))
def test_f32_forced_tier(tier, flags_name):
    import paper_1504_05022_b200 as sg
    us = [2, 3, 7, 16, 30, 32, 40, 100, 300, 700, 1500, 3000, 6000, 9000]
    A, B = gen.forced_u_pair(us, n=12000, seed=tier + 200, mode="real", dup=0.5)
    sg.set_debug(tier, 256 if tier == 20 else 0, 40 if tier == 20 else 0)
    g = run_gpu(A, B, flags=getattr(sg, flags_name) if flags_name else 0, fp32=True)
    _exact(g, oracle.spgemm(A, B, fp32=True))


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
def test_f32_rmat_and_stencil(flags_name):
    import paper_1504_05022_b200 as sg
    flags = getattr(sg, flags_name) if flags_name else 0
    for A in (gen.rmat(13, 16, (0.57, 0.19, 0.19, 0.05), seed=gen.SEED, mode="real"),
              gen.stencil("3d27", 20, mode="real")):
        g = run_gpu(A, A, flags=flags, fp32=True)
        _exact(g, oracle.spgemm(A, A, fp32=True))


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
def test_f32_long_multi_tile(flags_name):
    import paper_1504_05022_b200 as sg
    B = gen.random_rows(2000, 400_000, np.full(2000, 64), seed=41, mode="real")
    A = gen.random_rows(40, 2000, np.array([3, 20, 100, 300] * 10), seed=42, mode="real")
    sg.set_debug(-1, 64, 40)
    sg.set_debug_long_tile(8192)
    sg.set_debug_long_bucket(-1)  # the multi-tile rank / progressive path for every long row
    g = run_gpu(A, B, flags=getattr(sg, flags_name) if flags_name else 0, stats=True, fp32=True)
    assert g["stats"]["long_rows"] > 0
    _exact(g, oracle.spgemm(A, B, fp32=True))


def test_f32_galerkin_paper_level0():
    """The paper's SP Galerkin workload at its size: level 0 of the 2D 9-point 1024x1024
    hierarchy, P^T(AP), fp32 values, every row checked."""
    import paper_1504_05022_b200 as sg
    A, P, R = gen.amg_levels("2d9", 1024, 1)[0]
    gAP = run_gpu(A, P, flags=sg.FLAG_PRECISE, fp32=True)
    oAP = oracle.spgemm(A, P, fp32=True)
    _exact(gAP, oAP)
    AP32 = gen.Csr((A.shape[0], P.shape[1]), gAP["rp"], gAP["ci"], gAP["val"].astype(np.float64))
    g = run_gpu(R, AP32, flags=sg.FLAG_PRECISE, fp32=True)
    _exact(g, oracle.spgemm(R, AP32, fp32=True))


def test_f32_api_guards():
    import torch

    import paper_1504_05022_b200 as sg
    A = gen.random_csr(10, 10, 0.3, 4, mode="real")
    op = sg.SpGEMM(sg.DeviceCsr.from_host(A, dtype=torch.float32), sg.DeviceCsr.from_host(A, dtype=torch.float32))
    op.symbolic()
    lib = sg.load()
    c = torch.empty(11, dtype=torch.int64, device="cuda")
    assert lib.spgemm_numeric(op.h, c.data_ptr(), None, None) == 1   # fp64 numeric on an fp32 handle
    op.destroy()


@pytest.mark.parametrize("flags_name", ["FLAG_PRECISE", None])
def test_f32_long_bucket_path(flags_name):
    """SpSGEMM long rows on the bucket path (every long row, via the knob)."""
    import paper_1504_05022_b200 as sg
    B = gen.random_rows(2000, 400_000, np.full(2000, 64), seed=41, mode="real")
    A = gen.random_rows(40, 2000, np.array([3, 20, 100, 300] * 10), seed=42, mode="real")
    sg.set_debug(-1, 0, 40)
    sg.set_debug_long_bucket(1)
    g = run_gpu(A, B, flags=getattr(sg, flags_name) if flags_name else 0, stats=True, fp32=True)
    assert g["stats"]["tier_rows"].get("long", 0) > 0
    _exact(g, oracle.spgemm(A, B, fp32=True))
