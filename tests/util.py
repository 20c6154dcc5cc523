"""Shared test helpers: run the CUDA path through the C ABI and compare with the oracle."""
import numpy as np

import oracle

TOL = 1e-12  # north star: |Δc_ij| <= 1e-12 · Σ_k |a_ik||b_kj|


def run_gpu(A, B, flags=0, stats=False, fp32=False):
    import torch

    import paper_1504_05022_b200 as sg
    dt = torch.float32 if fp32 else torch.float64
    dA = sg.DeviceCsr.from_host(A, dtype=dt)
    dB = dA if B is A else sg.DeviceCsr.from_host(B, dtype=dt)
    op = sg.SpGEMM(dA, dB, flags)
    nnz = op.symbolic()
    C = op.numeric()
    torch.cuda.synchronize()
    st = op.stats() if stats else None
    u, t = op.debug_u()
    out = dict(rp=C.rp.cpu().numpy(), ci=C.ci.cpu().numpy(), val=C.val.cpu().numpy(), nnz=nnz,
               u=u.cpu().numpy(), tier=t.cpu().numpy(), stats=st)
    op.destroy()
    return out


def compare(g, R, exact=False, r0=0, what=""):
    """Structure bit-exact; values exact (int/dyadic modes) or within TOL·bound."""
    rp = g["rp"] - g["rp"][0] if r0 else g["rp"]
    np.testing.assert_array_equal(rp, R.rp, err_msg="row_ptr mismatch " + what)
    np.testing.assert_array_equal(g["ci"], R.ci, err_msg="col_idx mismatch " + what)
    if exact:
        bad = np.nonzero(g["val"] != R.val)[0]
        assert bad.size == 0, "%s: %d values differ, first at %d: %r vs %r" % (
            what, bad.size, bad[0], g["val"][bad[0]], R.val[bad[0]])
    else:
        err = np.abs(g["val"] - R.val)
        lim = TOL * R.bound
        bad = np.nonzero(~(err <= lim))[0]
        assert bad.size == 0, "%s: %d values outside 1e-12·bound, first at %d: %r vs %r (bound %r)" % (
            what, bad.size, bad[0], g["val"][bad[0]], R.val[bad[0]], R.bound[bad[0]])
