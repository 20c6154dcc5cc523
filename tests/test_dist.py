"""Multi-GPU row-block path.

CPU (gloo, world size 2): the host protocol of the dist_* entry points, through the
library's exported steps — partition by the prefix sum of u (spgemm_partition_rows), block
entry ranges (spgemm_dist_block_entries), placement of sharded B slices
(spgemm_dist_slice_layout), stitching offsets (spgemm_dist_offsets) — with gloo moving the
data where libspgemm uses NCCL, reproduces the single-process CSR bit for bit in both the root
and the sharded input modes.  The local multiply in this CPU test is the oracle (no GPU here);
on the GPU box the protocol runs inside libspgemm (NCCL) with one rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    """The dist_* protocol of libspgemm with gloo standing in for NCCL (CPU): every host-side
    step is the library's own exported function; only the local multiply is the oracle."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1504_05022_b200 as sg
    A = gen.rmat(10, 16, (0.57, 0.19, 0.19, 0.05), seed=5, mode="real")
    m = A.shape[0]
    # --- root mode: partition on rank 0, block entry ranges, send / recv, rebase ---------
    if rank == 0:
        u, _ = oracle.upper_bound(A, A)
        splits = sg.partition_rows(np.cumsum(u), world)
        bounds = sg.dist_block_entries(A.rp[splits])
        pack = torch.tensor(np.concatenate([splits, bounds.reshape(-1)]), dtype=torch.int64)
    else:
        pack = torch.zeros((world + 1) + 2 * world, dtype=torch.int64)
    dist.broadcast(pack, 0)
    splits = pack[:world + 1].numpy()
    bounds = pack[world + 1:].numpy().reshape(world, 2)
    r0, r1 = int(splits[rank]), int(splits[rank + 1])
    e0, e1 = int(bounds[rank, 0]), int(bounds[rank, 1])
    if rank == 0:
        for r in range(1, world):
            a, b = int(splits[r]), int(splits[r + 1])
            ea, eb = int(bounds[r, 0]), int(bounds[r, 1])
            dist.send(torch.from_numpy(A.rp[a:b + 1].copy()), r)
            dist.send(torch.from_numpy(A.ci[ea:eb].copy()), r)
            dist.send(torch.from_numpy(A.val[ea:eb].copy()), r)
        blk = gen.Csr((r1 - r0, A.shape[1]), A.rp[r0:r1 + 1] - e0, A.ci[e0:e1], A.val[e0:e1])
    else:
        rp = torch.zeros(r1 - r0 + 1, dtype=torch.int64)
        ci = torch.zeros(e1 - e0, dtype=torch.int32)
        val = torch.zeros(e1 - e0, dtype=torch.float64)
        for t in (rp, ci, val):
            dist.recv(t, 0)
        blk = gen.Csr((r1 - r0, A.shape[1]), rp.numpy() - e0, ci.numpy(), val.numpy())  # rebase
    R = oracle.spgemm(blk, A, with_bound=False)                  # local rows (stand-in for the GPU)
    local = torch.tensor([int(R.rp[-1])], dtype=torch.int64)
    allnnz = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allnnz, local)                               # the stitching collective
    off, tot = sg.dist_offsets([int(x) for x in allnnz], rank)
    root_block = (r0, r1, (R.rp[:-1] + off).tolist(), R.ci.tolist(), R.val.tolist(), tot)
    # --- sharded mode: B arrives as row slices; the library places them -----------------
    k = A.shape[0]
    b0, b1 = (rank * k) // world, ((rank + 1) * k) // world
    mine = torch.tensor([b0, b1, int(A.rp[b1] - A.rp[b0])], dtype=torch.int64)
    meta = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(meta, mine)
    meta = torch.stack(meta).numpy()
    base = sg.dist_slice_layout(meta[:, 0], meta[:, 1], meta[:, 2], k)
    slices = [None] * world
    dist.all_gather_object(slices, (A.rp[b0:b1] - A.rp[b0], A.ci[A.rp[b0]:A.rp[b1]], A.val[A.rp[b0]:A.rp[b1]]))
    rp = np.zeros(k + 1, dtype=np.int64)
    for r, (srp, sci, sval) in enumerate(slices):
        rp[meta[r, 0]:meta[r, 1]] = srp + base[r]                # rebase to the global entry offset
    rp[k] = base[world]
    ci = np.concatenate([x[1] for x in slices])
    val = np.concatenate([x[2] for x in slices])
    Bfull = gen.Csr(A.shape, rp, ci, val)
    a0, a1 = (rank * m) // world, ((rank + 1) * m) // world      # the caller's partition of A
    ablk = gen.Csr((a1 - a0, k), A.rp[a0:a1 + 1] - A.rp[a0], A.ci[A.rp[a0]:A.rp[a1]], A.val[A.rp[a0]:A.rp[a1]])
    S = oracle.spgemm(ablk, Bfull, with_bound=False)
    sn = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sn, torch.tensor([int(S.rp[-1])], dtype=torch.int64))
    soff, stot = sg.dist_offsets([int(x) for x in sn], rank)
    sharded_block = ((S.rp[:-1] + soff).tolist(), S.ci.tolist(), S.val.tolist(), stot)
    ok_b = (np.array_equal(Bfull.rp, A.rp) and np.array_equal(Bfull.ci, A.ci) and
            np.array_equal(Bfull.val.view(np.int64), A.val.view(np.int64)))
    blocks = [None] * world
    dist.all_gather_object(blocks, (root_block, sharded_block, ok_b))
    if rank == 0:
        q.put(blocks)
    dist.barrier()
    dist.destroy_process_group()


def test_rowblock_protocol_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    blocks = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    A = gen.rmat(10, 16, (0.57, 0.19, 0.19, 0.05), seed=5, mode="real")
    R = oracle.spgemm(A, A, with_bound=False)
    roots = [b[0] for b in blocks]
    rp = sum((b[2] for b in roots), []) + [roots[-1][5]]
    ci = sum((b[3] for b in roots), [])
    val = sum((b[4] for b in roots), [])
    assert roots[0][0] == 0 and roots[0][1] == roots[1][0] and roots[1][1] == A.shape[0]
    np.testing.assert_array_equal(np.array(rp), R.rp)
    np.testing.assert_array_equal(np.array(ci), R.ci)
    np.testing.assert_array_equal(np.array(val).view(np.int64), R.val.view(np.int64))
    # products are balanced within max u_i
    u, tot = oracle.upper_bound(A, A)
    cs = np.cumsum(u)
    left = cs[roots[0][1] - 1]
    assert abs(left - tot / 2) <= u.max()
    # sharded mode: every rank rebuilt B exactly, and the stitched C is the 1-process C
    assert all(b[2] for b in blocks)
    sh = [b[1] for b in blocks]
    np.testing.assert_array_equal(np.array(sum((b[0] for b in sh), []) + [sh[-1][3]]), R.rp)
    np.testing.assert_array_equal(np.array(sum((b[1] for b in sh), [])), R.ci)
    np.testing.assert_array_equal(np.array(sum((b[2] for b in sh), [])).view(np.int64), R.val.view(np.int64))


def test_protocol_host_functions():
    """Argument checks of the exported protocol steps (INVALID_VALUE / INVALID_CSR)."""
    import paper_1504_05022_b200 as sg
    np.testing.assert_array_equal(sg.dist_block_entries([0, 5, 5, 9]), [[0, 5], [5, 5], [5, 9]])
    with pytest.raises(sg.SpgemmError):
        sg.dist_block_entries([0, 5, 3])
    np.testing.assert_array_equal(sg.dist_slice_layout([0, 3, 3], [3, 3, 7], [10, 0, 20], 7), [0, 10, 10, 30])
    with pytest.raises(sg.SpgemmError):
        sg.dist_slice_layout([0, 4], [3, 7], [1, 1], 7)        # gap between slices
    with pytest.raises(sg.SpgemmError):
        sg.dist_slice_layout([0, 3], [3, 6], [1, 1], 7)        # does not cover k
    assert sg.dist_offsets([4, 0, 7], 0) == (0, 11)
    assert sg.dist_offsets([4, 0, 7], 2) == (4, 11)


@pytest.mark.gpu
@pytest.mark.parametrize("replicated", [True, False])
@pytest.mark.parametrize("precise", [False, True])
def test_dist_single_rank_gpu(replicated, precise):
    """dist_* with one rank on the GPU box: the NCCL communicator, partition, (broadcast /
    send-recv paths of rank 0) and stitching reproduce the single-GPU result exactly."""
    import paper_1504_05022_b200 as sg
    A = gen.rmat(12, 16, (0.45, 0.15, 0.15, 0.25), seed=7, mode="real")
    dA = sg.DeviceCsr.from_host(A)
    uid = sg.nccl_unique_id()
    flags = (sg.FLAG_INPUTS_REPLICATED if replicated else 0) | (sg.FLAG_PRECISE if precise else 0)
    op = sg.DistSpGEMM(0, 1, uid, A.shape[0], A.shape[1], A.shape[1], dA, dA, flags)
    rb, re_, ln, gn = op.symbolic()
    C = op.numeric()
    torch.cuda.synchronize()
    op.destroy()
    R = oracle.spgemm(A, A)
    assert (rb, re_) == (0, A.shape[0]) and ln == gn == int(R.rp[-1])
    np.testing.assert_array_equal(C.rp.cpu().numpy(), R.rp)
    np.testing.assert_array_equal(C.ci.cpu().numpy(), R.ci)
    assert np.all(np.abs(C.val.cpu().numpy() - R.val) <= 1e-12 * R.bound)


@pytest.mark.gpu
@pytest.mark.parametrize("precise", [False, True])
def test_dist_sharded_single_rank_gpu(precise):
    """spgemm_dist_create_sharded with one rank: B given as a slice (row pointers starting at
    an offset), A as a row block; the all-gather, rebasing and value stream reproduce the
    single-GPU result exactly (c5's input shape at a small n)."""
    import paper_1504_05022_b200 as sg
    n = 1 << 14
    A = gen.band(n, mode="real")
    B = gen.uniform_rows(n, n, 64, mode="real")
    dA, dB = sg.DeviceCsr.from_host(A), sg.DeviceCsr.from_host(B)
    # row pointers that do not start at 0: entries of the block are ci[e - rp[0]]
    dB2 = sg.DeviceCsr(dB.rows, dB.cols, dB.rp + 1000, dB.ci, dB.val)
    uid = sg.nccl_unique_id()
    op = sg.DistSpGEMM(0, 1, uid, n, n, n, dA, dB2, sg.FLAG_PRECISE if precise else 0,
                       a_rows=(0, n), b_rows=(0, n))
    rb, re_, ln, gn = op.symbolic()
    C = op.numeric()
    torch.cuda.synchronize()
    op.destroy()
    R = oracle.spgemm(A, B)
    assert (rb, re_) == (0, n) and ln == gn == int(R.rp[-1])
    np.testing.assert_array_equal(C.rp.cpu().numpy(), R.rp)
    np.testing.assert_array_equal(C.ci.cpu().numpy(), R.ci)
    assert np.all(np.abs(C.val.cpu().numpy() - R.val) <= 1e-12 * R.bound)


@pytest.mark.gpu
def test_device_partition_matches_host_rule():
    """The partition kernel of dist_symbolic (device) equals spgemm_partition_rows (host) on
    random and degenerate scans, for 1..8 ranks."""
    import paper_1504_05022_b200 as sg
    rng = np.random.default_rng(3)
    cases = [rng.integers(0, 50, size=1000), np.zeros(17, dtype=np.int64), np.array([5]),
             rng.integers(0, 3, size=100) * rng.integers(0, 1000, size=100), np.array([0, 0, 9, 0])]
    for u in cases:
        scan = np.cumsum(u).astype(np.int64)
        d = torch.from_numpy(scan).cuda()
        for P in range(1, 9):
            np.testing.assert_array_equal(sg.debug_partition(d, P), sg.partition_rows(scan, P))
