"""Multi-GPU row-block path.

CPU (gloo, world size 2): the host protocol — partition by the prefix sum of u with the
library's own rule (spgemm_partition_rows), per-rank rows, allgather of per-rank nnz,
global row-pointer stitching — reproduces the single-process CSR bit for bit.  The local
multiply in this CPU test is the oracle (no GPU here); on the GPU box the same protocol runs
inside libspgemm (dist_* entry points, NCCL), tested with one rank per available GPU.
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
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1504_05022_b200 as sg
    A = gen.rmat(10, 16, (0.57, 0.19, 0.19, 0.05), seed=5, mode="real")
    u, _ = oracle.upper_bound(A, A)
    splits = sg.partition_rows(np.cumsum(u), world)
    r0, r1 = int(splits[rank]), int(splits[rank + 1])
    R = oracle.spgemm(A, A, r0, r1, with_bound=False)       # local rows (stand-in for the GPU)
    local = torch.tensor([int(R.rp[-1])], dtype=torch.int64)
    allnnz = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allnnz, local)                           # the stitching collective
    off = int(sum(int(x) for x in allnnz[:rank]))
    rp = R.rp + off                                          # global row offsets
    blocks = [None] * world
    dist.all_gather_object(blocks, (r0, r1, rp[:-1].tolist(), R.ci.tolist(), R.val.tolist(),
                                    int(sum(int(x) for x in allnnz))))
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
    rp = sum((b[2] for b in blocks), []) + [blocks[-1][5]]
    ci = sum((b[3] for b in blocks), [])
    val = sum((b[4] for b in blocks), [])
    assert blocks[0][0] == 0 and blocks[0][1] == blocks[1][0] and blocks[1][1] == A.shape[0]
    np.testing.assert_array_equal(np.array(rp), R.rp)
    np.testing.assert_array_equal(np.array(ci), R.ci)
    np.testing.assert_array_equal(np.array(val).view(np.int64), R.val.view(np.int64))
    # products are balanced within max u_i
    u, tot = oracle.upper_bound(A, A)
    cs = np.cumsum(u)
    left = cs[blocks[0][1] - 1]
    assert abs(left - tot / 2) <= u.max()


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
