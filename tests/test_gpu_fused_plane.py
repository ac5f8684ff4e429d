"""The cross-GPU sum data planes under a test a 1-GPU box runs.

A 1-rank NCCL communicator with TSQR_FUSED_ALLREDUCE=1 routes every allreduce of the
factorisation through `k_reduce_allreduce` (symmetric NCCL window, LSA barrier, epoch-parity
halves); with TSQR_NCCL_ALLREDUCE=1 through `k_reduce` + `ncclAllReduce`.  On one rank the
cross-GPU sum is the identity and both kernels form the local split-row sum in the same fixed
order, so Q and R must be BITWISE equal to the plan without a communicator ('local' plane) --
over several CUDA-graph replays (the window half alternates with the barrier epoch, which
persists across replays) and for every algorithm (the calls alternate b x b Gram, b x N_j Y and
(j-1)b x b C blocks, so consecutive calls use different block shapes in the two halves).
"""
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def comm1():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.distributed as dist
    import paper_2405_04237_b200 as t
    torch.cuda.set_device(0)
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    c = t.NcclComm(0, 1, 0)
    yield t, c
    torch.cuda.synchronize()
    c.close()
    if own:
        dist.destroy_process_group()


def _plan(t, comm, m, n, b, algo, plane):
    old = {k: os.environ.get(k) for k in ("TSQR_FUSED_ALLREDUCE", "TSQR_NCCL_ALLREDUCE", "TSQR_CLUSTER_PATH")}
    os.environ["TSQR_FUSED_ALLREDUCE"] = "1" if plane == "fused" else "0"
    os.environ["TSQR_NCCL_ALLREDUCE"] = "1" if plane == "nccl" else "0"
    os.environ["TSQR_CLUSTER_PATH"] = "0"  # the same (streaming) kernels on every plane
    try:
        p = t.Plan(m, n, b, algo, comm=comm if plane != "local" else None)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert p.data_plane() == plane
    return p


@pytest.mark.parametrize("plane", ["fused", "nccl"])
@pytest.mark.parametrize("algo,m,n,b,kappa", [("mcqr2gs", 65536 + 37, 512, 64, 1e15),
                                               ("mcqr2gs", 4096, 64, 16, 1e8),
                                               ("cqr2gs", 20000, 256, 32, 1e6),
                                               ("cqr2", 70001, 128, 128, 1e4),
                                               ("scqr3", 65536, 128, 128, 1e12),
                                               ("mcqr2gs", 50000, 1024, 256, 1e12)])
def test_one_rank_plane_bitwise_equals_local(comm1, plane, algo, m, n, b, kappa):
    import torch
    t, c = comm1
    A, _, _ = synth.generate_np(m, n, kappa, seed=5, chunk=m if m % 65536 else 65536)
    A0 = t.to_colmajor(A)
    ref = _plan(t, c, m, n, b, algo, "local")
    Aref = A0.clone()
    Rref = ref.factor(Aref)
    calls_ref = ref.counts()[0]
    ref.close()
    p = _plan(t, c, m, n, b, algo, plane)
    X = t.colmajor_empty(m, n)
    for rep in range(4):  # graph capture + 3 replays: both window halves, epochs 0..(4 * calls)
        X.copy_(A0)
        R = p.factor(X)
        torch.cuda.synchronize()
        assert torch.equal(R, Rref), (plane, rep)
        assert torch.equal(X, Aref), (plane, rep)
        assert p.counts()[0] == calls_ref
    p.close()


def test_one_rank_fused_breakdown_keeps_barriers_matched(comm1):
    """A zero column breaks the first Cholesky down; every later fused call must still run its
    barrier (the status is uniform), so the NEXT factorisation on the same plan is correct."""
    import torch
    t, c = comm1
    m, n, b = 8192, 128, 32
    A, _, _ = synth.generate_np(m, n, 1e4, seed=6, chunk=m)
    p = _plan(t, c, m, n, b, "mcqr2gs", "fused")
    ref = _plan(t, c, m, n, b, "mcqr2gs", "local")
    Aref = t.to_colmajor(A)
    Rref = ref.factor(Aref)
    ref.close()
    bad = A.copy()
    bad[:, 3] = 0.0
    ref = _plan(t, c, m, n, b, "mcqr2gs", "local")
    with pytest.raises(t.TsqrError) as e0:
        ref.factor(t.to_colmajor(bad))
    ref.close()
    with pytest.raises(t.TsqrError) as e:
        p.factor(t.to_colmajor(bad))
    assert e.value.status == t.TSQR_ERR_BREAKDOWN
    assert e.value.info == e0.value.info and e.value.info["pivot"] == 3
    X = t.to_colmajor(A)
    R = p.factor(X)
    torch.cuda.synchronize()
    assert torch.equal(R, Rref) and torch.equal(X, Aref)
    p.close()
