"""Multi-GPU (one process per GPU, NCCL through the C ABI) tests; skipped unless >= 2 GPUs.
  - R is bitwise identical on every rank (redundant Cholesky / R assembly);
  - 4k-2 allreduces per factorisation;
  - the distributed factorisation of the global matrix meets the accuracy gates and matches
    the single-GPU factorisation of the same global matrix (kappa <= 1e8: 1e-10 in R).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, m_local, n, b, kappa, algo, cuts=None):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _work(rank, world, q, m_local, n, b, kappa, algo, cuts)
    except BaseException as e:  # report instead of leaving the parent waiting on the queue
        q.put((rank, {"error": repr(e)}))
        raise
    finally:
        dist.destroy_process_group()


def _work(rank, world, q, m_local, n, b, kappa, algo, cuts):
    import torch
    import torch.distributed as dist
    import paper_2405_04237_b200 as t
    import synth
    from harness import verify
    comm = t.NcclComm(rank, world, rank)
    m = m_local * world
    chunk = min(m_local, 65536)  # generator chunk of the global matrix (independent of the split)
    if cuts is None:  # equal block rows
        A = t.colmajor_empty(m_local, n, device=f"cuda:{rank}")
        synth.generate_torch(A, m, rank * m_local, n, kappa, seed=1, chunk=chunk)
    else:  # uneven block rows [cuts[rank], cuts[rank+1]) of the same global matrix
        Af = t.colmajor_empty(m, n, device=f"cuda:{rank}")
        synth.generate_torch(Af, m, 0, n, kappa, seed=1, chunk=chunk)
        m_local = cuts[rank + 1] - cuts[rank]
        A = t.colmajor_empty(m_local, n, device=f"cuda:{rank}")
        A.copy_(Af[cuts[rank]:cuts[rank + 1]])
        del Af
    A0 = A.clone()
    plan = t.Plan(m_local, n, b, algo, comm=comm, device=f"cuda:{rank}")
    R = plan.factor(A)
    calls, _ = plan.counts()
    Rc = R.cpu().contiguous()
    Rs = [torch.empty_like(Rc) for _ in range(world)]
    dist.all_gather(Rs, Rc)
    orth = verify.orthogonality(A.cpu(), group=dist.group.WORLD)
    res = verify.residual(A0.cpu(), A.cpu(), R.cpu(), group=dist.group.WORLD)
    out = {"R": [r.numpy() for r in Rs], "calls": calls, "orth": orth, "res": res}
    if rank == 0:
        Af = t.colmajor_empty(m, n, device="cuda:0")
        synth.generate_torch(Af, m, 0, n, kappa, seed=1, chunk=chunk)
        out["R1"] = t.factor(Af, b, algo).cpu().numpy()
    plan.close()
    torch.cuda.synchronize()
    comm.close()
    q.put((rank, out))


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("algo,n,b,kappa", [("mcqr2gs", 256, 64, 1e8), ("mcqr2gs", 512, 64, 1e15),
                                             ("cqr2gs", 128, 32, 1e6), ("cqr2", 64, 64, 1e4),
                                             ("scqr3", 128, 128, 1e12)])
def test_two_rank_factorisation(algo, n, b, kappa):
    _run_ranks(algo, n, b, kappa)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_uneven_block_rows():
    """m_local may differ per rank (tsqr_create sums it collectively): ragged, non-multiple-
    of-64 block rows of the same global matrix give the same R as the single-GPU run."""
    world = min(_ngpu(), 4)
    m = world << 17
    cuts = [0] + [int(m * (r + 1) / world) + (1000 * (r + 1) if r + 1 < world else 0) - 37 * r
                  for r in range(world - 1)] + [m]
    _run_ranks("mcqr2gs", 256, 64, 1e6, cuts=cuts)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_rank_with_no_rows():
    """A rank may own zero rows (m_local = 0): it still takes part in every allreduce with
    zero partial sums and receives the same R."""
    world = min(_ngpu(), 4)
    m = world << 17
    cuts = [0, 0] + [int(m * (r + 1) / world) for r in range(1, world - 1)] + [m]
    _run_ranks("mcqr2gs", 128, 32, 1e6, cuts=cuts)


def _run_ranks(algo, n, b, kappa, cuts=None):
    import torch.multiprocessing as mp
    world = min(_ngpu(), 4)
    m_local = 1 << 17
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, m_local, n, b, kappa, algo, cuts))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = {}
    for _ in range(world):
        r, v = q.get(timeout=600)
        if "error" in v:  # a rank failed: the others may be blocked in a collective
            for p in procs:
                p.kill()
            pytest.fail(f"rank {r}: {v['error']}")
        outs[r] = v
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    o = outs[0]
    for r in range(1, world):
        assert np.array_equal(o["R"][0], o["R"][r])
    k = n // b
    assert o["calls"] == {"cqr2": 2, "scqr3": 3}.get(algo, 4 * k - 2)
    assert o["orth"] <= 1e-13 and o["res"] <= 1e-14, (o["orth"], o["res"])
    if kappa <= 1e8:
        R, R1 = o["R"][0], o["R1"]
        assert np.linalg.norm(R - R1) / np.linalg.norm(R1) <= 1e-10
