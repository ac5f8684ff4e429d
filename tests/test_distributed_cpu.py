"""world_size-2 gloo tests of the multi-rank host logic on CPU:
  - the seeded generator is independent of the rank count (each rank builds only its own
    row chunks, synth.generate_torch), so every P factors the same global matrix;
  - the per-rank algorithms with one allreduce per reduction (tests/dist_emulation.py) match
    the single-address-space oracle and issue 4k-2 allreduces (Appendix A.2 of SURVEY);
  - R is bitwise identical on every rank (redundant Cholesky / R assembly);
  - bench.py's cross-rank reduction of step times is a max.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, v = q.get(timeout=300)
        out[r] = v
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _entry(fn, rank, world, port, q, args):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world, *args)))
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------- workers (module level: spawn)
def _gen_worker(rank, world, m, n, kappa, chunk):
    import synth
    m_local = m // world
    A = torch.empty((n, m_local), dtype=torch.float64).T
    synth.generate_torch(A, m, rank * m_local, n, kappa, seed=3, chunk=chunk)
    return A.numpy().copy()


def _algo_worker(rank, world, m, n, b, kappa, algo):
    import synth
    from tests import dist_emulation as de
    A, _, _ = synth.generate_np(m, n, kappa, seed=0, chunk=m)
    m_local = m // world
    Al = np.array(A[rank * m_local:(rank + 1) * m_local], order="F")
    comm = de.Comm()
    R = de.mcqr2gs(Al, b, comm) if algo == "mcqr2gs" else de.cqr2gs(Al, b, comm)
    return {"R": R, "Q": Al, "calls": comm.calls}


def _max_worker(rank, world):
    import bench  # noqa: F401  (import check: bench.py must import on CPU)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- tests
def test_generator_independent_of_rank_count():
    m, n, chunk = 8192, 32, 2048
    out = _run(_gen_worker, 2, m, n, 1e6, chunk)
    A2 = np.vstack([out[0], out[1]])
    A1 = _run(_gen_worker, 1, m, n, 1e6, chunk)[0]
    assert np.array_equal(A1, A2)
    # rows of an orthonormal U times Sigma V^T: the planted spectrum is recovered
    s = np.linalg.svd(A1, compute_uv=False)
    assert abs(s[0] - 1.0) < 1e-12 and abs(s[-1] / 1e-6 - 1.0) < 1e-6


@pytest.mark.parametrize("algo", ["mcqr2gs", "cqr2gs"])
def test_distributed_algorithm_matches_oracle(orc, algo):
    m, n, b, kappa = 4096, 64, 16, 1e6
    out = _run(_algo_worker, 2, m, n, b, kappa, algo)
    assert np.array_equal(out[0]["R"], out[1]["R"])  # bitwise replicated R
    assert out[0]["calls"] == 4 * (n // b) - 2
    import synth
    A, _, _ = synth.generate_np(m, n, kappa, seed=0, chunk=m)
    _, Ro, _ = orc.factor(A, b, algo)
    R = out[0]["R"]
    assert np.linalg.norm(R - Ro) / np.linalg.norm(Ro) <= 1e-10
    Q = np.vstack([out[0]["Q"], out[1]["Q"]])
    assert orc.orthogonality(Q) <= 1e-13
    assert orc.residual(A, Q, R) <= 1e-14


def test_bench_step_time_is_max_over_ranks():
    out = _run(_max_worker, 2)
    assert out[0] == out[1] == 2.0
