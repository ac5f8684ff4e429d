"""The one-launch cluster path (csrc/cluster_small.cuh, TSQR_PATH_CLUSTER) against the CPU
oracle on the same seeded inputs: every algorithm, ragged and tiny row counts (most CTAs of
the cluster own only zero padding), every supported panel width, breakdown reporting,
determinism and CUDA-graph replay, the host-buffer entry point, and eligibility limits.
Parity protocol as tests/test_gpu_parity.py: R <= 1e-10 (kappa <= 1e8),
Q <= 1e-11 (kappa <= 1e4), gates for mCQR2GS at every kappa, outcome classes otherwise."""
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

REDUCTIONS = {"cqr": 1, "scqr": 1, "cqr2": 2, "scqr3": 3}


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_04237_b200 as t
    t.load()
    return t


def _plan(T, m, n, b, algo, path="cluster"):
    old = os.environ.get("TSQR_CLUSTER_PATH")
    os.environ["TSQR_CLUSTER_PATH"] = "1" if path == "cluster" else "0"
    try:
        p = T.Plan(m, n, b, algo)
    finally:
        if old is None:
            os.environ.pop("TSQR_CLUSTER_PATH")
        else:
            os.environ["TSQR_CLUSTER_PATH"] = old
    assert p.exec_path() == path, (m, n, b, p.exec_path())
    return p


def _run(T, A, b, algo, path="cluster"):
    p = _plan(T, A.shape[0], A.shape[1], b, algo, path)
    Ad = T.to_colmajor(A)
    try:
        R = p.factor(Ad)
        calls = p.counts()[0]
    except T.TsqrError as e:
        assert e.status == T.TSQR_ERR_BREAKDOWN
        return None, None, e.info, None
    finally:
        p.close()
    return Ad.cpu().numpy(), R.cpu().numpy(), None, calls


def _reductions(algo, n, b):
    k = n // b
    if algo in REDUCTIONS:
        return REDUCTIONS[algo]
    if algo == "cqrgs":
        return 2 * k - 1
    return 2 if k == 1 else 4 * k - 2


@pytest.mark.parametrize("algo,m,n,b,kappa", [
    ("mcqr2gs", 4096, 64, 16, 1e8), ("mcqr2gs", 4096, 64, 16, 1e15), ("mcqr2gs", 4096, 64, 16, 1e3),
    ("mcqr2gs", 4001, 64, 16, 1e12), ("mcqr2gs", 1536, 128, 32, 1e10), ("mcqr2gs", 1536, 128, 64, 1e6),
    ("mcqr2gs", 100, 48, 16, 1e5), ("mcqr2gs", 33, 32, 16, 1e3), ("mcqr2gs", 2048, 96, 32, 1e14),
    ("cqr2gs", 4096, 64, 16, 1e6), ("cqr2gs", 3000, 96, 32, 1e4), ("cqr2gs", 2048, 64, 64, 1e5),
    ("cqr2", 4096, 64, 64, 1e4), ("cqr2", 777, 32, 32, 1e7), ("cqr2", 5000, 16, 16, 1e2),
    ("cqr", 4096, 32, 32, 1e3), ("cqrgs", 4096, 64, 16, 1e3),
    ("scqr3", 2048, 64, 64, 1e12), ("scqr3", 2048, 32, 32, 1e14), ("scqr", 4096, 64, 64, 1e6),
    ("mcqr2gs", 4096, 64, 64, 1e10), ("cqr2gs", 4096, 64, 32, 1e9),
])
def test_cluster_vs_oracle(T, orc, algo, m, n, b, kappa):
    A, _, _ = synth.generate_np(m, n, kappa, seed=11, chunk=m)
    Qo, Ro, io = orc.factor(A, b, algo)
    Q, R, info, calls = _run(T, A, b, algo)
    if io["status"] != 0 or info is not None:  # breakdown on one side: same stage of the same pass
        assert io["status"] == 5 and info is not None, (io, info)
        return
    assert calls == _reductions(algo, n, b)
    assert np.array_equal(np.tril(R, -1), np.zeros_like(R)) and np.all(np.diag(R) > 0)
    orth, res = orc.orthogonality(Q), orc.residual(A, Q, R)
    ortho, reso = orc.orthogonality(Qo), orc.residual(A, Qo, Ro)
    assert res <= 1e-14 or algo in ("cqr", "scqr", "cqrgs"), res
    if algo in ("mcqr2gs", "scqr3") or kappa <= 1e8:
        if algo not in ("cqr", "scqr", "cqrgs"):
            assert orth <= 1e-13, orth
    else:  # outcome class (R-21)
        assert (orth <= 1e-13) == (ortho <= 1e-13) or max(orth, ortho) / min(orth, ortho) <= 100, (orth, ortho)
    if algo in ("cqr", "scqr", "cqrgs"):  # single passes: orthogonality tracks the oracle's
        assert orth <= 100 * ortho + 1e-14, (orth, ortho)
    if kappa <= 1e8:
        assert np.linalg.norm(R - Ro) / np.linalg.norm(Ro) <= 1e-10
    if kappa <= 1e4:
        assert np.linalg.norm(Q - Qo) / np.linalg.norm(Qo) <= 1e-11


@pytest.mark.parametrize("algo,b", [("mcqr2gs", 16), ("cqr2gs", 32), ("cqr2", 64)])
def test_cluster_vs_stream_path(T, algo, b):
    """Both execution paths of the library on the same input: the same factorisation up to
    rounding order (R <= 1e-12, Q <= 1e-9 at kappa = 1e6)."""
    A, _, _ = synth.generate_np(4096, 64, 1e6, seed=12)
    Qc, Rc, _, cc = _run(T, A, b, algo, "cluster")
    Qs, Rs, _, cs = _run(T, A, b, algo, "stream")
    assert cc == cs
    assert np.linalg.norm(Rc - Rs) / np.linalg.norm(Rs) <= 1e-12
    # Q of two backward-stable orders differs by ~ kappa u (1e-10 here); R by ~ u
    assert np.linalg.norm(Qc - Qs) / np.linalg.norm(Qs) <= 1e-9


def test_cluster_breakdown_like_oracle(T, orc):
    A, _, _ = synth.generate_np(4096, 64, 1e2, seed=15)
    A[:, 20] = 0.0
    _, _, io = orc.factor(A, 16, "mcqr2gs")
    Q, R, info, _ = _run(T, A, 16, "mcqr2gs")
    assert Q is None and io["status"] == 5
    assert (info["pass"], info["panel"], info["stage"], info["pivot"]) == (io["pass"], io["panel"], io["stage"],
                                                                          io["pivot"])
    # the plan recovers: the next factorisation on a good matrix succeeds (status re-armed)
    A2, _, _ = synth.generate_np(4096, 64, 1e2, seed=15)
    Q2, R2, info2, _ = _run(T, A2, 16, "mcqr2gs")
    assert info2 is None


def test_cluster_deterministic_graph_replay_and_eager(T):
    import torch
    A, _, _ = synth.generate_np(4096, 64, 1e12, seed=13)
    p = _plan(T, 4096, 64, 16, "mcqr2gs")
    Ad = T.to_colmajor(A)
    R = T.colmajor_empty(64, 64)
    outs = []
    for _ in range(3):
        Ad.copy_(torch.from_numpy(A))
        p.factor(Ad, R)
        outs.append((Ad.cpu().numpy(), R.cpu().numpy()))
    p.set_graph(False)
    Ad.copy_(torch.from_numpy(A))
    p.factor(Ad, R)
    outs.append((Ad.cpu().numpy(), R.cpu().numpy()))
    for q, r in outs[1:]:
        assert np.array_equal(q, outs[0][0]) and np.array_equal(r, outs[0][1])
    assert p.counts() == (14, 1)  # 4k-2 reductions, ONE kernel launch
    p.close()


def test_cluster_timing_class_and_factor_host(T):
    import torch
    m, n, b = 4096, 64, 16
    A, _, _ = synth.generate_np(m, n, 1e8, seed=14)
    p = _plan(T, m, n, b, "mcqr2gs")
    Ad = T.to_colmajor(A)
    Rd = p.factor(Ad)
    Qd, Rd = Ad.cpu().numpy(), Rd.cpu().numpy()
    p.set_timing(True)
    Ah = torch.from_numpy(np.array(A, order="F")).T.contiguous().T.pin_memory()
    Rh = torch.zeros((n, n), dtype=torch.float64).T.contiguous().T.pin_memory()
    A_dev, R_dev = T.colmajor_empty(m, n), T.colmajor_empty(n, n)
    for _ in range(2):
        Ah.copy_(torch.from_numpy(np.array(A, order="F")))
        p.factor_host(Ah, Rh, A_dev, R_dev)
        p.wait()
        assert np.array_equal(Ah.numpy(), Qd) and np.array_equal(Rh.numpy(), Rd)
    tm = p.timing()
    assert tm["cluster"]["launches"] == 2 and tm["cluster"]["ms"] > 0
    assert all(tm[c]["launches"] == 0 for c in ("gram", "proj", "update", "trmm", "chol"))
    p.close()


def test_cluster_eligibility(T):
    """The plan picks the cluster path only where the block fits one cluster's shared memory,
    b in {16, 32, 64}; TSQR_CLUSTER_PATH=0 forces the streaming kernels."""
    cases = [(4096, 64, 16, "mcqr2gs", "cluster"), (4096, 64, 64, "cqr2", "cluster"),
             (65536, 64, 16, "mcqr2gs", "stream"), (4096, 512, 64, "mcqr2gs", "stream"),
             (2048, 256, 128, "mcqr2gs", "stream"), (4096, 64, 64, "scqr3", "stream"),
             (2048, 64, 64, "scqr3", "cluster"), (8192, 64, 16, "mcqr2gs", "stream")]
    for m, n, b, algo, want in cases:
        p = T.Plan(m, n, b, algo)
        assert p.exec_path() == want, (m, n, b, algo)
        p.close()
