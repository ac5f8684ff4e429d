"""Runtime-adaptive repetition (TSQR_MCQR2GS_ADAPTIVE, DESIGN R-23) on
the GPU against the CPU oracle's mcqr2gs_adaptive (same rule, same default tau = 2^-50):
  * tau = 0 is the GPU's mCQR2GS bitwise, tau = inf its CQRGS bitwise (the skipped kernels
    return at once; R_jj = I U1 and R += 0 U1 are exact);
  * at the default tau the number of skipped panels equals the oracle's, R matches it
    (<= 1e-10, kappa <= 1e8) and the gates hold over a kappa sweep;
  * a breakdown is reported as for mCQR2GS; graph replays re-decide every call."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_04237_b200 as t
    t.load()
    return t


def _run(T, A, b, algo, tau=None, reps=1):
    import torch
    m, n = A.shape
    p = T.Plan(m, n, b, algo)
    if tau is not None:
        p.set_adapt_tau(tau)
    A0 = T.to_colmajor(A)
    X = T.colmajor_empty(m, n)
    try:
        for _ in range(reps):
            X.copy_(A0)
            R = p.factor(X)
        sk = p.skipped_panels()
    except T.TsqrError as e:
        p.close()
        return None, None, e.info, None
    torch.cuda.synchronize()
    p.close()
    return X.cpu().numpy(), R.cpu().numpy(), None, sk


@pytest.mark.parametrize("m,n,b,kappa", [(65536 + 37, 512, 64, 1e3), (20000, 1024, 128, 1e6), (20000, 1024, 256, 1e2),
                                         (8192, 256, 32, 1e12)])
def test_adaptive_limits_bitwise(T, m, n, b, kappa):
    A, _, _ = synth.generate_np(m, n, kappa, seed=3, chunk=m if m % 65536 else 65536)
    Q0, R0, _, s0 = _run(T, A, b, "mcqr2gs_adaptive", tau=0.0)
    Qm, Rm, _, _ = _run(T, A, b, "mcqr2gs")
    assert s0 == 0
    assert np.array_equal(Q0, Qm) and np.array_equal(R0, Rm)
    Qi, Ri, _, si = _run(T, A, b, "mcqr2gs_adaptive", tau=np.inf, reps=2)
    Qc, Rc, _, _ = _run(T, A, b, "cqrgs")
    assert si == n // b
    assert np.array_equal(Qi, Qc) and np.array_equal(Ri, Rc)


@pytest.mark.parametrize("kappa", [1.0, 1e2, 1e3, 1e4, 1e6, 1e8, 1e12, 1e15])
def test_adaptive_vs_oracle(T, orc, kappa):
    m, n, b = 1 << 15, 256, 32
    A, _, _ = synth.generate_np(m, n, kappa, seed=1)
    Qo, Ro, io = orc.factor(A, b, "mcqr2gs_adaptive")
    so = orc.adapt_skipped()
    Q, R, info, sk = _run(T, A, b, "mcqr2gs_adaptive", reps=2)
    assert io["status"] == 0 and info is None
    assert sk == so, (sk, so)
    assert np.array_equal(np.tril(R, -1), 0 * R) and np.all(np.diag(R) > 0)
    assert orc.orthogonality(Q) <= 1e-13 and orc.residual(A, Q, R) <= 1e-14
    if kappa <= 1e8:
        assert np.linalg.norm(R - Ro) / np.linalg.norm(Ro) <= 1e-10


def test_adaptive_breakdown_and_recovery(T, orc):
    A, _, _ = synth.generate_np(4096, 64, 1e2, seed=15)
    bad = A.copy()
    bad[:, 20] = 0.0
    _, _, io = orc.factor(bad, 16, "mcqr2gs_adaptive")
    Q, R, info, _ = _run(T, bad, 16, "mcqr2gs_adaptive")
    assert Q is None and io["status"] == 5
    assert (info["pass"], info["panel"], info["stage"], info["pivot"]) == (io["pass"], io["panel"], io["stage"],
                                                                          io["pivot"])
    Q, R, info, sk = _run(T, A, 16, "mcqr2gs_adaptive")
    assert info is None and orc.orthogonality(Q) <= 1e-13
