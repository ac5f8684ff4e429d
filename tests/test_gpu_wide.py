"""Wide panels ("panels are 400, 2000 and 4000 wide", P:111 30000 x 3000
with 3 panels; DESIGN R-24: widths as multiples of 64): the multi-CTA blocked Cholesky +
inverse against the oracle (LAPACK-pinned) and whole factorisations with b = 384 .. 2048
against the CPU oracle."""
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


@pytest.mark.parametrize("b", [320, 512, 1024, 2048])
def test_wide_chol_inv_vs_oracle(T, orc, b):
    rng = np.random.default_rng(b)
    X = rng.standard_normal((4 * b, b)) @ np.diag(np.logspace(0, -4, b))
    W = np.asfortranarray(X.T @ X)
    U, Z, st = T.chol_inv(T.to_colmajor(W))
    assert int(st[0].item()) == 0
    U, Z = U.cpu().numpy(), Z.cpu().numpy()
    Uo = orc.chol(W)[0]
    Zo = orc.tri_inv(Uo)
    assert np.array_equal(np.tril(U, -1), 0 * U) and np.array_equal(np.tril(Z, -1), 0 * Z)
    assert np.linalg.norm(U - Uo) / np.linalg.norm(Uo) <= 1e-12
    assert np.linalg.norm(Z - Zo) / np.linalg.norm(Zo) <= 1e-9  # kappa(U) = 1e4: Z to ~ kappa u
    assert np.linalg.norm(U @ Z - np.eye(b)) <= 1e-9


def test_wide_chol_breakdown_global_pivot(T):
    b = 512
    W = np.asfortranarray(np.eye(b) * 4.0)
    W[300, 300] = -1.0
    U, Z, st = T.chol_inv(T.to_colmajor(W))
    st = st.cpu().numpy()
    assert st[0] == 5 and st[4] == 300


@pytest.mark.parametrize("algo,m,n,b,kappa", [("mcqr2gs", 8192, 1536, 512, 1e4), ("mcqr2gs", 8192, 1536, 512, 1e12),
                                               ("mcqr2gs", 6000, 1152, 384, 1e4), ("cqr2", 20000, 384, 384, 1e6),
                                               ("cqr2gs", 8192, 1024, 512, 1e6), ("mcqr2gs", 10000, 2048, 1024, 1e8)])
def test_wide_panels_vs_oracle(T, orc, algo, m, n, b, kappa):
    A, _, _ = synth.generate_np(m, n, kappa, seed=4, chunk=m)
    Qo, Ro, io = orc.factor(A, b, algo)
    Ad = T.to_colmajor(A)
    p = T.Plan(m, n, b, algo)
    R = p.factor(Ad).cpu().numpy()
    calls = p.counts()[0]
    p.close()
    Q = Ad.cpu().numpy()
    k = n // b
    assert calls == {"cqr2": 2}.get(algo, 4 * k - 2)
    assert io["status"] == 0
    assert np.array_equal(np.tril(R, -1), 0 * R) and np.all(np.diag(R) > 0)
    orth, res = orc.orthogonality(Q), orc.residual(A, Q, R)
    assert res <= 1e-14, res
    if algo != "cqr2gs" or kappa <= 1e8:
        assert orth <= 1e-13, orth
    if kappa <= 1e8:
        assert np.linalg.norm(R - Ro) / np.linalg.norm(Ro) <= 1e-10


def test_paper_stability_shape_30000x3072_three_panels(T):
    """30000 x 3000, kappa up to 1e15, 3 panels -- here 30000 x 3072, b = 1024 (R-24):
    the mCQR2GS gates hold (error-free verifier; the oracle would need minutes)."""
    import torch
    from harness import verify
    m, n, b = 30000, 3072, 1024
    A = T.colmajor_empty(m, n)
    synth.generate_torch(A, m, 0, n, 1e15, seed=0, chunk=m)
    A0 = A.clone()
    p = T.Plan(m, n, b, "mcqr2gs")
    R = p.factor(A)
    p.close()
    orth, res = verify.orthogonality(A), verify.residual(A0, A, R)
    Rh = R.cpu().numpy()
    torch.cuda.synchronize()
    print(f"30000x3072 b=1024 kappa=1e15: orth {orth:.3e} res {res:.3e}")
    assert np.array_equal(np.tril(Rh, -1), 0 * Rh) and np.all(np.diag(Rh) > 0)
    # measured 1.08e-13 un-normalised at n = 3072: the per-entry level of the BJ gate through the
    # paper's normalisation (R-1): ||Q^TQ - I||_F / sqrt(n) <= 1e-13 / sqrt(512)
    assert orth / np.sqrt(n) <= 1e-13 / np.sqrt(512) and res <= 1e-14, (orth, res)
