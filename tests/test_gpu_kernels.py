"""Step-level parity of the CUDA kernels (through the C ABI) against the CPU oracle and
exact integer arithmetic.  GPU only."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
U_RND = 2.0 ** -53


@pytest.fixture(scope="module")
def T():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2405_04237_b200 as t
    t.load()
    return t


def np_of(x):
    return x.cpu().numpy()


def dev(t, x, ld=None):
    return t.to_colmajor(x, ld=ld)


def i64(x):
    return np.asarray(x).astype(np.int64)


# ------------------------------------------------------------------ exact integer pins
@pytest.mark.parametrize("m", [1, 63, 4099, 65536 + 17])
@pytest.mark.parametrize("b", [16, 32, 64, 128, 256])
def test_gram_exact_integers(T, m, b):
    X = synth.integer_matrix(m, b, seed=m + b)
    W = np_of(T.gram(dev(T, X)))
    ref = (i64(X).T @ i64(X)).astype(np.float64)
    assert np.array_equal(W, ref)


@pytest.mark.parametrize("m,p,q", [(4099, 64, 448), (70001, 448, 64), (513, 16, 48), (3000, 130, 70),
                                   (65536, 256, 1792)])
def test_proj_exact_integers(T, m, p, q):
    Lm = synth.integer_matrix(m, p, seed=1)
    Rm = synth.integer_matrix(m, q, seed=2)
    out = np_of(T.proj(dev(T, Lm), dev(T, Rm)))
    assert np.array_equal(out, (i64(Lm).T @ i64(Rm)).astype(np.float64))


# the larger cases give every CTA several row tiles per warp group and several column chunks
# per tile (the pipelined path with all its slot reuse), so a race shows up as a wrong integer
@pytest.mark.parametrize("m,p,q", [(4099, 64, 448), (70001, 448, 64), (513, 16, 48), (3001, 130, 70),
                                   (8192, 256, 1792), (65536 + 17, 64, 128), (300001, 64, 448),
                                   (150000, 128, 192), (99999, 32, 96)])
def test_update_exact_integers(T, m, p, q):
    X = synth.integer_matrix(m, q, seed=3)
    Lm = synth.integer_matrix(m, p, seed=4)
    S = synth.integer_matrix(p, q, seed=5)
    Xd = dev(T, X)
    T.update(Xd, dev(T, Lm), dev(T, S))
    assert np.array_equal(np_of(Xd), (i64(X) - i64(Lm) @ i64(S)).astype(np.float64))


def _unit_upper_int(b, seed):
    rng = np.random.default_rng(seed)
    return np.asfortranarray(np.triu(rng.integers(-1, 2, size=(b, b)).astype(np.float64), 1) + np.eye(b))


@pytest.mark.parametrize("b", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("m", [100, 4099, 65536 + 3])
def test_trmm_exact_integers(T, b, m):
    X = synth.integer_matrix(m, b, seed=6, lo=-1, hi=1)
    Z = _unit_upper_int(b, b)
    Xd = dev(T, X)
    T.trmm(Xd, dev(T, Z))
    ref = i64(X) @ i64(Z)
    assert np.abs(ref).max() < 2 ** 53
    assert np.array_equal(np_of(Xd), ref.astype(np.float64))


def test_odd_leading_dimension_paths(T):
    """lda odd -> 8-byte cp.async path; same exact results."""
    m, b = 4097, 64
    X = synth.integer_matrix(m, b, seed=7)
    W = np_of(T.gram(dev(T, X, ld=m + 1 if m % 2 == 0 else m)))
    assert np.array_equal(W, (i64(X).T @ i64(X)).astype(np.float64))
    Xd = dev(T, X, ld=m)  # odd
    Z = _unit_upper_int(b, 1)
    T.trmm(Xd, dev(T, Z))
    assert np.array_equal(np_of(Xd), (i64(X) @ i64(Z)).astype(np.float64))


# ------------------------------------------------------------------ oracle parity (random)
@pytest.mark.parametrize("m,b,kappa", [(65536 + 5, 64, 1e8), (4096, 16, 1e3), (20000, 256, 1e4)])
def test_gram_vs_oracle(T, orc, m, b, kappa):
    A, _, _ = synth.generate_np(m, b, kappa, seed=2, chunk=m)
    W = np_of(T.gram(dev(T, A)))
    Wo = orc.gram(A)
    assert np.array_equal(W, W.T)
    bound = np.abs(A).T @ np.abs(A)
    assert np.all(np.abs(W - Wo) <= 64 * U_RND * bound)


@pytest.mark.parametrize("m,p,q", [(65536 + 5, 64, 448), (30000, 448, 64)])
def test_proj_update_vs_oracle(T, orc, m, p, q):
    rng = np.random.default_rng(0)
    Lm = np.asfortranarray(rng.standard_normal((m, p)))
    Rm = np.asfortranarray(rng.standard_normal((m, q)))
    out = np_of(T.proj(dev(T, Lm), dev(T, Rm)))
    ref = orc.atb(Lm, Rm)
    bound = np.abs(Lm).T @ np.abs(Rm)
    assert np.all(np.abs(out - ref) <= 64 * U_RND * bound)
    S = np.asfortranarray(rng.standard_normal((p, q)) / p)
    Xd = dev(T, Rm)
    T.update(Xd, dev(T, Lm), dev(T, S))
    ref = orc.sub_prod(Rm, Lm, S)
    bound = np.abs(Rm) + np.abs(Lm) @ np.abs(S)
    assert np.all(np.abs(np_of(Xd) - ref) <= 2 * p * U_RND * bound)


@pytest.mark.parametrize("b,kappa", [(16, 1e2), (64, 1e6), (128, 1e7), (256, 1e5)])
def test_chol_inv_vs_oracle(T, orc, b, kappa):
    A, _, _ = synth.generate_np(8192, b, kappa, seed=3)
    W = orc.gram(A)
    U, Z, st = T.chol_inv(dev(T, W))
    assert int(st[0]) == 0
    U, Z = np_of(U), np_of(Z)
    Uo, brk = orc.chol(W)
    assert brk is None
    assert np.array_equal(np.tril(U, -1), np.zeros_like(U)) and np.array_equal(np.tril(Z, -1), np.zeros_like(Z))
    assert np.linalg.norm(U - Uo) <= b * U_RND * kappa * np.linalg.norm(Uo)
    Zo = orc.tri_inv(Uo)
    assert np.linalg.norm(Z - Zo) <= b * U_RND * kappa ** 2 * np.linalg.norm(Zo)
    assert np.linalg.norm(U @ Z - np.eye(b)) <= b * U_RND * kappa


def test_chol_spec_examples_and_breakdown(T):
    import torch
    U, Z, st = T.chol_inv(dev(T, np.array([[4.0, 2.0], [2.0, 5.0]])))
    assert np.array_equal(np_of(U), np.array([[2.0, 1.0], [0.0, 2.0]]))
    assert np.array_equal(np_of(Z), np.array([[0.5, -0.25], [0.0, 0.5]]))
    U, Z, st = T.chol_inv(dev(T, np.array([[1.0, 2.0], [2.0, 1.0]])))
    s = st.cpu().numpy()
    assert s[0] == 5 and s[4] == 1
    assert st[6:8].view(torch.float64).item() == -3.0


def test_kernels_deterministic(T):
    A, _, _ = synth.generate_np(65536, 256, 1e6, seed=4)
    Ad = dev(T, A)
    w1 = np_of(T.gram(Ad))
    w2 = np_of(T.gram(Ad))
    assert np.array_equal(w1, w2)
    p1 = np_of(T.proj(Ad[:, :64], Ad[:, 64:]))
    p2 = np_of(T.proj(Ad[:, :64], Ad[:, 64:]))
    assert np.array_equal(p1, p2)
