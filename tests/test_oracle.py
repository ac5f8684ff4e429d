"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself:
worked examples printed in SPEC.md (tests/golden), exact integer arithmetic, LAPACK
(numpy/scipy) as an independent third party, closed forms, invariants, metamorphic
identities and the paper's stated accuracy claims. No test here retypes the oracle's
formulas. CPU only.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
U_RND = 2.0 ** -53


def M(x):
    return np.asfortranarray(np.array(x, dtype=np.float64))


# ---------------------------------------------------------------- SPEC worked examples
def test_spec_gram(orc):
    for ex in GOLD["gram"]:
        assert np.array_equal(orc.gram(M(ex["a"])), M(ex["expect"])), ex["cite"]


def test_spec_projection_and_update(orc):
    for ex in GOLD["matmul_t"]:
        assert np.array_equal(orc.atb(M(ex["a"]), M(ex["b"])), M(ex["expect"])), ex["cite"]
    for ex in GOLD["sub_prod"]:
        assert np.array_equal(orc.sub_prod(M(ex["c"]), M(ex["q"]), M(ex["y"])), M(ex["expect"])), ex["cite"]


def test_spec_cholesky(orc):
    for ex in GOLD["chol"]:
        U, brk = orc.chol(M(ex["w"]))
        if "breakdown_pivot" in ex:
            assert U is None and brk == (ex["breakdown_pivot"], ex["pivot_value"]), ex["cite"]
        else:
            assert brk is None and np.array_equal(U, M(ex["expect"])), ex["cite"]


def test_spec_rsolve_trimul(orc):
    for ex in GOLD["rsolve"]:
        assert np.array_equal(orc.rsolve(M(ex["a"]), M(ex["u"])), M(ex["expect"])), ex["cite"]
    for ex in GOLD["tri_mul"]:
        assert np.array_equal(orc.tri_mul(M(ex["r2"]), M(ex["r1"])), M(ex["expect"])), ex["cite"]


def test_spec_cqr_and_householder(orc):
    for ex in GOLD["cqr"]:
        Q, R, info = orc.factor(M(ex["a"]), 1, "cqr")
        assert info["status"] == 0
        assert np.array_equal(R, M(ex["r"]))
        np.testing.assert_allclose(Q, M(ex["q"]), rtol=0, atol=2 * U_RND)
    for ex in GOLD["householder"]:
        Q, R = orc.householder(M(ex["a"]))
        np.testing.assert_allclose(R, M(ex["r"]), rtol=0, atol=8 * U_RND)
        np.testing.assert_allclose(Q, M(ex["q"]), rtol=0, atol=4 * U_RND)


def test_spec_metrics(orc):
    for ex in GOLD["orthogonality_unnormalised"]:
        assert orc.orthogonality(M(ex["q"])) == pytest.approx(ex["expect"], abs=1e-15), ex["cite"]
    for ex in GOLD["residual"]:
        r = orc.residual(M(ex["a"]), M(ex["q"]), M(ex["r"]))
        if "expect" in ex:
            assert r == ex["expect"], ex["cite"]
        else:
            assert r <= ex["expect_max"], ex["cite"]


# ---------------------------------------------------------------- exact integer pins
@pytest.mark.parametrize("m,p,q", [(1000, 16, 16), (4099, 7, 33), (777, 64, 5)])
def test_atb_exact_integers(orc, m, p, q):
    """Entries in [-3,3]: every partial sum is an integer < 2^53, so any summation
    order is exact; compare bitwise with int64 arithmetic."""
    X = synth.integer_matrix(m, p, seed=1)
    Y = synth.integer_matrix(m, q, seed=2)
    ref = (X.astype(np.int64).T @ Y.astype(np.int64)).astype(np.float64)
    assert np.array_equal(orc.atb(X, Y), ref)
    G = (X.astype(np.int64).T @ X.astype(np.int64)).astype(np.float64)
    W = orc.gram(X)
    assert np.array_equal(W, G) and np.array_equal(W, W.T)


def test_sub_prod_exact_integers(orc):
    X = synth.integer_matrix(513, 40, seed=3)
    Q = synth.integer_matrix(513, 24, seed=4)
    Y = synth.integer_matrix(24, 40, seed=5)
    ref = (X.astype(np.int64) - Q.astype(np.int64) @ Y.astype(np.int64)).astype(np.float64)
    assert np.array_equal(orc.sub_prod(X, Q, Y), ref)


def _unit_upper_int(b, seed):
    rng = np.random.default_rng(seed)
    U = np.triu(rng.integers(-2, 3, size=(b, b)).astype(np.float64), 1) + np.eye(b)
    return np.asfortranarray(U)


def test_rsolve_exact(orc):
    """X = Z U with integer Z and unit upper-triangular integer U: rsolve(X,U) must give Z
    exactly (every intermediate is a small integer)."""
    b = 12
    U = _unit_upper_int(b, 0)
    Z = synth.integer_matrix(300, b, seed=6)
    X = (Z.astype(np.int64) @ U.astype(np.int64)).astype(np.float64)
    assert np.array_equal(orc.rsolve(X, U), Z)


def test_tri_inv_exact(orc):
    """A unit upper-triangular integer matrix has an integer inverse: U Z = I exactly."""
    for b in (8, 16):
        U = _unit_upper_int(b, b)
        Z = orc.tri_inv(U)
        assert np.array_equal(Z, np.round(Z))
        assert np.array_equal(U.astype(np.int64) @ Z.astype(np.int64), np.eye(b, dtype=np.int64))
        assert np.array_equal(np.tril(Z, -1), np.zeros((b, b)))


# ---------------------------------------------------------------- LAPACK pins
@pytest.mark.parametrize("b,kappa", [(16, 1e2), (64, 1e6), (128, 1e7)])
def test_cholesky_vs_lapack(orc, b, kappa):
    A, _, _ = synth.generate_np(4096, b, kappa, seed=3)
    W = A.T @ A
    W = np.triu(W) + np.triu(W, 1).T  # exactly symmetric
    U, brk = orc.chol(W)
    assert brk is None
    Ul = sla.cholesky(W, lower=False)  # LAPACK dpotrf
    assert np.array_equal(np.tril(U, -1), np.zeros_like(U))
    assert np.all(np.diag(U) > 0)
    assert np.linalg.norm(U.T @ U - W) <= 10 * U_RND * np.linalg.norm(W) * b
    # forward error relative to LAPACK: first-order bound b * u * cond(U) with cond(U) = kappa
    assert np.linalg.norm(U - Ul) <= b * U_RND * kappa * np.linalg.norm(Ul)


def test_tri_inv_vs_lapack(orc):
    A, _, _ = synth.generate_np(2048, 64, 1e4, seed=4)
    U = np.linalg.qr(A, mode="r")
    U = np.asfortranarray(U * np.sign(np.diag(U))[:, None])
    Z = orc.tri_inv(U)
    Zl = sla.lapack.dtrtri(U, lower=0)[0]
    cond = np.linalg.cond(U)
    assert np.linalg.norm(Z - Zl) <= 64 * U_RND * cond * np.linalg.norm(Zl)


def test_householder_vs_numpy(orc):
    rng = np.random.default_rng(7)
    for _ in range(10):
        m, n = int(rng.integers(20, 200)), int(rng.integers(2, 20))
        A = np.asfortranarray(rng.standard_normal((m, n)))
        Q, R = orc.householder(A)
        Qn, Rn = np.linalg.qr(A)
        s = np.sign(np.diag(Rn))
        Qn, Rn = Qn * s, Rn * s[:, None]
        np.testing.assert_allclose(R, Rn, atol=1e-12 * np.linalg.norm(A))
        np.testing.assert_allclose(Q, Qn, atol=1e-12)
        assert orc.orthogonality(Q) / math.sqrt(n) <= 50 * U_RND
        assert orc.residual(A, Q, R) <= 50 * U_RND


# ---------------------------------------------------------------- whole algorithms
ALL = ["cqr", "cqr2", "cqrgs", "cqr2gs", "mcqr2gs"]


def test_algorithms_match_householder_small(orc):
    """S:362 / S:596: on 50 small well-conditioned inputs every algorithm's R equals the
    (unique, sign-normalised) Householder R within 1e-10 ||A||_F entrywise."""
    rng = np.random.default_rng(11)
    for t in range(50):
        m, n = int(rng.integers(40, 200)), int(rng.integers(2, 20))
        kappa = 10.0 ** rng.uniform(0, 3)
        A, _, _ = synth.generate_np(m, n, kappa, seed=100 + t, chunk=m)
        _, Rh = orc.householder(A)
        b = int(rng.integers(1, n + 1))
        for algo in ALL:
            Q, R, info = orc.factor(A, b, algo)
            assert info["status"] == 0, (algo, info)
            assert np.max(np.abs(R - Rh)) <= 1e-10 * np.linalg.norm(A), algo
            assert orc.residual(A, Q, R) <= 1e-13, algo


def test_degeneracies_bitwise(orc):
    """P:357 / S:334: with one panel CQR2GS and mCQR2GS are CQR2, CQRGS is CQR."""
    A, _, _ = synth.generate_np(2048, 48, 1e6, seed=5)
    Q2, R2, _ = orc.factor(A, 48, "cqr2")
    for algo in ("cqr2gs", "mcqr2gs"):
        Q, R, _ = orc.factor(A, 48, algo)
        assert np.array_equal(Q, Q2) and np.array_equal(R, R2), algo
    Q1, R1, _ = orc.factor(A, 48, "cqr")
    Q, R, _ = orc.factor(A, 48, "cqrgs")
    assert np.array_equal(Q, Q1) and np.array_equal(R, R1)


def test_orthonormal_input(orc):
    """kappa = 1: R = I and Q = A within 10u."""
    A, _, _ = synth.generate_np(4096, 64, 1.0, seed=6)
    for algo, b in [("cqr2", 64), ("cqr2gs", 16), ("mcqr2gs", 16), ("mcqr2gs", 32)]:
        Q, R, info = orc.factor(A, b, algo)
        assert info["status"] == 0
        assert np.max(np.abs(R - np.eye(64))) <= 10 * U_RND * 8
        assert np.max(np.abs(Q - A)) <= 10 * U_RND * 8


def test_column_power_of_two_scaling_bitwise(orc):
    """Metamorphic pin: scaling columns by D = diag(2^e) commutes exactly with every
    rounded step, so Q(AD) = Q(A) and R(AD) = R(A) D bitwise (an index or transposition
    error in Gram, update, re-orthogonalisation or R assembly breaks this)."""
    A, _, _ = synth.generate_np(4096, 64, 1e12, seed=8)
    e = np.random.default_rng(0).integers(-6, 7, size=64)
    D = np.ldexp(1.0, e)
    AD = np.asfortranarray(A * D)
    for algo, b in [("cqr2gs", 16), ("mcqr2gs", 16), ("mcqr2gs", 32)]:
        Q, R, i1 = orc.factor(A, b, algo)
        QD, RD, i2 = orc.factor(AD, b, algo)
        assert i1["status"] == 0 and i2["status"] == 0
        assert np.array_equal(Q, QD), algo
        assert np.array_equal(R * D, RD), algo


def test_r_equals_r_of_sigma_vt(orc):
    """A = U (Sigma V^T) with orthonormal U, so R(A) = R(Sigma V^T), an n x n matrix
    factored here by LAPACK (numpy.linalg.qr) -- an m-free, implementation-free pin."""
    n = 64
    for kappa in (1e2, 1e5, 1e8):
        A, sigma, V = synth.generate_np(8192, n, kappa, seed=9, chunk=4096)
        B = sigma[:, None] * V.T
        Rb = np.linalg.qr(B, mode="r")
        Rb = Rb * np.sign(np.diag(Rb))[:, None]
        for algo, b in [("cqr2", n), ("cqr2gs", 16), ("mcqr2gs", 16)]:
            _, R, info = orc.factor(A, b, algo)
            assert info["status"] == 0
            rel = np.linalg.norm(R - Rb) / np.linalg.norm(Rb)
            assert rel <= 1e-12, (kappa, algo, rel)


def test_determinant_identity(orc):
    """|det R| = prod sigma_i, i.e. sum log R_ii = -(n/2) log kappa (closed form)."""
    n = 64
    for kappa, tol in ((1e4, 1e-9), (1e8, 1e-6), (1e15, 1.0)):
        A, _, _ = synth.generate_np(4096, n, kappa, seed=10)
        _, R, info = orc.factor(A, 16, "mcqr2gs")
        assert info["status"] == 0
        assert abs(np.sum(np.log(np.diag(R))) + 0.5 * n * math.log(kappa)) <= tol


def test_invariants_and_counts(orc):
    """R strictly upper with exact zeros and positive diagonal; Allreduce count
    4k-2 for CQR2GS and mCQR2GS, 2 for CQR2, 2k-1 for CQRGS (Appendix A.2 of SURVEY,
    S:331)."""
    n, b = 64, 16
    k = n // b
    A, _, _ = synth.generate_np(4096, n, 1e8, seed=12)
    for algo, expect in [("cqr2", 2), ("cqr", 1), ("cqrgs", 2 * k - 1), ("cqr2gs", 4 * k - 2),
                         ("mcqr2gs", 4 * k - 2)]:
        orc.reset_reduction_count()
        Q, R, info = orc.factor(A, b, algo)
        assert orc.reduction_count() == expect, algo
        assert info["status"] == 0
        assert np.array_equal(np.tril(R, -1), np.zeros_like(R))
        assert np.all(np.diag(R) > 0)


def test_ragged_panels(orc):
    """the last panel may be narrower; results stay accurate."""
    A, _, _ = synth.generate_np(4096, 50, 1e10, seed=13)
    for algo in ("cqr2gs", "mcqr2gs"):
        Q, R, info = orc.factor(A, 16, algo)
        assert info["status"] == 0
        assert orc.orthogonality(Q) <= 1e-13 and orc.residual(A, Q, R) <= 1e-14


def test_thread_count_independence(orc):
    A, _, _ = synth.generate_np(65536, 64, 1e12, seed=14)
    old = orc.get_threads()
    try:
        orc.set_threads(1)
        Q1, R1, _ = orc.factor(A, 16, "mcqr2gs")
        orc.set_threads(max(2, old))
        Q2, R2, _ = orc.factor(A, 16, "mcqr2gs")
    finally:
        orc.set_threads(old)
    assert np.array_equal(Q1, Q2) and np.array_equal(R1, R2)


def test_breakdown_reporting(orc):
    """A zero column makes the Gram singular with an exactly zero pivot: CQR's Cholesky
    breaks down; the oracle reports it as a value with (panel, stage, pivot)."""
    A, _, _ = synth.generate_np(1024, 16, 1e2, seed=15)
    A[:, 5] = 0.0
    Q, R, info = orc.factor(A, 16, "cqr2")
    assert Q is None and info["status"] == 5
    assert info["panel"] == 1 and info["stage"] == 1 and info["pivot"] == 5
    assert not (info["pivot_value"] > 0)
    A2, _, _ = synth.generate_np(1024, 32, 1e2, seed=15)
    A2[:, 20] = 0.0
    _, _, info2 = orc.factor(A2, 16, "mcqr2gs")
    assert info2["status"] == 5 and info2["panel"] == 2 and info2["stage"] == 1 and info2["pivot"] == 4


# ---------------------------------------------------------------- paper's accuracy claims
def _run(orc, A, b, algo):
    Q, R, info = orc.factor(A, b, algo)
    if info["status"] != 0:
        return None
    return orc.orthogonality(Q) / math.sqrt(A.shape[1])


@pytest.mark.parametrize("kappa", [1e0, 1e4, 1e8, 1e12, 1e15])
def test_paper_claim_mcqr2gs_three_panels(orc, kappa):
    """mCQR2GS with 3 panels reaches O(u) orthogonality and residual through
    kappa = 1e15 (SPEC's desk-scale 3000 x 300)."""
    A, _, _ = synth.generate_np(3000, 300, kappa, seed=0, chunk=3000)
    Q, R, info = orc.factor(A, 100, "mcqr2gs")
    assert info["status"] == 0
    assert orc.orthogonality(Q) / math.sqrt(300) <= 1e-13
    assert orc.residual(A, Q, R) <= 1e-13


def test_paper_claim_cqr2_fails_beyond_1e8(orc):
    """CQR2 is stable to kappa ~ 1e8 and fails (breakdown or loss of
    orthogonality) beyond."""
    A, _, _ = synth.generate_np(3000, 300, 1e4, seed=0, chunk=3000)
    assert _run(orc, A, 300, "cqr2") <= 1e-13
    A, _, _ = synth.generate_np(3000, 300, 1e12, seed=0, chunk=3000)
    o = _run(orc, A, 300, "cqr2")
    assert o is None or o > 1e-8


def test_paper_claim_mcqr2gs_two_panels_break(orc):
    """with 2 panels mCQR2GS breaks down at very high kappa, 3 panels do not
    (S:355). Frozen desk-scale observation (R-17): at 6000 x 600 the
    2-panel breakdown appears at kappa = 1e16, one decade above the paper's 1e15 at
    30000 x 3000 -- inside SPEC's +-1 decade allowance."""
    A, _, _ = synth.generate_np(6000, 600, 1e16, seed=0, chunk=6000)
    o = _run(orc, A, 300, "mcqr2gs")
    assert o is None or o > 1e-8
    assert _run(orc, A, 200, "mcqr2gs") <= 1e-13


def test_paper_claim_cqr2gs_needs_more_panels(orc):
    """at kappa = 1e15 CQR2GS needs many panels; k=1 always breaks down
    (S:594). Frozen desk-scale observation: k = 10 passes."""
    A, _, _ = synth.generate_np(3000, 300, 1e15, seed=0, chunk=3000)
    assert _run(orc, A, 300, "cqr2gs") is None
    assert _run(orc, A, 30, "cqr2gs") <= 1e-13
    A, _, _ = synth.generate_np(6000, 600, 1e16, seed=0, chunk=6000)
    for b in (600, 300):
        o = _run(orc, A, b, "cqr2gs")
        assert o is None or o > 1e-8
    assert _run(orc, A, 60, "cqr2gs") <= 1e-13


def test_interlacing_panel_condition(orc):
    """Eq. 7: cond(A) >= cond(A_1) >= sigma_{1+(n-b)} / sigma_b for the leading
    panel A_1 of the generated matrices."""
    n = 30
    for kappa in (1e0, 1e4, 1e8):
        A, sigma, _ = synth.generate_np(300, n, kappa, seed=1, chunk=300)
        for b in (3, 15):
            c = np.linalg.cond(A[:, :b])
            lower = sigma[n - b] / sigma[b - 1]
            assert c <= kappa * 1.05 + 1e-9 and c * 1.05 >= lower


# ---------------------------------------------------------------- shifted CholeskyQR3
def test_scqr3_matches_householder_small(orc):
    """Uniqueness of the thin QR: on well-conditioned inputs sCQR3's R equals the
    sign-normalised Householder R (LAPACK-free here: the oracle's own Householder is pinned
    against numpy above)."""
    rng = np.random.default_rng(21)
    for t in range(20):
        m, n = int(rng.integers(60, 300)), int(rng.integers(2, 24))
        A, _, _ = synth.generate_np(m, n, 10.0 ** rng.uniform(0, 4), seed=300 + t, chunk=m)
        _, Rh = orc.householder(A)
        Q, R, info = orc.factor(A, n, "scqr3")
        assert info["status"] == 0
        assert np.max(np.abs(R - Rh)) <= 1e-10 * np.linalg.norm(A)
        assert orc.residual(A, Q, R) <= 1e-13


@pytest.mark.parametrize("kappa", [1e8, 1e12, 1e15])
def test_paper_claim_scqr3_ill_conditioned(orc, kappa):
    """P:254-256 and Fig. orthoscqr3: with the conservative Frobenius shift sCQR3
    completes through kappa = 1e15 with O(u) orthogonality and residual, where CQR2 (no
    shift) fails beyond 1e8."""
    A, _, _ = synth.generate_np(3000, 300, kappa, seed=0, chunk=3000)
    Q, R, info = orc.factor(A, 300, "scqr3")
    assert info["status"] == 0
    assert orc.orthogonality(Q) / math.sqrt(300) <= 1e-13
    assert orc.residual(A, Q, R) <= 1e-13


def test_scqr_shift_makes_singular_gram_factorable(orc):
    """The shift is what makes the Cholesky succeed (Alg. 4 l.2-3): with an exactly
    repeated column the unshifted Gram is singular and CQR breaks down, sCQR does not, and
    its first diagonal entry obeys u_11^2 = g_11 + s with 0 < s << g_11."""
    A, _, _ = synth.generate_np(2048, 16, 1e3, seed=13)
    A = np.asfortranarray(np.hstack([A, A[:, :1]]))
    _, _, info = orc.factor(A, 17, "cqr")
    assert info["status"] == 5
    Q, R, info = orc.factor(A, 17, "scqr")
    assert info["status"] == 0
    g11 = float(np.dot(A[:, 0], A[:, 0]))
    s = R[0, 0] ** 2 - g11
    assert 0.0 < s < 1e-10 * g11


def test_scqr3_power_of_two_scaling_bitwise(orc):
    """Metamorphic pin: s scales with ||A||_F^2, so scaling A by 2^e scales every Gram, shift
    and Cholesky factor exactly: Q(2^e A) = Q(A) and R(2^e A) = 2^e R(A) bitwise."""
    A, _, _ = synth.generate_np(4096, 64, 1e14, seed=14)
    Q, R, i1 = orc.factor(A, 64, "scqr3")
    Qs, Rs, i2 = orc.factor(np.asfortranarray(np.ldexp(A, 5)), 64, "scqr3")
    assert i1["status"] == 0 and i2["status"] == 0
    assert np.array_equal(Q, Qs) and np.array_equal(np.ldexp(R, 5), Rs)


def test_scqr3_allreduce_count(orc):
    """Three Gram reductions (sCQR + CQR2, Alg. 5; "communication 50% higher than CQR2",
    P:264)."""
    A, _, _ = synth.generate_np(4096, 32, 1e6, seed=15)
    orc.reset_reduction_count()
    _, _, info = orc.factor(A, 32, "scqr3")
    assert info["status"] == 0 and orc.reduction_count() == 3


# ---------------------------------------------------------------- round-2 pins
def test_spec_matmul_and_accumulate_exact(orc):
    """orc_matmul's general mode, used for R := R2 R1 and for R_{1:j-1,j} += C U1 (R-8):
    SPEC's printed examples and an integer-exact accumulate case against int64."""
    for ex in GOLD["matmul"]:
        assert np.array_equal(orc.matmul(M(ex["a"]), M(ex["b"])), M(ex["expect"])), ex["cite"]
    A = synth.integer_matrix(37, 23, seed=21)
    B = synth.integer_matrix(23, 11, seed=22)
    C0 = synth.integer_matrix(37, 11, seed=23)
    want = C0.astype(np.int64) + A.astype(np.int64) @ B.astype(np.int64)
    got = orc.matmul(A, B, C=C0)
    assert np.array_equal(got, want.astype(np.float64))
    assert np.array_equal(orc.matmul(A, B), (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64))


@pytest.mark.parametrize("m,c0,b", [(4096, 48, 16), (2048, 64, 32)])
def test_mcqr2gs_panel_r_assembly_closed_form(orc, m, c0, b):
    """Alg. 8 lines 6-8 with the R bookkeeping of R-8 on a panel that is NOT orthogonal to the
    earlier panels.  Mathematics fixes the answer for any panel P: A_j = V1 U1 and
    V1 = Q_{1:j-1} C + Q_j U2, so R_{1:j-1,j} gains exactly Q_{1:j-1}^T P and R_jj is the R
    factor of the projected panel (I - Q Q^T) P (LAPACK, sign-normalised).  Inside the full
    algorithm the earlier lines make Q_{1:j-1}^T P a rounding-level quantity, which is why the
    C U1 term cannot be seen there; here it is O(1), so dropping it, flipping its sign or
    transposing an operand fails by orders of magnitude."""
    rng = np.random.default_rng(31)
    Qprev = np.asfortranarray(np.linalg.qr(rng.standard_normal((m, c0)))[0])
    N, _, _ = synth.generate_np(m, b, 1e3, seed=32, chunk=m)
    G = rng.standard_normal((c0, b)) * 4.0
    P = np.asfortranarray(Qprev @ G + N)
    Y0 = rng.standard_normal((c0, b))
    Qj, Rcol, Rjj, info = orc.mcqr2gs_panel(Qprev, P, R_col=Y0)
    assert info["status"] == 0
    want_col = Y0 + Qprev.T @ P
    assert np.linalg.norm(Rcol - want_col) <= 1e-12 * np.linalg.norm(want_col)
    Pp = P - Qprev @ (Qprev.T @ P)
    Qh, Rh = np.linalg.qr(Pp)
    Rh = np.sign(np.diag(Rh))[:, None] * Rh
    assert np.linalg.norm(Rjj - Rh) <= 1e-12 * np.linalg.norm(Rh)
    # the panel identity itself: P = Q_{1:j-1} (R_{1:j-1,j} - Y0) + Q_j R_jj
    assert np.linalg.norm(P - Qprev @ (Rcol - Y0) - Qj @ Rjj) <= 1e-14 * np.linalg.norm(P)
    # one block-GS pass against an O(1) component: cross-orthogonality at the u * kappa(P) level
    assert np.linalg.norm(Qprev.T @ Qj) <= 1e-9


def test_scqr_shift_value_closed_form(orc):
    """The value of the sCQR shift (Alg. 4 l.2: s = sqrt(m) u ||A||_F^2, m the row
    count, u = 2^-53).  For A with orthonormal columns G = I + O(u) and ||A||_F^2 = n, so
    W = (1 + s) I and every R_ii^2 - 1 = s = sqrt(m) u n.  At m = 2^18, n = 64, s = 32768 u:
    the rounding of G and R (a few u) is resolved to well under 1%; sqrt(b) for sqrt(m),
    ||A||_F for ||A||_F^2 or u = 2^-52 are off by 2x or more."""
    m, n = 1 << 18, 64
    A = synth.orthonormal_np(m, n, seed=1)
    Q, R, info = orc.factor(A, n, "scqr")
    assert info["status"] == 0
    s = math.sqrt(m) * U_RND * n
    d = np.diag(R) ** 2 - 1.0
    assert np.max(np.abs(d / s - 1.0)) <= 0.01, (d.min() / s, d.max() / s)


# ---------------------------------------------------------------- NEXT-f4: adaptive repetition
# oracle.c mcqr2gs_adaptive (DESIGN R-23).  Pins: the two limits of the threshold are
# existing algorithms bitwise; the estimate has closed forms; the default threshold keeps the
# gates over a kappa sweep (frozen desk-scale observation) while skipping where kappa is small.

@pytest.fixture
def tau_guard(orc):
    t = orc.get_adapt_tau()
    yield
    orc.set_adapt_tau(t)


@pytest.mark.parametrize("m,n,b,kappa", [(4096, 128, 32, 1e3), (3001, 96, 32, 1e10), (2048, 64, 64, 1e2),
                                         (5000, 100, 32, 1e6)])
def test_adaptive_tau_zero_is_mcqr2gs_bitwise(orc, tau_guard, m, n, b, kappa):
    A, _, _ = synth.generate_np(m, n, kappa, seed=2, chunk=m)
    orc.set_adapt_tau(0.0)
    Qa, Ra, ia = orc.factor(A, b, "mcqr2gs_adaptive")
    Qm, Rm, im = orc.factor(A, b, "mcqr2gs")
    assert orc.adapt_skipped() == 0
    assert np.array_equal(Qa, Qm) and np.array_equal(Ra, Rm)


@pytest.mark.parametrize("m,n,b,kappa", [(4096, 128, 32, 1e3), (3001, 96, 32, 1e10), (5000, 100, 32, 1e6)])
def test_adaptive_tau_inf_is_cqrgs_bitwise(orc, tau_guard, m, n, b, kappa):
    A, _, _ = synth.generate_np(m, n, kappa, seed=2, chunk=m)
    orc.set_adapt_tau(math.inf)
    Qa, Ra, _ = orc.factor(A, b, "mcqr2gs_adaptive")
    Qc, Rc, _ = orc.factor(A, b, "cqrgs")
    assert orc.adapt_skipped() == -(-n // b)
    assert np.array_equal(Qa, Qc) and np.array_equal(Ra, Rc)


def test_adaptive_estimate_closed_forms(orc):
    """E = max(u nu(U)^2 nu(Z)^2, u nu([Rcol; U]) nu(Z)), nu(M) = ||M||_F / sqrt(b):
    U = I, no column above: E = u exactly; U = diag(s): own = u (sum s^2/b)(sum s^-2/b);
    a column block above adds to nu([Rcol; U]) only."""
    import ctypes
    L = orc.lib()
    L.orc_adapt_estimate.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int64]
    L.orc_adapt_estimate.restype = ctypes.c_double
    P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    u = 2.0 ** -53
    b = 8
    I = np.asfortranarray(np.eye(b))
    dummy = np.zeros((1, b), order="F")
    assert L.orc_adapt_estimate(P(I), b, P(dummy), 1, 0) == u
    s = 2.0 ** np.arange(b)  # powers of two: every sum below is exact
    D = np.asfortranarray(np.diag(s))
    own = u * (np.sum(s ** 2) / b) * (np.sum(s ** -2.0) / b)
    assert L.orc_adapt_estimate(P(D), b, P(dummy), 1, 0) == pytest.approx(own, rel=1e-15)
    Rc = np.asfortranarray(np.full((3, b), 4.0))  # ||Rcol||_F^2 = 3 b 16
    across = u * math.sqrt((3 * b * 16 + b) / b) * 1.0
    assert L.orc_adapt_estimate(P(I), b, P(Rc), 3, 3) == pytest.approx(across, rel=1e-15)
    assert orc.kappa_f(D) == pytest.approx(math.sqrt(np.sum(s ** 2) * np.sum(s ** -2.0)), rel=1e-15)
    assert orc.diag_ratio(D) == s[-1] / s[0]


def test_adaptive_default_threshold_keeps_gates(orc, tau_guard):
    """Frozen desk-scale observation (R-23): with the default tau = 2^-50 every case of the
    kappa sweep meets the BJ gates; orthonormal-column inputs skip every repetition, kappa = 1e2
    at least half of them (6 of 8 measured); at
    kappa >= 1e12 nothing is skipped and the result is mCQR2GS bitwise."""
    assert orc.get_adapt_tau() == 2.0 ** -50
    m, n, b = 1 << 14, 256, 32
    k = n // b
    for kappa in (1.0, 1e2, 1e4, 1e8, 1e12, 1e15):
        A, _, _ = synth.generate_np(m, n, kappa, seed=1)
        Q, R, info = orc.factor(A, b, "mcqr2gs_adaptive")
        sk = orc.adapt_skipped()
        assert info["status"] == 0
        assert orc.orthogonality(Q) <= 1e-13 and orc.residual(A, Q, R) <= 1e-14, kappa
        assert np.array_equal(np.tril(R, -1), 0 * R) and np.all(np.diag(R) > 0)
        if kappa == 1.0:
            assert sk == k, sk
        if kappa == 1e2:
            assert sk >= k // 2, sk
        if kappa >= 1e12:
            assert sk == 0
            Qm, Rm, _ = orc.factor(A, b, "mcqr2gs")
            assert np.array_equal(Q, Qm) and np.array_equal(R, Rm)
