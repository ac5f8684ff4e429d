"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE. Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package. The CUDA
product path (``paper_2405_04237_b200``) never imports it and shares no code with it.

All matrices are numpy float64 arrays in Fortran (column-major) order, matching the
oracle's ``X[r + c*ldx]`` convention. Functions cite the paper through oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CQR2, CQR2GS, MCQR2GS, CQR, CQRGS, SCQR3, SCQR, MCQR2GS_ADAPTIVE = 0, 1, 2, 3, 4, 5, 6, 7
ALGOS = {"cqr2": CQR2, "cqr2gs": CQR2GS, "mcqr2gs": MCQR2GS, "cqr": CQR, "cqrgs": CQRGS, "scqr3": SCQR3,
         "scqr": SCQR, "mcqr2gs_adaptive": MCQR2GS_ADAPTIVE}
OK, ERR_ARG, ERR_BREAKDOWN, ERR_NOMEM = 0, 1, 5, 6

BUILD_CMD = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
             "-std=c99", "-Wall", "-o", _LIB, _SRC, "-lm"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2 -ffp-contract=off: no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(BUILD_CMD, check=True)
    return _LIB


class Info(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("pass_", ctypes.c_int32), ("panel", ctypes.c_int32),
                ("stage", ctypes.c_int32), ("pivot", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("pivot_value", ctypes.c_double)]

    def as_dict(self):
        return {"status": self.status, "pass": self.pass_, "panel": self.panel, "stage": self.stage,
                "pivot": self.pivot, "pivot_value": self.pivot_value}


_lib = None
_P = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_set_adapt_tau.argtypes = [ctypes.c_double]
        L.orc_get_adapt_tau.restype = ctypes.c_double
        L.orc_adapt_skipped.restype = ctypes.c_int64
        L.orc_diag_ratio.argtypes = [_P, _I64, _I64]
        L.orc_diag_ratio.restype = ctypes.c_double
        L.orc_kappa_f.argtypes = [_P, _I64, _I64]
        L.orc_kappa_f.restype = ctypes.c_double
        L.orc_get_threads.restype = ctypes.c_int
        L.orc_gram.argtypes = [_P, _I64, _I64, _I64, _P, _I64]
        L.orc_atb.argtypes = [_P, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64]
        L.orc_chol.argtypes = [_P, _I64, _I64, _P, _I64, ctypes.POINTER(ctypes.c_int32), _P]
        L.orc_rsolve.argtypes = [_P, _I64, _I64, _I64, _P, _I64]
        L.orc_rsolve.restype = None
        L.orc_tri_inv.argtypes = [_P, _I64, _I64, _P, _I64]
        L.orc_tri_inv.restype = None
        L.orc_matmul.argtypes = [_P, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64, ctypes.c_int, ctypes.c_int]
        L.orc_matmul.restype = None
        L.orc_mcqr2gs_panel.argtypes = [_P, _I64, _I64, _I64, _I64, _P, _I64, ctypes.c_int, ctypes.POINTER(Info)]
        L.orc_mcqr2gs_panel.restype = ctypes.c_int
        L.orc_sub_prod.argtypes = [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64]
        L.orc_sub_prod.restype = None
        L.orc_factor.argtypes = [_P, _I64, _I64, _I64, _I64, ctypes.c_int, _P, _I64, ctypes.POINTER(Info)]
        L.orc_householder.argtypes = [_P, _I64, _I64, _I64, _P, _I64, _P, _I64]
        L.orc_orthogonality.argtypes = [_P, _I64, _I64, _I64]
        L.orc_orthogonality.restype = ctypes.c_double
        L.orc_residual.argtypes = [_P, _I64, _P, _I64, _P, _I64, _I64, _I64]
        L.orc_residual.restype = ctypes.c_double
        L.orc_reduction_count.restype = ctypes.c_int64
        L.orc_reset_reduction_count.restype = None
        L.orc_set_threads(len(os.sched_getaffinity(0)))
    return _lib


def _f(a: np.ndarray) -> np.ndarray:
    a = np.asfortranarray(a, dtype=np.float64)
    return a


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.f_contiguous
    return a.ctypes.data_as(_P)


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def reduction_count() -> int:
    """Sigma_rows reductions since the last reset (= Allreduce calls of the distributed form)."""
    return int(lib().orc_reduction_count())


def reset_reduction_count() -> None:
    lib().orc_reset_reduction_count()


def gram(X):
    X = _f(X)
    m, b = X.shape
    W = np.zeros((b, b), order="F")
    rc = lib().orc_gram(_p(X), m, m, b, _p(W), b)
    assert rc == OK
    return W


def atb(X, Y):
    X, Y = _f(X), _f(Y)
    m, p = X.shape
    q = Y.shape[1]
    out = np.zeros((p, q), order="F")
    rc = lib().orc_atb(_p(X), m, _p(Y), m, m, p, q, _p(out), p)
    assert rc == OK
    return out


def chol(W):
    """Upper Cholesky; returns (U, None) or (None, (pivot, pivot_value))."""
    W = _f(W)
    b = W.shape[0]
    U = np.zeros((b, b), order="F")
    piv = ctypes.c_int32(-1)
    pv = ctypes.c_double(0.0)
    rc = lib().orc_chol(_p(W), b, b, _p(U), b, ctypes.byref(piv), ctypes.byref(pv))
    if rc == ERR_BREAKDOWN:
        return None, (piv.value, pv.value)
    assert rc == OK
    return U, None


def rsolve(X, U):
    X = np.array(X, dtype=np.float64, order="F", copy=True)
    U = _f(U)
    m, b = X.shape
    lib().orc_rsolve(_p(X), m, m, b, _p(U), b)
    return X


def tri_inv(U):
    U = _f(U)
    b = U.shape[0]
    Z = np.zeros((b, b), order="F")
    lib().orc_tri_inv(_p(U), b, b, _p(Z), b)
    return Z


def tri_mul(A, B):
    """Product of two upper-triangular matrices (skips the known-zero region)."""
    A, B = _f(A), _f(B)
    n = A.shape[0]
    C = np.zeros((n, n), order="F")
    lib().orc_matmul(_p(A), n, _p(B), n, n, n, n, _p(C), n, 1, 0)
    return C


def matmul(A, B, C=None):
    """A @ B (plain triple loop); with C given, returns C + A @ B (the accumulate mode used for
    R_{1:j-1,j} += C U1, R-8)."""
    A, B = _f(A), _f(B)
    p, r = A.shape
    q = B.shape[1]
    acc = C is not None
    C = np.array(C, dtype=np.float64, order="F", copy=True) if acc else np.zeros((p, q), order="F")
    lib().orc_matmul(_p(A), p, _p(B), r, p, r, q, _p(C), p, 0, 1 if acc else 0)
    return C


def sub_prod(X, Q, Y):
    X = np.array(X, dtype=np.float64, order="F", copy=True)
    Q, Y = _f(Q), _f(Y)
    m, q = X.shape
    p = Q.shape[1]
    lib().orc_sub_prod(_p(X), m, _p(Q), m, _p(Y), p, m, p, q)
    return X


def factor(A, b: int, algo: str | int):
    """Run one of the paper's algorithms on a copy of A.

    Returns (Q, R, info_dict). On breakdown Q and R are None and info holds
    (pass, panel, stage, pivot, pivot_value).
    """
    algo_id = ALGOS[algo] if isinstance(algo, str) else int(algo)
    Q = np.array(A, dtype=np.float64, order="F", copy=True)
    m, n = Q.shape
    R = np.zeros((n, n), order="F")
    info = Info()
    rc = lib().orc_factor(_p(Q), m, m, n, int(b), algo_id, _p(R), n, ctypes.byref(info))
    d = info.as_dict()
    if rc != OK:
        return None, None, d
    return Q, R, d


def mcqr2gs_panel(Qprev, P, R_col=None):
    """Lines 6-8 of Alg. 8 plus the R bookkeeping (R-8) for one panel P (m x b) given the
    earlier panels' Q_{1:j-1} = Qprev (m x c0).  R_col (c0 x b) is the incoming R_{1:j-1,j}
    (zeros if None).  Returns (Q_j, R_{1:j-1,j}, R_jj, info)."""
    Qprev, P = _f(Qprev), _f(P)
    m, c0 = Qprev.shape
    b = P.shape[1]
    X = np.asfortranarray(np.hstack([Qprev, P]))
    n = c0 + b
    R = np.zeros((n, n), order="F")
    if R_col is not None:
        R[:c0, c0:] = R_col
    info = Info()
    rc = lib().orc_mcqr2gs_panel(_p(X), m, m, c0, b, _p(R), n, 2, ctypes.byref(info))
    d = info.as_dict()
    d["status"] = rc
    if rc != OK:
        return None, None, None, d
    return X[:, c0:], R[:c0, c0:].copy(), R[c0:, c0:].copy(), d


def set_adapt_tau(tau: float) -> None:
    """Threshold of the adaptive repetition rule (NEXT-f4, oracle.c mcqr2gs_adaptive)."""
    lib().orc_set_adapt_tau(float(tau))


def get_adapt_tau() -> float:
    return float(lib().orc_get_adapt_tau())


def adapt_skipped() -> int:
    """Panels whose CholeskyQR repetition the last adaptive factorisation skipped."""
    return int(lib().orc_adapt_skipped())


def diag_ratio(U) -> float:
    U = _f(U)
    return float(lib().orc_diag_ratio(_p(U), U.shape[0], U.shape[0]))


def kappa_f(U) -> float:
    """||U||_F ||U^{-1}||_F of an upper-triangular U (the adaptive rule's estimate)."""
    U = _f(U)
    return float(lib().orc_kappa_f(_p(U), U.shape[0], U.shape[0]))


def householder(A):
    A = _f(A)
    m, n = A.shape
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n), order="F")
    rc = lib().orc_householder(_p(A), m, m, n, _p(Q), m, _p(R), n)
    assert rc == OK
    return Q, R


def orthogonality(Q) -> float:
    """||Q^T Q - I||_F, un-normalised (divide by sqrt(n) for the paper's P:104 form)."""
    Q = _f(Q)
    m, n = Q.shape
    return float(lib().orc_orthogonality(_p(Q), m, m, n))


def residual(A, Q, R) -> float:
    """||A - Q R||_F / ||A||_F."""
    A, Q, R = _f(A), _f(Q), _f(R)
    m, n = A.shape
    return float(lib().orc_residual(_p(A), m, _p(Q), m, _p(R), n, m, n))
