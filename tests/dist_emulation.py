"""Per-rank (distributed) form of the paper's algorithms on CPU, for world_size > 1 tests of
the multi-rank host logic with the gloo backend.  TEST INFRASTRUCTURE.

Each rank owns a contiguous block of rows (1-D block-row layout, Fig. distA);
every cross-rank sum is one torch.distributed.all_reduce (the Allreduce of Alg. 2 l.4,
Alg. 7 l.3/l.8, Alg. 8 l.3/l.6/l.7/l.8); Cholesky and R assembly are redundant on every rank
(P:140).  The same placement and count of collectives as libtsqr's tsqr_factor.  Local
arithmetic is plain numpy FP64.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class Comm:
    def __init__(self, group=None):
        self.group = group
        self.calls = 0

    def allreduce(self, x: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t, group=self.group)
        self.calls += 1
        return t.numpy()


def _chol(W):
    U = np.linalg.cholesky(W).T  # LAPACK; upper factor W = U^T U
    return U


def cqr(X, comm: Comm):
    W = comm.allreduce(X.T @ X)
    W = np.triu(W) + np.triu(W, 1).T
    U = _chol(W)
    X[:] = np.linalg.solve(U.T, X.T).T  # X U^{-1}
    return U


def cqr2(X, comm):
    U1 = cqr(X, comm)
    U2 = cqr(X, comm)
    return np.triu(U2 @ U1)


def mcqr2gs(A, b, comm):
    """Alg. 8 per rank; returns the replicated R, A overwritten by Q."""
    m, n = A.shape
    k = n // b
    R = np.zeros((n, n))
    R[:b, :b] = cqr2(A[:, :b], comm)
    for j in range(1, k):
        p, c0 = (j - 1) * b, j * b
        Y = comm.allreduce(A[:, p:c0].T @ A[:, c0:])
        A[:, c0:] -= A[:, p:c0] @ Y
        R[p:c0, c0:] = Y
        U1 = cqr(A[:, c0:c0 + b], comm)
        C = comm.allreduce(A[:, :c0].T @ A[:, c0:c0 + b])
        A[:, c0:c0 + b] -= A[:, :c0] @ C
        U2 = cqr(A[:, c0:c0 + b], comm)
        R[c0:c0 + b, c0:c0 + b] = np.triu(U2 @ U1)
        R[:c0, c0:c0 + b] += C @ U1
    return R


def cqr2gs(A, b, comm):
    """Two passes of Alg. 7, R = R2 R1."""
    def cqrgs(X):
        m, n = X.shape
        Rp = np.zeros((n, n))
        for j in range(n // b):
            c0, c1 = j * b, (j + 1) * b
            Rp[c0:c1, c0:c1] = cqr(X[:, c0:c1], comm)
            if c1 < n:
                Y = comm.allreduce(X[:, c0:c1].T @ X[:, c1:])
                X[:, c1:] -= X[:, c0:c1] @ Y
                Rp[c0:c1, c1:] = Y
        return Rp
    R1 = cqrgs(A)
    R2 = cqrgs(A)
    return np.triu(R2 @ R1)
