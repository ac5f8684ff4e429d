"""Accuracy metrics of a computed factorisation on the GPU, for sizes the CPU
oracle's double-double metrics cannot reach in seconds.

Q^T Q and A - QR are accumulated in fixed 8192-row chunks (cuBLAS FP64 inside a chunk)
and the chunk results are combined by a pairwise tree, so the verifier's own error stays
at a few u per entry -- far below the 1e-13 / 1e-14 gates (a single K = 2^22 GEMM would
not be: sequential accumulation over m rows leaves ~u sqrt(m) per diagonal entry).
Multi-rank: the per-rank Gram / residual sums are all-reduced over torch.distributed.
"""
from __future__ import annotations

import math

import torch

CHUNK = 8192


def _pairwise(parts):
    while len(parts) > 1:
        nxt = [parts[i] + parts[i + 1] for i in range(0, len(parts) - 1, 2)]
        if len(parts) % 2:
            nxt.append(parts[-1])
        parts = nxt
    return parts[0]


class _Tree:
    """Streaming pairwise sum (binary counter) with O(log N) live partials."""

    def __init__(self):
        self.stack = []  # (level, tensor)

    def add(self, t):
        lvl = 0
        while self.stack and self.stack[-1][0] == lvl:
            _, s = self.stack.pop()
            t = s + t
            lvl += 1
        self.stack.append((lvl, t))

    def total(self):
        return _pairwise([t for _, t in self.stack])


def local_gram(Q, chunk: int = CHUNK):
    m, n = Q.shape
    tree = _Tree()
    if m == 0:
        return torch.zeros((n, n), dtype=torch.float64, device=Q.device)
    for r0 in range(0, m, chunk):
        Qc = Q[r0:r0 + chunk]
        tree.add(Qc.T @ Qc)
    return tree.total()


def orthogonality(Q, group=None, chunk: int = CHUNK) -> float:
    """||Q^T Q - I||_F (un-normalised; divide by sqrt(n) for P:104's form)."""
    G = local_gram(Q, chunk)
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(G, group=group)
    n = Q.shape[1]
    E = G - torch.eye(n, dtype=torch.float64, device=Q.device)
    return float(torch.linalg.norm(E))


def residual(A0, Q, R, group=None, chunk: int = CHUNK) -> float:
    """||A0 - Q R||_F / ||A0||_F."""
    m = A0.shape[0]
    num, den = _Tree(), _Tree()
    Ru = torch.triu(R)
    for r0 in range(0, m, chunk):
        a = A0[r0:r0 + chunk]
        d = a - Q[r0:r0 + chunk] @ Ru
        num.add((d * d).sum().reshape(1))
        den.add((a * a).sum().reshape(1))
    z = torch.zeros(1, dtype=torch.float64, device=A0.device)
    nn = num.total() if num.stack else z
    dd = den.total() if den.stack else z
    v = torch.cat([nn, dd])
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(v, group=group)
    return math.sqrt(float(v[0]) / float(v[1]))
