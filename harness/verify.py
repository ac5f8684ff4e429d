"""Accuracy metrics of a computed factorisation on the GPU, for sizes the CPU
oracle's double-double metrics cannot reach in seconds.  Measurement harness, not the
product path: plain torch ops (cuBLAS DGEMM on the GPU, any BLAS on the CPU).

Both metrics are computed ERROR-FREE up to the final rounding, so they agree with the
oracle's double-double `orc_orthogonality` / `orc_residual` to ~1e-30 (pinned by
tests/test_verify.py against the oracle) -- an fp64 GEMM alone would not do: Q^T Q - I and
A - QR are differences of O(1) quantities that cancel to O(u), so ordinary fp64
accumulation carries an error the size of the quantity measured (~3e-16 measured).

Method (Ozaki-style error-free splitting):
  * every operand is split into slices X = X_1 + X_2 + ... whose entries are integers of at
    most BITS bits times a power-of-two quantum that is common along the contraction's
    OUTER index (per column of Q for Q^T Q, per row of Q / per column of R for Q R);
  * a GEMM of two slices then sums products that are integer multiples of one common quantum
    with |integer| < 2^(2*BITS) each; with the contraction length <= 2^(53 - 2*BITS) every
    partial sum is an exactly representable fp64 number, so the GEMM is EXACT whatever its
    summation order (cuBLAS, MKL, blocked or not);
  * the exact slice products (and A, and the identity shares) are accumulated elementwise in
    double-double (TwoSum), and only the final (hi + lo) is rounded.
Rows are processed in chunks of CHUNK (Gram: the contraction over rows is chunked, so the
chunk length bounds it); Q^T Q - I is accumulated as sum_chunks (Q_c^T Q_c - (c/m) I) so the
double-double sums stay near 0.  Multi-rank: the per-rank double-double shares of
Q^T Q - I are all-gathered over torch.distributed and summed in rank order in double-double;
the residual's squared sums (relative accuracy suffices) are all-reduced in fp64.
"""
from __future__ import annotations

import math
from fractions import Fraction

import torch

CHUNK = 4096     # rows per Gram chunk: 2^12 terms of < 2^40 -> < 2^52, exact
BITS_G = 20      # slice width for the Gram (contraction over <= CHUNK rows)
RCHUNK = 8192    # rows per residual chunk (contraction over n <= 4096 = 2^12 columns)
BITS_R = 20
MAX_SLICES = 8   # 8 x 20 bits: anything left is below 2^-160 of the row / column maximum


def _split(X: torch.Tensor, dim: int, bits: int) -> list[torch.Tensor]:
    """X = sum of the returned slices (exactly, up to < 2^-(MAX_SLICES*bits) of the max along
    `dim`); slice s holds integers of <= bits bits times 2^(e - bits*(s+1)), e the exponent
    of the max |entry| along `dim` (common to all entries sharing the other index)."""
    amax = X.abs().amax(dim=dim, keepdim=True)
    e = torch.frexp(amax).exponent.to(torch.float64)  # amax < 2^e (0 for a zero line)
    out, r = [], X
    for s in range(MAX_SLICES):
        q = torch.exp2(e - bits * (s + 1))
        hi = torch.round(r / q) * q  # r / q is exact (power-of-two scaling); |.| <= 2^bits
        out.append(hi)
        r = r - hi                   # exact
        if not bool(torch.any(r != 0)):
            break
    return out


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


class _DD:
    """Elementwise double-double accumulator."""

    def __init__(self, hi):
        self.hi = hi.clone()
        self.lo = torch.zeros_like(hi)

    def add(self, x):
        s, e = _two_sum(self.hi, x)
        e = e + self.lo
        self.hi, self.lo = _two_sum(s, e)

    def value(self):
        return self.hi + self.lo


def _exact_gram_shift(Qc: torch.Tensor, share: tuple[float, float] | None, acc: _DD):
    """acc += Q_c^T Q_c - share*I exactly (share = (hi, lo) double-double)."""
    S = _split(Qc, 0, BITS_G)
    for i, a in enumerate(S):
        for j, b in enumerate(S):
            acc.add(a.T @ b)
    if share is not None:
        n = Qc.shape[1]
        eye = torch.eye(n, dtype=torch.float64, device=Qc.device)
        acc.add(-share[0] * eye)
        acc.add(-share[1] * eye)


def _dd_fraction(num: int, den: int) -> tuple[float, float]:
    f = Fraction(num, den)
    hi = float(f)
    return hi, float(f - Fraction(hi))


def local_gram(Q, chunk: int = CHUNK, m_global: int | None = None, dd: bool = False):
    """sum over row chunks of Q_c^T Q_c (exact up to the final rounding); with m_global, the
    rank's share of Q^T Q - I: sum of (Q_c^T Q_c - (c/m_global) I).  dd=True returns the
    unrounded double-double (hi, lo)."""
    m, n = Q.shape
    acc = _DD(torch.zeros((n, n), dtype=torch.float64, device=Q.device))
    chunk = min(chunk, CHUNK)
    for r0 in range(0, m, chunk):
        Qc = Q[r0:r0 + chunk]
        _exact_gram_shift(Qc, _dd_fraction(Qc.shape[0], m_global) if m_global else None, acc)
    return (acc.hi, acc.lo) if dd else acc.value()


def _comm_device(group, dev):
    """Tensors passed to torch.distributed collectives live where the group's backend wants them."""
    import torch.distributed as dist
    return dev if dist.get_backend(group) == "nccl" else torch.device("cpu")


def orthogonality(Q, group=None, chunk: int = CHUNK) -> float:
    """||Q^T Q - I||_F (un-normalised; divide by sqrt(n) for P:104's form)."""
    m = Q.shape[0]
    if group is not None:
        import torch.distributed as dist
        mt = torch.tensor([float(m)], dtype=torch.float64, device=_comm_device(group, Q.device))
        dist.all_reduce(mt, group=group)
        m = int(mt.item())
    n = Q.shape[1]
    if m == 0:
        return math.sqrt(n)
    hi, lo = local_gram(Q, chunk, m_global=m, dd=True)
    if group is None:
        E = hi + lo
    else:  # the rank shares are O(sqrt(m_r)/m), not small: gather them unrounded, sum in rank order
        import torch.distributed as dist
        w = dist.get_world_size(group)
        cd = _comm_device(group, Q.device)
        his = [torch.empty((n, n), dtype=torch.float64, device=cd) for _ in range(w)]
        los = [torch.empty((n, n), dtype=torch.float64, device=cd) for _ in range(w)]
        dist.all_gather(his, hi.to(cd).contiguous(), group=group)
        dist.all_gather(los, lo.to(cd).contiguous(), group=group)
        acc = _DD(torch.zeros((n, n), dtype=torch.float64, device=cd))
        for h, l in zip(his, los):
            acc.add(h)
            acc.add(l)
        E = acc.value()
    return float(torch.linalg.norm(E))


def residual(A0, Q, R, group=None, chunk: int = RCHUNK) -> float:
    """||A0 - Q R||_F / ||A0||_F, with R's upper triangle (A - QR formed exactly per entry, then
    rounded once; the squares are summed in fp64 -- relative accuracy is all that matters there)."""
    m, n = A0.shape
    Ru = torch.triu(R.to(A0.device))
    SR = _split(Ru, 0, BITS_R)  # per column of R
    num = torch.zeros((), dtype=torch.float64, device=A0.device)
    den = torch.zeros((), dtype=torch.float64, device=A0.device)
    for r0 in range(0, m, chunk):
        a = A0[r0:r0 + chunk]
        acc = _DD(a)
        for qs in _split(Q[r0:r0 + chunk], 1, BITS_R):  # per row of Q
            for rs in SR:
                acc.add(-(qs @ rs))
        d = acc.value()
        num = num + (d * d).sum()
        den = den + (a * a).sum()
    v = torch.stack([num, den])
    if group is not None:
        import torch.distributed as dist
        v = v.to(_comm_device(group, A0.device))
        dist.all_reduce(v, group=group)
    v = v.cpu()
    return math.sqrt(float(v[0]) / float(v[1])) if float(v[1]) > 0 else 0.0
