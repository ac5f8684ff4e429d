"""Seeded generators for the paper's ill-conditioned test matrices.

Shared by the oracle tests and the CUDA tests/bench; contains no CholeskyQR arithmetic.
numpy.linalg.qr / torch.linalg.qr (LAPACK / cuSOLVER Householder) are used here only
to draw Haar-orthonormal factors, as the paper draws them from an SVD.
"""
from __future__ import annotations

import math

import numpy as np

DEFAULT_CHUNK = 65536


def chunk_rows(m: int, chunk: int = DEFAULT_CHUNK) -> int:
    """Row-chunk size c used for U: c = min(m, chunk); must divide m."""
    c = min(m, chunk)
    if m % c != 0:
        raise ValueError(f"m={m} must be a multiple of the chunk size {c}")
    return c


def spectrum(n: int, kappa: float) -> np.ndarray:
    """sigma_i = kappa^{-(i-1)/(n-1)}, i = 1..n  ((1, s^{1/(n-1)}, ..., s) with s = 1/kappa)."""
    if n == 1:
        return np.ones(1)
    e = np.arange(n, dtype=np.float64) / (n - 1)
    return np.power(float(kappa), -e)


def _rng(seed: int, *stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed) & 0xFFFFFFFF, *stream])))


def _signed_q(G: np.ndarray) -> np.ndarray:
    Q, R = np.linalg.qr(G)
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return Q * s


_STREAM_V, _STREAM_U = 1, 2


def right_factor(n: int, kappa: float, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """(sigma, V): the planted spectrum and the n x n orthogonal right factor."""
    V = _signed_q(_rng(seed, _STREAM_V).standard_normal((n, n)))
    return spectrum(n, kappa), V


def generate_np(m: int, n: int, kappa: float, seed: int = 0, chunk: int = DEFAULT_CHUNK):
    """Global m x n test matrix as a Fortran-ordered float64 numpy array.

    Returns (A, sigma, V). Deterministic in (m, n, kappa, seed, chunk).
    """
    if m < n:
        raise ValueError("need m >= n")
    c = chunk_rows(m, chunk)
    if c < n:
        raise ValueError(f"chunk {c} must be >= n={n}")
    sigma, V = right_factor(n, kappa, seed)
    B = sigma[:, None] * V.T  # Sigma V^T
    A = np.empty((m, n), order="F")
    scale = 1.0 / math.sqrt(m // c)
    for t in range(m // c):
        Ut = _signed_q(_rng(seed, _STREAM_U, t).standard_normal((c, n)))
        if scale != 1.0:
            Ut = Ut * scale
        A[t * c:(t + 1) * c, :] = Ut @ B
    return A, sigma, V


def generate_torch(out, m_global: int, row0: int, n: int, kappa: float, seed: int = 0,
                   chunk: int = DEFAULT_CHUNK):
    """Fill `out` (a CUDA float64 view of shape (m_local, n), column-major strides (1, lda))
    with rows [row0, row0 + m_local) of the global test matrix, generated on the device.

    Same recipe as generate_np (sigma and V are drawn on the host with numpy, so they are
    bit-identical on every rank); the Gaussian chunks of U are drawn with torch's CUDA
    generator seeded per (seed, chunk index), so the matrix is independent of the number
    of ranks but not bit-identical to generate_np. Used for sizes the oracle cannot run.
    """
    import torch

    m_local = out.shape[0]
    c = chunk_rows(m_global, chunk)
    if row0 % c or m_local % c:
        raise ValueError("rank row range must be aligned to the U chunk size")
    sigma, V = right_factor(n, kappa, seed)
    B = torch.from_numpy(np.ascontiguousarray(sigma[:, None] * V.T)).to(out.device)
    scale = 1.0 / math.sqrt(m_global // c)
    g = torch.Generator(device=out.device)
    for t in range(row0 // c, (row0 + m_local) // c):
        g.manual_seed((int(seed) * 1_000_003 + t * 7919 + 17) & 0x7FFFFFFFFFFFFFFF)
        G = torch.randn((c, n), generator=g, dtype=torch.float64, device=out.device)
        Q, R = torch.linalg.qr(G)
        s = torch.sign(torch.diagonal(R))
        s[s == 0] = 1.0
        Q = Q * (s * scale)
        r = t * c - row0
        out[r:r + c, :].copy_(Q @ B)
    return sigma, V


def identity_scaled(m: int, n: int, scale: float = 1.0) -> np.ndarray:
    """m x n matrix with orthonormal columns (first n rows = I) times `scale`."""
    A = np.zeros((m, n), order="F")
    A[np.arange(n), np.arange(n)] = scale
    return A


def integer_matrix(m: int, n: int, seed: int = 0, lo: int = -3, hi: int = 3) -> np.ndarray:
    """Small-integer entries in [lo, hi]: every product and partial sum of a Gram or
    projection over m <= 2^40 rows is an exact integer below 2^53 (exact-arithmetic pin)."""
    return np.asfortranarray(_rng(seed, 99).integers(lo, hi + 1, size=(m, n)).astype(np.float64))


def generate_panel_conditioned_np(m: int, n: int, b: int, panel_kappas, seed: int = 0):
    """m x n matrix whose panels (b columns each) are mutually orthogonal in exact arithmetic,
    panel j having its own planted condition number panel_kappas[j]:
        A = U blockdiag(Sigma_1 V_1^T, ..., Sigma_k V_k^T),  U^T U = I (m x n, Haar),
    Sigma_j = spectrum(b, panel_kappas[j]), V_j Haar b x b.  Used to make the rounding-level
    terms of the mCQR2GS R assembly (R-8) large: after the line-3 projection panel j keeps a
    component ~u along Q_{1:j-1}, which the first CQR's U1^{-1} amplifies by kappa_j.
    Returns (A, [sigma_j]).  Contains no CholeskyQR arithmetic (numpy QR draws Haar factors)."""
    k = n // b
    if k * b != n or len(panel_kappas) != k:
        raise ValueError("need n = k b and one kappa per panel")
    U = _signed_q(_rng(seed, 7, 1).standard_normal((m, n)))
    B = np.zeros((n, n))
    sig = []
    for j, kap in enumerate(panel_kappas):
        s = spectrum(b, kap)
        Vj = _signed_q(_rng(seed, 7, 2 + j).standard_normal((b, b)))
        B[j * b:(j + 1) * b, j * b:(j + 1) * b] = s[:, None] * Vj.T
        sig.append(s)
    return np.asfortranarray(U @ B), sig


def orthonormal_np(m: int, n: int, seed: int = 0) -> np.ndarray:
    """m x n Haar matrix with orthonormal columns (kappa = 1)."""
    return np.asfortranarray(_signed_q(_rng(seed, 8).standard_normal((m, n))))
