"""Seeded synthetic test matrices (the paper's test-matrix suite).

This module holds NONE of the method's arithmetic: it only draws the inputs that
both the CPU oracle (tests) and the CUDA path (tests, bench) consume.

Recipe (normalised per DESIGN.md reading R-3b):
    A = U diag(sigma) V^T,  sigma_i = kappa^{-(i-1)/(n-1)}  (sigma_1 = 1, sigma_n = 1/kappa)
    V = sign-normalised Q factor of an n x n N(0,1) matrix (stream (seed, "V"))
    U = Q factors of c x n N(0,1) chunks (stream (seed, "U", t)), scaled by 1/sqrt(m/c),
        so U^T U = sum_t U_t^T U_t = I with no dependence on how rows are sharded.
For m <= chunk this is exactly "U and V ... obtained from the SVD of a random input
matrix" in distribution (Haar-distributed orthonormal factors).
"""
from .matrices import (spectrum, generate_np, generate_torch, right_factor, chunk_rows,
                       identity_scaled, integer_matrix, generate_panel_conditioned_np, orthonormal_np)

__all__ = ["spectrum", "generate_np", "generate_torch", "right_factor", "chunk_rows",
           "identity_scaled", "integer_matrix", "generate_panel_conditioned_np", "orthonormal_np"]
