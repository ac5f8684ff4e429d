"""Measurement harness shared by tests/ and bench.py (not part of the product path):
GPU-side accuracy metrics computed with plain torch ops."""
