"""Seeded dwell-time / adjoint vectors for the fluence products.

No fluence arithmetic here: these are inputs t (dwell times, s) and y (row
weights) for μ = A·t and g = Aᵀ·y.
"""
from __future__ import annotations

import numpy as np


def sparse_plan(K: int, seed: int = 0, frac: float = 0.02, t_max: float = 1800.0) -> np.ndarray:
    """A sparse LP-like plan: nnz ≈ frac·K columns, Σt = T_max."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nnz = max(1, int(round(frac * K)))
    idx = rng.choice(K, size=nnz, replace=False)
    w = rng.uniform(0.5, 1.5, size=nnz)
    t = np.zeros(K, np.float64)
    t[idx] = w / w.sum() * t_max
    return t


def dense_iterate(K: int, seed: int = 0, t_max: float = 1800.0) -> np.ndarray:
    """Initial PDHG-style iterate t_k = (T_max/K)·U(0,2)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (t_max / K) * rng.uniform(0.0, 2.0, size=K)


def row_weights(N: int, seed: int = 0) -> np.ndarray:
    """Non-negative y for Aᵀ·y (benchmarks use y ≥ 0)."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    return rng.uniform(0.0, 1.0, size=N)
