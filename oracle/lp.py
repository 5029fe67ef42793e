"""Oracle for NEXT-1, the relaxed dwell-time LP (TEST INFRASTRUCTURE ONLY).

Only tests/ and tools that time the oracle may import this module; it never
imports the product package and the product never imports it.

The problem is Eq. 9 of the paper (§IV-D "Approximate
Two-Stage Optimization"):

    minimise   Σ_k t_k + Σ_i p_i σ_i
    subject to μ_i + σ_i ≥ μ_min      for every patch i   (μ = A·t, Eq. 5)
               Σ_k t_k ≤ T_max                              (time budget)
               t ≥ 0, σ ≥ 0

with A[i, k] = I_i(x_k) the irradiance matrix (W/m²), t in s, μ_min in J/m²
(280), p_i the infeasibility penalty ("p_i > ‖I‖_F").

Its dual (standard LP duality, y ≥ 0 the multipliers of the N coverage rows
and of the budget row):

    maximise   μ_min Σ_i y_i − T_max y_b
    subject to (Aᵀ y)_k − y_b ≤ 1  for every k,   y_i ≤ p_i,   y ≥ 0, y_b ≥ 0.

* `solve`     — the LP through scipy's HiGHS solver (a library primitive used
                as one step; SPEC's in-repo simplex is a CPU-program choice,
                S:394), returning primal t, σ, the duals and both objectives.
* `vertices`  — brute force for tiny instances: every basic solution (every
                choice of K+N linearly independent active constraints) is
                solved and the best feasible one kept.  This is the pin that
                does not depend on HiGHS ("vertex-enumeration oracle").
* `kkt`       — primal/dual residuals and the duality gap of any candidate,
                written from the two programs above.
"""
from __future__ import annotations

import itertools

import numpy as np


def _as_penalty(p, n):
    p = np.asarray(p, dtype=np.float64)
    return np.full(n, float(p)) if p.ndim == 0 else p.astype(np.float64)


def solve(A, mu_min, p, t_max):
    """Eq. 9 by HiGHS.  A: (N, K) array (rows = patches, columns = vantage
    configurations).  Returns dict(t, sigma, y, y_budget, obj, dual_obj, status)."""
    from scipy.optimize import linprog

    A = np.asarray(A, dtype=np.float64)
    n, k = A.shape
    p = _as_penalty(p, n)
    c = np.concatenate([np.ones(k), p])
    # A_ub x <= b_ub:  -(A t + σ) <= -μ_min ;  Σ t <= T_max
    a_ub = np.zeros((n + 1, k + n))
    a_ub[:n, :k] = -A
    a_ub[:n, k:] = -np.eye(n)
    a_ub[n, :k] = 1.0
    b_ub = np.concatenate([np.full(n, -float(mu_min)), [float(t_max)]])
    res = linprog(c, A_ub=a_ub, b_ub=b_ub, bounds=[(0, None)] * (k + n), method="highs")
    if res.status != 0:
        raise RuntimeError(f"HiGHS status {res.status}: {res.message}")
    y_all = -np.asarray(res.ineqlin.marginals)  # multipliers of the <= rows, sign-flipped to y >= 0
    y, yb = y_all[:n], y_all[n]
    return {"t": res.x[:k], "sigma": res.x[k:], "y": y, "y_budget": float(yb), "obj": float(res.fun),
            "dual_obj": float(mu_min * y.sum() - t_max * yb), "status": "optimal"}


def vertices(A, mu_min, p, t_max, tol=1e-9):
    """Brute-force optimum of Eq. 9 over all basic solutions (K + N <= ~8)."""
    A = np.asarray(A, dtype=np.float64)
    n, k = A.shape
    p = _as_penalty(p, n)
    nv = k + n
    # all constraints as G x >= h: coverage rows, budget row (-Σt >= -T_max), x >= 0
    G = np.zeros((n + 1 + nv, nv))
    h = np.zeros(n + 1 + nv)
    G[:n, :k] = A
    G[:n, k:] = np.eye(n)
    h[:n] = mu_min
    G[n, :k] = -1.0
    h[n] = -t_max
    G[n + 1:, :] = np.eye(nv)
    c = np.concatenate([np.ones(k), p])
    best, best_x = np.inf, None
    for rows in itertools.combinations(range(G.shape[0]), nv):
        M = G[list(rows)]
        if abs(np.linalg.det(M)) < 1e-12:
            continue
        x = np.linalg.solve(M, h[list(rows)])
        if np.all(G @ x - h >= -tol * (1.0 + np.abs(h))):
            v = float(c @ x)
            if v < best:
                best, best_x = v, x
    return {"obj": best, "t": best_x[:k], "sigma": best_x[k:]}


def kkt(A, mu_min, p, t_max, t, sigma, y, y_budget):
    """Residuals of a candidate (t, σ; y, y_b): absolute primal infeasibility
    (2-norm of the violated rows), dual infeasibility (2-norm of the violated
    reduced costs) and |primal − dual objective|, plus both objectives."""
    A = np.asarray(A, dtype=np.float64)
    n, k = A.shape
    p = _as_penalty(p, n)
    t, sigma, y = (np.asarray(v, dtype=np.float64) for v in (t, sigma, y))
    mu = A @ t
    rp = np.concatenate([np.maximum(0.0, mu_min - mu - sigma), [max(0.0, t.sum() - t_max)],
                         np.maximum(0.0, -t), np.maximum(0.0, -sigma)])
    rd = np.concatenate([np.maximum(0.0, A.T @ y - y_budget - 1.0), np.maximum(0.0, y - p),
                         np.maximum(0.0, -y), [max(0.0, -y_budget)]])
    po = float(t.sum() + p @ sigma)
    do = float(mu_min * y.sum() - t_max * y_budget)
    return {"primal_res": float(np.linalg.norm(rp)), "dual_res": float(np.linalg.norm(rd)),
            "gap": abs(po - do), "primal_obj": po, "dual_obj": do}
