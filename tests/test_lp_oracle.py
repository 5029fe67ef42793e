"""Pins of the LP oracle (NEXT-1, Eq. 9) — CPU only.

The oracle (`oracle/lp.py`) solves the relaxed dwell-time LP with HiGHS; these
tests tie it to things that do not depend on HiGHS: closed forms printed in
SPEC, a brute-force vertex enumeration on tiny instances
(S:376), LP duality, the paper's stated behaviour of the penalty,
and monotonicity.
"""
import numpy as np
import pytest

from conftest import golden
from synth import configs


@pytest.fixture(scope="module")
def lp():
    pytest.importorskip("scipy")
    from oracle import lp as m
    return m


def test_one_patch_dwell_printed(lp):
    """one patch, one vantage, I = 6.3662 W/m², μ_min = 280 → t = 43.98 s, σ = 0."""
    g = golden("point_source.txt")
    A = np.array([[g["E_at_1m_facing"]]])
    r = lp.solve(A, g["mu_min"], p=1e3, t_max=1e6)
    assert abs(r["t"][0] - g["dwell_at_6_3662"]) < 5e-3
    assert r["sigma"][0] == 0.0
    assert abs(r["obj"] - r["dual_obj"]) < 1e-9 * r["obj"]


def test_invisible_patch_takes_full_slack(lp):
    """S:384 / P:272: a patch seen from no vantage gets σ_i = μ_min; t is unchanged."""
    rng = np.random.default_rng(0)
    A = rng.uniform(0.5, 5.0, (5, 3))
    base = lp.solve(A, 280.0, p=100.0, t_max=1e6)
    A2 = np.vstack([A, np.zeros((1, 3))])
    r = lp.solve(A2, 280.0, p=100.0, t_max=1e6)
    assert abs(r["sigma"][-1] - 280.0) < 1e-9
    assert abs(r["obj"] - (base["obj"] + 100.0 * 280.0)) < 1e-7 * r["obj"]
    assert abs(r["t"].sum() - base["t"].sum()) < 1e-7 * base["t"].sum()


def test_closed_forms(lp):
    """Hand-solvable instances: (i) one patch, two vantages → all time on the
    brighter one, t = μ_min / max I; (ii) N patches each lit by its own
    vantage only → t_k = μ_min / A_kk; (iii) budget-bound single patch with
    p > 1/I → t = T_max and σ = μ_min − I·T_max."""
    r = lp.solve(np.array([[2.0, 5.0]]), 280.0, p=100.0, t_max=1e6)
    assert np.allclose(r["t"], [0.0, 56.0], atol=1e-9) and abs(r["obj"] - 56.0) < 1e-9
    d = np.array([1.0, 2.0, 4.0, 8.0])
    r = lp.solve(np.diag(d), 280.0, p=100.0, t_max=1e6)
    assert np.allclose(r["t"], 280.0 / d, rtol=1e-12) and not r["sigma"].any()
    r = lp.solve(np.array([[2.0]]), 280.0, p=10.0, t_max=100.0)
    assert abs(r["t"][0] - 100.0) < 1e-9 and abs(r["sigma"][0] - 80.0) < 1e-9
    assert abs(r["obj"] - (100.0 + 10.0 * 80.0)) < 1e-9


def _tiny(rng, n, k, budget_bound):
    A = rng.uniform(0.0, 6.0, (n, k)) * (rng.uniform(size=(n, k)) < 0.7)
    p = rng.uniform(0.5, 3.0, n)
    t_max = rng.uniform(20.0, 60.0) if budget_bound else 1e5
    return A, p, t_max


def test_vertex_enumeration_agrees(lp):
    """50 random instances (≤ 7 variables): HiGHS optimum = the best
    basic feasible solution by brute force, within 1e-6."""
    rng = np.random.default_rng(1)
    for it in range(50):
        n, k = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        A, p, t_max = _tiny(rng, n, k, budget_bound=it % 3 == 0)
        h = lp.solve(A, 280.0, p, t_max)
        v = lp.vertices(A, 280.0, p, t_max)
        assert abs(h["obj"] - v["obj"]) <= 1e-6 * max(1.0, v["obj"]), (it, h["obj"], v["obj"])


def test_duality_and_kkt_residuals(lp):
    """Strong duality at the HiGHS optimum, and `kkt` flags a perturbed
    candidate (so the residual code cannot pass everything)."""
    rng = np.random.default_rng(2)
    A = rng.uniform(0, 10, (40, 12)) * (rng.uniform(size=(40, 12)) < 0.5)
    r = lp.solve(A, 280.0, p=50.0, t_max=600.0)
    k = lp.kkt(A, 280.0, 50.0, 600.0, r["t"], r["sigma"], r["y"], r["y_budget"])
    scale = 1.0 + abs(k["primal_obj"])
    assert k["primal_res"] < 1e-7 * 280 and k["dual_res"] < 1e-7 * 50 and k["gap"] < 1e-7 * scale
    t_bad = r["t"].copy()
    t_bad[np.argmax(t_bad)] *= 0.5
    kb = lp.kkt(A, 280.0, 50.0, 600.0, t_bad, r["sigma"], r["y"], r["y_budget"])
    assert kb["primal_res"] > 1.0 and kb["gap"] > 1.0


def test_penalty_above_frobenius_gives_zero_slack(lp, orc):
    """with p_i > ‖I‖_F and a large T_max, every σ_i = 0 when all
    patches are visible (empty 5×5 room C1, oracle A), so coverage is 100 %."""
    c = configs.c1()
    pat = orc.extruded_patches(c["scene"])
    v = orc.vantage(c["scene"], c["vantage"])
    A = orc.irradiance_matrix(pat, v["samples"][v["feasible"]])["A"]  # (N, K)
    p = 10.0 * np.linalg.norm(A)
    r = lp.solve(A, 280.0, p, t_max=1e6)
    assert not r["sigma"].any()
    mu = A @ r["t"]
    assert (mu >= 280.0 * (1 - 1e-9)).all()
    assert r["t"].sum() < 1e6


def test_budget_binds_and_monotonicity(lp):
    """A tight T_max binds (Σt = T_max, some σ > 0); raising μ_min never lowers
    the optimum; adding a vantage column never raises it."""
    rng = np.random.default_rng(3)
    A = rng.uniform(0, 4, (30, 8)) * (rng.uniform(size=(30, 8)) < 0.6)
    A[:, 0] += 0.1  # every patch visible from some vantage
    r = lp.solve(A, 280.0, p=100.0, t_max=50.0)
    assert abs(r["t"].sum() - 50.0) < 1e-7 and r["sigma"].max() > 1.0
    objs = [lp.solve(A, m, p=100.0, t_max=1e4)["obj"] for m in (100.0, 200.0, 280.0, 400.0)]
    assert all(b >= a - 1e-9 for a, b in zip(objs, objs[1:]))
    base = lp.solve(A[:, :6], 280.0, p=100.0, t_max=1e4)["obj"]
    more = lp.solve(A, 280.0, p=100.0, t_max=1e4)["obj"]
    assert more <= base + 1e-9
