"""Pins of the NEXT-4 static single-point baseline oracle (P:7, P:290, P:293;
S:538–541) — CPU only."""
import numpy as np
import pytest

from synth import configs


def test_hand_built_choice_and_dwell(orc):
    """Three configurations over four unit-area patches: the one seeing the
    most area wins; among equal areas the shorter dwell; dwell = μ_min / min A."""
    area = np.array([1.0, 1.0, 2.0, 1.0])
    A = np.array([[4.0, 0.0, 1.0],
                  [2.0, 8.0, 1.0],
                  [0.0, 1.0, 2.0],
                  [0.0, 0.5, 0.0]])
    r = orc.static_baseline(A, area, t_budget=100.0, mu_min=280.0)
    assert list(r["visible_area"]) == [2.0, 4.0, 4.0]
    assert r["column"] == 2 and abs(r["dwell_s"] - 280.0) < 1e-12      # tie: 280/1 < 280/0.5
    assert list(r["covered_at_budget"]) == [1.0, 1.0, 0.0]             # A·100 >= 280
    assert r["best_budget_column"] == 0


def test_empty_room_sees_everything(orc):
    """Convex room (C1): every wall patch is visible from every interior
    configuration, so the static lamp's visible area is the whole wall
    area and its coverage after its dwell is 100 %."""
    c = configs.c1()
    pat = orc.extruded_patches(c["scene"])
    v = orc.vantage(c["scene"], c["vantage"])
    A = orc.irradiance_matrix(pat, v["samples"][v["feasible"]], mode="2d")["A"]
    r = orc.static_baseline(A, pat["area"])
    assert np.allclose(r["visible_area"], pat["area"].sum(), rtol=1e-12)
    mu = A[:, r["column"]] * r["dwell_s"]
    assert (mu >= 280.0 * (1 - 1e-12)).all()


def test_static_never_beats_the_lp_plan(orc):
    """the LP plan covers at least as much as the best static lamp with
    the same budget, on the C3 worlds (oracle A, HiGHS)."""
    pytest.importorskip("scipy")
    from oracle import lp
    for seed in range(3):
        c = configs.c3(seed)
        pat = orc.extruded_patches(c["scene"])
        v = orc.vantage(c["scene"], c["vantage"])
        A = orc.irradiance_matrix(pat, v["samples"][v["feasible"]], mode="2d")["A"]
        r = orc.static_baseline(A, pat["area"], t_budget=configs.T_MAX)
        plan = lp.solve(A, configs.MU_MIN, 10 * np.linalg.norm(A), configs.T_MAX)
        mu = A @ plan["t"]
        covered = pat["area"][mu >= configs.MU_MIN * (1 - 1e-9)].sum()
        assert covered >= r["covered_at_budget"].max() - 1e-9
