"""Pins of the NEXT-2 oracle (area-integrated irradiance, Eq. 4 as written,
P:159–162 and P:248; reading Q23) — CPU only.

They tie `oracle.irradiance_area_*` to closed forms that do not depend on it:
the point-to-rectangle solid angle, Σ Ω = 4π inside a closed convex enclosure
(the flux of an isotropic lamp is P), the analytic flux through a partially
shadowed patch (convergence in the subdivision level), and the small-patch
limit (the centroid point model of a6).
"""
import math

import numpy as np
import pytest

from synth import configs, rooms, ward


def rect_solid_angle(a, b, h):
    """Solid angle of an a×b rectangle seen from a point at height h above one
    corner (standard closed form: atan(ab / (h √(a²+b²+h²))))."""
    return math.atan(a * b / (h * math.sqrt(a * a + b * b + h * h)))


def quad_scene(x0, x1, y0, y1, z=0.0, up=True):
    """Two triangles tiling [x0,x1]×[y0,y1] at height z, normal ±z."""
    V = np.array([[x0, y0, z], [x1, y0, z], [x1, y1, z], [x0, y1, z]], np.float32)
    F = np.array([[0, 1, 2], [0, 2, 3]] if up else [[0, 2, 1], [0, 3, 2]], np.int32)
    return V, F


def test_solid_angle_rectangle_closed_form(orc):
    """Van Oosterom–Strackee on the two triangles of a rectangle = the
    rectangle formula, for corner views at several aspect ratios/heights."""
    for a, b, h in ((1.0, 1.0, 1.0), (2.0, 0.5, 0.3), (0.1, 3.0, 2.0), (5.0, 5.0, 0.01)):
        p = [0.0, 0.0, h]
        A, B, C, D = [0, 0, 0], [a, 0, 0], [a, b, 0], [0, b, 0]
        om = orc.solid_angle(p, A, B, C) + orc.solid_angle(p, A, C, D)
        assert abs(om - rect_solid_angle(a, b, h)) < 1e-13
    # a point over the middle: 4 corner rectangles
    om = orc.solid_angle([0, 0, 1], [-1, -1, 0], [1, -1, 0], [1, 1, 0]) + \
        orc.solid_angle([0, 0, 1], [-1, -1, 0], [1, 1, 0], [-1, 1, 0])
    assert abs(om - 4 * rect_solid_angle(1, 1, 1)) < 1e-13
    # large solid angles (denominator < 0 branch): a hemisphere-like view
    om = orc.solid_angle([0, 0, 1e-3], [-100, -100, 0], [100, -100, 0], [100, 100, 0]) + \
        orc.solid_angle([0, 0, 1e-3], [-100, -100, 0], [100, 100, 0], [-100, 100, 0])
    assert abs(om - 2 * math.pi) < 1e-4


def test_rectangle_patch_flux_exact(orc):
    """Two unoccluded triangle patches tiling a rectangle: Σ|s|·A = P Ω/(4π)
    exactly, for every subdivision level (Σ_s Ω_s = Ω)."""
    V, F = quad_scene(0.0, 2.0, 0.0, 0.5)
    pat = orc.trimesh_patches(V, F)
    lam = np.array([[[0.0, 0.0, 0.3]]], np.float32)
    h = float(np.float32(0.3))
    for m in (0, 1, 3):
        r = orc.irradiance_area_matrix(pat, lam, m=m)
        flux = (pat["area"] * r["A"][:, 0]).sum()
        assert abs(flux - 80.0 / (4 * math.pi) * rect_solid_angle(2.0, 0.5, h)) < 1e-12 * flux
        assert (r["nvis"][:, 0] == 4 ** m).all()


@pytest.mark.parametrize("m", [0, 1, 2])
def test_closed_enclosure_total_flux_is_P(orc, m):
    """A lamp inside a closed convex enclosure: every patch is lit, Σ_i Ω_i = 4π,
    so Σ_i |s_i| A_ij = P exactly (to rounding) at any tessellation — unlike the
    centroid model's O(h²) error (test_oracle_pins)."""
    mm = ward._Mesh()
    mm.box((0, 0, 0), (1, 1, 1), 0.25, np.eye(4), inward=True)
    V, F = np.concatenate(mm.V).astype(np.float32), np.concatenate(mm.F).astype(np.int32)
    pat = orc.trimesh_patches(V, F)
    lam = np.array([[[0.5, 0.5, 0.5]], [[0.3, 0.6, 0.45]], [[0.9, 0.1, 0.2]]], np.float32)
    r = orc.irradiance_area_matrix(pat, lam, m=m)
    flux = (pat["area"][:, None] * r["A"]).sum(0)
    assert np.allclose(flux, 80.0, rtol=1e-12, atol=0)


def test_partial_shadow_converges_to_analytic(orc):
    """A 1×1 floor square (two patches) under a lamp at (0.5, 0.5, 2); an
    opaque plate at z = 1 covering x ≤ 0.6 casts its edge at x = 0.7 on the
    floor.  The visible region [0.7, 1]×[0, 1] has an exact solid angle; the
    area model converges to it as the subdivision level m grows."""
    Vf, Ff = quad_scene(0.0, 1.0, 0.0, 1.0)
    Vp, Fp = quad_scene(-3.0, 0.6, -3.0, 4.0, z=1.0, up=False)
    V = np.concatenate([Vf, Vp]).astype(np.float32)
    F = np.concatenate([Ff, Fp + 4]).astype(np.int32)
    pat = orc.trimesh_patches(V, F)
    lamp = np.float32([0.5, 0.5, 2.0])
    lam = lamp.reshape(1, 1, 3)
    x_s = 0.5 + (float(np.float32(0.6)) - 0.5) * 2.0      # shadow edge on the floor
    p = lamp.astype(np.float64)
    om = (orc.solid_angle(p, [x_s, 0, 0], [1, 0, 0], [1, 1, 0]) +
          orc.solid_angle(p, [x_s, 0, 0], [1, 1, 0], [x_s, 1, 0]))
    exact = 80.0 / (4 * math.pi) * om
    errs = []
    for m in (1, 2, 3, 4, 5):
        r = orc.irradiance_area_pairs(pat, lam, [0, 1], [0, 0], m=m)
        flux = (pat["area"][:2] * r["A"]).sum()
        errs.append(abs(flux - exact) / exact)
    assert errs[-1] < 0.02
    assert all(b < a for a, b in zip(errs[1:], errs[2:]))   # monotone once resolved
    assert errs[-1] < errs[0] / 4


def test_small_patch_limit_is_the_point_model(orc):
    """For patches small against the lamp distance the area model tends to the
    centroid point model of a6 (Eq. 7): the largest relative difference over a
    tessellated floor tile shrinks as O(h²) with the triangle size h."""
    lam = np.array([[[0.13, 0.07, 0.6]]], np.float32)
    errs = []
    for e in (0.1, 0.05, 0.025):
        mm = ward._Mesh()
        mm.box((0, 0, -0.01), (0.4, 0.4, 0.0), e, np.eye(4))
        V, F = np.concatenate(mm.V).astype(np.float32), np.concatenate(mm.F).astype(np.int32)
        pat = orc.trimesh_patches(V, F)
        top = np.nonzero(pat["normal"][:, 2] > 0.5)[0]      # the tile's upper face
        pt = orc.irradiance_pairs(pat, lam, top, np.zeros_like(top))
        ar = orc.irradiance_area_pairs(pat, lam, top, np.zeros_like(top), m=0)
        assert pt["vis"].all() and (ar["nvis"] == 1).all()
        errs.append(np.abs(ar["A"] / pt["A"] - 1).max())
    assert errs[-1] < 2e-3
    assert errs[0] / errs[1] > 3.0 and errs[1] / errs[2] > 3.0


def test_2d_and_3d_area_oracles_agree(orc):
    """On an extruded world the floorplan visibility and the triangle
    visibility give the same area-model matrix on non-degenerate pairs."""
    sc = dict(rooms.random_room(2), patch_res=0.25)
    pat = orc.extruded_patches(sc)
    v = orc.vantage(sc, configs.DISC_OPTS)
    lam = v["samples"][v["feasible"]][[3, 17, 40]]
    a2 = orc.irradiance_area_matrix(pat, lam, m=1, mode="2d")
    a3 = orc.irradiance_area_matrix(pat, lam, m=1, mode="3d")
    ok = ~(a2["deg"] | a3["deg"])
    assert ok.mean() > 0.95 and (a2["A"][ok] > 0).mean() > 0.05
    assert np.allclose(a2["A"][ok], a3["A"][ok], rtol=1e-12, atol=0)
