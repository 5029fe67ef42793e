"""Pins of the NEXT-3 oracle: the paper's visibility-cube method
by brute force — CPU only.  Closed forms: the pixel solid angles tile the
sphere (each face 1/6 of it: the emission texture E sums to P);
a closed enclosure receives exactly P; a symmetric room under a
centred lamp receives symmetric flux; the cube estimate converges to the
exact area integral (NEXT-2) as the face resolution grows."""
import math

import numpy as np
import pytest

from synth import ward


def test_pixel_solid_angles_tile_the_sphere(orc):
    for R in (1, 2, 7, 64):
        tot = sum(orc.pixel_solid_angle(R, a, b) for a in range(R) for b in range(R))
        assert abs(tot - 2 * math.pi / 3) < 1e-12          # one face = 4π/6
    # a corner pixel is smaller than a centre pixel (cos³ falloff)
    assert orc.pixel_solid_angle(16, 0, 0) < orc.pixel_solid_angle(16, 8, 8)
    # centre pixel ≈ (2/R)² at distance 1
    R = 256
    assert abs(orc.pixel_solid_angle(R, R // 2, R // 2) / (2.0 / R) ** 2 - 1) < 1e-4


def cube_room(e):
    m = ward._Mesh()
    m.box((0, 0, 0), (1, 1, 1), e, np.eye(4), inward=True)
    return orc_patches(np.concatenate(m.V).astype(np.float32), np.concatenate(m.F).astype(np.int32))


def orc_patches(V, F):
    from oracle import oracle as O
    return O.trimesh_patches(V, F)


def test_closed_enclosure_receives_P(orc):
    """Every pixel ray of a lamp inside a closed room hits a front face, so
    Σ_i F_i = P exactly (to rounding), at any face resolution."""
    pat = cube_room(0.25)
    lam = np.array([[[0.5, 0.5, 0.5]], [[0.31, 0.62, 0.47]]], np.float32)
    for R in (4, 16):
        r = orc.cubemap(pat, lam, R=R)
        assert np.allclose(r["F"].sum(0), 80.0, rtol=1e-12, atol=0)


def test_centred_lamp_one_face_per_wall(orc):
    """Lamp at the centre of the unit cube room, cube faces aligned with the
    walls: each wall's pixels are exactly one cube face, so every wall
    receives P/6 (the emission texture's face sum)."""
    pat = cube_room(0.25)
    lam = np.array([[[0.5, 0.5, 0.5]]], np.float32)
    r = orc.cubemap(pat, lam, R=16)
    n = pat["normal"]
    for ax in range(3):
        for s in (-1, 1):
            wall = np.abs(n[:, ax] - s) < 1e-6
            assert abs(r["F"][wall, 0].sum() - 80.0 / 6) < 1e-9


def test_cube_converges_to_the_area_integral(orc):
    """The cube estimate of the mean irradiance tends to the exact area
    integral of NEXT-2 (unoccluded room: exact solid angles) as the face
    resolution R grows: the error is pixel quantisation at triangle edges,
    O(1/R)."""
    pat = cube_room(0.5)
    lam = np.array([[[0.37, 0.55, 0.46]]], np.float32)
    exact = orc.irradiance_area_matrix(pat, lam, m=0)["A"][:, 0]
    errs = []
    for R in (24, 48, 96):
        cube = orc.cubemap(pat, lam, R=R)["A"][:, 0]
        errs.append(np.mean(np.abs(cube - exact) / exact))
        assert abs((pat["area"] * cube).sum() - (pat["area"] * exact).sum()) < 1e-9   # both = P
    assert errs[2] < 0.02
    assert errs[0] / errs[1] > 1.5 and errs[1] / errs[2] > 1.5


def test_occluded_patch_gets_nothing(orc):
    """A patch hidden behind a plate receives no pixel (P:246 nearest surface)."""
    V = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                  [-1, -1, 1], [2, -1, 1], [2, 2, 1], [-1, 2, 1]], np.float32)
    F = np.array([[0, 1, 2], [0, 2, 3], [4, 5, 6], [4, 6, 7]], np.int32)   # plate faces up, to the lamp
    pat = orc_patches(V, F)
    lam = np.array([[[0.5, 0.5, 2.0]]], np.float32)
    r = orc.cubemap(pat, lam, R=16, hits=True)
    assert r["F"][0, 0] == 0 and r["F"][1, 0] == 0          # the floor is shadowed
    assert r["F"][2:, 0].sum() > 0                            # the plate's top is lit
