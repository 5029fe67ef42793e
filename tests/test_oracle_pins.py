"""Pins for the fp64 oracle against what the paper and mathematics fix
(closed forms, invariants, symmetries, hand-built occlusion, an independent
ray-marching check).  CPU only.

Each test states the passage it follows; the oracle is never compared with
itself.
"""
import math

import numpy as np
import pytest

from conftest import golden
from synth import configs, rooms, ward


# ---------------------------------------------------------------- helpers ---
def one_triangle_scene():
    """A single triangle in z=0 whose centroid is exactly the origin (binary
    fractions), normal +z."""
    s = 1.0 / 64
    V = np.array([[-s, -s, 0], [2 * s, -s, 0], [-s, 2 * s, 0]], np.float32)
    F = np.array([[0, 1, 2]], np.int32)
    return V, F


def cube_room(e):
    """Closed unit cube with inward normals (a convex enclosure), tessellated at e."""
    m = ward._Mesh()
    m.box((0, 0, 0), (1, 1, 1), e, np.eye(4), inward=True)
    return np.concatenate(m.V).astype(np.float32), np.concatenate(m.F).astype(np.int32)


def lamps_of(points):
    return np.asarray(points, np.float32).reshape(-1, 1, 3)


# ------------------------------------------------------ a6: closed forms ---
def test_point_source_closed_form_printed_values(orc):
    """6.3662 W/m² at 1 m, 1.59155 at 2 m, 0 at cosθ = 0 (P=80 W)."""
    g = golden("point_source.txt")
    V, F = one_triangle_scene()
    p = orc.trimesh_patches(V, F)
    assert p["centroid"].tolist() == [[0.0, 0.0, 0.0]]
    assert p["normal"].tolist() == [[0.0, 0.0, 1.0]]
    r = orc.irradiance_matrix(p, lamps_of([[0, 0, 1], [0, 0, 2], [0.5, 0, 0]]), P=g["P_watts"])
    A = r["A"][0]
    assert abs(A[0] - g["E_at_1m_facing"]) < g["print_tol"] * g["E_at_1m_facing"]
    assert abs(A[1] - g["E_at_2m_facing"]) < g["print_tol"] * g["E_at_2m_facing"]
    assert A[2] == g["E_cos_zero"]
    assert r["deg"][0, 2, 0]          # cosθ = 0 exactly is flagged degenerate (Q8)
    # inverse-square law: quarter at twice the distance
    assert abs(A[1] / A[0] - 0.25) < 1e-15


def test_back_face_and_cos_falloff(orc):
    """visible only if <y - x_k, n> > 0 (back faces give 0);
    Eq. 7 numerator <., n>/d: equal-distance lamps scale with cosθ."""
    V, F = one_triangle_scene()
    p = orc.trimesh_patches(V, F)
    pts = [[0, 0, 1], [0, 0, -1], [0.6, 0, 0.8], [0.8, 0, 0.6], [0, -0.28, 0.96]]
    r = orc.irradiance_matrix(p, lamps_of(pts))
    A = r["A"][0]
    assert A[1] == 0.0 and not r["vis"][0, 1, 0]
    lam = np.asarray(pts, np.float32).astype(np.float64)
    for j, cos in ((2, 0.8), (3, 0.6), (4, 0.96)):
        d = np.linalg.norm(lam[j])       # |lamp| = 1 up to fp32 rounding of the coordinates
        assert abs(d - 1) < 1e-7
        assert abs(A[j] / A[0] - cos) < 1e-6


def test_dwell_sanity(orc):
    """t = μ_min / I = 280 / 6.3662 = 43.98 s reaches μ_min exactly."""
    g = golden("point_source.txt")
    V, F = one_triangle_scene()
    p = orc.trimesh_patches(V, F)
    r = orc.irradiance_matrix(p, lamps_of([[0, 0, 1]]))
    t = np.array([g["mu_min"] / r["A"][0, 0]])
    assert abs(t[0] - g["dwell_at_6_3662"]) < 5e-3
    mu = orc.fluence(r["A"], t)
    cov = orc.coverage(mu * (1 + 1e-15), p["area"], g["mu_min"])
    assert cov[0] == cov[1]


def test_linearity_in_power_is_exact(orc):
    """doubling P doubles every entry exactly (power-of-two scaling)."""
    sc = rooms.random_room(3)
    p = orc.extruded_patches(sc)
    lam = lamps_of([[1.1, 2.3, 1.0], [3.2, 0.7, 1.0]])
    a1 = orc.irradiance_matrix(p, lam, P=80.0)["A"]
    a2 = orc.irradiance_matrix(p, lam, P=160.0)["A"]
    assert np.array_equal(a2, 2 * a1)


def test_flux_conservation_converges(orc):
    """Σ_i |s_i| A_ij -> P for a lamp inside a closed convex enclosure
    (each term is P·Ω_i/4π with ΣΩ = 4π; midpoint rule error O(h²)).
    Pins Eq. 7's 1/(4π d²)·cosθ, the areas and the normal signs together."""
    errs = []
    for e in (1 / 8, 1 / 16, 1 / 32):
        V, F = cube_room(e)
        p = orc.trimesh_patches(V, F)
        r = orc.irradiance_matrix(p, lamps_of([[0.5, 0.5, 0.5], [0.3, 0.6, 0.45]]))
        flux = (p["area"][:, None] * r["A"]).sum(0)
        assert r["vis"].all()            # convex: every front-facing pair visible
        errs.append(np.abs(flux / 80.0 - 1).max())
    assert errs[-1] < 2e-3
    assert errs[0] / errs[1] > 3.0 and errs[1] / errs[2] > 3.0   # O(h²)


# --------------------------------------------------- a1: patch attributes ---
def test_extruded_counts_and_areas(orc):
    """empty 5×5 room, h=2, res=0.125 -> 160 patches, area 40 m²;
    S:48/S:66: patch areas sum to the total wall area."""
    g = golden("counts.txt")
    p = orc.extruded_patches(rooms.empty_room())
    assert p["N"] == g["c1_patches"]
    assert abs(p["area"].sum() - g["c1_area"]) < 1e-12
    for seed in range(5):
        sc = rooms.random_room(seed)
        p = orc.extruded_patches(sc)
        per = 16.0
        for poly in sc["obstacles"]:
            q = poly.astype(np.float64)
            per += np.linalg.norm(np.roll(q, -1, 0) - q, axis=1).sum()
        assert abs(p["area"].sum() - per * 2.0) < 1e-9 * per * 2
        # equal-width patches, each no wider than res
        w = np.linalg.norm(p["seg"][:, 2:] - p["seg"][:, :2], axis=1)
        assert (w <= 0.125 + 1e-6).all()


def test_extruded_normals_face_free_space(orc):
    """Q2/Q14: boundary normals point into the room, obstacle normals out of the
    obstacle; the triangles' right-hand normals equal the patch normal."""
    sc = rooms.random_room(11)
    p = orc.extruded_patches(sc)
    c, n = p["centroid"].astype(np.float64), p["normal"].astype(np.float64)
    assert np.allclose(np.linalg.norm(n, axis=1), 1, atol=1e-7)
    nb = 4 * 32  # 4 boundary walls of 4 m at 0.125 m
    probe = c + 0.01 * n
    assert ((probe[:nb, :2] > 0) & (probe[:nb, :2] < 4)).all()
    back = c - 0.01 * n
    assert (((back[:nb, :2] < 0) | (back[:nb, :2] > 4)).any(1)).all()


def test_extruded_normals_face_free_space_pip(orc):
    """Same as above with an explicit point-in-polygon check on obstacles."""
    sc = rooms.random_room(11)
    p = orc.extruded_patches(sc)
    c, n = p["centroid"].astype(np.float64), p["normal"].astype(np.float64)
    i = 4 * 32
    for poly in sc["obstacles"]:
        q = poly.astype(np.float64)
        nseg = 0
        for k in range(len(q)):
            L = np.linalg.norm(q[(k + 1) % len(q)] - q[k])
            nseg += math.ceil(L / 0.125)
        for r in range(i, i + nseg):
            out = c[r, :2] + 1e-3 * n[r, :2]
            inn = c[r, :2] - 1e-3 * n[r, :2]
            assert not _pip(out, q) and _pip(inn, q)
        i += nseg
    tri = p["tri"].reshape(-1, 3, 3).astype(np.float64)
    tn = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
    tn /= np.linalg.norm(tn, axis=1)[:, None]
    assert np.allclose(tn, np.repeat(n, 2, 0), atol=1e-6)


def _pip(pt, poly):
    x, y = pt
    inside = False
    for k in range(len(poly)):
        (ax, ay), (bx, by) = poly[k], poly[(k + 1) % len(poly)]
        if (ay > y) != (by > y) and x < ax + (y - ay) * (bx - ax) / (by - ay):
            inside = not inside
    return inside


def test_trimesh_patches_closed_solids(orc):
    """Divergence theorem: (1/3)Σ|s_i|(c_i·n_i) = volume for each closed,
    outward-wound solid, and minus the room volume for the inward shell —
    pins the centroid, normal and area formulas of a1."""
    w = ward.ward(seed=0, n_bays=1, e=0.25)
    p = orc.trimesh_patches(w["vertices"], w["tris"])
    c = p["centroid"].astype(np.float64)
    n = p["normal"].astype(np.float64)
    flux = p["area"] * (c * n).sum(1) / 3.0
    vol = np.bincount(w["solid"], weights=flux)
    L = 10.0 / 3.0
    assert abs(vol[0] + L * 7.0 * 3.0) < 1e-4 * L * 21   # shell: inward normals
    assert (vol[1:] > 0).all()
    # bed frame 0.9 m x 2.0 m, its height jittered by the generator (yaw leaves z alone)
    zf = w["vertices"][np.unique(w["tris"][w["solid"] == 1]), 2].astype(np.float64)
    assert abs(zf.max() - zf.min() - 0.5) < 0.5 * 0.016
    assert abs(vol[1] - 0.9 * 2.0 * (zf.max() - zf.min())) < 1e-4   # bed frame volume


def test_trimesh_rejects_degenerate(orc):
    V = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], np.float32)
    with pytest.raises(ValueError):
        orc.trimesh_patches(V, np.array([[0, 1, 2]], np.int32))


# ------------------------------------------------------------- a5: occlusion ---
def test_empty_room_all_visible_and_d4_symmetry(orc):
    """convex room -> every front-facing pair visible; the empty
    5×5 room's A is invariant under its 8 symmetries (BASELINE north_star)."""
    c = configs.c1()
    p = orc.extruded_patches(c["scene"])
    v = orc.vantage(c["scene"], c["vantage"])
    lam = v["samples"][v["feasible"]]
    r = orc.irradiance_matrix(p, lam)
    assert r["vis"].all() and not r["deg"].any()
    A = r["A"]
    cen = p["centroid"][:, :2].astype(np.float64) - 2.5
    lxy = lam[:, 0, :2].astype(np.float64) - 2.5
    for (a, b, cc, d) in ((0, -1, 1, 0), (-1, 0, 0, -1), (0, 1, -1, 0), (1, 0, 0, -1),
                          (-1, 0, 0, 1), (0, 1, 1, 0), (0, -1, -1, 0)):
        M = np.array([[a, b], [cc, d]], float)
        sp = _match(cen @ M.T, cen)
        sl = _match(lxy @ M.T, lxy)
        assert np.allclose(A[np.ix_(sp, sl)], A, rtol=1e-13, atol=0)


def _match(X, Y):
    idx = np.empty(len(X), int)
    for k, x in enumerate(X):
        d = np.abs(Y - x).sum(1)
        idx[k] = int(np.argmin(d))
        assert d[idx[k]] < 1e-9
    return idx


def test_box_occludes(orc):
    """a box between light and patch -> not visible; removing the box
    restores Eq. 7's value (monotonicity)."""
    sc = rooms.box_room()
    p = orc.extruded_patches(sc)
    p0 = orc.extruded_patches(rooms.empty_room(4.0, 2.0, 0.25))
    lam = lamps_of([[2.0, 0.5, 1.0]])
    # patch on the far wall (y = 4) straight behind the box
    far = [i for i in range(p["N"]) if abs(p["centroid"][i, 1] - 4) < 1e-6 and abs(p["centroid"][i, 0] - 2.125) < 1e-6]
    far0 = [i for i in range(p0["N"]) if abs(p0["centroid"][i, 1] - 4) < 1e-6 and abs(p0["centroid"][i, 0] - 2.125) < 1e-6]
    assert len(far) == 1 and len(far0) == 1
    r = orc.irradiance_pairs(p, lam, far, [0])
    r0 = orc.irradiance_pairs(p0, lam, far0, [0])
    assert r["A"][0] == 0.0 and not r["vis"][0, 0] and not r["deg"][0, 0]
    assert r0["A"][0] > 0 and r0["vis"][0, 0]
    # monotonicity over the whole matrix: the box only removes light
    lam2 = lamps_of([[0.5, 0.5, 1.0], [3.5, 3.3, 1.0], [2.0, 0.4, 1.0]])
    A = orc.irradiance_matrix(p, lam2)["A"]
    A0 = orc.irradiance_matrix(p0, lam2)["A"]
    wall = np.array([_find(p0, c) for c in p["centroid"][:p0["N"]]])
    assert (A[:p0["N"]] <= A0[wall] + 1e-15).all()
    assert (A[:p0["N"]] < A0[wall]).any()


def _find(p, c):
    d = np.abs(p["centroid"] - c).sum(1)
    k = int(np.argmin(d))
    assert d[k] < 1e-6
    return k


def test_partitioned_room_sees_nothing_across(orc):
    """lights on one side of a full partition see no patches on the other
    (rays whose crossing of the divider is away from the 2 cm end slits)."""
    sc = rooms.partitioned_room()
    p = orc.extruded_patches(sc)
    lam = lamps_of([[x, y, 1.0] for x in (0.5, 1.7, 3.3) for y in (0.4, 1.2)])
    A = orc.irradiance_matrix(p, lam)["A"]
    c = p["centroid"].astype(np.float64)
    for j, L in enumerate(lam[:, 0].astype(np.float64)):
        for i in range(p["N"]):
            if c[i, 1] > 2.1:
                tc = (2.0 - L[1]) / (c[i, 1] - L[1])
                xc = L[0] + tc * (c[i, 0] - L[0])
                if 0.1 < xc < 3.9:
                    assert A[i, j] == 0.0


def test_2d_and_3d_oracles_agree(orc):
    """Independent floorplan oracle (P:292 midpoint visibility graph) vs the 3D
    triangle oracle on extruded worlds: identical visibility on every pair that
    neither flags as degenerate, identical entries where visible."""
    for seed in (0, 5, 17):
        sc = rooms.random_room(seed)
        p = orc.extruded_patches(sc)
        v = orc.vantage(sc, configs.DISC_OPTS)
        lam = v["samples"][v["feasible"]][::3]
        r3 = orc.irradiance_matrix(p, lam, mode="3d")
        r2 = orc.irradiance_matrix(p, lam, mode="2d")
        ok = ~(r3["deg"] | r2["deg"])
        assert ok.mean() > 0.999
        assert np.array_equal(r3["vis"][ok], r2["vis"][ok])
        both = ok[..., 0] & r3["vis"][..., 0]
        assert np.array_equal(r3["A"][both], r2["A"][both])
        assert 0.05 < r3["vis"].mean() < 0.95


def test_ray_marching_agreement(orc):
    """agreement with a brute-force ray-marching check on random pairs
    (point-in-polygon sampling along the segment; independent of the
    segment-intersection algebra), excluding near-tangent pairs."""
    rng = np.random.default_rng(0)
    sc = rooms.random_room(2)
    p = orc.extruded_patches(sc)
    v = orc.vantage(sc, configs.DISC_OPTS)
    lam = v["samples"][v["feasible"]]
    pi = rng.integers(0, p["N"], 400)
    pj = rng.integers(0, len(lam), 400)
    r = orc.irradiance_pairs(p, lam, pi, pj, want_margin=True)
    polys = [q.astype(np.float64) for q in sc["obstacles"]]
    ts = np.linspace(0, 1, 4001)[1:-1]
    checked = 0
    for q in range(400):
        c = p["centroid"][pi[q]].astype(np.float64)
        n = p["normal"][pi[q]].astype(np.float64)
        L = lam[pj[q], 0].astype(np.float64)
        if (L - c) @ n <= 0:
            assert not r["vis"][q, 0]
            continue
        if abs(r["S"][q, 0]) < 2e-3:       # within marching resolution of tangency
            continue
        pts = L[None, :2] + ts[:, None] * (c[:2] - L[:2])[None, :]
        pts = pts[ts < 1 - 1e-3]           # stop short of the target's own wall
        hit = any(_pip_many(pts, poly).any() for poly in polys)
        assert hit == (not r["vis"][q, 0]), q
        checked += 1
    assert checked > 150


def _pip_many(pts, poly):
    x, y = pts[:, 0], pts[:, 1]
    inside = np.zeros(len(pts), bool)
    for k in range(len(poly)):
        (ax, ay), (bx, by) = poly[k], poly[(k + 1) % len(poly)]
        cond = (ay > y) != (by > y)
        with np.errstate(divide="ignore", invalid="ignore"):
            xi = ax + (y - ay) * (bx - ax) / (by - ay)
        inside ^= cond & (x < xi)
    return inside


def test_self_and_endpoint_cut(orc):
    """Q6/Q15: the target's own triangles never occlude; an occluder within
    0.1 mm of the target is ignored, one at 1 mm is not."""
    V, F = one_triangle_scene()
    s = 1.0 / 64
    for gap, blocked in ((5e-5, False), (1e-3, True)):
        V2 = np.concatenate([V, V + np.array([0, 0, gap], np.float32)])
        # the second triangle faces down (reversed winding) and covers the first
        F2 = np.array([[0, 1, 2], [3, 5, 4]], np.int32)
        p = orc.trimesh_patches(V2, F2)
        r = orc.irradiance_pairs(p, lamps_of([[0, 0, 1]]), [0], [0])
        assert r["vis"][0, 0] == (not blocked)
    del s


# --------------------------------------------------------------- a3: vantage ---
def test_vantage_grid_counts(orc):
    """Q9: cell-centred grid — 400 raw / 324 feasible in C1 (0.15 m dilated disc),
    64 at 0.5 m in a 4 m room, 13 440 raw Floatbot cells in the ward."""
    g = golden("counts.txt")
    v = orc.vantage(rooms.empty_room(), configs.DISC_OPTS)
    assert len(v["points"]) == g["c1_grid_raw"]
    assert v["feasible"].sum() == g["c1_grid_feasible"] and not v["ambiguous"].any()
    v = orc.vantage(rooms.random_room(0, n_obstacles=0), configs.DISC_OPTS_COARSE)
    assert len(v["points"]) == g["room4_grid05"] and v["feasible"].all()
    cand = orc.vantage_candidates(configs.c4_scene(), configs.FLOAT_OPTS)
    assert len(cand["points"]) == g["ward_float_raw"]


def test_vantage_obstacles_removed(orc):
    """an obstacle filling the room centre removes interior grid points;
    no feasible point lies inside an obstacle or closer than the clearance."""
    sc = rooms.box_room(box=(1.0, 1.0, 3.0, 3.0))
    v = orc.vantage(sc, configs.DISC_OPTS)
    P = v["points"][v["feasible"]]
    inside = (P[:, 0] > 1) & (P[:, 0] < 3) & (P[:, 1] > 1) & (P[:, 1] < 3)
    assert not inside.any()
    # 4 m room: 14×14 clear of the walls, minus 8×8 inside the box, minus 4×8 within 0.15 m of it
    assert v["feasible"].sum() == 196 - 64 - 32 and not v["ambiguous"].any()


def test_vantage_3d_free_space(orc):
    """Q20: points inside a closed solid are not free even when far from its
    faces; points in the room are free."""
    m = ward._Mesh()
    m.box((0, 0, 0), (4, 4, 3), 0.5, np.eye(4), inward=True)
    m.box((1, 1, 0), (3, 3, 2), 0.3, np.eye(4))
    V = np.concatenate(m.V).astype(np.float32)
    F = np.concatenate(m.F).astype(np.int32)
    sc = dict(vertices=V, tris=F)
    v = orc.vantage(sc, configs.vopts(configs.FLOAT3D, 0.5, 0.05))
    P = v["points"]
    inside = (P[:, 0] > 1) & (P[:, 0] < 3) & (P[:, 1] > 1) & (P[:, 1] < 3) & (P[:, 2] < 2)
    assert not (v["feasible"] & inside).any()
    assert v["feasible"][~inside].all()
    assert not v["ambiguous"].any()


# --------------------------------------------------------- a7/a8: fluence ---
def test_fluence_linearity_and_coverage(orc):
    """zero dwell -> coverage 0; doubling dwell doubles μ exactly."""
    rng = np.random.default_rng(1)
    A = rng.uniform(0, 5, (50, 7)).astype(np.float32)
    A[rng.uniform(size=A.shape) < 0.5] = 0
    t = rng.uniform(0, 100, 7)
    mu = orc.fluence(A, t)
    assert np.array_equal(orc.fluence(A, 2 * t), 2 * mu)
    area = rng.uniform(0.1, 1, 50)
    assert orc.coverage(np.zeros(50), area)[0] == 0.0
    cov = orc.coverage(mu, area, 280.0, rowsum=orc.fluence(A, np.ones(7)))
    assert cov[0] <= cov[2] <= cov[1]
    # brute-force sums
    assert abs(mu[3] - sum(float(A[3, k]) * t[k] for k in range(7))) < 1e-9 * abs(mu[3]) + 1e-300
    y = rng.uniform(0, 1, 50)
    g = orc.fluence_t(A, y)
    assert abs(g[2] - sum(float(A[i, 2]) * y[i] for i in range(50))) < 1e-12 * g[2]
