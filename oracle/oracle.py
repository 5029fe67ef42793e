"""Python face of the fp64 CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module.  It never imports the product
package `paper_2103_14137_b200` and the product never imports it.

* liboracle.so (uvd_oracle.c, plain C fp64, -ffp-contract=off) does rows a1,
  a3 (per-point feasibility), a4–a6 (brute force: every ray against every
  triangle) and the 2D floorplan oracle.
* This file adds the cell-centred vantage grid (a3, Q9), the Armbot reach proxy
  (Q12) and rows a7/a8 (Eq. 5 fluence and coverage) with numpy fp64.

Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; Q# = DESIGN.md readings.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "uvd_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

DISC2D, TOWER, FLOAT3D, ARM = 0, 1, 2, 3
DEG_BAND = 1e-6


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain IEEE fp64 semantics (no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-pthread", "-o", LIB, SRC, "-lm"]
        subprocess.check_call(cmd)
    return LIB


_lib = None
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.orc_default_threads.restype = C.c_int
        L.orc_extruded_count.restype = C.c_int64
        L.orc_extruded_count.argtypes = [_f32p, _f32p, _i32p, C.c_int, C.c_float]
        L.orc_extruded_patches.restype = None
        L.orc_extruded_patches.argtypes = [_f32p, C.c_float, _f32p, _i32p, C.c_int, C.c_float,
                                           _f32p, _f32p, _f32p, _f64p, _f32p, _i32p]
        L.orc_trimesh_patches.restype = C.c_int64
        L.orc_trimesh_patches.argtypes = [_f32p, C.c_int64, _i32p, C.c_int64, _f32p, _f32p, _f64p]
        irr = [_f32p, _i32p, C.c_int64, _f32p, _f32p, C.c_int64, _f32p, C.c_int64, C.c_int,
               C.c_double, _i64p, _i64p, C.c_int64, _f64p, _u8p, _u8p, _f64p, C.c_int, C.c_int]
        L.orc_irradiance_3d.restype = C.c_int
        L.orc_irradiance_3d.argtypes = irr
        L.orc_irradiance_2d.restype = C.c_int
        L.orc_irradiance_2d.argtypes = [_f32p, _f32p, _f32p, C.c_int64, _f32p, C.c_int64, C.c_int,
                                        C.c_double, _i64p, _i64p, C.c_int64, _f64p, _u8p, _u8p,
                                        _f64p, C.c_int, C.c_int]
        L.orc_vantage_eval_3d.restype = None
        L.orc_vantage_eval_3d.argtypes = [_f32p, C.c_int64, _f32p, C.c_int64, C.c_int, C.c_double,
                                          C.c_int, _u8p, _u8p, _f64p, C.c_int]
        L.orc_vantage_eval_2d.restype = None
        L.orc_vantage_eval_2d.argtypes = [_f32p, _f32p, _i32p, C.c_int, _f32p, C.c_int64,
                                          C.c_double, _u8p, _u8p]
        L.orc_irradiance_area.restype = C.c_int
        L.orc_irradiance_area.argtypes = [C.c_int, _f32p, _i32p, C.c_int64, _f32p, C.c_int64, _f32p, _i64p,
                                          _i32p, _f32p, _f32p, _f64p, _f32p, C.c_int, C.c_double, C.c_int,
                                          _i64p, _i64p, C.c_int64, _f64p, _u8p, _i32p, _i32p, C.c_int]
        L.orc_cubemap.restype = None
        L.orc_cubemap.argtypes = [_f32p, _i32p, C.c_int64, C.c_int64, _f32p, C.c_int, C.c_double, C.c_int,
                                  _i64p, C.c_int64, _f64p, C.c_void_p, C.c_void_p, _f64p, C.c_int]
        L.orc_pixel_solid_angle.restype = C.c_double
        L.orc_pixel_solid_angle.argtypes = [C.c_int, C.c_int, C.c_int]
        L.orc_solid_angle.restype = C.c_double
        L.orc_solid_angle.argtypes = [_f64p, _f64p, _f64p, _f64p]
        _lib = L
    return _lib


def default_threads() -> int:
    return int(lib().orc_default_threads())


# --------------------------------------------------------------------------- #
# a1 — patches                                                                 #
# --------------------------------------------------------------------------- #
def _polys(scene):
    obs = scene["obstacles"]
    poly_n = np.array([len(p) for p in obs], np.int32) if obs else np.zeros(1, np.int32)
    poly_xy = (np.concatenate([np.asarray(p, np.float32).reshape(-1, 2) for p in obs]).ravel()
               if obs else np.zeros(2, np.float32))
    return np.ascontiguousarray(poly_xy, np.float32), poly_n, len(obs)


def extruded_patches(scene: dict) -> dict:
    """Canonical 2.5D wall patches."""
    bounds = np.ascontiguousarray(scene["bounds"], np.float32)
    poly_xy, poly_n, n_poly = _polys(scene)
    res = float(scene["patch_res"])
    N = int(lib().orc_extruded_count(bounds, poly_xy, poly_n, n_poly, res))
    seg = np.zeros((N, 4), np.float32)
    cen = np.zeros((N, 3), np.float32)
    nrm = np.zeros((N, 3), np.float32)
    area = np.zeros(N, np.float64)
    tri = np.zeros((2 * N, 9), np.float32)
    tp = np.zeros(2 * N, np.int32)
    lib().orc_extruded_patches(bounds, float(scene["wall_height"]), poly_xy, poly_n, n_poly, res,
                               seg, cen, nrm, area, tri, tp)
    return dict(seg=seg, centroid=cen, normal=nrm, area=area, tri=tri, tri_patch=tp, N=N)


def trimesh_patches(V: np.ndarray, F: np.ndarray) -> dict:
    """Canonical 3D patches: patch i = triangle i."""
    V = np.ascontiguousarray(V, np.float32)
    F = np.ascontiguousarray(F, np.int32)
    nt = len(F)
    cen = np.zeros((nt, 3), np.float32)
    nrm = np.zeros((nt, 3), np.float32)
    area = np.zeros(nt, np.float64)
    bad = int(lib().orc_trimesh_patches(V, len(V), F, nt, cen, nrm, area))
    if bad >= 0:
        raise ValueError(f"zero-area triangle {bad} (S:32)")
    tri = np.ascontiguousarray(V[F].reshape(nt, 9))
    return dict(centroid=cen, normal=nrm, area=area, tri=tri,
                tri_patch=np.arange(nt, dtype=np.int32), N=nt)


def scene_patches(scene: dict) -> dict:
    if "vertices" in scene:
        return trimesh_patches(scene["vertices"], scene["tris"])
    return extruded_patches(scene)


# --------------------------------------------------------------------------- #
# a4–a6 — irradiance entries                                                   #
# --------------------------------------------------------------------------- #
def irradiance_pairs(patches: dict, lamps: np.ndarray, pi, pj, P: float = 80.0,
                     mode: str = "3d", early_exit: bool = True, n_threads: int = 0,
                     want_margin: bool = False) -> dict:
    """A[i_q, j_q] for each pair q, plus per-(pair, lamp sample) visibility,
    degeneracy flags (|S| < 1e-6 or |cosθ| < 1e-6, Q8) and optionally margins.

    lamps: (K, L, 3) float32.  mode "3d" = brute force against every triangle;
    "2d" = floorplan segment oracle (extruded worlds only)."""
    lamps = np.ascontiguousarray(lamps, np.float32)
    K, L = lamps.shape[0], lamps.shape[1]
    pi = np.ascontiguousarray(pi, np.int64)
    pj = np.ascontiguousarray(pj, np.int64)
    n = len(pi)
    A = np.zeros(n, np.float64)
    vis = np.zeros(n * L, np.uint8)
    deg = np.zeros(n * L, np.uint8)
    S = np.zeros(n * L, np.float64)
    if mode == "3d":
        rc = lib().orc_irradiance_3d(patches["tri"], patches["tri_patch"], len(patches["tri"]),
                                     patches["centroid"], patches["normal"], patches["N"],
                                     lamps.reshape(-1), K, L, P, pi, pj, n, A, vis, deg, S,
                                     int(early_exit and not want_margin), n_threads)
    else:
        rc = lib().orc_irradiance_2d(patches["seg"], patches["centroid"], patches["normal"],
                                     patches["N"], lamps.reshape(-1), K, L, P, pi, pj, n, A, vis,
                                     deg, S, int(early_exit and not want_margin), n_threads)
    if rc != 0:
        raise ArithmeticError("lamp–surface distance < 1e-9 m (S:160)")
    out = dict(A=A, vis=vis.reshape(n, L).astype(bool), deg=deg.reshape(n, L).astype(bool))
    if want_margin:
        out["S"] = S.reshape(n, L)
    return out


def irradiance_matrix(patches: dict, lamps: np.ndarray, P: float = 80.0, mode: str = "3d",
                      n_threads: int = 0) -> dict:
    """Full N×K matrix (small cases only): A[i, j], vis[i, j, l], deg[i, j, l]."""
    N, K = patches["N"], lamps.shape[0]
    ii, jj = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    r = irradiance_pairs(patches, lamps, ii.ravel(), jj.ravel(), P, mode, n_threads=n_threads)
    L = lamps.shape[1]
    return dict(A=r["A"].reshape(N, K), vis=r["vis"].reshape(N, K, L), deg=r["deg"].reshape(N, K, L))


def solid_angle(p, a, b, c) -> float:
    """Van Oosterom–Strackee solid angle of triangle abc seen from p (fp64)."""
    f = [np.ascontiguousarray(v, np.float64) for v in (p, a, b, c)]
    return float(lib().orc_solid_angle(*f))


def irradiance_area_pairs(patches: dict, lamps: np.ndarray, pi, pj, m: int = 1, P: float = 80.0,
                          mode: str = "3d", n_threads: int = 0) -> dict:
    """NEXT-2, Eq. 4 as written (reading Q23): mean irradiance
    over patch i from configuration j, each patch triangle split into 4^m
    sub-triangles (edge midpoints), solid angle per sub-triangle (Van
    Oosterom–Strackee), visibility of each sub-triangle's fp32 centroid."""
    lamps = np.ascontiguousarray(lamps, np.float32)
    K, L = lamps.shape[0], lamps.shape[1]
    pi = np.ascontiguousarray(pi, np.int64)
    pj = np.ascontiguousarray(pj, np.int64)
    n, N = len(pi), patches["N"]
    per = 2 if "seg" in patches else 1           # 2.5D: the wall quad's two triangles
    pfirst = np.arange(N, dtype=np.int64) * per
    pcount = np.full(N, per, np.int32)
    A = np.zeros(n, np.float64)
    deg = np.zeros(n, np.uint8)
    nvis = np.zeros(n, np.int32)
    nsub = np.zeros(n, np.int32)
    seg = patches.get("seg", np.zeros((1, 4), np.float32))
    rc = lib().orc_irradiance_area(0 if mode == "3d" else 1, patches["tri"], patches["tri_patch"],
                                   len(patches["tri"]), np.ascontiguousarray(seg, np.float32), len(seg),
                                   patches["tri"], pfirst, pcount, patches["centroid"], patches["normal"],
                                   patches["area"], lamps.reshape(-1), L, P, int(m), pi, pj, n, A, deg,
                                   nvis, nsub, n_threads)
    if rc != 0:
        raise ArithmeticError("lamp–surface distance < 1e-9 m (S:160)")
    return dict(A=A, deg=deg.astype(bool), nvis=nvis, nsub=nsub)


def irradiance_area_matrix(patches: dict, lamps: np.ndarray, m: int = 1, P: float = 80.0, mode: str = "3d",
                           n_threads: int = 0) -> dict:
    N, K = patches["N"], lamps.shape[0]
    ii, jj = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    r = irradiance_area_pairs(patches, lamps, ii.ravel(), jj.ravel(), m, P, mode, n_threads)
    return dict(A=r["A"].reshape(N, K), deg=r["deg"].reshape(N, K), nvis=r["nvis"].reshape(N, K))


# --------------------------------------------------------------------------- #
# a3 — vantage sampling                                                        #
# --------------------------------------------------------------------------- #
def grid_axis(lo: float, hi: float, rho: float) -> np.ndarray:
    """Cell-centred grid x = lo + (a + 1/2)·ρ, a = 0..floor((hi-lo)/ρ)-1 (Q9),
    computed in fp64 from the fp32 inputs and stored as fp32."""
    lo, hi, rho = float(np.float32(lo)), float(np.float32(hi)), float(np.float32(rho))
    n = int(np.floor((hi - lo) / rho))
    return (lo + (np.arange(n, dtype=np.float64) + 0.5) * rho).astype(np.float32)


def _mesh_bbox(scene):
    V = np.asarray(scene["vertices"], np.float32)
    return V.min(0), V.max(0)


def vantage_candidates(scene: dict, opts: dict) -> dict:
    """Raw grid candidates (x fastest, then y, then z) with their lamp sample points."""
    rho = opts["spacing"]
    if opts["robot"] == DISC2D:
        b = scene["bounds"]
        xs, ys = grid_axis(b[0], b[2], rho), grid_axis(b[1], b[3], rho)
        zs = np.array([opts["lamp_z"]], np.float32)
    else:
        lo, hi = _mesh_bbox(scene)
        xs, ys = grid_axis(lo[0], hi[0], rho), grid_axis(lo[1], hi[1], rho)
        if opts["robot"] == FLOAT3D:
            zs = grid_axis(lo[2], hi[2], rho)
        elif opts["robot"] == ARM:
            zs = grid_axis(opts["zmin"], opts["zmax"], rho)
        else:
            zs = np.array([0.0], np.float32)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1).astype(np.float32)
    if opts["robot"] == TOWER:   # cylinder samples z_l = z0 + (l + 1/2)·H/L (Q11)
        L = int(opts["lamp_samples"])
        z0, z1 = float(np.float32(opts["lamp_z0"])), float(np.float32(opts["lamp_z1"]))
        zl = (z0 + (np.arange(L) + 0.5) * (z1 - z0) / L).astype(np.float32)
        sub = np.repeat(pts[:, None, :], L, 1)
        sub[:, :, 2] = zl[None, :]
        return dict(points=pts, samples=np.ascontiguousarray(sub), L=L)
    return dict(points=pts, samples=pts[:, None, :].copy(), L=1)


def vantage(scene: dict, opts: dict, idx=None, n_threads: int = 0) -> dict:
    """Feasibility + ambiguity of every raw candidate (or of the subset `idx`).

    Returns dict(points (R,3), samples (R,L,3), feasible (R,), ambiguous (R,), idx)."""
    cand = vantage_candidates(scene, opts)
    idx = np.arange(len(cand["points"])) if idx is None else np.asarray(idx, np.int64)
    samples = np.ascontiguousarray(cand["samples"][idx])
    R = len(idx)
    feas = np.zeros(R, np.uint8)
    amb = np.zeros(R, np.uint8)
    if opts["robot"] == DISC2D:
        poly_xy, poly_n, n_poly = _polys(scene)
        lib().orc_vantage_eval_2d(np.ascontiguousarray(scene["bounds"], np.float32), poly_xy,
                                  poly_n, n_poly, np.ascontiguousarray(samples[:, 0, :]), R,
                                  float(opts["clearance"]), feas, amb)
    else:
        tri = np.ascontiguousarray(np.asarray(scene["vertices"], np.float32)[scene["tris"]].reshape(-1, 9))
        md = np.zeros(R, np.float64)
        lib().orc_vantage_eval_3d(tri, len(tri), samples.reshape(-1), R, samples.shape[1],
                                  float(opts["clearance"]), 1, feas, amb, md, n_threads)
        if opts["robot"] == ARM:
            reach_ok, reach_amb = arm_reach(scene, opts, samples[:, 0, :], tri, n_threads)
            feas &= reach_ok.astype(np.uint8)
            amb |= reach_amb.astype(np.uint8)
    return dict(points=cand["points"][idx], samples=samples, feasible=feas.astype(bool),
                ambiguous=amb.astype(bool), idx=idx)


def arm_bases(scene: dict, opts: dict, tri=None, n_threads: int = 0, near=None) -> dict:
    """Armbot base positions: floor grid at z = base_z, feasible iff clearance
    base_clearance from every triangle and in free space (Q12).  near: optional
    (R, 3) points; only bases within reach + 1e-3 m of one of them are
    evaluated (the others cannot decide the reach proxy for those points)."""
    lo, hi = _mesh_bbox(scene)
    rho = opts["spacing"]
    xs, ys = grid_axis(lo[0], hi[0], rho), grid_axis(lo[1], hi[1], rho)
    Y, X = np.meshgrid(ys, xs, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel(), np.full(X.size, np.float32(opts["base_z"]))], 1)
    pts = np.ascontiguousarray(pts, np.float32)
    if near is not None:
        lim = float(np.float32(opts["reach"])) + 1e-3
        Q = np.asarray(near, np.float64)
        keep = np.zeros(len(pts), bool)
        for s in range(0, len(Q), 256):
            d2 = ((Q[s:s + 256, None, :] - pts[None, :, :].astype(np.float64)) ** 2).sum(-1)
            keep |= (d2 <= lim * lim).any(0)
        pts = np.ascontiguousarray(pts[keep])
    if tri is None:
        tri = np.ascontiguousarray(np.asarray(scene["vertices"], np.float32)[scene["tris"]].reshape(-1, 9))
    R = len(pts)
    feas = np.zeros(R, np.uint8)
    amb = np.zeros(R, np.uint8)
    md = np.zeros(R, np.float64)
    lib().orc_vantage_eval_3d(tri, len(tri), pts.reshape(-1), R, 1, float(opts["base_clearance"]),
                              1, feas, amb, md, n_threads)
    return dict(points=pts, feasible=feas.astype(bool), ambiguous=amb.astype(bool))


def arm_reach(scene, opts, lamp_pts, tri=None, n_threads: int = 0):
    """Reach proxy (Q12): lamp p is reachable iff |p − b| ≤ reach (fp64) for some
    feasible base b.  Ambiguous if the decision depends on an ambiguous base or a
    distance within 1e-6 of the reach."""
    bases = arm_bases(scene, opts, tri, n_threads, near=lamp_pts)
    B = bases["points"].astype(np.float64)
    reach = float(np.float32(opts["reach"]))
    ok = np.zeros(len(lamp_pts), bool)
    amb = np.zeros(len(lamp_pts), bool)
    P = np.asarray(lamp_pts, np.float64)
    for s in range(0, len(P), 256):
        d = np.sqrt(((P[s:s + 256, None, :] - B[None, :, :]) ** 2).sum(-1))
        clear_in = (d <= reach) & bases["feasible"][None, :] & ~bases["ambiguous"][None, :]
        near = (np.abs(d - reach) < DEG_BAND) | ((d <= reach) & bases["ambiguous"][None, :])
        ok[s:s + 256] = ((d <= reach) & bases["feasible"][None, :]).any(1)
        amb[s:s + 256] = ~clear_in.any(1) & near.any(1)
    return ok, amb


# --------------------------------------------------------------------------- #
# a7 / a8 — fluence and coverage                                               #
# --------------------------------------------------------------------------- #
def fluence(A: np.ndarray, t: np.ndarray) -> np.ndarray:
    """μ_i = Σ_k I_i(x_k) t_k  (Eq. 5), fp64.  A is (N, K)."""
    return np.asarray(A, np.float64) @ np.asarray(t, np.float64)


def fluence_t(A: np.ndarray, y: np.ndarray) -> np.ndarray:
    """g_k = Σ_i A[i, k] y_i (the LP's adjoint product), fp64."""
    return np.asarray(A, np.float64).T @ np.asarray(y, np.float64)


def coverage(mu: np.ndarray, area: np.ndarray, mu_min: float = 280.0,
             rowsum: np.ndarray | None = None) -> np.ndarray:
    """(covered, total, visible_total) areas: covered = Σ|s_i|·[μ_i ≥ μ_min]
    (inclusive, Q16; P:9 "fraction of the surface area"), total = Σ|s_i|,
    visible_total = Σ|s_i|·[row i ever nonzero]."""
    mu = np.asarray(mu, np.float64)
    area = np.asarray(area, np.float64)
    covered = float(area[mu >= mu_min].sum())
    total = float(area.sum())
    vis_total = float(area[np.asarray(rowsum) > 0].sum()) if rowsum is not None else total
    return np.array([covered, total, vis_total])


# --------------------------------------------------------------------------- #
# NEXT-4 — static single-point baseline                                        #
# --------------------------------------------------------------------------- #
def static_baseline(A: np.ndarray, area: np.ndarray, t_budget: float = 1800.0, mu_min: float = 280.0) -> dict:
    """The paper's static illumination strategy (P:7):
    put the lamp at the vantage configuration whose visible patch area is
    largest and leave it until every visible patch has μ_min, i.e. for
    max_i μ_min / A_ij over the visible patches; ties (equal visible area) go
    to the shorter dwell, then the lower index (reading Q24).  Also the area a
    static lamp covers within `t_budget` at each configuration.
    A: (N, K) in W/m²."""
    A = np.asarray(A, np.float64)
    N, K = A.shape
    vis = np.array([area[A[:, j] > 0].sum() for j in range(K)])
    mn = np.array([A[A[:, j] > 0, j].min() if (A[:, j] > 0).any() else np.inf for j in range(K)])
    cov = np.array([area[A[:, j] * t_budget >= mu_min].sum() for j in range(K)])
    dwell = np.array([mu_min / m if np.isfinite(m) else np.inf for m in mn])
    best = min(range(K), key=lambda j: (-vis[j], dwell[j], j))
    return dict(visible_area=vis, min_irradiance=mn, covered_at_budget=cov, column=best, dwell_s=dwell[best],
                best_budget_column=min(range(K), key=lambda j: (-cov[j], j)))


# --------------------------------------------------------------------------- #
# NEXT-3 — the paper's visibility cube                                          #
# --------------------------------------------------------------------------- #
def pixel_solid_angle(R: int, a: int, b: int) -> float:
    """Exact solid angle of cube-face pixel (a, b) of an R×R face."""
    return float(lib().orc_pixel_solid_angle(int(R), int(a), int(b)))


def cubemap(patches: dict, lamps: np.ndarray, cols=None, R: int = 32, P: float = 80.0, hits: bool = False,
            n_threads: int = 0) -> dict:
    """The paper's §IV-C pipeline by brute force: per lamp sample 6
    R×R cube faces, each pixel's nearest triangle (closest hit) receives the
    pixel's power (P/L)·Ω_px/(4π) when front-facing; A = F/|s|.
    Returns A (N, n_cols), F, the energy on degenerate pixels per column and,
    with hits=True, per-pixel winner ids (n_cols, L, 6, R, R) (-1 none,
    -2 back-facing) and degeneracy flags."""
    lamps = np.ascontiguousarray(lamps, np.float32)
    K, L = lamps.shape[0], lamps.shape[1]
    cols = np.arange(K, dtype=np.int64) if cols is None else np.ascontiguousarray(cols, np.int64)
    n, N = len(cols), patches["N"]
    F = np.zeros(n * N, np.float64)
    deg_e = np.zeros(n, np.float64)
    hit = np.zeros(n * L * 6 * R * R, np.int32) if hits else None
    deg = np.zeros(n * L * 6 * R * R, np.uint8) if hits else None
    lib().orc_cubemap(patches["tri"], patches["tri_patch"], len(patches["tri"]), N, lamps.reshape(-1), L, P, R,
                      cols, n, F, hit.ctypes.data if hits else None, deg.ctypes.data if hits else None, deg_e,
                      n_threads)
    F = F.reshape(n, N).T
    out = dict(A=F / patches["area"][:, None], F=F, deg_energy=deg_e)
    if hits:
        out["hit"] = hit.reshape(n, L, 6, R, R)
        out["deg"] = deg.reshape(n, L, 6, R, R).astype(bool)
    return out
