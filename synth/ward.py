"""Synthetic hospital-ward triangle mesh (workloads C4/C5).

The paper's ward is a GrabCAD asset decimated to 60k triangles;
it is not available, so this generator builds a ward-SHAPED scene of closed,
consistently wound solids:

* shell  W×D×H box (floor, ceiling, 4 walls), normals pointing INTO the room;
* per bay and side: a bed (frame 2.0×0.9×0.5 m, mattress, headboard), a bedside
  cabinet (0.5×0.45×0.8 m), a chair (seat, 4 legs, back), an over-bed table,
  an IV pole (cylinder r=0.02 m, h=1.8 m);
* a nurse counter, a sink unit, a door panel and window frames on the walls.

Every furniture solid is closed with OUTWARD winding; each item (group of
solids) is jittered by ±2 cm and ±3° yaw, and its height scaled by 1 ± 1.5 % (wall
fittings shifted ±1 cm; seeded) so grid-aligned rays and lamp planes do not
systematically hit edges.  Faces are tessellated uniformly into
cells of edge ≤ e, two triangles per cell, giving ≈ 2·A_surf/e² triangles.

Output dict: vertices float32 (nv,3), tris int32 (nt,3), plus bookkeeping
(solid id per triangle, solid volume list) used only by generator tests.
PRNG: numpy PCG64(seed).
"""
from __future__ import annotations

import math

import numpy as np


class _Mesh:
    def __init__(self):
        self.V: list[np.ndarray] = []
        self.F: list[np.ndarray] = []
        self.solid: list[np.ndarray] = []
        self.nv = 0
        self.n_solids = 0

    def add(self, V: np.ndarray, F: np.ndarray, solid: int):
        self.V.append(V)
        self.F.append(F + self.nv)
        self.solid.append(np.full(len(F), solid, np.int32))
        self.nv += len(V)

    def quad_grid(self, o, u, v, e, solid):
        """Rectangle o + a·u + b·v, a,b∈[0,1]; normal = u×v; cells of edge ≤ e."""
        o, u, v = (np.asarray(x, np.float64) for x in (o, u, v))
        nu = max(1, math.ceil(np.linalg.norm(u) / e - 1e-9))
        nv = max(1, math.ceil(np.linalg.norm(v) / e - 1e-9))
        a = np.arange(nu + 1) / nu
        b = np.arange(nv + 1) / nv
        P = o[None, None, :] + a[:, None, None] * u[None, None, :] + b[None, :, None] * v[None, None, :]
        V = P.reshape(-1, 3)
        idx = np.arange((nu + 1) * (nv + 1)).reshape(nu + 1, nv + 1)
        p00 = idx[:-1, :-1].ravel(); p10 = idx[1:, :-1].ravel()
        p11 = idx[1:, 1:].ravel(); p01 = idx[:-1, 1:].ravel()
        F = np.concatenate([np.stack([p00, p10, p11], 1), np.stack([p00, p11, p01], 1)])
        self.add(V, F.astype(np.int64), solid)

    def box(self, lo, hi, e, xform, inward=False):
        """Closed axis-aligned box in local coords, then xform (4×4 affine)."""
        s = self.n_solids
        self.n_solids += 1
        x0, y0, z0 = lo
        x1, y1, z1 = hi
        X, Y, Z = x1 - x0, y1 - y0, z1 - z0
        faces = [((x0, y0, z0), (0, Y, 0), (X, 0, 0)),   # -z
                 ((x0, y0, z1), (X, 0, 0), (0, Y, 0)),   # +z
                 ((x0, y0, z0), (X, 0, 0), (0, 0, Z)),   # -y
                 ((x0, y1, z0), (0, 0, Z), (X, 0, 0)),   # +y
                 ((x0, y0, z0), (0, 0, Z), (0, Y, 0)),   # -x
                 ((x1, y0, z0), (0, Y, 0), (0, 0, Z))]   # +x
        R, t = xform[:3, :3], xform[:3, 3]
        for o, u, v in faces:
            o2 = R @ np.asarray(o, float) + t
            u2 = R @ np.asarray(u, float)
            v2 = R @ np.asarray(v, float)
            if inward:
                u2, v2 = v2, u2
            self.quad_grid(o2, u2, v2, e, s)
        return s

    def cylinder(self, cxy, r, z0, z1, e, xform):
        s = self.n_solids
        self.n_solids += 1
        nseg = max(8, math.ceil(2 * math.pi * r / e))
        nh = max(1, math.ceil((z1 - z0) / e - 1e-9))
        th = 2 * math.pi * np.arange(nseg) / nseg
        ring = np.stack([cxy[0] + r * np.cos(th), cxy[1] + r * np.sin(th)], 1)
        zs = z0 + (z1 - z0) * np.arange(nh + 1) / nh
        P = np.concatenate([np.repeat(ring, nh + 1, 0), np.tile(zs, nseg)[:, None]], 1)  # (nseg*(nh+1),3)
        idx = np.arange(nseg * (nh + 1)).reshape(nseg, nh + 1)
        k = np.arange(nseg)
        k1 = (k + 1) % nseg
        a = idx[k][:, :-1].ravel(); b = idx[k1][:, :-1].ravel()
        c = idx[k1][:, 1:].ravel(); d = idx[k][:, 1:].ravel()
        F = [np.stack([a, b, c], 1), np.stack([a, c, d], 1)]
        ctop = len(P); cbot = len(P) + 1
        P = np.concatenate([P, [[cxy[0], cxy[1], z1], [cxy[0], cxy[1], z0]]])
        F.append(np.stack([np.full(nseg, ctop), idx[k, nh], idx[k1, nh]], 1))
        F.append(np.stack([np.full(nseg, cbot), idx[k1, 0], idx[k, 0]], 1))
        R, t = xform[:3, :3], xform[:3, 3]
        self.add(P @ R.T + t, np.concatenate(F).astype(np.int64), s)
        return s


def _xform(yaw: float, tx: float, ty: float, sz: float = 1.0, tz: float = 0.0) -> np.ndarray:
    c, s = math.cos(yaw), math.sin(yaw)
    M = np.eye(4)
    M[:3, :3] = [[c, -s, 0], [s, c, 0], [0, 0, sz]]
    M[:3, 3] = [tx, ty, tz]
    return M


def ward(seed: int = 0, n_bays: int = 3, e: float = 0.06, width: float = 7.0,
         height: float = 3.0) -> dict:
    """Ward with `n_bays` bed bays per long wall (3 bays → 10 m × 7 m × 3 m, 6 beds)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    # heights: a second stream (the xy / yaw jitter above is unchanged by it);
    # item heights scaled by 1 ± 1.5 % and wall fittings shifted by ± 1 cm, so
    # no horizontal face sits exactly in a lamp-grid plane (e.g. a 0.8 m
    # cabinet top and the Armbot grid's z = 0.8 m plane: cos θ = 0 exactly,
    # a degenerate pair of SURVEY §8c for every such patch and lamp)
    rng_h = np.random.Generator(np.random.PCG64(seed + 1000))

    def hz():
        return rng_h.uniform(0.985, 1.015)
    bay = 10.0 / 3.0
    length = bay * n_bays
    m = _Mesh()
    m.box((0, 0, 0), (length, width, height), e, np.eye(4), inward=True)  # shell

    def jit():
        return (math.radians(rng.uniform(-3, 3)), rng.uniform(-0.02, 0.02), rng.uniform(-0.02, 0.02))

    def X(yaw, tx, ty):  # placement with the height jitter
        return _xform(yaw, tx, ty, hz())

    for side in (0, 1):
        for b in range(n_bays):
            cx = bay * (b + 0.5)
            # local frame: origin at the middle of the bed head, +y away from the wall
            flip = side == 1
            base_y = 0.15 if not flip else width - 0.15
            yaw0 = 0.0 if not flip else math.pi
            dyaw, dx, dy = jit()
            M = X(yaw0 + dyaw, cx + dx, base_y + dy)
            m.box((-0.45, 0.05, 0.0), (0.45, 2.05, 0.5), e, M)          # bed frame
            m.box((-0.425, 0.075, 0.5), (0.425, 2.025, 0.65), e, M)     # mattress
            m.box((-0.45, 0.0, 0.0), (0.45, 0.05, 1.0), e, M)           # headboard
            dyaw, dx, dy = jit()
            M = X(yaw0 + dyaw, cx + dx, base_y + dy)
            m.box((0.6, 0.0, 0.0), (1.1, 0.45, 0.8), e, M)              # bedside cabinet
            dyaw, dx, dy = jit()
            M = X(yaw0 + dyaw, cx + dx, base_y + dy)
            sx, sy = 0.75, 1.0                                          # chair
            m.box((sx, sy, 0.45), (sx + 0.45, sy + 0.45, 0.5), e, M)    # seat
            for lx, ly in ((0, 0), (0.41, 0), (0, 0.41), (0.41, 0.41)):
                m.box((sx + lx, sy + ly, 0.0), (sx + lx + 0.04, sy + ly + 0.04, 0.45), e, M)
            m.box((sx + 0.41, sy, 0.5), (sx + 0.45, sy + 0.45, 0.95), e, M)  # back
            dyaw, dx, dy = jit()
            M = X(yaw0 + dyaw, cx + dx, base_y + dy)
            tx, ty = -1.2, 1.6                                          # over-bed table
            m.box((tx, ty, 0.0), (tx + 0.6, ty + 0.4, 0.03), e, M)
            m.box((tx + 0.05, ty + 0.175, 0.03), (tx + 0.1, ty + 0.225, 0.9), e, M)
            m.box((tx, ty, 0.9), (tx + 0.8, ty + 0.4, 0.93), e, M)
            dyaw, dx, dy = jit()
            M = X(yaw0 + dyaw, cx + dx, base_y + dy)
            m.cylinder((-0.7, 0.3), 0.02, 0.0, 1.8, e, M)              # IV pole
    # nurse counter and sink unit in the middle / against the x=0 wall
    for b in range(max(1, n_bays // 3)):
        dyaw, dx, dy = jit()
        cx0 = length - 2.0 - b * 10.0
        M = X(dyaw, cx0 + dx, width / 2 + dy)
        m.box((-0.75, -0.35, 0.0), (0.75, 0.35, 1.1), e, M)
        dyaw, dx, dy = jit()
        M = X(dyaw, 0.4 + b * 10.0 + dx, width / 2 + dy)
        m.box((-0.3, -0.5, 0.0), (0.3, 0.5, 0.9), e, M)
    # door panel on the x=length wall, window frames on the y=width wall
    m.box((length - 0.04, width / 2 - 0.6, 0.0), (length - 0.001, width / 2 + 0.6, 2.1), e, _xform(0, 0, 0, hz()))
    for b in range(n_bays):
        cx = bay * (b + 0.5)
        m.box((cx - 0.6, width - 0.031, 1.2), (cx + 0.6, width - 0.001, 2.3), e,
              _xform(0, 0, 0, 1.0, rng_h.uniform(-0.01, 0.01)))
    V = np.concatenate(m.V).astype(np.float32)
    F = np.concatenate(m.F).astype(np.int32)
    solid = np.concatenate(m.solid)
    return dict(vertices=V, tris=F, solid=solid, n_solids=m.n_solids,
                bbox=np.array([0, 0, 0, length, width, height], np.float32))
