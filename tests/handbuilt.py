"""Hand-built scenes and their closed-form expectations, shared by the oracle
pins (tests/test_oracle_pins_r2.py) and the GPU checks against the same
constructions (tests/test_gpu_vantage_pins.py).  No oracle and no CUDA code here."""
import math

import numpy as np

from synth import configs, ward

def _mesh(boxes):
    """boxes: list of (lo, hi, inward); each face one quad (2 triangles)."""
    m = ward._Mesh()
    for lo, hi, inward in boxes:
        m.box(lo, hi, 100.0, np.eye(4), inward=inward)
    V = np.concatenate(m.V).astype(np.float32)
    F = np.concatenate(m.F).astype(np.int32)
    return V, F


def _line_scene(h=0.75, zc=1.0):
    """A small triangle in the plane x = 0 facing +x with centroid (0, 0, zc)
    exactly, plus a helper triangle behind it (x = -1) that widens the bbox so
    the Towerbot grid has a column at (h, 0); the helper cannot occlude
    segments from x = h > 0 to the patch."""
    s = 1.0 / 64
    V = np.array([[0, -s, zc - s], [0, 2 * s, zc - s], [0, -s, zc + 2 * s],
                  [-1.0, -0.25, 0.0], [-1.0, 0.25, 0.0], [-1.0, 0.0, 2.5],
                  [1.0, 0.0, 0.0]], np.float32)
    # helper: facing -x (away from the lamps); a zero-area-free sliver to x = 1
    F = np.array([[0, 1, 2], [3, 5, 4], [3, 6, 4]], np.int32)
    return dict(vertices=V, tris=F)


def clearance_scene():
    """Room [0,2]³ (inward shell) with three boxes placed so FLOAT3D grid points
    (cell centres 0.125 + 0.25 a) sit 0.05 ± 1e-3 m from a face (box A), from a
    corner (box B, vertex region) and from an edge (box C)."""
    e, f = 0.049, 0.051
    boxes = [((0.0, 0.0, 0.0), (2.0, 2.0, 2.0), True),
             ((0.875 + e, 0.875 + f, 0.875 + e), (1.375 - f, 1.375 - e, 1.375 - f), False),   # A
             ((0.375 + e / math.sqrt(3),) * 3, (0.375 + e / math.sqrt(3) + 0.15,) * 3, False),   # B
             ((1.625 + f / math.sqrt(2), 0.375 + f / math.sqrt(2), 0.3),
              (1.625 + f / math.sqrt(2) + 0.15, 0.375 + f / math.sqrt(2) + 0.15, 0.45), False)]  # C
    V, F = _mesh(boxes)
    return dict(vertices=V, tris=F), len(boxes)


def clearance_expected(sc, n_boxes, pts):
    """Closed-form distance of each point to the room shell and the boxes, from
    the fp32 vertices (12 triangles per box in generation order), and whether
    it lies inside an obstacle."""
    V = sc["vertices"].astype(np.float64)
    P = np.asarray(pts, np.float64)
    per = len(V) // n_boxes
    d = np.full(len(P), np.inf)
    inside = np.zeros(len(P), bool)
    for k in range(n_boxes):
        B = V[k * per:(k + 1) * per]
        lo, hi = B.min(0), B.max(0)
        if k == 0:   # shell: points are inside the room
            d = np.minimum(d, np.minimum(P - lo, hi - P).min(1))
        else:
            dd = np.sqrt((np.maximum(np.maximum(lo - P, P - hi), 0.0) ** 2).sum(1))
            ins = ((P > lo) & (P < hi)).all(1)
            inside |= ins
            d = np.minimum(d, np.where(ins, np.minimum(P - lo, hi - P).min(1), dd))
    return d, inside


def corridor_scene():
    """Corridor room x ∈ [0,1], y ∈ [0,0.75], z ∈ [0,2.5] (inward shell) and a
    small plate hanging 0.25 m above base b2.  With ρ = 0.25, base_z = 0.4 and
    base clearance 0.325 (Q10/Q12) the floor grid (x, y ∈ {0.125, 0.375, ...})
    has exactly two bases clear of the walls, b1 = (0.375, 0.375, 0.4) and
    b2 = (0.625, 0.375, 0.4); the plate is 0.25 m from b2 (blocked) and
    √(0.245² + 0.25²) = 0.35 m from b1 (free)."""
    boxes = [((0.0, 0.0, 0.0), (1.0, 0.75, 2.5), True),
             ((0.62, 0.35, 0.65), (0.70, 0.40, 0.70), False)]
    V, F = _mesh(boxes)
    return dict(vertices=V, tris=F)


ARM_CORRIDOR = configs.vopts(configs.ARM, 0.25, 0.05, zmin=0.3, zmax=1.9, reach=0.85,
                             base_clearance=0.325, base_z=0.4)
B1 = np.array([0.375, 0.375, np.float32(0.4)], np.float64)   # fp32 grid values, exact in fp64
B2 = np.array([0.625, 0.375, np.float32(0.4)], np.float64)
