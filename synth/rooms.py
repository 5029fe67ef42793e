"""2.5D random-room generator (workloads C1–C3).

Follows SPEC worldgen.generate_random_room and the paper's
random-room description ("randomly generate 25 2.5D rooms in a 4 m × 4 m
area ... between 7 and 19 obstacles ... scaling, shearing and displacing regular
polygons").  Parameter ranges the paper leaves open are SPEC's defaults
(circumradius U[0.2, 0.8] m, shear U[-0.5, 0.5]); see DESIGN.md §Readings.

Output is a plain dict (the C-ABI's EXTRUDED scene description):
  bounds      (x0, y0, x1, y1) float32 metres
  wall_height float32 metres
  obstacles   list of float32 arrays (n_k, 2), CCW, strictly inside bounds
  patch_res   float32 metres
PRNG: numpy PCG64 seeded with `seed` (documented, platform independent).
"""
from __future__ import annotations

import numpy as np

MARGIN = 0.01  # obstacles kept this far inside the bounds ("strictly inside")


def empty_room(size: float = 5.0, wall_height: float = 2.0, patch_res: float = 0.125) -> dict:
    """C1: empty size×size room."""
    return dict(bounds=np.array([0.0, 0.0, size, size], np.float32),
                wall_height=np.float32(wall_height), obstacles=[],
                patch_res=np.float32(patch_res))


def _regular_polygon(k: int) -> np.ndarray:
    ang = 2.0 * np.pi * np.arange(k) / k
    return np.stack([np.cos(ang), np.sin(ang)], axis=1)  # CCW, unit circumradius


def random_room(seed: int, size: float = 4.0, n_obstacles: int | None = None,
                wall_height: float = 2.0, patch_res: float = 0.125,
                max_retry: int = 1000) -> dict:
    """C2/C3: one random 2.5D world.  n_obstacles ~ U{7..19} unless given."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if n_obstacles is None:
        n_obstacles = int(rng.integers(7, 20))
    lo, hi = MARGIN, size - MARGIN
    obstacles = []
    for _ in range(n_obstacles):
        k = int(rng.integers(3, 9))
        base = _regular_polygon(k)
        for _attempt in range(max_retry):
            r = rng.uniform(0.2, 0.8)
            sh = rng.uniform(-0.5, 0.5)
            th = rng.uniform(0.0, 2.0 * np.pi)
            rot = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
            shear = np.array([[1.0, sh], [0.0, 1.0]])  # det 1: keeps CCW
            poly = (base * r) @ shear.T @ rot.T
            ext_lo, ext_hi = poly.min(0), poly.max(0)
            if np.any(ext_hi - ext_lo >= hi - lo):
                continue
            cx = rng.uniform(lo - ext_lo[0], hi - ext_hi[0])
            cy = rng.uniform(lo - ext_lo[1], hi - ext_hi[1])
            poly = (poly + np.array([cx, cy])).astype(np.float32)
            if poly.min() > lo and poly.max() < hi:
                obstacles.append(poly)
                break
        else:
            raise RuntimeError(f"random_room(seed={seed}): placement failed after {max_retry} retries")
    return dict(bounds=np.array([0.0, 0.0, size, size], np.float32),
                wall_height=np.float32(wall_height), obstacles=obstacles,
                patch_res=np.float32(patch_res))


def partitioned_room(size: float = 4.0, wall_height: float = 2.0, patch_res: float = 0.25,
                     thickness: float = 0.1) -> dict:
    """A room split in two by a full-width thin wall (S:106, S:115 pin).

    The divider is a thin rectangle spanning the room from x=MARGIN to x=size-MARGIN,
    leaving MARGIN-wide slits; lamps on either side see nothing on the other side
    except through the slits, so tests only look at patches away from them."""
    y0 = size / 2 - thickness / 2
    y1 = size / 2 + thickness / 2
    a, b = MARGIN * 2, size - MARGIN * 2
    poly = np.array([[a, y0], [b, y0], [b, y1], [a, y1]], np.float32)
    return dict(bounds=np.array([0.0, 0.0, size, size], np.float32),
                wall_height=np.float32(wall_height), obstacles=[poly],
                patch_res=np.float32(patch_res))


def box_room(size: float = 4.0, box=(1.6, 1.6, 2.4, 2.4), wall_height: float = 2.0,
             patch_res: float = 0.25) -> dict:
    """An empty room with one square obstacle ("a box between light and patch")."""
    x0, y0, x1, y1 = box
    poly = np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], np.float32)
    return dict(bounds=np.array([0.0, 0.0, size, size], np.float32),
                wall_height=np.float32(wall_height), obstacles=[poly],
                patch_res=np.float32(patch_res))
