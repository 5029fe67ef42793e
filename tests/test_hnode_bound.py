"""The fp16 H-node slab test is conservative (csrc/hnodes.cu header,
csrc/assemble.cu H branch): for segments that meet an fp32 node box, the
kernel's half-precision arithmetic — h = fl16(1/d), constants fl16(−(o − c)·h),
one HFMA2 per plane of the box padded by 1.25·2⁻¹⁰·L_axis + 1e-4 m and rounded
outward to fp16, t range rounded outward — never rejects the box.  Emulated
exactly here (rational arithmetic, explicit round-to-nearest-even and directed
roundings onto the binary16 / binary32 grids) on grazing segments aimed at box
faces, edges and corners; a negative control shows the check has teeth (no
padding: some grazing segments are rejected).  CPU only."""
import math
import random
from fractions import Fraction as F

import numpy as np


def _round_grid(x: F, mant: int, emin: int, mode: str) -> F:
    """Round x onto a binary floating-point grid with `mant` fraction bits and
    minimum normal exponent emin (subnormals below), mode rn / rd / ru."""
    if x == 0:
        return F(0)
    e = max(math.floor(math.log2(abs(x))), emin)
    # correct a floor(log2) off by one from float rounding
    while abs(x) >= F(2) ** (e + 1):
        e += 1
    while e > emin and abs(x) < F(2) ** e:
        e -= 1
    ulp = F(2) ** (e - mant)
    q = x / ulp
    if mode == "rd":
        n = math.floor(q)
    elif mode == "ru":
        n = math.ceil(q)
    else:
        n = math.floor(q)
        r = q - n
        if r > F(1, 2) or (r == F(1, 2) and n % 2 == 1):
            n += 1
    return n * ulp


def h16(x, mode="rn"):
    return _round_grid(F(x), 10, -14, mode)


def f32(x, mode="rn"):
    return _round_grid(F(x), 23, -126, mode)


def _kernel_accepts(box, o, d, tmin, tmax, ctr, half, pad_on=True, ix_err=0):
    """The H branch of lane_walk32 for one child box (exact emulation)."""
    planes = []
    for ax in range(3):
        L = 2 * half[ax]
        pad = F(1.25) / 1024 * F(L) + F(1, 10000) if pad_on else F(0)
        # build: outward rounding of the padded plane (relative to the centre)
        lo = h16(F(box[ax][0]) - F(ctr[ax]) - pad, "rd")
        hi = h16(F(box[ax][1]) - F(ctr[ax]) + pad, "ru")
        # walk: fp32 reciprocal (rcp.approx: relative error <= 2^-23), then fp16
        ix = f32(F(1) / F(d[ax]) * (1 + F(ix_err[ax]) / 2 ** 23) if ix_err else F(1) / F(d[ax]))
        hix = h16(ix)
        orx = f32(F(o[ax]) - F(ctr[ax]))
        hb = h16(-f32(orx * hix))
        ta, tb = h16(lo * hix + hb), h16(hi * hix + hb)  # HFMA2: one rounding each
        planes.append((min(ta, tb), max(ta, tb)))  # the octant copy stores (entry, exit)
    en = max(max(p[0] for p in planes), h16(F(tmin), "rd"))
    ex = min(min(p[1] for p in planes), h16(F(tmax), "ru"))
    return en <= ex


def _exact_meets(box, o, d, tmin, tmax):
    lo_t, hi_t = F(tmin), F(tmax)
    for ax in range(3):
        a = (F(box[ax][0]) - F(o[ax])) / F(d[ax])
        b = (F(box[ax][1]) - F(o[ax])) / F(d[ax])
        lo_t, hi_t = max(lo_t, min(a, b)), min(hi_t, max(a, b))
    return lo_t <= hi_t


def _cases(n, seed):
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        half = [rng.uniform(1.0, 15.0) for _ in range(3)]
        ctr = [float(np.float32(rng.uniform(-20, 20))) for _ in range(3)]
        # an fp32 box inside the scene, sizes from 1 cm to metres
        box = []
        for ax in range(3):
            s = 10 ** rng.uniform(-2, math.log10(half[ax]))
            a = rng.uniform(ctr[ax] - half[ax], ctr[ax] + half[ax] - s)
            box.append((float(np.float32(a)), float(np.float32(a + s))))
        o = [float(np.float32(rng.uniform(ctr[k] - half[k], ctr[k] + half[k]))) for k in range(3)]
        # aim at a point on a face, an edge or a corner of the box
        p = [rng.uniform(*box[k]) for k in range(3)]
        for k in rng.sample(range(3), rng.randint(1, 3)):
            p[k] = box[k][rng.randint(0, 1)]
        t0 = rng.uniform(0.05, 0.95)
        d = [float(np.float32((p[k] - o[k]) / t0)) for k in range(3)]
        if min(abs(x) for x in d) < 1.0 / 2048 or any(abs(o[k] - ctr[k]) > half[k] for k in range(3)):
            continue  # the H path is taken only for |1/d| <= 2048 and lamps in the scene box
        tmin = float(np.float32(max(0.0, t0 - rng.choice([0.0, 1e-6, 1e-3, 0.1]))))
        tmax = float(np.float32(min(1.0, t0 + rng.choice([0.0, 1e-6, 1e-3, 0.1]))))
        if not _exact_meets(box, o, d, tmin, tmax):
            continue
        out.append((box, o, d, tmin, tmax, ctr, half, [rng.choice([-1, 0, 1]) for _ in range(3)]))
    return out


def test_hnode_test_never_rejects_a_box_the_segment_meets():
    cases = _cases(1500, 11)
    rejected = [c for c in cases if not _kernel_accepts(*c[:7], pad_on=True, ix_err=c[7])]
    assert not rejected, f"{len(rejected)} grazing segments rejected by the padded fp16 test"


def test_hnode_negative_control_unpadded_boxes_fail():
    """Without the padding the same emulation rejects some grazing segments
    (so the check above can fail)."""
    cases = _cases(600, 12)
    rejected = sum(not _kernel_accepts(*c[:7], pad_on=False, ix_err=c[7]) for c in cases)
    assert rejected > 0


def test_rounding_helpers_match_numpy():
    rng = np.random.default_rng(0)
    for x in rng.standard_normal(300) * 10.0 ** rng.integers(-6, 4, 300):
        assert float(h16(x)) == float(np.float16(x)) or abs(x) > 65504
        assert float(f32(x)) == float(np.float32(x))
        assert h16(x, "rd") <= F(x) <= h16(x, "ru")
