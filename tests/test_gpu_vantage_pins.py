"""The CUDA path on the hand-built constructions that pin the oracle
(tests/handbuilt.py, tests/test_oracle_pins_r2.py): expectations come from
closed forms, not from the oracle, so a misreading shared by the oracle and
the kernels would fail here too.

* clearance (Q10): FLOAT3D feasibility on the room whose box faces,
  edges and corners sit 0.05 ± 1e-3 m from grid points;
* reach proxy (Q12): ARM feasibility on the corridor with one blocked
  base;
* lamp split (Q11): the GPU's L-sample entries = the mean of its
  single-point entries (with a partial shadow), converging to the analytic
  line source.
"""
import math

import numpy as np
import pytest

from handbuilt import ARM_CORRIDOR, B1, B2, _line_scene, clearance_expected, clearance_scene, corridor_scene
from synth import configs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def uvd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd as U
    return U


def _grid(scene, opts):
    """Raw candidate grid (x fastest, then y, then z; Q9) written out here."""
    V = scene["vertices"]
    lo, hi = V.min(0), V.max(0)
    rho = float(np.float32(opts["spacing"]))

    def axis(a, b):
        a, b = float(np.float32(a)), float(np.float32(b))
        return (a + (np.arange(int(np.floor((b - a) / rho))) + 0.5) * rho).astype(np.float32)
    xs, ys = axis(lo[0], hi[0]), axis(lo[1], hi[1])
    zs = axis(lo[2], hi[2]) if opts["robot"] == configs.FLOAT3D else axis(opts["zmin"], opts["zmax"])
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)


def _feasible_mask(uvd, scene, opts):
    sc = uvd.Scene(scene)
    lamps, raw = sc.vantage(opts)
    pts = _grid(scene, opts)
    g = np.zeros(len(pts), bool)
    g[raw.cpu().numpy()] = True
    assert np.array_equal(lamps[:, 0].cpu().numpy(), pts[g])
    sc.close()
    return pts, g


def test_gpu_clearance_threshold(uvd):
    scene, nb = clearance_scene()
    opts = configs.vopts(configs.FLOAT3D, 0.25, 0.05)
    pts, g = _feasible_mask(uvd, scene, opts)
    d, inside = clearance_expected(scene, nb, pts)
    assert np.array_equal(g, (d >= 0.05) & ~inside)
    near = np.abs(d - 0.05) < 1.5e-3
    assert g[near].any() and (~g[near]).any()


def test_gpu_reach_proxy_corridor(uvd):
    scene = corridor_scene()
    pts, g = _feasible_mask(uvd, scene, ARM_CORRIDOR)
    P = pts.astype(np.float64)
    d, inside = clearance_expected(scene, 2, P)
    reach = np.linalg.norm(P - B1, axis=1) <= np.float32(0.85)
    assert np.array_equal(g, (d >= 0.05) & ~inside & reach)
    # points reachable only from the blocked base b2 are rejected
    only_b2 = (d >= 0.05) & ~inside & ~reach & (np.linalg.norm(P - B2, axis=1) <= 0.85)
    assert only_b2.any() and not g[only_b2].any()


def _column(scene, L, h=0.75):
    V = scene["vertices"]
    lo, hi = V.min(0), V.max(0)
    xs = (lo[0] + (np.arange(int((hi[0] - lo[0]) / 0.5)) + 0.5) * 0.5)
    assert np.any(np.abs(xs - h) < 1e-7)
    f0, f1 = float(np.float32(0.37)), float(np.float32(1.57))
    z = np.array([f0 + (l + 0.5) * (f1 - f0) / L for l in range(L)], np.float32)
    lam = np.zeros((1, L, 3), np.float32)
    lam[0, :, 0] = h
    lam[0, :, 2] = z
    return lam


def test_gpu_lamp_split(uvd):
    base = _line_scene()
    V, F = base["vertices"], base["tris"]
    Vp = np.array([[0.3, -0.3, 0.8], [0.5, -0.3, 0.8], [0.5, 0.3, 0.8], [0.3, 0.3, 0.8]], np.float32)
    Fp = np.array([[0, 1, 2], [0, 2, 3]], np.int32) + len(V)
    shadowed = dict(vertices=np.concatenate([V, Vp]), tris=np.concatenate([F, Fp]))
    h, zc = 0.75, 1.0
    f0, f1 = float(np.float32(0.37)), float(np.float32(1.57))

    def prim(z):
        u = z - zc
        return u / (h * math.sqrt(h * h + u * u))
    exact = 80.0 / (4 * math.pi * (f1 - f0)) * (prim(f1) - prim(f0))
    errs = []
    for scene in (base, shadowed):
        sc = uvd.Scene(scene)
        row = int(np.nonzero(sc.patches()["orig_id"].cpu().numpy() == 0)[0][0])
        for L in (1, 3, 10, 16, 64):
            lam = torch.from_numpy(_column(scene, L)).cuda()
            r = sc.irradiance(lam, vis_bits=True)
            singles = sc.irradiance(lam.reshape(L, 1, 3), vis_bits=True)
            sc.sync_status()
            a = float(r["A"][0, row])
            s = singles["A"][:, row].double().cpu().numpy()
            assert abs(a - s.sum() / L) <= 1e-6 * max(a, 1e-30)   # fp32 storage of each side
            bits = r["vis_bits"].cpu().numpy().view(np.uint32)[0, :, row // 32] >> (row % 32) & 1
            sb = singles["vis_bits"].cpu().numpy().view(np.uint32)[:, 0, row // 32] >> (row % 32) & 1
            assert np.array_equal(bits, sb)
            if scene is base and L >= 16:
                errs.append(abs(a - exact) / exact)
            if scene is shadowed and L == 10:
                assert 0 < bits.sum() < L
        sc.close()
    assert errs[0] / errs[1] > 3.5 and errs[1] < 2e-4, errs
