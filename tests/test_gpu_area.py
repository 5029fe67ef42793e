"""GPU parity of NEXT-2, the area-integrated irradiance model (Eq. 4 as
written; reading Q23), through the C-ABI
(uvd_irradiance_matrix with UVD_MODEL_AREA) against the oracle's
`irradiance_area_*` on the same seeded inputs.

Bars: entries within 1e-5 relative (fp64 solid angles, one fp32 rounding) on
pairs the oracle does not flag degenerate (a sub-ray with |margin| < 1e-6 or
|cosθ| < 1e-6); the degenerate fraction stays < 1e-3 of pairs; closed forms
(Σ|s|A = P in a closed enclosure, the analytic partial shadow) hold on the
GPU's own output.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from synth import configs, rooms, ward  # noqa: E402

REL = 1e-5


@pytest.fixture(scope="module")
def uvd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd as U
    return U


def gpu_area(U, desc, lamps_np, m, vis_bits=False):
    sc = U.Scene(desc)
    lam = torch.from_numpy(np.ascontiguousarray(lamps_np, np.float32)).cuda()
    r = sc.irradiance(lam, area_subdiv=m, vis_bits=vis_bits)
    sc.sync_status()
    orig = sc.patches()["orig_id"].cpu().numpy()
    A = np.zeros((sc.N, lam.shape[0]))
    A[orig] = r["A"][:, :sc.N].T.double().cpu().numpy()
    return sc, r, A, orig


def compare(A, ref, deg_gate=1e-3):
    deg = ref["deg"]
    assert deg.mean() < deg_gate, deg.mean()
    ok = ~deg
    err = np.abs(A[ok] - ref["A"][ok])
    assert (err <= REL * np.abs(ref["A"][ok]) + 1e-30).all(), err.max()
    assert (A[ok] > 0).mean() > 0.05


@pytest.mark.parametrize("m", [0, 1, 2])
def test_area_c1_full_matrix(uvd, m):
    c = configs.c1()
    v = O.vantage(c["scene"], c["vantage"])
    lam = v["samples"][v["feasible"]][::4]
    sc, r, A, orig = gpu_area(uvd, c["scene"], lam, m)
    ref = O.irradiance_area_matrix(O.extruded_patches(c["scene"]), lam, m=m, mode="2d")
    compare(A, ref)
    assert (A > 0).all()       # convex room: every patch lit


@pytest.mark.parametrize("seed", [0, 5, 11])
def test_area_c2_full_matrix(uvd, seed):
    c = configs.c2(seed)
    v = O.vantage(c["scene"], c["vantage"])
    lam = v["samples"][v["feasible"]][::3]
    sc, r, A, orig = gpu_area(uvd, c["scene"], lam, 1, vis_bits=True)
    pat = O.extruded_patches(c["scene"])
    ref = O.irradiance_area_matrix(pat, lam, m=1, mode="2d")
    compare(A, ref)
    # vis bit = some sub-triangle seen (non-degenerate pairs)
    vb = r["vis_bits"].cpu().numpy().view(np.uint32)[:, 0, :]
    bits = ((vb[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(vb.shape[0], -1)[:, :sc.N].T
    gvis = np.zeros_like(bits)
    gvis[orig] = bits
    ok = ~ref["deg"]
    assert np.array_equal(gvis.astype(bool)[ok], (ref["nvis"] > 0)[ok])


def test_area_small_ward_sampled(uvd):
    """3D triangles (every occluder a triangle), Towerbot L = 10 samples,
    sampled pairs against the brute-force oracle."""
    w = ward.ward(seed=4, n_bays=1, e=0.3)
    opts = dict(configs.TOWER_OPTS, spacing=0.5)
    v = O.vantage(w, opts)
    lam = v["samples"][v["feasible"]]
    sc, r, A, orig = gpu_area(uvd, w, lam, 1)
    pat = O.trimesh_patches(w["vertices"], w["tris"])
    rng = np.random.default_rng(0)
    pi = rng.integers(0, sc.N, 600)
    pj = rng.integers(0, lam.shape[0], 600)
    ref = O.irradiance_area_pairs(pat, lam, pi, pj, m=1)
    ok = ~ref["deg"]
    assert ok.mean() > 0.99
    got = A[pi, pj]
    assert (np.abs(got[ok] - ref["A"][ok]) <= REL * ref["A"][ok] + 1e-30).all()
    assert (got[ok] > 0).mean() > 0.05


def test_area_closed_enclosure_flux(uvd):
    """Σ_i |s_i| A_ij = P for lamps inside a closed convex enclosure, on the
    GPU's own output (exact solid angles; fp32 storage of A)."""
    mm = ward._Mesh()
    mm.box((0, 0, 0), (1, 1, 1), 0.125, np.eye(4), inward=True)
    desc = {"vertices": np.concatenate(mm.V).astype(np.float32), "tris": np.concatenate(mm.F).astype(np.int32)}
    lam = np.array([[[0.5, 0.5, 0.5]], [[0.3, 0.6, 0.45]], [[0.9, 0.1, 0.2]]], np.float32)
    sc, r, A, orig = gpu_area(uvd, desc, lam, 1)
    area = O.trimesh_patches(desc["vertices"], desc["tris"])["area"]
    flux = (area[:, None] * A).sum(0)
    assert np.allclose(flux, 80.0, rtol=2e-7, atol=0)


def test_area_partial_shadow_analytic(uvd):
    """The oracle pin's partial shadow (tests/test_area_oracle.py) on the GPU:
    the flux through the half-shadowed floor converges to the analytic
    solid angle of its lit part."""
    V = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                  [-3, -3, 1], [0.6, -3, 1], [0.6, 4, 1], [-3, 4, 1]], np.float32)
    F = np.array([[0, 1, 2], [0, 2, 3], [4, 6, 5], [4, 7, 6]], np.int32)
    desc = {"vertices": V, "tris": F}
    lamp = np.float32([0.5, 0.5, 2.0]).reshape(1, 1, 3)
    x_s = 0.5 + (float(np.float32(0.6)) - 0.5) * 2.0
    p = lamp.reshape(3).astype(np.float64)
    om = (O.solid_angle(p, [x_s, 0, 0], [1, 0, 0], [1, 1, 0]) + O.solid_angle(p, [x_s, 0, 0], [1, 1, 0], [x_s, 1, 0]))
    exact = 80.0 / (4 * math.pi) * om
    area = O.trimesh_patches(V, F)["area"]
    errs = []
    for m in (2, 4, 6):
        sc, r, A, orig = gpu_area(uvd, desc, lamp, m)
        errs.append(abs((area[:2] * A[:2, 0]).sum() - exact) / exact)
    assert errs[-1] < 0.015 and errs[-1] < errs[0]   # O(h) boundary error: 0.7 sits 0.8 into a 1/64 column


def test_area_model_rejects_csc_and_bad_level(uvd):
    c = configs.c1()
    sc = uvd.Scene(c["scene"])
    lam, _ = sc.vantage(c["vantage"])
    with pytest.raises(uvd.UvdError):
        sc.irradiance(lam, area_subdiv=7)
    import ctypes as C
    m = uvd._MatrixOut()
    m.format = uvd.CSC
    m.colptr = torch.zeros(lam.shape[0] + 1, dtype=torch.int64, device="cuda").data_ptr()
    lamp = uvd._Lamp(80.0, 1, 1, 1)
    rc = uvd.lib().uvd_irradiance_matrix(sc.handle, uvd._ptr(lam), lam.shape[0], None, lam.shape[0],
                                         C.byref(lamp), C.byref(m), uvd._stream())
    assert rc == uvd.UVD_ERR_INVALID


def test_area_c4_floatbot_sampled(uvd):
    """The area model at C4 size (the timing configuration): sampled pairs
    against the brute-force oracle (oracle's own vantage samples)."""
    desc = configs.c4_scene()
    sc = uvd.Scene(desc)
    lamps, raw = sc.vantage(configs.FLOAT_OPTS)
    K = lamps.shape[0]
    cols = np.arange(0, K, 64)
    r = sc.irradiance(lamps, cols=list(cols), area_subdiv=1)
    sc.sync_status()
    orig = sc.patches()["orig_id"].cpu().numpy()
    rng = np.random.default_rng(3)
    ri = rng.integers(0, sc.N, 300)
    ci = rng.integers(0, len(cols), 300)
    got = r["A"][torch.from_numpy(ci).cuda(), torch.from_numpy(ri).cuda()].double().cpu().numpy()
    uc = np.unique(ci)
    v = O.vantage(desc, configs.FLOAT_OPTS, idx=raw.cpu().numpy()[cols[uc]])
    lam_o = np.zeros((len(cols), 1, 3), np.float32)
    lam_o[uc] = v["samples"]
    assert np.array_equal(lam_o[uc], lamps.cpu().numpy()[cols[uc]])
    ref = O.irradiance_area_pairs(O.scene_patches(desc), lam_o, orig[ri], ci, m=1)
    ok = ~ref["deg"]
    assert ok.mean() > 0.98
    assert (np.abs(got[ok] - ref["A"][ok]) <= REL * ref["A"][ok] + 1e-30).all()
    assert 0.05 < (got[ok] > 0).mean() < 0.95
