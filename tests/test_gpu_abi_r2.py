"""ABI behaviour added in round 2: coverage on
several streams at once, the atomic error-flag read of uvd_sync_status, call
scratch through the caller's allocator, the static baseline's choice made
in the library, and the fix-up list export."""
import ctypes as C
import threading

import numpy as np
import pytest

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


def test_coverage_concurrent_streams(uvd):
    c = configs.c2(2)
    sc = uvd.Scene(c["scene"])
    lamps, _ = sc.vantage(c["vantage"])
    A = sc.irradiance(lamps)["A"]
    K = lamps.shape[0]
    mus = [uvd.fluence(A, sc.N, torch.full((K,), float(tv), dtype=torch.float64, device="cuda"))
           for tv in (5.0, 40.0, 400.0)]
    torch.cuda.synchronize()
    ref = [sc.coverage(m, configs.MU_MIN) for m in mus]
    assert len({tuple(r) for r in ref}) == 3
    errs = []

    def worker(k):
        s = torch.cuda.Stream()
        try:
            for _ in range(40):
                got = sc.coverage(mus[k], configs.MU_MIN, stream=s)
                if not np.array_equal(got, ref[k]):
                    errs.append((k, got, ref[k]))
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=worker, args=(k,)) for k in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs[:3]


def test_sync_status_reports_errors_from_other_streams(uvd):
    c = configs.c1()
    sc = uvd.Scene(c["scene"])
    lam = sc.patches()["centroid"][7:8].reshape(1, 1, 3).contiguous()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        sc.irradiance(lam, stream=s1)
    s1.synchronize()
    with pytest.raises(uvd.UvdError) as e:
        sc.sync_status(stream=s2)
    assert e.value.code == uvd.UVD_ERR_DOMAIN
    sc.sync_status(stream=s2)  # read and cleared in one atomic: clean now


def test_fluence_scratch_through_allocator(uvd):
    calls = {"alloc": 0, "free": 0}

    @uvd._ALLOC_FN
    def alloc(nbytes, device, stream, ctx):
        calls["alloc"] += 1
        return torch.cuda.caching_allocator_alloc(int(nbytes), device, stream)

    @uvd._FREE_FN
    def free(ptr, device, stream, ctx):
        calls["free"] += 1
        torch.cuda.caching_allocator_delete(ptr)
    al = uvd._Allocator(alloc, free, None)
    c = configs.c2(1)
    sc = uvd.Scene(c["scene"])
    lamps, _ = sc.vantage(c["vantage"])
    A = sc.irradiance(lamps)["A"]
    K = lamps.shape[0]
    t = torch.rand(K, dtype=torch.float64, device="cuda")
    m = uvd._dense_desc(A)
    m.allocator = C.pointer(al)
    out = torch.empty(sc.N, dtype=torch.float64, device="cuda")
    uvd._check(uvd.lib().uvd_fluence(C.byref(m), sc.N, K, 0, uvd._ptr(t), uvd._ptr(out), uvd._stream()))
    torch.cuda.synchronize()
    assert calls["alloc"] >= 1 and calls["alloc"] == calls["free"]
    assert torch.equal(out, uvd.fluence(A, sc.N, t))
    # the default (no allocator: cudaMallocAsync) gives the same bits
    m.allocator = C.POINTER(uvd._Allocator)()
    out2 = torch.empty_like(out)
    uvd._check(uvd.lib().uvd_fluence(C.byref(m), sc.N, K, 0, uvd._ptr(t), uvd._ptr(out2), uvd._stream()))
    assert torch.equal(out, out2)


def test_static_choice_in_library(uvd):
    """The choice (reading Q24) comes from uvd_static_columns: it matches the
    lexicographic rule applied to the per-column outputs."""
    c = configs.c2(9)
    sc = uvd.Scene(c["scene"])
    lamps, _ = sc.vantage(c["vantage"])
    A = sc.irradiance(lamps)["A"]
    g = sc.static_baseline(A, t_budget=configs.T_MAX)
    vis, mn, cov = g["visible_area"], g["min_irradiance"], g["covered_at_budget"]
    dwell = np.where(np.isfinite(mn), configs.MU_MIN / mn, np.inf)
    K = len(vis)
    assert g["column"] == min(range(K), key=lambda j: (-vis[j], dwell[j], j))
    assert g["best_budget_column"] == min(range(K), key=lambda j: (-cov[j], j))
    assert g["dwell_s"] == dwell[g["column"]]


def test_fixup_list_export(uvd):
    """The exported fix-up entries are exactly the entries left undecided: the
    instrumented kernel's count equals the list's count, and the entries are
    distinct and in range; a capacity below the count truncates the list but
    not the count."""
    sc = uvd.Scene(configs.c4_scene())
    lamps, _ = sc.vantage(configs.FLOAT_OPTS)
    cols = list(range(0, lamps.shape[0], 40))
    r = sc.irradiance(lamps, cols=cols, fixups=1 << 20)
    rc = sc.irradiance(lamps, cols=cols, counters=True)
    n = r["fixup_count"]
    assert n > 0 and n == int(rc["counters"][4].item()) == len(r["fixups"])
    fl = r["fixups"].cpu().numpy().astype(np.uint64)
    assert len(np.unique(fl)) == n
    assert ((fl >> np.uint64(32)) < len(cols)).all() and ((fl & np.uint64(0xffffffff)) < sc.N).all()
    r2 = sc.irradiance(lamps, cols=cols, fixups=5)
    assert r2["fixup_count"] == n and len(r2["fixups"]) == 5
    assert torch.equal(r2["A"], r["A"])


@pytest.mark.parametrize("which", ["ward", "c2"])
def test_scene_export_import_roundtrip(uvd, which):
    """uvd_scene_export / uvd_scene_import (the multi-rank scene broadcast,
    SURVEY §8e): the imported scene is the same scene — patches, BVH, vantage
    samples, A, visibility bits and the fix-up list bit for bit — and a
    corrupted image is refused."""
    from synth import ward
    if which == "ward":
        desc, vo = ward.ward(seed=3, n_bays=1, e=0.2), configs.vopts(configs.FLOAT3D, 0.5, 0.05)
    else:
        c = configs.c2(6)
        desc, vo = c["scene"], c["vantage"]
    a = uvd.Scene(desc)
    img = a.export()
    b = uvd.Scene.from_image(img)
    assert (a.N, a.M, a.total_area) == (b.N, b.M, b.total_area) and np.array_equal(a.bbox, b.bbox)
    pa, pb = a.patches(), b.patches()
    for k in pa:
        assert torch.equal(pa[k], pb[k])
    ba, bb = a.bvh(), b.bvh()
    assert ba["root"] == bb["root"] and torch.equal(ba["nodes"], bb["nodes"]) and torch.equal(ba["tri"], bb["tri"])
    la, ra = a.vantage(vo)
    lb, rb = b.vantage(vo)
    assert torch.equal(la, lb) and torch.equal(ra, rb)
    xa = a.irradiance(la, vis_bits=True, fixups=1 << 16)
    xb = b.irradiance(la, vis_bits=True, fixups=1 << 16)
    a.sync_status()
    b.sync_status()
    assert torch.equal(xa["A"], xb["A"]) and torch.equal(xa["vis_bits"], xb["vis_bits"])
    assert xa["fixup_count"] == xb["fixup_count"]
    bad = img.clone()
    bad[:8] = 0
    with pytest.raises(uvd.UvdError) as e:
        uvd.Scene.from_image(bad)
    assert e.value.code == uvd.UVD_ERR_INVALID
    with pytest.raises(uvd.UvdError):
        uvd.Scene.from_image(img[:200].contiguous())


def test_lamp_outside_padding_range_is_reported(uvd):
    """A lamp farther than the scene's largest coordinate + 50 m (beyond what
    the fp32 box padding covers) or non-finite makes uvd_sync_status return
    INVALID; lamps inside the range do not."""
    c = configs.c2(2)
    sc = uvd.Scene(c["scene"])
    lamps, _ = sc.vantage(c["vantage"])
    sc.irradiance(lamps)
    sc.sync_status()
    for bad in (1000.0, float("nan")):
        far = lamps.clone()
        far[3, 0, 2] = bad
        sc.irradiance(far)
        with pytest.raises(Exception, match="validated range"):
            sc.sync_status()
        sc.sync_status()  # the flag was cleared by the read
    sc.close()
