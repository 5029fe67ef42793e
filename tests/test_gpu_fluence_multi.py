"""uvd_fluence_multi: μ = A·x, A·𝟙 and Aᵀ·y in one pass over A (a7).  Against
the single-product uvd_fluence calls on the same A: A·x and A·𝟙 bit for bit
when uvd_fluence does not split its columns (same column-order fp64 sums),
else within 1e-13,
Aᵀ·y within 1e-12 relative (row blocks summed in another fixed order); every
output subset, ragged sizes (n not a multiple of 4 or of the 2048-row block,
k not a multiple of the 8 columns in flight), determinism, an fp64 CPU
reference of the same products, and the argument checks."""
import numpy as np
import pytest

from synth import configs, vectors

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


def _rand_A(n, k, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    ld = (n + 31) // 32 * 32
    A = torch.rand((k, ld), generator=g, dtype=torch.float32)
    A[:, n:] = 0.0
    A[torch.rand((k, ld), generator=g) < 0.4] = 0.0  # occluded entries
    return A.cuda()


@pytest.mark.parametrize("n,k", [(1, 1), (5, 3), (2047, 9), (2049, 17), (4099, 64), (70001, 37)])
def test_multi_matches_single_products(uvd, n, k):
    A = _rand_A(n, k, n + k)
    x = torch.from_numpy(vectors.sparse_plan(k, seed=1)).cuda()
    y = torch.rand(n, dtype=torch.float64, device="cuda")
    ax, a1, aty = uvd.fluence_multi(A, n, x=x, y=y, rowsum=True)
    ref_ax = uvd.fluence(A, n, x)
    ref_a1 = uvd.fluence(A, n, torch.ones(k, dtype=torch.float64, device="cuda"))
    ref_g = uvd.fluence(A, n, y, transpose=True)
    if k < 16:  # uvd_fluence sums in one column chunk: the same order
        assert torch.equal(ax, ref_ax) and torch.equal(a1, ref_a1)
    assert torch.allclose(ax, ref_ax, rtol=1e-13, atol=0) and torch.allclose(a1, ref_a1, rtol=1e-13, atol=0)
    assert torch.allclose(aty, ref_g, rtol=1e-12, atol=0)
    # an independent fp64 reference
    Ad = A[:, :n].double().cpu().numpy()
    assert np.allclose(ax.cpu().numpy(), Ad.T @ x.cpu().numpy(), rtol=1e-12, atol=1e-300)
    assert np.allclose(a1.cpu().numpy(), Ad.sum(0), rtol=1e-12)
    assert np.allclose(aty.cpu().numpy(), Ad @ y.cpu().numpy(), rtol=1e-12)
    # deterministic
    ax2, a12, aty2 = uvd.fluence_multi(A, n, x=x, y=y, rowsum=True)
    assert torch.equal(ax, ax2) and torch.equal(a1, a12) and torch.equal(aty, aty2)


def test_multi_output_subsets(uvd):
    n, k = 5003, 21
    A = _rand_A(n, k, 7)
    x = torch.rand(k, dtype=torch.float64, device="cuda")
    y = torch.rand(n, dtype=torch.float64, device="cuda")
    full = uvd.fluence_multi(A, n, x=x, y=y, rowsum=True)
    for xx, yy, rs in ((x, None, False), (None, None, True), (None, y, False), (x, y, False), (None, y, True),
                       (x, None, True)):
        got = uvd.fluence_multi(A, n, x=xx, y=yy, rowsum=rs)
        for g, f, want in zip(got, full, (xx is not None, rs, yy is not None)):
            assert (g is not None) == want
            if want:
                assert torch.equal(g, f)


def test_multi_on_assembled_matrix(uvd):
    c = configs.c2(5)
    sc = uvd.Scene(c["scene"])
    lamps, _ = sc.vantage(c["vantage"])
    A = sc.irradiance(lamps)["A"]
    K, N = lamps.shape[0], sc.N
    t = torch.from_numpy(vectors.sparse_plan(K, seed=3)).cuda()
    y = torch.rand(N, dtype=torch.float64, device="cuda")
    mu, rs, g = uvd.fluence_multi(A, N, x=t, y=y, rowsum=True)
    assert torch.allclose(mu, uvd.fluence(A, N, t), rtol=1e-13, atol=0)
    assert torch.allclose(rs, uvd.fluence(A, N, torch.ones(K, dtype=torch.float64, device="cuda")), rtol=1e-13, atol=0)
    assert torch.allclose(g, uvd.fluence(A, N, y, transpose=True), rtol=1e-12, atol=0)


def test_multi_argument_checks(uvd):
    A = _rand_A(100, 4, 1)
    with pytest.raises(Exception):
        uvd.fluence_multi(A, 100)  # no output at all
    m = uvd._dense_desc(A)
    out = torch.empty(100, dtype=torch.float64, device="cuda")
    import ctypes as C
    rc = uvd.lib().uvd_fluence_multi(C.byref(m), 100, 4, None, None, C.c_void_p(out.data_ptr()), None, None, None)
    assert rc == uvd.UVD_ERR_INVALID  # A·x without x


def test_multi_fallback_matches(uvd, monkeypatch):
    """When the warp partials of Aᵀ·y would exceed the cap (4 GB; lowered here
    through UVD_MULTI_PART_MAX) the call runs one pass per product: results
    then equal the single-product calls bit for bit."""
    n, k = 3001, 40
    A = _rand_A(n, k, 9)
    x = torch.rand(k, dtype=torch.float64, device="cuda")
    y = torch.rand(n, dtype=torch.float64, device="cuda")
    monkeypatch.setenv("UVD_MULTI_PART_MAX", "64")
    ax, a1, aty = uvd.fluence_multi(A, n, x=x, y=y, rowsum=True)
    assert torch.equal(ax, uvd.fluence(A, n, x))
    assert torch.equal(a1, uvd.fluence(A, n, torch.ones(k, dtype=torch.float64, device="cuda")))
    assert torch.equal(aty, uvd.fluence(A, n, y, transpose=True))


def test_multi_empty_shapes(uvd):
    """An empty column shard (k = 0): A·x = A·𝟙 = 0 and Aᵀ·y is empty; n = 0:
    nothing to compute."""
    n = 70
    A = torch.zeros((0, 96), dtype=torch.float32, device="cuda")
    x = torch.zeros(0, dtype=torch.float64, device="cuda")
    y = torch.rand(n, dtype=torch.float64, device="cuda")
    ax, a1, aty = uvd.fluence_multi(A, n, x=x, y=y, rowsum=True)
    assert ax.shape == (n,) and a1.shape == (n,) and aty.shape == (0,)
    assert not ax.any() and not a1.any()
