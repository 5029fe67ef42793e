"""Structural pins of row a2 (the BVH) through uvd_scene_bvh: whatever tree the
builder makes, occlusion is exact only if (i) every triangle sits in exactly
one leaf, (ii) no node is reached twice from the root (a tree), (iii) every
child box contains all vertices of its subtree, (iv) the leaf-ordered
triangles are the input triangles, unchanged, and (v) the depth fits the
traversal stack (64).  Checked here on a 2.5D room, a small ward and C4."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from synth import configs, rooms, ward  # noqa: E402

LEAF = np.int64(0x80000000)


@pytest.fixture(scope="module")
def uvd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd as U
    return U


def check_tree(sc, input_tris=None):
    b = sc.bvh()
    words = b["nodes"].cpu().numpy()
    boxes = words.view(np.float32)
    refs = words[:, 12:14].astype(np.int64) & 0xFFFFFFFF
    tri = b["tri"].cpu().numpy()
    M = tri.shape[0]
    verts = tri.reshape(M, 3, 4)[:, :, :3]
    seen_tri = np.zeros(M, np.int32)
    seen_node = np.zeros(len(words), np.int32)
    # iterative DFS from the root with subtree vertex bounds checked bottom-up
    root = b["root"]
    assert root == 0
    stack = [(0, 1)]
    max_depth = 0
    lo_of = {}
    order = []
    while stack:
        n, dep = stack.pop()
        seen_node[n] += 1
        max_depth = max(max_depth, dep)
        order.append(n)
        for side in (0, 1):
            r = refs[n, side]
            if r & LEAF:
                start, cnt = (r & 0x7FFFFFFF) >> 3, (r & 7) + 1
                seen_tri[start:start + cnt] += 1
            else:
                assert r > n  # depth-first preorder: children after their parent
                stack.append((int(r), dep + 1))
    # collapsed subtrees (leaves of up to 2 triangles) leave some node records
    # unreferenced; a reached node is reached once, and reached nodes = leaves - 1
    n_leaves = int(((refs[seen_node == 1] & LEAF) != 0).sum())
    assert seen_node.max() == 1, "no node reached twice"
    assert int((seen_node == 1).sum()) == n_leaves - 1 or len(words) == 1
    assert (seen_tri == 1).all(), "every triangle in exactly one leaf"
    assert max_depth < 64
    # boxes contain their subtrees: compute subtree bounds in reverse preorder
    lo = np.full((len(words), 3), np.inf, np.float32)
    hi = np.full((len(words), 3), -np.inf, np.float32)
    for n in reversed(order):
        for side in (0, 1):
            r = refs[n, side]
            if r & LEAF:
                start, cnt = (r & 0x7FFFFFFF) >> 3, (r & 7) + 1
                v = verts[start:start + cnt].reshape(-1, 3)
                clo, chi = v.min(0), v.max(0)
            else:
                clo, chi = lo[int(r)], hi[int(r)]
            bx = boxes[n]
            if side == 0:
                blo = np.array([bx[0], bx[2], bx[8]]); bhi = np.array([bx[1], bx[3], bx[9]])
            else:
                blo = np.array([bx[4], bx[6], bx[10]]); bhi = np.array([bx[5], bx[7], bx[11]])
            if r & LEAF and cnt == 1 and len(words) == 1 and side == 1:
                continue  # the empty second child of a single-leaf tree
            assert (blo <= clo).all() and (bhi >= chi).all(), (n, side)
            lo[n] = np.minimum(lo[n], clo)
            hi[n] = np.maximum(hi[n], chi)
    if input_tris is not None:
        orig = tri[:, 7].view(np.int32)
        assert np.array_equal(np.sort(orig), np.arange(M))
        assert np.array_equal(verts[np.argsort(orig)], input_tris)
    return b


def test_bvh_room_2p5d(uvd):
    sc = uvd.Scene(rooms.random_room(3))
    check_tree(sc)


def test_bvh_small_ward(uvd):
    w = ward.ward(seed=4, n_bays=1, e=0.3)
    sc = uvd.Scene(w)
    check_tree(sc, w["vertices"][w["tris"]])


@pytest.mark.slow
def test_bvh_c4(uvd):
    w = configs.c4_scene()
    sc = uvd.Scene(w)
    check_tree(sc, w["vertices"][w["tris"]])


def test_bvh_tiny(uvd):
    s = 1.0 / 64
    V = np.array([[-s, -s, 0], [2 * s, -s, 0], [-s, 2 * s, 0]], np.float32)
    sc = uvd.Scene(dict(vertices=V, tris=np.array([[0, 1, 2]], np.int32)))
    b = sc.bvh()
    assert b["nodes"].shape[0] == 1


@pytest.mark.parametrize("builder", ["sah", "sah-chunked", "ploc", "karras"])
def test_builders_give_identical_matrices(uvd, builder, monkeypatch):
    """The three builders (binned SAH default, PLOC, Karras LBVH) make
    different trees; the occlusion decisions — hence A and the visibility bits
    in input row order — are identical (exact tests, tree-independent).
    "sah-chunked" forces the SAH builder's multi-CTA path for nodes above 1000
    triangles, in chunks of 300 positions (ragged last chunks)."""
    w = ward.ward(seed=5, n_bays=1, e=0.25)
    if builder == "sah-chunked":
        monkeypatch.setenv("UVD_SAH_HUGE", "1000")
        monkeypatch.setenv("UVD_SAH_CHUNK", "300")
        builder = "sah"
    monkeypatch.setenv("UVD_BVH", builder)
    sc = uvd.Scene(w)
    check_tree(sc, w["vertices"][w["tris"]])
    lam, _ = sc.vantage(configs.vopts(configs.FLOAT3D, 0.6, 0.05))
    r = sc.irradiance(lam)
    orig = sc.patches()["orig_id"].cpu().numpy()
    A = np.zeros((sc.N, lam.shape[0]), np.float32)
    A[orig] = r["A"][:, :sc.N].T.cpu().numpy()
    monkeypatch.setenv("UVD_BVH", "sah")
    monkeypatch.delenv("UVD_SAH_HUGE", raising=False)
    monkeypatch.delenv("UVD_SAH_CHUNK", raising=False)
    ref_sc = uvd.Scene(w)
    rr = ref_sc.irradiance(lam)
    ro = ref_sc.patches()["orig_id"].cpu().numpy()
    R = np.zeros_like(A)
    R[ro] = rr["A"][:, :ref_sc.N].T.cpu().numpy()
    assert np.array_equal(A, R)


def test_sah_chunked_same_tree(uvd, monkeypatch):
    """The multi-CTA (chunked) SAH path bins the same centroids into the same
    bins as the one-CTA path, and picks the split by the same sweep: the trees
    have the same SAH split decisions, so the same leaf order of triangles."""
    w = ward.ward(seed=6, n_bays=1, e=0.2)
    monkeypatch.setenv("UVD_BVH", "sah")
    a = uvd.Scene(w).bvh()
    monkeypatch.setenv("UVD_SAH_HUGE", "64")
    monkeypatch.setenv("UVD_SAH_CHUNK", "100")
    sc = uvd.Scene(w)
    b = check_tree(sc, w["vertices"][w["tris"]])
    # the leaf order can differ only where a bin's atomic box merge order differs
    # (it cannot: min / max are order-free), so the triangle order is identical
    ta = a["tri"].cpu().numpy()[:, 7].view(np.int32)
    tb = b["tri"].cpu().numpy()[:, 7].view(np.int32)
    assert np.array_equal(ta, tb)


@pytest.mark.parametrize("builder", ["sah", "ploc", "karras"])
def test_build_deterministic(uvd, builder, monkeypatch):
    """Every rank builds the scene from the same input: the build's
    atomics (bin counts, min/max, child-id allocation) must not leak into the
    result — two builds give byte-identical node arrays and triangle order."""
    w = ward.ward(seed=10, n_bays=1, e=0.25)
    monkeypatch.setenv("UVD_BVH", builder)
    monkeypatch.setenv("UVD_SAH_HUGE", "2000")  # exercise the multi-CTA levels too
    a = uvd.Scene(w).bvh()
    b = uvd.Scene(w).bvh()
    assert torch.equal(a["nodes"], b["nodes"])
    assert torch.equal(a["tri"], b["tri"])
