"""GPU parity of NEXT-1, the relaxed dwell-time LP (Eq. 9), through
the C-ABI (uvd_lp_solve), against the HiGHS oracle (`oracle/lp.py`).

The LP optimum value is unique but the optimal (t, σ) need not be (Q17), so
the bar is: the GPU objective equals the oracle's within 1e-5 relative, the
GPU point is feasible for the oracle's own A within 1e-5 relative (every
coverage row, the budget), and the GPU's reported KKT residuals meet its eps.
Inputs: seeded synthetic matrices (fp32 values, the same numbers on both
sides) and the C3 worlds end to end (GPU scene → GPU A → GPU LP vs oracle A →
HiGHS).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
pytest.importorskip("scipy")

from oracle import lp as OLP  # noqa: E402
from oracle import oracle as O  # noqa: E402
from synth import configs  # noqa: E402

REL_OBJ = 1e-5


@pytest.fixture(scope="module")
def uvd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd as U
    return U


def dense_gpu(A_nk):
    """(N, K) fp32 numpy -> the library's dense layout: (K, ld) with ld = N rounded to 32."""
    n, k = A_nk.shape
    ld = (n + 31) // 32 * 32
    out = torch.zeros((k, ld), dtype=torch.float32)
    out[:, :n] = torch.from_numpy(np.ascontiguousarray(A_nk.T))
    return out.cuda()


def synth_matrix(seed, n, k, density=0.5, zero_rows=0):
    rng = np.random.default_rng(seed)
    A = (rng.uniform(0.0, 8.0, (n, k)) * (rng.uniform(size=(n, k)) < density)).astype(np.float32)
    A[np.arange(n), rng.integers(0, k, n)] += rng.uniform(0.5, 2.0, n).astype(np.float32)  # every patch seen...
    if zero_rows:
        A[:zero_rows] = 0.0  # ...except `zero_rows` invisible ones
    return A


def check(uvd, A32, mu_min, p, t_max, eps=1e-8, **kw):
    n, k = A32.shape
    r = uvd.lp_solve(dense_gpu(A32), n, mu_min=mu_min, t_max=t_max, penalty=p, eps=eps, **kw)
    ref = OLP.solve(A32.astype(np.float64), mu_min, p, t_max)
    assert r["status"] == 0, r
    t, s = r["t"].cpu().numpy(), r["sigma"].cpu().numpy()
    y, yb = r["y"].cpu().numpy(), float(r["y_budget"].cpu().numpy()[0])
    kk = OLP.kkt(A32.astype(np.float64), mu_min, p, t_max, t, s, y, yb)
    scale = 1.0 + abs(ref["obj"])
    assert abs(kk["primal_obj"] - ref["obj"]) <= REL_OBJ * scale, (kk["primal_obj"], ref["obj"])
    assert abs(kk["dual_obj"] - ref["obj"]) <= REL_OBJ * scale
    qn = np.sqrt(n * mu_min ** 2 + t_max ** 2)
    assert kk["primal_res"] <= REL_OBJ * (1 + qn)
    assert max(r["rel_primal_res"], r["rel_dual_res"], r["rel_gap"]) <= eps
    return r, ref, t, s


def test_lp_one_patch_printed_dwell(uvd):
    """I = 6.3662 W/m², μ_min = 280 → t = 43.98 s, σ = 0."""
    A = np.array([[6.3662]], np.float32)
    r, ref, t, s = check(uvd, A, 280.0, 1e3, 1e6)
    assert abs(t[0] - 43.98) < 5e-3 and s[0] < 1e-6


def test_lp_closed_forms(uvd):
    """Diagonal instance t_k = μ_min/A_kk; budget-bound single patch t = T_max, σ = μ_min − I·T_max."""
    d = np.array([1.0, 2.0, 4.0, 8.0], np.float32)
    r, ref, t, s = check(uvd, np.diag(d), 280.0, 100.0, 1e6)
    assert np.allclose(t, 280.0 / d, rtol=1e-6)
    r, ref, t, s = check(uvd, np.array([[2.0]], np.float32), 280.0, 10.0, 100.0)
    assert abs(t[0] - 100.0) < 1e-4 and abs(s[0] - 80.0) < 1e-4


def test_lp_invisible_patches_take_full_slack(uvd):
    """rows seen from no vantage end with σ_i = μ_min."""
    A = synth_matrix(1, 120, 24, zero_rows=3)
    r, ref, t, s = check(uvd, A, 280.0, 50.0, 1e6)
    assert np.allclose(s[:3], 280.0, rtol=1e-6)


@pytest.mark.parametrize("seed,n,k,t_max", [(2, 200, 40, 1e6), (3, 500, 64, 300.0), (4, 333, 17, 1e6),
                                            (5, 64, 200, 1800.0)])
def test_lp_random_instances(uvd, seed, n, k, t_max):
    A = synth_matrix(seed, n, k, density=0.3)
    p = 10.0 * float(np.linalg.norm(A.astype(np.float64)))
    r, ref, t, s = check(uvd, A, 280.0, p, t_max)
    if t_max < 1e5:
        assert r["sum_t"] <= t_max * (1 + 1e-6)


def test_lp_graph_and_stream_launches_identical(uvd):
    """The CUDA-graph replay and plain launches run the same kernels in the same
    order: bit-identical results."""
    A = synth_matrix(6, 300, 48, density=0.4)
    g = dense_gpu(A)
    s = torch.cuda.Stream()
    a = uvd.lp_solve(g, 300, penalty=100.0, eps=1e-7, use_graph=True, stream=s)
    b = uvd.lp_solve(g, 300, penalty=100.0, eps=1e-7, use_graph=False, stream=s)
    torch.cuda.synchronize()
    assert a["iterations"] == b["iterations"]
    assert torch.equal(a["t"], b["t"]) and torch.equal(a["y"], b["y"]) and torch.equal(a["sigma"], b["sigma"])


def test_lp_penalty_vector_and_csc(uvd):
    """Per-patch penalties (prioritised patches) as a device vector, and
    the CSC form of A, reach the oracle's optimum."""
    n, k = 150, 30
    A = synth_matrix(7, n, k, density=0.3, zero_rows=2)
    rng = np.random.default_rng(7)
    p = rng.uniform(5.0, 50.0, n)
    r = uvd.lp_solve(dense_gpu(A), n, penalty=torch.from_numpy(p).cuda(), t_max=400.0, eps=1e-8)
    ref = OLP.solve(A.astype(np.float64), 280.0, p, 400.0)
    assert abs(r["primal_obj"] - ref["obj"]) <= REL_OBJ * (1 + ref["obj"])
    cols = [np.nonzero(A[:, j])[0] for j in range(k)]
    colptr = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    csc = {"colptr": torch.from_numpy(colptr).cuda(),
           "rowidx": torch.from_numpy(np.concatenate(cols).astype(np.int32)).cuda(),
           "values": torch.from_numpy(np.concatenate([A[c, j] for j, c in enumerate(cols)])).cuda(),
           "nnz": int(colptr[-1])}
    rc = uvd.lp_solve(csc, n, penalty=torch.from_numpy(p).cuda(), t_max=400.0, eps=1e-8)
    assert abs(rc["primal_obj"] - ref["obj"]) <= REL_OBJ * (1 + ref["obj"])


def test_lp_c3_end_to_end(uvd):
    """C3 worlds end to end: GPU scene → GPU A → GPU LP, against oracle A →
    HiGHS, with p = 10‖A‖_F and T_max = 30 min."""
    for seed in range(4):
        c = configs.c3(seed)
        sc = uvd.Scene(c["scene"])
        lam, _ = sc.vantage(c["vantage"])
        r = sc.irradiance(lam, col_sumsq=True)
        sc.sync_status()
        fro = float(np.sqrt(r["col_sumsq"].sum().item()))
        N = sc.N
        res = uvd.lp_solve(r["A"], N, penalty=10.0 * fro, t_max=configs.T_MAX, eps=1e-8)
        assert res["status"] == 0
        pat = O.extruded_patches(c["scene"])
        v = O.vantage(c["scene"], c["vantage"])
        lam_o = v["samples"][v["feasible"]]  # the oracle's own vantage set ...
        assert np.array_equal(lam_o, lam.cpu().numpy())  # ... identical to the GPU's
        ref_A = O.irradiance_matrix(pat, lam_o, mode="2d")
        assert not ref_A["deg"].any()
        An = ref_A["A"]  # (N, K) in the oracle's (input) row order
        ref = OLP.solve(An, configs.MU_MIN, 10.0 * np.linalg.norm(An), configs.T_MAX)
        assert abs(res["primal_obj"] - ref["obj"]) <= REL_OBJ * (1 + ref["obj"]), (seed, res, ref["obj"])
        # the GPU plan is feasible for the oracle's A (rows mapped to input order)
        orig = sc.patches()["orig_id"].cpu().numpy()
        sig = np.zeros(N)
        sig[orig] = res["sigma"].cpu().numpy()
        t = res["t"].cpu().numpy()
        viol = np.maximum(0.0, configs.MU_MIN - An @ t - sig)
        assert viol.max() <= 1e-4 * configs.MU_MIN


def test_lp_two_column_shards(uvd):
    """Multi-process path of uvd_lp_solve (columns sharded) exercised by
    two solver threads on two streams of this one GPU: the allreduce callback
    sums the two shards' partials through host memory behind a host barrier (no
    kernel ever waits on another).  The sharded solve reaches the single-process
    objective; the union of the shards' dwell times is a feasible plan."""
    import threading
    n, k = 240, 36
    A = synth_matrix(9, n, k, density=0.35, zero_rows=1)
    p = 10.0 * float(np.linalg.norm(A.astype(np.float64)))
    ref = OLP.solve(A.astype(np.float64), 280.0, p, 300.0)
    shards = [[j for j in range(k) if (j // 4) % 2 == r] for r in range(2)]
    bar = threading.Barrier(2)
    slots = [None, None]
    out = [None, None]

    def reducer(rank):
        def red(x, op):
            torch.cuda.current_stream().synchronize()
            slots[rank] = x.cpu()
            bar.wait()
            o = slots[1 - rank]
            tot = torch.maximum(slots[rank], o) if op == "max" else (slots[0] + slots[1])  # same order on both
            bar.wait()
            x.copy_(tot.to(x.device))
            torch.cuda.current_stream().synchronize()
        return red

    def run(rank):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            g = dense_gpu(np.ascontiguousarray(A[:, shards[rank]]))
            out[rank] = uvd.lp_solve(g, n, penalty=p, t_max=300.0, eps=1e-8, allreduce=reducer(rank), stream=s)
            s.synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert out[0] is not None and out[1] is not None
    assert out[0]["status"] == 0 and out[0]["iterations"] == out[1]["iterations"]
    assert abs(out[0]["primal_obj"] - ref["obj"]) <= REL_OBJ * (1 + ref["obj"])
    assert out[0]["primal_obj"] == out[1]["primal_obj"]
    t = np.zeros(k)
    for r in range(2):
        t[shards[r]] = out[r]["t"].cpu().numpy()
    assert t.sum() <= 300.0 * (1 + 1e-6)
    s = out[0]["sigma"].cpu().numpy()
    viol = np.maximum(0.0, 280.0 - A.astype(np.float64) @ t - s)
    assert viol.max() <= 1e-4 * 280.0


def test_lp_degenerate_inputs(uvd):
    """No light at all (an all-zero A, and an empty column shard): every patch
    takes the full slack σ = μ_min, t = 0, objective p·N·μ_min; a bad
    argument fails loudly."""
    n = 40
    r = uvd.lp_solve(dense_gpu(np.zeros((n, 5), np.float32)), n, penalty=3.0, t_max=100.0, eps=1e-9)
    assert r["status"] == 0
    assert np.allclose(r["sigma"].cpu().numpy(), 280.0, rtol=1e-7) and not r["t"].cpu().numpy().any()
    assert abs(r["primal_obj"] - 3.0 * n * 280.0) <= 1e-6 * 3.0 * n * 280.0
    empty = torch.zeros((0, 64), dtype=torch.float32, device="cuda")
    r = uvd.lp_solve(empty, n, penalty=3.0, t_max=100.0, eps=1e-9)
    assert np.allclose(r["sigma"].cpu().numpy(), 280.0, rtol=1e-7)
    with pytest.raises(uvd.UvdError):
        uvd.lp_solve(dense_gpu(np.ones((n, 5), np.float32)), n, penalty=-1.0)
