"""Hard-case parity at full size (VERDICT r1 "What's missing" 2): the entries
the fp32 traversal left undecided — the ones k_fixup re-traces with exact fp64
triangle tests, ≈0.05 % of C5's entries — drawn from the library's own fix-up
list (uvd_matrix_out.fixup_list) at the bench's launch configuration, checked
one by one against the fp64 oracle (P:242 visibility, S:121 agreement with a
brute-force oracle outside the degenerate set).  Plus the degenerate fraction
measured on random pairs of the same launches (gate < 1e-4, north_star).
"""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import parity
from synth import configs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

DEG_GATE = 1e-4


@pytest.fixture(scope="module")
def uvd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd as U
    return U


def _gpu_pick(r, ci, ri, L):
    """GPU values and visibility bits of local (column, row) pairs."""
    gA = r["A"][torch.from_numpy(ci).cuda(), torch.from_numpy(ri).cuda()].double().cpu().numpy()
    vb = r["vis_bits"].cpu().numpy().view(np.uint32)
    gvis = np.stack([(vb[ci, l, ri // 32] >> (ri % 32).astype(np.uint32)) & 1 for l in range(L)], 1).astype(bool)
    return gA, gvis


def _run(uvd, desc, vopts, n_fix, n_rand, seed, cols_frac=None):
    sc = uvd.Scene(desc)
    lamps, raw = sc.vantage(vopts)
    K, L = lamps.shape[0], lamps.shape[1]
    rng = np.random.default_rng(seed)
    cols = None
    if cols_frac is not None:
        cols = np.sort(rng.choice(K, max(1, int(K * cols_frac)), replace=False))
    r = sc.irradiance(lamps, cols=cols, vis_bits=True, fixups=1 << 24)
    sc.sync_status()
    orig = sc.patches()["orig_id"].cpu().numpy()
    n_cols = r["A"].shape[0]
    fl = r["fixups"].cpu().numpy().astype(np.uint64)
    assert r["fixup_count"] == len(fl) > 0
    # the list holds distinct, in-range entries
    fc, fr = (fl >> np.uint64(32)).astype(np.int64), (fl & np.uint64(0xffffffff)).astype(np.int64)
    assert (fc < n_cols).all() and (fr < sc.N).all() and len(np.unique(fl)) == len(fl)
    pick = rng.choice(len(fl), min(n_fix, len(fl)), replace=False)
    sets = {"fixup": (fc[pick], fr[pick]),
            "random": (rng.integers(0, n_cols, n_rand), rng.integers(0, sc.N, n_rand))}
    gcol_all = np.arange(K) if cols is None else cols
    pat = O.scene_patches(desc)
    out = {}
    for name, (ci, ri) in sets.items():
        gA, gvis = _gpu_pick(r, ci, ri, L)
        gcol = gcol_all[ci]
        uc, inv = np.unique(gcol, return_inverse=True)
        ol = parity.oracle_lamps(desc, vopts, raw.cpu().numpy()[uc])
        # the GPU's columns are the oracle's feasible candidates (or ambiguous ones)
        assert (ol["feasible"] | ol["ambiguous"]).all()
        assert np.array_equal(ol["samples"], lamps.cpu().numpy()[uc])
        st = parity.compare_pairs(pat, ol["samples"], orig[ri], inv, gA, gvis)
        assert st["mismatches"] == 0, (name, st)
        assert st["entries_beyond_tol"] == 0, (name, st)
        out[name] = st
    print({k: {q: v[q] for q in ("pairs", "rays", "degenerate_rays", "degenerate_cos", "degenerate_margin",
                                 "degenerate_fraction", "max_rel_err", "visible_fraction")} for k, v in out.items()},
          "fixup_count", r["fixup_count"], "entries", sc.N * n_cols)
    assert out["random"]["degenerate_fraction"] < DEG_GATE
    sc.close()
    return out, r["fixup_count"]


def test_c4_towerbot_fixups(uvd):
    out, n = _run(uvd, configs.c4_scene(), configs.TOWER_OPTS, 2000, 3000, 11)
    # the undecided entries are where the degenerate rays live: most fix-up
    # entries are still decidable (and decided correctly), some are degenerate
    assert out["fixup"]["entries_checked"] > 0.5 * out["fixup"]["pairs"]


def test_c4_floatbot_fixups(uvd):
    out, n = _run(uvd, configs.c4_scene(), configs.FLOAT_OPTS, 2000, 20000, 12)
    assert out["fixup"]["entries_checked"] > 0.5 * out["fixup"]["pairs"]


@pytest.mark.slow
def test_c5_armbot_fixups(uvd):
    """The bench workload (all 12 546 columns, one launch)."""
    out, n = _run(uvd, configs.c5_scene(), configs.ARM_OPTS, 2000, 4000, 13)
    assert out["fixup"]["entries_checked"] > 0.5 * out["fixup"]["pairs"]
