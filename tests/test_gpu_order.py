"""The work order of k_assemble_lane (column-major, or super-tiles of tiles with
every column of a super-tile first, `item_to_tile` in csrc/assemble.cu) changes
only which warp computes an entry (UVD_ASM_SUPER = log2 of the tiles per
super-tile, < 0 column-major): A and the visibility bits are bit-identical
for every order, including a ragged last super-tile and a super-tile larger than
the column."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from synth import configs, ward  # noqa: E402


@pytest.fixture(scope="module")
def uvd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd as U
    return U


@pytest.mark.parametrize("super_log2", ["0", "1", "3", "16"])
def test_work_order_bit_identical(uvd, super_log2, monkeypatch):
    w = ward.ward(seed=7, n_bays=1, e=0.25)
    sc = uvd.Scene(w)
    lam, _ = sc.vantage(configs.vopts(configs.FLOAT3D, 0.6, 0.05))
    cols = list(range(0, lam.shape[0], 3))
    monkeypatch.setenv("UVD_ASM_SUPER", "-1")
    ref = sc.irradiance(lam, cols=cols, vis_bits=True)
    monkeypatch.setenv("UVD_ASM_SUPER", super_log2)
    got = sc.irradiance(lam, cols=cols, vis_bits=True)
    sc.sync_status()
    assert torch.equal(ref["A"], got["A"])
    assert torch.equal(ref["vis_bits"], got["vis_bits"])
    assert float(ref["A"].abs().sum()) > 0


def test_octant_copies_off_bit_identical(uvd, monkeypatch):
    """Scenes whose octant node copies would exceed their memory cap (or with
    UVD_OCT=0) traverse the one node array with a min/max per slab: the same
    boxes, hence the same decisions, bit for bit, for both models."""
    w = ward.ward(seed=8, n_bays=1, e=0.25)
    lam_opts = configs.vopts(configs.FLOAT3D, 0.6, 0.05)
    monkeypatch.delenv("UVD_OCT", raising=False)
    sc = uvd.Scene(w)
    lam, _ = sc.vantage(lam_opts)
    cols = list(range(0, lam.shape[0], 2))
    ref = sc.irradiance(lam, cols=cols, vis_bits=True)
    ref_area = sc.irradiance(lam, cols=cols[:6], area_subdiv=1)
    monkeypatch.setenv("UVD_OCT", "0")
    sc0 = uvd.Scene(w)
    got = sc0.irradiance(lam, cols=cols, vis_bits=True)
    got_area = sc0.irradiance(lam, cols=cols[:6], area_subdiv=1)
    sc.sync_status()
    sc0.sync_status()
    assert torch.equal(ref["A"], got["A"])
    assert torch.equal(ref["vis_bits"], got["vis_bits"])
    assert torch.equal(ref_area["A"], got_area["A"])


@pytest.mark.parametrize("cap", ["1", "5"])
def test_fixup_list_overflow_bit_identical(uvd, cap, monkeypatch):
    """Entries the fp32 pass leaves undecided go to a list re-traced by
    k_fixup_run; beyond the list's capacity they stay pending and
    k_fixup_overflow re-traces them.  Both routes give the same exact decisions
    (UVD_FIXUP_CAP shrinks the list to force the second)."""
    w = ward.ward(seed=9, n_bays=1, e=0.25)
    sc = uvd.Scene(w)
    lam, _ = sc.vantage(configs.vopts(configs.FLOAT3D, 0.5, 0.05))
    monkeypatch.delenv("UVD_FIXUP_CAP", raising=False)
    ref = sc.irradiance(lam, vis_bits=True, counters=True)
    assert int(ref["counters"][4]) > 5, "the scene must flag some entries for the exact re-trace"
    monkeypatch.setenv("UVD_FIXUP_CAP", cap)
    got = sc.irradiance(lam, vis_bits=True)
    sc.sync_status()
    assert torch.equal(ref["A"], got["A"])
    assert torch.equal(ref["vis_bits"], got["vis_bits"])


