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
