"""fp16 top-of-tree nodes (csrc/hnodes.cu): they change which boxes the walk
visits, never a decision.  The assembly with H nodes (default) and without
(UVD_HNODES=0, read per call) must give the same A and visibility bits bit for
bit, and the same fix-up entries (the fp32 triangle filter decides the same
rays), on scenes of each workload family, at several H depths."""
import os

import numpy as np
import pytest

from synth import configs, ward

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


def _assemble(sc, lamps, hnodes):
    old = os.environ.get("UVD_HNODES")
    os.environ["UVD_HNODES"] = "1" if hnodes else "0"
    try:
        r = sc.irradiance(lamps, vis_bits=True, fixups=1 << 22)
        sc.sync_status()
    finally:
        if old is None:
            os.environ.pop("UVD_HNODES")
        else:
            os.environ["UVD_HNODES"] = old
    fl = np.sort(r["fixups"].cpu().numpy().astype(np.uint64))
    return r["A"][:, :sc.N].cpu().numpy(), r["vis_bits"].cpu().numpy(), fl


CASES = {
    "c2": lambda: (configs.c2(1)["scene"], configs.c2(1)["vantage"]),
    "ward_float": lambda: (ward.ward(seed=4, n_bays=1, e=0.12), configs.FLOAT_OPTS),
    "ward_tower": lambda: (ward.ward(seed=5, n_bays=1, e=0.12), configs.TOWER_OPTS),
    "ward_arm": lambda: (ward.ward(seed=6, n_bays=1, e=0.12), configs.ARM_OPTS),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("depth", ["2", "6", "9"])
def test_hnodes_do_not_change_decisions(uvd, name, depth, monkeypatch):
    monkeypatch.setenv("UVD_HDEPTH", depth)  # read when the scene is built
    desc, vopts = CASES[name]()
    sc = uvd.Scene(desc)
    lamps, _ = sc.vantage(vopts)
    a0, v0, f0 = _assemble(sc, lamps, False)
    a1, v1, f1 = _assemble(sc, lamps, True)
    assert np.array_equal(v0, v1), "visibility bits differ with H nodes"
    assert np.array_equal(a0.view(np.uint32), a1.view(np.uint32)), "A differs with H nodes"
    assert np.array_equal(f0, f1), "fix-up entries differ with H nodes"
    sc.close()


def test_hnodes_survive_export_import(uvd):
    c = configs.c2(3)
    sc = uvd.Scene(c["scene"])
    lamps, _ = sc.vantage(c["vantage"])
    img = sc.export()
    sc2 = uvd.Scene.from_image(img)
    a0, v0, _ = _assemble(sc, lamps, True)
    a1, v1, _ = _assemble(sc2, lamps, True)
    assert np.array_equal(v0, v1) and np.array_equal(a0.view(np.uint32), a1.view(np.uint32))
