"""Measured parity at full size: for each workload, one
full assembly in the bench's launch configuration, then the fp64 oracle on
(a) uniformly random (patch, configuration) pairs and (b) entries drawn from
the library's fix-up list (the rays the fp32 pass left undecided).  Reports
mismatches, the degenerate fraction (gate < 1e-4) and the max relative error.

usage: python tools/parity_sample.py [out.json] [--c4 N] [--tower N] [--c5 N] [--fix N]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import parity  # noqa: E402
from synth import configs  # noqa: E402


def run(uvd, name, desc, vopts, n_rand, n_fix, seed):
    t0 = time.time()
    sc = uvd.Scene(desc)
    lamps, raw = sc.vantage(vopts)
    K, L = lamps.shape[0], lamps.shape[1]
    r = sc.irradiance(lamps, vis_bits=True, fixups=1 << 24)
    sc.sync_status()
    orig = sc.patches()["orig_id"].cpu().numpy()
    fl = r["fixups"].cpu().numpy().astype(np.uint64)
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(fl), min(n_fix, len(fl)), replace=False)
    sets = {"random": (rng.integers(0, K, n_rand), rng.integers(0, sc.N, n_rand)),
            "fixup": ((fl[pick] >> np.uint64(32)).astype(np.int64), (fl[pick] & np.uint64(0xffffffff)).astype(np.int64))}
    pat = O.scene_patches(desc)
    vb = r["vis_bits"].cpu().numpy().view(np.uint32)
    res = {"workload": name, "N": sc.N, "K": K, "L": L, "entries": sc.N * K, "fixup_count": r["fixup_count"],
           "fixup_fraction": r["fixup_count"] / (sc.N * K)}
    for nm, (ci, ri) in sets.items():
        gA = r["A"][torch.from_numpy(ci).cuda(), torch.from_numpy(ri).cuda()].double().cpu().numpy()
        gvis = np.stack([(vb[ci, l, ri // 32] >> (ri % 32).astype(np.uint32)) & 1 for l in range(L)], 1).astype(bool)
        uc, inv = np.unique(ci, return_inverse=True)
        ol = parity.oracle_lamps(desc, vopts, raw.cpu().numpy()[uc])
        ok_cols = ol["feasible"] | ol["ambiguous"]
        assert ok_cols.all() and np.array_equal(ol["samples"], lamps.cpu().numpy()[uc])
        st = parity.compare_pairs(pat, ol["samples"], orig[ri], inv, gA, gvis)
        st.pop("mismatch_at", None)
        st.pop("bad_at", None)
        res[nm] = st
    res["seconds"] = time.time() - t0
    sc.close()
    del r
    torch.cuda.empty_cache()
    print(json.dumps(res), flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default=os.path.join(ROOT, "gpurun_out", "parity.json"))
    ap.add_argument("--c4", type=int, default=100000)
    ap.add_argument("--tower", type=int, default=20000)
    ap.add_argument("--c5", type=int, default=20000)
    ap.add_argument("--fix", type=int, default=2000)
    a = ap.parse_args()
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd
    out = {"threads": O.default_threads(), "runs": []}
    out["runs"].append(run(uvd, "C4 Floatbot", configs.c4_scene(), configs.FLOAT_OPTS, a.c4, a.fix, 1))
    out["runs"].append(run(uvd, "C4 Towerbot (L=10)", configs.c4_scene(), configs.TOWER_OPTS, a.tower, a.fix, 2))
    out["runs"].append(run(uvd, "C5 Armbot", configs.c5_scene(), configs.ARM_OPTS, a.c5, a.fix, 3))
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
