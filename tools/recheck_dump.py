"""Offline parity re-check of uvd-shard/1 dumps (shard.dump_shard; bench.py
--dump): for every rank's shard, regenerate the seeded workload's scene, let
the fp64 oracle recompute the patches and the lamp samples of sampled
columns from their grid-candidate ids, and compare sampled entries (values
and visibility bits) — no GPU needed.  usage:
  python tools/recheck_dump.py PREFIX [--pairs N] [--seed S]"""
import argparse
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from oracle import parity  # noqa: E402
from paper_2103_14137_b200.shard import load_shard  # noqa: E402


def recheck(prefix, pairs=2000, seed=0):
    import bench
    ranks = sorted(int(p.rsplit(".rank", 1)[1][:-5]) for p in glob.glob(prefix + ".rank*.json"))
    if not ranks:
        raise SystemExit(f"no shards at {prefix}.rank*.json")
    out = []
    for rk in ranks:
        head, sec = load_shard(prefix, rk)
        wl = bench.workload(head["workload"])
        desc = wl["scene"]
        pat = O.scene_patches(desc)
        rng = np.random.default_rng(seed + rk)
        n = min(pairs, head["n_cols"] * head["n_rows"])
        ci = rng.integers(0, head["n_cols"], n)
        ri = rng.integers(0, head["n_rows"], n)
        uc, inv = np.unique(ci, return_inverse=True)
        raw = np.asarray(head["raw"], np.int64)[uc]
        ol = parity.oracle_lamps(desc, wl["vantage"], raw)
        assert (ol["feasible"] | ol["ambiguous"]).all(), "a dumped column the oracle rejects"
        assert np.array_equal(ol["samples"], np.asarray(sec["lamps"])[uc]), "lamp samples differ from the oracle's"
        gA = np.asarray(sec["A"])[ci, ri].astype(np.float64)
        L = head["L"]
        if "vis_bits" in sec:
            vb = np.asarray(sec["vis_bits"])
            gvis = np.stack([(vb[ci, l, ri // 32] >> (ri % 32).astype(np.uint32)) & 1 for l in range(L)], 1).astype(bool)
        else:  # values only: visibility inferred from A > 0 (L = 1)
            gvis = (gA > 0)[:, None]
        orig = np.asarray(sec["orig_id"])
        st = parity.compare_pairs(pat, ol["samples"], orig[ri], inv, gA, gvis, P=head["power_w"])
        st.pop("mismatch_at", None)
        st.pop("bad_at", None)
        st.update(rank=rk, workload=head["workload"], n_cols=head["n_cols"], n_rows=head["n_rows"])
        out.append(st)
        print(json.dumps(st), flush=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("prefix")
    ap.add_argument("--pairs", type=int, default=2000)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    res = recheck(a.prefix, a.pairs, a.seed)
    sys.exit(0 if all(r["mismatches"] == 0 for r in res) else 1)
