"""Traversal statistics of k_assemble_lane's walk (tools/walkstats.c) on
sampled work items of a workload: visits per ray by node depth and the union
of nodes a work item's 32 lanes visit (what a warp-shared traversal of those
levels would still have to visit).  usage: python tools/walkstats.py [C5|C4-float] [n_items]"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import __graft_entry__  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    n_items = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd
    wl = bench.workload(name)
    sc = uvd.Scene(wl["scene"])
    lam, _ = sc.vantage(wl["vantage"])
    assert lam.shape[1] == 1
    b = sc.bvh()
    p = sc.patches()
    d = tempfile.mkdtemp()
    files = {}
    for k, t in (("nodes", b["nodes"]), ("tri", b["tri"]), ("cen", p["centroid"]), ("nrm", p["normal"]),
                 ("lamps", lam[:, 0, :].contiguous())):
        files[k] = os.path.join(d, k + ".bin")
        t.cpu().numpy().tofile(files[k])
    K, N = lam.shape[0], sc.N
    rng = np.random.default_rng(0)
    items = np.stack([rng.integers(0, K, n_items), rng.integers(0, (N + 31) // 32, n_items)], 1).astype(np.int64)
    files["items"] = os.path.join(d, "items.bin")
    items.tofile(files["items"])
    exe = os.path.join(d, "walkstats")
    defs = [a for a in os.environ.get("WALKSTATS_DEFS", "").split() if a]
    subprocess.check_call(["gcc", "-O2", *defs, "-o", exe, os.path.join(ROOT, "tools", "walkstats.c"), "-lm"])
    out = subprocess.check_output([exe, files["nodes"], files["tri"], files["cen"], files["nrm"], files["lamps"],
                                   files["items"], str(N), str(sc.M), str(b["nodes"].shape[0]), str(K),
                                   str(b["root"]), str(n_items)], text=True)
    res = json.loads(out)
    res["workload"] = wl["name"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
