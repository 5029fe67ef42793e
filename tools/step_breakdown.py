"""Per-phase timing of one bench step (host wall clock around synchronized
phases) to locate non-kernel time.  usage: python tools/step_breakdown.py [C5]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import configs, vectors  # noqa: E402

wl = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "C5")
dev = torch.device("cuda", 0)
V = torch.from_numpy(np.ascontiguousarray(wl["scene"]["vertices"], np.float32)).to(dev)
F = torch.from_numpy(np.ascontiguousarray(wl["scene"]["tris"], np.int32)).to(dev)
desc = dict(vertices=V, tris=F)
sc = uvd.Scene(desc)
lam, _ = sc.vantage(wl["vantage"])
N, K = sc.N, lam.shape[0]
A = torch.empty((K, sc.ld()), dtype=torch.float32, device=dev)
t = torch.from_numpy(vectors.sparse_plan(K)).to(dev)
ones = torch.ones(K, dtype=torch.float64, device=dev)
y = torch.from_numpy(vectors.row_weights(N)).to(dev)
sc.close()
for rep in range(3):
    T = {}
    def tick(name, t0):
        torch.cuda.synchronize()
        T[name] = time.perf_counter() - t0
        return time.perf_counter()
    t0 = time.perf_counter()
    sc = uvd.Scene(desc); t0 = tick("scene", t0)
    lam, _ = sc.vantage(wl["vantage"]); t0 = tick("vantage", t0)
    sc.irradiance(lam, out=A); t0 = tick("irradiance", t0)
    mu = uvd.fluence(A, N, t); t0 = tick("A.t", t0)
    rs = uvd.fluence(A, N, ones); t0 = tick("A.1", t0)
    g = uvd.fluence(A, N, y, transpose=True); t0 = tick("At.y", t0)
    cov = sc.coverage(mu, 280.0, rs); t0 = tick("coverage", t0)
    sc.sync_status(); sc.close(); t0 = tick("close", t0)
    print({k: round(v * 1e3, 1) for k, v in T.items()}, "ms")
