"""Host-time diagnosis of the coverage / sync_status / close tail of a step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import vectors  # noqa: E402

wl = bench.workload("C5")
dev = torch.device("cuda", 0)
V = torch.from_numpy(np.ascontiguousarray(wl["scene"]["vertices"], np.float32)).to(dev)
F = torch.from_numpy(np.ascontiguousarray(wl["scene"]["tris"], np.int32)).to(dev)
desc = dict(vertices=V, tris=F)
sc = uvd.Scene(desc)
lam, _ = sc.vantage(wl["vantage"])
N, K = sc.N, lam.shape[0]
cols = list(range(K))
A = torch.empty((K, sc.ld()), dtype=torch.float32, device=dev)
t = torch.from_numpy(vectors.sparse_plan(K)).to(dev)
ones = torch.ones(K, dtype=torch.float64, device=dev)
sc.close()
for rep in range(4):
    sc = uvd.Scene(desc)
    lam, _ = sc.vantage(wl["vantage"])
    sc.irradiance(lam, cols=cols, out=A)
    mu = uvd.fluence(A, N, t)
    rs = uvd.fluence(A, N, ones)
    torch.cuda.synchronize()
    h = {}
    t0 = time.perf_counter(); cov = sc.coverage(mu, 280.0, rs); h["coverage"] = time.perf_counter() - t0
    t0 = time.perf_counter(); sc.sync_status(); h["sync_status"] = time.perf_counter() - t0
    t0 = time.perf_counter(); sc.close(); h["close"] = time.perf_counter() - t0
    t0 = time.perf_counter(); torch.cuda.synchronize(); h["sync"] = time.perf_counter() - t0
    print({k: round(v * 1e3, 2) for k, v in h.items()}, "ms", flush=True)
