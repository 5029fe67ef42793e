"""Run k_assemble on a column subset of a workload (for ncu captures).

usage: python tools/profile_assemble.py [C5|C4-float|C4-tower] [n_cols] [repeats]
env: CONTIG=1 contiguous middle columns; AREA=m the NEXT-2 area model at subdivision m
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_14137_b200 import uvd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n_cols = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl = bench.workload(name)
sc = uvd.Scene(wl["scene"])
lamps, _ = sc.vantage(wl["vantage"])
K = lamps.shape[0]
if os.environ.get("CONTIG"):
    s0 = K // 3
    cols = list(range(s0, min(K, s0 + n_cols)))
else:
    step = max(1, K // n_cols)
    cols = list(range(0, K, step))[:n_cols]
A = torch.empty((len(cols), sc.ld()), dtype=torch.float32, device="cuda")
area = int(os.environ["AREA"]) if os.environ.get("AREA") else None
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(reps):
    e0.record()
    sc.irradiance(lamps, cols=cols, out=A, area_subdiv=area)
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {r}: {e0.elapsed_time(e1):.2f} ms for {len(cols)} cols x {sc.N} rows "
          f"= {len(cols) * sc.N / e0.elapsed_time(e1) / 1e6:.3f} G entries/s")
sc.sync_status()
r = sc.irradiance(lamps, cols=cols, out=A, counters=True, area_subdiv=area)
print("counters (rays, box tests, tri tests, node fetches, fp64 fixups, cache hits):", r["counters"].tolist())
