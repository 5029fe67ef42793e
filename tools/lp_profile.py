"""A short LP run on C4 Floatbot for ncu (development tool): builds A, then
one uvd_lp_solve of `iters` iterations without graphs (so every kernel is a
separate launch ncu can attribute).

usage: python tools/lp_profile.py [iters]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import configs  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = uvd.Scene(configs.c4_scene())
lam, _ = sc.vantage(configs.FLOAT_OPTS)
a = sc.irradiance(lam, col_sumsq=True)
sc.sync_status()
p = 10.0 * float(np.sqrt(a["col_sumsq"].sum().item()))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r = uvd.lp_solve(a["A"], sc.N, penalty=p, t_max=configs.T_MAX, eps=1e-12, max_iter=iters, check_every=32,
                 use_graph=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("iterations", r["iterations"], "obj", r["primal_obj"])
