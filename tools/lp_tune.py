"""LP heuristic tuning runs on C4 Floatbot (development tool): one A, several
uvd_lp_solve runs under UVD_LP_* overrides (the library reads them per call).

usage: python tools/lp_tune.py [eps] [max_iter]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import configs  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-4
mx = int(sys.argv[2]) if len(sys.argv) > 2 else 60000
sc = uvd.Scene(configs.c4_scene())
lam, _ = sc.vantage(configs.FLOAT_OPTS)
a = sc.irradiance(lam, col_sumsq=True)
sc.sync_status()
p = 10.0 * float(np.sqrt(a["col_sumsq"].sum().item()))
variants = [json.loads(v) for v in sys.argv[3:]] if len(sys.argv) > 3 else [
    {}, {"UVD_LP_THETA": "0.2"}, {"UVD_LP_THETA": "0.8"}, {"UVD_LP_RHO": "0.5"}, {"UVD_LP_ART": "0.2"},
    {"UVD_LP_NEC": "0.9"}]
for var in variants:
    for k in ("UVD_LP_THETA", "UVD_LP_RHO", "UVD_LP_ART", "UVD_LP_NEC", "UVD_LP_SUFF"):
        os.environ.pop(k, None)
    os.environ.update(var)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = uvd.lp_solve(a["A"], sc.N, penalty=p, t_max=configs.T_MAX, eps=eps, max_iter=mx)
    dt = time.perf_counter() - t0
    print(json.dumps({"var": var, "status": r["status"], "it": r["iterations"], "s": round(dt, 1),
                      "obj": r["primal_obj"], "res": [r["rel_primal_res"], r["rel_dual_res"], r["rel_gap"]]}),
          flush=True)
