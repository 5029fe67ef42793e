"""The paper's §V-A comparison on the GPU (P:9): the 25 random
2.5D rooms, the LP-planned mobile lamp (NEXT-1, "time until full
disinfection": Eq. 9 with a non-binding budget) against the best static lamp
(NEXT-4: the configuration seeing the most area, left on until every patch it
sees has μ_min).  The paper reports 100 % vs 35 % coverage and ~2 orders of
magnitude more time for the static lamp.

usage: python tools/compare_static.py [--rooms 25] [--grid 0.25] [--out profiles/static_r01.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import configs, rooms  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rooms", type=int, default=25)
    ap.add_argument("--grid", type=float, default=0.25)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for seed in range(a.rooms):
        sc = uvd.Scene(rooms.random_room(seed, 4.0))
        lam, _ = sc.vantage(configs.vopts(configs.DISC2D, a.grid, 0.15, lamp_z=1.0))
        K = int(lam.shape[0])
        r = sc.irradiance(lam, col_sumsq=True)
        sc.sync_status()
        A = r["A"]
        ones = torch.ones(K, dtype=torch.float64, device="cuda")
        rowsum = uvd.fluence(A, sc.N, ones)
        total = sc.coverage(rowsum, 1e300, rowsum)  # [0, total area, ever-visible area]
        # mobile: LP plan, budget not binding ("time until full disinfection")
        p = 10.0 * float(np.sqrt(r["col_sumsq"].sum().item()))
        plan = uvd.lp_solve(A, sc.N, penalty=p, t_max=1e7, eps=1e-7, max_iter=400000)
        mu = uvd.fluence(A, sc.N, plan["t"])
        cov_m = sc.coverage(mu * (1 + 1e-6), configs.MU_MIN, rowsum)  # tolerance of the LP's eps
        # static: the best single configuration, left on until its visible patches reach μ_min
        st = sc.static_baseline(A, t_budget=configs.T_MAX)
        j = st["column"]
        tj = torch.zeros(K, dtype=torch.float64, device="cuda")
        tj[j] = st["dwell_s"]
        cov_s = sc.coverage(uvd.fluence(A, sc.N, tj) * (1 + 1e-12), configs.MU_MIN, rowsum)
        rows.append({"seed": seed, "N": sc.N, "K": K, "total_area": total[1], "visible_area": total[2],
                     "mobile_cov_total": cov_m[0] / cov_m[1], "mobile_cov_visible": cov_m[0] / cov_m[2],
                     "mobile_dwell_s": plan["sum_t"], "lp_status": plan["status"],
                     "static_cov_total": cov_s[0] / cov_s[1], "static_cov_visible": cov_s[0] / cov_s[2],
                     "static_dwell_s": st["dwell_s"], "static_column": j})
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in rows[-1].items()}), flush=True)
    summ = {k: float(np.mean([r[k] for r in rows])) for k in
            ("mobile_cov_total", "mobile_cov_visible", "static_cov_total", "static_cov_visible")}
    summ["median_time_ratio_static_over_mobile"] = float(np.median([r["static_dwell_s"] / r["mobile_dwell_s"]
                                                                    for r in rows]))
    print(json.dumps(summ))
    if a.out:
        json.dump({"grid_m": a.grid, "rooms": rows, "summary": summ}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
