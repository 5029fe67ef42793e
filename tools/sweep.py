"""NEXT-4 resolution sweeps (PAPER App. II) on the GPU: the
paper's two 2.5D experiments over the 25 random rooms and its 3D grid sweep,
reusing the hot path (scene → vantage → A) and NEXT-1 (the LP).

* env-res: wall patch resolution 1/2 … 1/32 m at a 0.1 m grid;
* grid:    vantage grid 1/2 … 1/32 m at the 1/8 m "balanced" patch resolution;
* 3d:      Floatbot grid spacing 1000 … 250 mm on the C4 ward, 30-minute budget.

For each point: assembly time and entries/s (the throughput curve), the LP's
total dwell for full disinfection of the visible patches (Eq. 9 with a loose
budget) or the 30-minute coverage, normalised per room by the coarsest
resolution as the paper plots them (mean ± std over rooms).

usage: python tools/sweep.py [--rooms 25] [--no-3d] [--out profiles/sweep_r01.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import configs, rooms  # noqa: E402


def run_one(scene, vopts, t_max, eps):
    sc = uvd.Scene(scene)
    lam, _ = sc.vantage(vopts)
    K = int(lam.shape[0])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a = sc.irradiance(lam, col_sumsq=True)
    e1.record()
    sc.sync_status()
    ms = e0.elapsed_time(e1)
    A = a["A"]
    p = 10.0 * float(np.sqrt(a["col_sumsq"].sum().item()))
    rowsum = uvd.fluence(A, sc.N, torch.ones(K, dtype=torch.float64, device="cuda"))
    t0 = time.perf_counter()
    r = uvd.lp_solve(A, sc.N, penalty=p, t_max=t_max, eps=eps, max_iter=400000)
    lp_s = time.perf_counter() - t0
    mu = uvd.fluence(A, sc.N, r["t"])
    cov = sc.coverage(mu, configs.MU_MIN, rowsum)
    return {"N": sc.N, "K": K, "assemble_ms": ms, "entries_per_s": sc.N * K / (ms / 1e3),
            "dwell_s": r["sum_t"], "nnz_t": int((r["t"] > 0).sum().item()), "lp_status": r["status"],
            "lp_iterations": r["iterations"], "lp_s": lp_s,
            "coverage_total": cov[0] / cov[1], "coverage_visible": cov[0] / cov[2]}


def summarise(rows_by_level, key):
    """per-room normalisation by the first (coarsest) level, then mean/std per level"""
    levels = list(rows_by_level)
    base = np.array([r[key] for r in rows_by_level[levels[0]]])
    out = {}
    for lv in levels:
        v = np.array([r[key] for r in rows_by_level[lv]]) / base
        out[str(lv)] = {"mean": float(v.mean()), "std": float(v.std())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rooms", type=int, default=25)
    ap.add_argument("--no-3d", action="store_true")
    ap.add_argument("--eps", type=float, default=1e-7)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = {"gpu": torch.cuda.get_device_name(0), "rooms": a.rooms}
    loose = 1e6  # "time until full disinfection": the budget does not bind
    res_levels = [0.5, 0.25, 0.125, 0.0625, 0.03125]
    env = {lv: [] for lv in res_levels}
    for seed in range(a.rooms):
        for lv in res_levels:
            sc = rooms.random_room(seed, 4.0, patch_res=lv)
            env[lv].append(run_one(sc, configs.vopts(configs.DISC2D, 0.1, 0.15, lamp_z=1.0), loose, a.eps))
        print("env-res room", seed, [round(env[lv][-1]["dwell_s"], 1) for lv in res_levels], flush=True)
    out["env_res"] = {"levels_m": res_levels, "grid_m": 0.1,
                      "dwell_norm": summarise(env, "dwell_s"),
                      "raw": {str(k): v for k, v in env.items()}}
    grid_levels = [0.5, 0.25, 0.125, 0.0625, 0.03125]
    grid = {lv: [] for lv in grid_levels}
    for seed in range(a.rooms):
        for lv in grid_levels:
            sc = rooms.random_room(seed, 4.0, patch_res=0.125)
            grid[lv].append(run_one(sc, configs.vopts(configs.DISC2D, lv, 0.15, lamp_z=1.0), loose, a.eps))
        print("grid room", seed, [round(grid[lv][-1]["dwell_s"], 1) for lv in grid_levels], flush=True)
    out["grid"] = {"levels_m": grid_levels, "patch_res_m": 0.125,
                   "dwell_norm": summarise(grid, "dwell_s"),
                   "raw": {str(k): v for k, v in grid.items()}}
    if not a.no_3d:
        sp = [1.0, 0.75, 0.5, 0.4, 0.3, 0.25]
        rows = []
        for s in sp:
            r = run_one(configs.c4_scene(), dict(configs.FLOAT_OPTS, spacing=s), configs.T_MAX, 1e-4)
            r["spacing_m"] = s
            rows.append(r)
            print("3d", s, {k: r[k] for k in ("K", "assemble_ms", "coverage_total", "lp_iterations")}, flush=True)
        out["grid_3d"] = rows
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
