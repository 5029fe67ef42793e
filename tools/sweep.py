"""NEXT-4 resolution sweeps as throughput-scaling curves (PAPER App. II axes,
P:495–522): assembly time and entries/s of the hot path
(scene → vantage → A) as the paper's resolutions vary.  Only the throughput
axis is reproduced — the paper's dwell/coverage results need its planner and
asset and are out of scope.

* env-res: wall patch resolution 1/2 … 1/32 m at a 0.1 m grid on the random
  rooms;
* grid:    vantage grid 1/2 … 1/32 m at the 1/8 m patch resolution;
* 3d:      Floatbot grid spacing 1000 … 250 mm on the C4 ward.

Each point: best of 3 CUDA-event timings of uvd_irradiance_matrix after a
warm-up (the BVH prebuilt), N, K, entries/s.

usage: python tools/sweep.py [--rooms 25] [--no-3d] [--out profiles/sweep_r02.json]
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


def run_one(scene, vopts, reps=3):
    sc = uvd.Scene(scene)
    lam, _ = sc.vantage(vopts)
    K = int(lam.shape[0])
    A = torch.empty((K, sc.ld()), dtype=torch.float32, device="cuda")
    sc.irradiance(lam, out=A)
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sc.irradiance(lam, out=A)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    sc.sync_status()
    n = sc.N
    sc.close()
    return {"N": n, "K": K, "assemble_ms": best, "entries_per_s": n * K / (best / 1e3)}


def summary(rows):
    return {"N": int(np.median([r["N"] for r in rows])), "K": int(np.median([r["K"] for r in rows])),
            "assemble_ms_median": float(np.median([r["assemble_ms"] for r in rows])),
            "entries_per_s_median": float(np.median([r["entries_per_s"] for r in rows]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rooms", type=int, default=25)
    ap.add_argument("--no-3d", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    out = {"gpu": torch.cuda.get_device_name(0), "rooms": a.rooms, "timing": "best of 3 after a warm-up"}
    levels = [0.5, 0.25, 0.125, 0.0625, 0.03125]
    env = {lv: [run_one(rooms.random_room(s, 4.0, patch_res=lv), configs.vopts(configs.DISC2D, 0.1, 0.15, lamp_z=1.0))
                for s in range(a.rooms)] for lv in levels}
    out["env_res"] = {"grid_m": 0.1, "levels": {str(k): summary(v) for k, v in env.items()}}
    print("env-res", {k: round(v["entries_per_s_median"] / 1e9, 2) for k, v in out["env_res"]["levels"].items()})
    grid = {lv: [run_one(rooms.random_room(s, 4.0, patch_res=0.125), configs.vopts(configs.DISC2D, lv, 0.15, lamp_z=1.0))
                 for s in range(a.rooms)] for lv in levels}
    out["grid"] = {"patch_res_m": 0.125, "levels": {str(k): summary(v) for k, v in grid.items()}}
    print("grid", {k: round(v["entries_per_s_median"] / 1e9, 2) for k, v in out["grid"]["levels"].items()})
    if not a.no_3d:
        rows = []
        for s in [1.0, 0.75, 0.5, 0.4, 0.3, 0.25]:
            r = run_one(configs.c4_scene(), dict(configs.FLOAT_OPTS, spacing=s))
            r["spacing_m"] = s
            rows.append(r)
            print("3d", s, r, flush=True)
        out["grid_3d"] = rows
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
