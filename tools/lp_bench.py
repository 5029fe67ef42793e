"""Time NEXT-1 (the relaxed dwell-time LP of Eq. 9, uvd_lp_solve) on the GPU.

* C3 worlds (2.5D rooms at 0.5 m, ≈16–64 candidates): GPU solve
  time and µs/iteration (CUDA-graph replay), objective vs the HiGHS oracle on
  the oracle's own A, HiGHS wall time beside it.
* C4 Floatbot (215 940 patches × ≈8.5k candidates, dense A 7.4 GB): time to a
  1e-4 relative KKT point, iterations, µs/iteration and the HBM bandwidth of
  an iteration (one Aᵀ·y pass over A + the nonzero-t columns for A·t) against
  the measured HBM peak; coverage of the resulting plan.

usage: python tools/lp_bench.py [--c4] [--out profiles/lp_r01.json]
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
from synth import configs  # noqa: E402


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6537.6


def timed_solve(A, n, **kw):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    r = uvd.lp_solve(A, n, **kw)
    e1.record(s)
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1)


def c3(out):
    from oracle import lp as OLP
    from oracle import oracle as O
    rows = []
    for seed in range(10):
        c = configs.c3(seed)
        sc = uvd.Scene(c["scene"])
        lam, _ = sc.vantage(c["vantage"])
        a = sc.irradiance(lam, col_sumsq=True)
        sc.sync_status()
        p = 10.0 * float(np.sqrt(a["col_sumsq"].sum().item()))
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            uvd.lp_solve(a["A"], sc.N, penalty=p, t_max=configs.T_MAX, eps=1e-6, stream=s)  # warm-up
            r, ms = timed_solve(a["A"], sc.N, penalty=p, t_max=configs.T_MAX, eps=1e-6, stream=s)
        pat = O.extruded_patches(c["scene"])
        v = O.vantage(c["scene"], c["vantage"])
        An = O.irradiance_matrix(pat, v["samples"][v["feasible"]], mode="2d")["A"]
        t0 = time.perf_counter()
        ref = OLP.solve(An, configs.MU_MIN, 10.0 * np.linalg.norm(An), configs.T_MAX)
        t_h = time.perf_counter() - t0
        rows.append({"seed": seed, "N": sc.N, "K": int(lam.shape[0]), "iterations": r["iterations"],
                     "restarts": r["restarts"], "gpu_ms": ms, "us_per_iter": 1e3 * ms / max(1, r["iterations"]),
                     "obj_gpu": r["primal_obj"], "obj_highs": ref["obj"],
                     "rel_obj_diff": abs(r["primal_obj"] - ref["obj"]) / (1 + abs(ref["obj"])),
                     "highs_s": t_h, "status": r["status"]})
        print(json.dumps(rows[-1]), flush=True)
    out["c3"] = rows


def c4(out):
    sc = uvd.Scene(configs.c4_scene())
    lam, _ = sc.vantage(configs.FLOAT_OPTS)
    K, N = int(lam.shape[0]), sc.N
    a = sc.irradiance(lam, col_sumsq=True)
    sc.sync_status()
    A = a["A"]
    p = 10.0 * float(np.sqrt(a["col_sumsq"].sum().item()))
    s = torch.cuda.Stream()
    res = {}
    with torch.cuda.stream(s):
        # fixed-iteration run: per-iteration time and bandwidth
        r, ms = timed_solve(A, N, penalty=p, t_max=configs.T_MAX, eps=1e-12, max_iter=2048, stream=s)
        nnz = int((r["t"] != 0).sum().item())
        ld = A.shape[1]
        bytes_it = 4.0 * ld * K + 4.0 * ld * nnz + 8.0 * 15 * N  # Aᵀy pass + A·t over nonzero t + vectors
        res["fixed_2048"] = {"ms": ms, "us_per_iter": 1e3 * ms / r["iterations"], "nnz_t_final": nnz,
                             "bytes_per_iter_model": bytes_it,
                             "gbs": bytes_it / (ms / r["iterations"] / 1e3) / 1e9, "hbm_peak_gbs": hbm_peak()}
        res["fixed_2048"]["frac"] = res["fixed_2048"]["gbs"] / hbm_peak()
        print(json.dumps(res["fixed_2048"]), flush=True)
        for eps in (1e-4,):
            r, ms = timed_solve(A, N, penalty=p, t_max=configs.T_MAX, eps=eps, max_iter=100000, stream=s)
            mu = uvd.fluence(A, N, r["t"], stream=s)
            rowsum = uvd.fluence(A, N, torch.ones(K, dtype=torch.float64, device="cuda"), stream=s)
            cov = sc.coverage(mu, configs.MU_MIN, rowsum, stream=s)
            res[f"eps_{eps:g}"] = {"ms": ms, "iterations": r["iterations"], "restarts": r["restarts"],
                                   "status": r["status"], "obj": r["primal_obj"], "dual_obj": r["dual_obj"],
                                   "rel_primal_res": r["rel_primal_res"], "rel_dual_res": r["rel_dual_res"],
                                   "rel_gap": r["rel_gap"], "sum_t_s": r["sum_t"],
                                   "nnz_t": int((r["t"] > 0).sum().item()),
                                   "coverage_total": cov[0] / cov[1], "coverage_visible": cov[0] / cov[2]}
            print(json.dumps(res[f"eps_{eps:g}"]), flush=True)
    out["c4_floatbot"] = {"N": N, "K": K, "A_GB": K * A.shape[1] * 4 / 1e9, "penalty": p, **res}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c4", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = {"gpu": torch.cuda.get_device_name(0)}
    if not a.no_c3:
        c3(out)
    if a.c4:
        c4(out)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
