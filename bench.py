#!/usr/bin/env python
"""bench.py — irradiance-matrix entries/s on B200 (BASELINE.json metric).

One step = one pass of the whole hot path (SURVEY §8(a) rows a1–a8) over the
workload, inputs resident in HBM when the timed region starts:
  a1/a2  uvd_scene_create from the device-resident triangle soup (patch
         attributes + LBVH build)
  a3     uvd_vantage_sample (Armbot grid, clearance, free space, reach)
  a4–a6  uvd_irradiance_matrix (this rank's block-cyclic column shard)
  a7     uvd_fluence: μ = A·t (sparse LP-like plan), A·𝟙 (ever-visible rows),
         g = Aᵀ·y; NCCL all_reduce of μ and A·𝟙 when N > 1
  a8     uvd_coverage
value = N_patches · K_configs / (step time, max over ranks)  [dense-equivalent
entries decided per second; back-facing zeros count, SURVEY §8d].

`--impl reference` times the fp64 CPU oracle (oracle/, the only other place this
script executes it) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "irradiance-matrix entries/s (occlusion-tested)"
UNIT = "entries/s"
# FP32 roofline denominator for the traversal kernel (bound "alu"): guide unit
# counts × max clock = 148 SM × 128 FP32 lanes × 2 flop × 1.965 GHz.
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def _hbm_peak():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else
    the profiling guide's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6537.6


HBM_PEAK_GBS = _hbm_peak()
# algorithmic FP32-equivalent flops (fp64 op = 2) per counted unit
FLOP_PER_PAIR = 26.0      # a4: ray setup + front-face test per (patch, lamp sample)
FLOP_PER_RAY = 10.0       # a5/a6 per front-facing ray: t-range, Eq. 7 (fp64)
FLOP_PER_BOX = 12.0       # fp32 slab test of one child box
FLOP_PER_TRI = 80.0       # fp32 filtered division-free Möller–Trumbore with its error bounds (~80 ops)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="uvd", choices=["uvd", "reference"])
    ap.add_argument("--workload", default="C5", choices=["C5", "C4-float", "C4-tower", "C2"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostics: skip the nvidia-smi sampler")
    return ap.parse_args()


def workload(name):
    from synth import configs
    if name == "C5":
        return dict(name="C5: synthetic ward ≥1M triangles × Armbot configs at 0.25 m",
                    scene=configs.c5_scene(), vantage=configs.ARM_OPTS, L=1)
    if name == "C4-float":
        return dict(name="C4: synthetic ward ~216k triangles × Floatbot configs at 0.25 m",
                    scene=configs.c4_scene(), vantage=configs.FLOAT_OPTS, L=1)
    if name == "C4-tower":
        return dict(name="C4: synthetic ward ~216k triangles × Towerbot (L=10) at 0.25 m",
                    scene=configs.c4_scene(), vantage=configs.TOWER_OPTS, L=10)
    if name == "C2":
        return dict(name="C2: random 2.5D room seed 0, 0.25 m grid", scene=configs.c2(0)["scene"],
                    vantage=configs.DISC_OPTS, L=1)
    raise ValueError(name)


# --------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# -------------------------------------------------------------- oracle ---
def oracle_sample_setup(wl, n_lamps=48, seed=0):
    """Bounded oracle sample of the same workload: the oracle's own patches and
    lamp positions (grid candidates that pass the oracle's clearance and
    free-space test; the Armbot reach proxy is skipped for time)."""
    from oracle import oracle as O
    pat = O.scene_patches(wl["scene"])
    cand = O.vantage_candidates(wl["scene"], wl["vantage"])
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(cand["points"]), size=min(len(cand["points"]), 4 * n_lamps), replace=False)
    opts = dict(wl["vantage"])
    if opts["robot"] == O.ARM:
        opts = dict(opts, robot=O.FLOAT3D)   # reach proxy skipped in the timing sample
    if opts["robot"] == O.DISC2D:
        v = O.vantage(wl["scene"], opts, idx=np.sort(pick))
    else:
        tri = np.ascontiguousarray(np.asarray(wl["scene"]["vertices"], np.float32)[wl["scene"]["tris"]].reshape(-1, 9))
        samples = np.ascontiguousarray(cand["samples"][np.sort(pick)])
        R = len(samples)
        feas = np.zeros(R, np.uint8)
        amb = np.zeros(R, np.uint8)
        md = np.zeros(R, np.float64)
        O.lib().orc_vantage_eval_3d(tri, len(tri), samples.reshape(-1), R, samples.shape[1],
                                    float(opts["clearance"]), 1, feas, amb, md, 0)
        v = dict(samples=samples, feasible=feas.astype(bool))
    lamps = v["samples"][v["feasible"]][:n_lamps]
    return O, pat, np.ascontiguousarray(lamps, np.float32)


def oracle_time(O, pat, lamps, seconds, seed=1, batch=None):
    rng = np.random.default_rng(seed)
    threads = O.default_threads()
    batch = batch or 64 * threads
    done, t0 = 0, time.perf_counter()
    while True:
        pi = rng.integers(0, pat["N"], batch)
        pj = rng.integers(0, len(lamps), batch)
        O.irradiance_pairs(pat, lamps, pi, pj)
        done += batch
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    # each pair is one entry with L lamp samples (the lamps array carries L)
    return done / el, done, el, threads


# ---------------------------------------------------------------- main ---
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    wl = workload(args.workload)
    O, pat, lamps = oracle_sample_setup(wl)
    per_step = max(2.0, min(8.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_time(O, pat, lamps, per_step / 4)
    vals, tot_pairs, tot_t = [], 0, 0.0
    for s in range(args.steps):
        v, n, el, threads = oracle_time(O, pat, lamps, per_step, seed=100 + s)
        vals.append(v)
        tot_pairs += n
        tot_t += el
    value = tot_pairs / tot_t
    sample = (f"{tot_pairs} uniformly random (patch, configuration) pairs of {wl['name']} "
              f"({pat['N']} patches, {len(lamps)} oracle-feasible lamp positions), brute force fp64")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": wl["name"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    # one process per GPU; BENCH_BACKEND=gloo + fewer GPUs than ranks is only a
    # functional dry run of the multi-rank path (ranks then share a device)
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if ws > 1:
        dist.barrier()
    from paper_2103_14137_b200 import shard, uvd
    from synth import configs, vectors

    wl = workload(args.workload)
    sc_np = wl["scene"]
    dev = torch.device("cuda", local)
    is_mesh = "vertices" in sc_np
    if is_mesh:
        V_dev = torch.from_numpy(np.ascontiguousarray(sc_np["vertices"], np.float32)).to(dev)
        F_dev = torch.from_numpy(np.ascontiguousarray(sc_np["tris"], np.int32)).to(dev)
        desc_dev = dict(vertices=V_dev, tris=F_dev)
    else:
        desc_dev = sc_np
    # sizes (deterministic): one untimed pass
    scene = uvd.Scene(desc_dev)
    lamps, _ = scene.vantage(wl["vantage"])
    N, K, L = scene.N, lamps.shape[0], lamps.shape[1]
    ld = scene.ld()
    cols = shard.block_cyclic(K, ws, rank, 32)
    n_loc = len(cols)
    A = torch.empty((n_loc, ld), dtype=torch.float32, device=dev)
    t_glob = vectors.sparse_plan(K, seed=0)
    t_loc = torch.from_numpy(t_glob[cols]).to(dev)
    ones = torch.ones(n_loc, dtype=torch.float64, device=dev)
    y = torch.from_numpy(vectors.row_weights(N, 0)).to(dev)
    scene.close()
    del lamps
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev_k0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_k1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    phase_names = ("scene", "vantage", "irradiance", "fluence", "coverage")
    ev_ph = [[torch.cuda.Event(enable_timing=True) for _ in range(len(phase_names) + 1)]
             for _ in range(args.steps)]

    def step(i=None):
        ev = ev_ph[i] if i is not None else None
        if ev:
            ev[0].record(stream)
        sc = uvd.Scene(desc_dev)                              # a1, a2
        if ev:
            ev[1].record(stream)
        lam, _ = sc.vantage(wl["vantage"])                    # a3
        if ev:
            ev[2].record(stream)
            ev_k0[i].record(stream)
        sc.irradiance(lam, cols=cols, out=A)                  # a4–a6
        if ev:
            ev_k1[i].record(stream)
            ev[3].record(stream)
        mu = uvd.fluence(A, N, t_loc)                         # a7: μ = A·t
        rowsum = uvd.fluence(A, N, ones)                      #     A·𝟙 (ever-visible rows)
        g = uvd.fluence(A, N, y, transpose=True)              #     g = Aᵀ·y
        shard.reduce_partials(mu, rowsum)                     # NCCL all_reduce (N > 1)
        if ev:
            ev[4].record(stream)
        cov = sc.coverage(mu, configs.MU_MIN, rowsum)         # a8
        sc.sync_status()
        sc.close()
        if ev:
            ev[5].record(stream)
        return cov, g

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    if not args.no_clocks:
        clocks.start()
    n_launch0 = uvd.launch_count()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        cov, _ = step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    n_launch = uvd.launch_count() - n_launch0
    clk = clocks.stop()
    k_each = [a.elapsed_time(b) for a, b in zip(ev_k0, ev_k1)]
    k_ms = float(np.mean(k_each))
    k_sum = float(shard.sum_over_ranks([k_ms], device=dev)[0])
    ms_total, k_ms, k_med, k_best = shard.max_over_ranks(
        [ms_total, k_ms, float(np.median(k_each)), float(np.min(k_each))], device=dev)
    imbalance = k_ms / (k_sum / ws)  # slowest rank's assembly time over the mean
    ms_step = ms_total / args.steps
    value = N * K / (ms_step / 1e3)
    phases = {nm: float(np.mean([e[k].elapsed_time(e[k + 1]) for e in ev_ph]))
              for k, nm in enumerate(phase_names)}

    # roofline of the dominant kernel: algorithmic work from one instrumented launch
    sc = uvd.Scene(desc_dev)
    lam, _ = sc.vantage(wl["vantage"])
    r = sc.irradiance(lam, cols=cols, out=A, counters=True)
    cnt = r["counters"].cpu().numpy().astype(np.float64)
    sc.close()
    cnt = shard.sum_over_ranks(cnt, device=dev).cpu().numpy()
    pairs = float(N) * K * L
    flops = FLOP_PER_PAIR * pairs + FLOP_PER_RAY * cnt[0] + FLOP_PER_BOX * cnt[1] + FLOP_PER_TRI * cnt[2]
    achieved = flops / ws / (k_ms / 1e3) / 1e12
    traffic, traffic_note = None, None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic_r01.json")
    if os.path.exists(tfile) and args.workload == "C5":
        tr = json.load(open(tfile))
        traffic = tr["bytes_per_col"] * K  # per launch: all columns of the step
        traffic_note = (f"DRAM read+write of {tr['capture']} ({tr['cols']}-column launch), scaled per column "
                        f"to this {K}-column launch")
    roofline = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic, "traffic_note": traffic_note,
                "kernel": "k_assemble", "kernel_ms": k_ms, "kernel_ms_median": k_med,
                "kernel_ms_best": k_best, "imbalance": imbalance,
                "kernel_share": k_ms / ms_step,
                "rays_per_s": cnt[0] / (k_ms / 1e3),
                "per_launch": {"rays": cnt[0], "box_tests": cnt[1], "tri_tests": cnt[2],
                               "warp_node_fetches": cnt[3], "flops_fp32eq": flops},
                "peak_note": "148 SM x 128 FP32 lanes x 2 x 1.965 GHz (guide); measured FFMA 70.8 TFLOP/s"}

    # a7 (HBM-bound GEMVs) against the measured HBM peak: algorithmic bytes of
    # the step's three products = A's nonzero-t columns + A twice + vectors
    nnz_t = int((t_loc != 0).sum().item())
    a7_bytes = 4.0 * ld * (nnz_t + 2 * n_loc) + 8.0 * (4 * N + 2 * n_loc)
    a7_ms = phases["fluence"]
    a7 = {"kernels": "k_gemv_n (A·t, A·1), k_gemv_t (Aᵀ·y)", "bytes": a7_bytes, "ms": a7_ms,
          "achieved_gbs": a7_bytes / (a7_ms / 1e3) / 1e9, "peak_gbs": HBM_PEAK_GBS,
          "frac": a7_bytes / (a7_ms / 1e3) / 1e9 / HBM_PEAK_GBS,
          "note": "phase time includes the all_reduce for N > 1"}

    # end to end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(uvd, shard, configs, wl, sc_np, is_mesh, cols, n_loc, ld, N, K, t_glob, dev,
                      dist if ws > 1 else None, max(1, min(args.steps, 3)))

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        O, pat, olamps = oracle_sample_setup(wl)
        v, n, el, threads = oracle_time(O, pat, olamps, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{n} uniformly random (patch, configuration) pairs of the same workload, "
                         f"{len(olamps)} oracle-feasible lamp positions, {el:.1f} s on {threads} threads",
               "extrapolated_full_matrix_s": float(N) * K / v if v > 0 else None}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": wl["name"], "n_patches": N, "n_tris": int(len(sc_np["tris"])) if is_mesh else 2 * N,
                           "k_configs": K, "lamp_samples": L, "columns": "block-cyclic, blocks of 32",
                           "A_bytes": int(K) * ld * 4,
                           "l2": "inputs larger than L2: every step rebuilds the BVH and writes the "
                                 f"{K * ld * 4 / 1e9:.1f} GB dense A",
                           "precision": "fp32 conservative box tests; fp64 triangle tests and Eq. 7; A stored fp32",
                           "step": "scene_create+vantage+irradiance+fluence(A·t, A·1, Aᵀy)+coverage"},
                "phases_ms": phases, "roofline": roofline, "roofline_a7": a7, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(n_launch), "clocks": clk}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_e2e(uvd, shard, configs, wl, sc_np, is_mesh, cols, n_loc, ld, N, K, t_glob, dev, dist, steps):
    """Same metric through the public API with HOST inputs: the triangle soup
    and t are copied from pinned host memory and μ + coverage are read back
    inside the timed region (wall clock, max over ranks)."""
    import torch
    if is_mesh:
        Vh = torch.from_numpy(np.ascontiguousarray(sc_np["vertices"], np.float32)).pin_memory()
        Fh = torch.from_numpy(np.ascontiguousarray(sc_np["tris"], np.int32)).pin_memory()
        desc = dict(vertices=Vh.numpy(), tris=Fh.numpy())
        h2d_scene = Vh.numel() * 4 + Fh.numel() * 4
    else:
        desc = sc_np
        h2d_scene = 0
    th = torch.from_numpy(np.ascontiguousarray(t_glob[cols])).pin_memory()
    mu_h = torch.empty(N, dtype=torch.float64).pin_memory()
    A = torch.empty((n_loc, ld), dtype=torch.float32, device=dev)

    def one():
        sc = uvd.Scene(desc)
        lam, _ = sc.vantage(wl["vantage"])
        sc.irradiance(lam, cols=cols, out=A)
        t = th.to(dev, non_blocking=True)
        mu = uvd.fluence(A, N, t)
        shard.reduce_partials(mu)
        cov = sc.coverage(mu, configs.MU_MIN)
        mu_h.copy_(mu, non_blocking=True)
        torch.cuda.synchronize()
        sc.close()
        return cov

    one()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    el = time.perf_counter() - t0
    el = shard.max_over_ranks([el], device=dev)[0]
    return {"value": N * K / (el / steps), "unit": UNIT, "steps": steps,
            "h2d_bytes_per_step": int(h2d_scene + th.numel() * 8),
            "d2h_bytes_per_step": int(N * 8 + 3 * 8 + 8)}


if __name__ == "__main__":
    sys.exit(main())
