#!/usr/bin/env python
"""bench.py — irradiance-matrix entries/s on B200 (BASELINE.json metric).

One step = one pass of the whole hot path (SURVEY §8(a) rows a1–a8) over the
workload, inputs resident in HBM when the timed region starts:
  a1/a2  uvd_scene_create from the device-resident triangle soup (patch
         attributes + LBVH build)
  a3     uvd_vantage_sample (Armbot grid, clearance, free space, reach)
  a4–a6  uvd_irradiance_matrix (this rank's block-cyclic column shard)
  a7     uvd_fluence_multi: μ = A·t (sparse LP-like plan), A·𝟙 (ever-visible rows),
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


def _ffma_peak():
    """Our own FFMA microbenchmark on this B200 (tools/peaks.cu, profiles/peaks_r01.json)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "peaks_r01.json")))["fp32_ffma_tflops"])
    except Exception:  # noqa: BLE001
        return None


FFMA_MEASURED_TFLOPS = _ffma_peak()
# what the path computes in: fp32 conservative box tests and fp32 error-bounded
# triangle filter; exact fp64 triangle re-tests of undecided rays, fp64 ray
# setup / front-face test / Eq. 7; A stored fp32
DTYPE = "fp32+fp64"
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
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity sample")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank assembles a fixed 1/8 of the C5 configurations "
                         "(total K = N x K/8), instead of a share of the fixed full problem")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--dump", default=None, metavar="PREFIX",
                    help="after the timed region, every rank writes its A shard and visibility bits "
                         "(uvd-shard/1: PREFIX.rank<r>.json/.bin) for tools/recheck_dump.py")
    ap.add_argument("--no-bcast", action="store_true",
                    help="N > 1: every rank builds the scene instead of rank 0 building and broadcasting it")
    return ap.parse_args()


def workload(name):
    from synth import configs
    if name == "C5":
        return dict(name="C5: synthetic ward ≥1M triangles × Armbot configs (0.2 m grid)",
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
def oracle_sample_setup(wl, n_lamps=48, seed=0, gpu_raw=None):
    """Bounded oracle sample of the same workload (BASELINE configuration,
    Armbot reach proxy included): the oracle's own patches and the oracle's own
    feasibility verdict and lamp samples for `n_lamps` grid candidates — drawn
    from the GPU's feasible candidates when `gpu_raw` (their grid ids) is
    given, so the sample's entries can be compared with the GPU's columns, else
    from the whole grid.  Returns (O, patches, lamps (n, L, 3), raw ids)."""
    from oracle import oracle as O
    pat = O.scene_patches(wl["scene"])
    rng = np.random.default_rng(seed)
    if gpu_raw is not None:
        raw = np.sort(rng.choice(gpu_raw, size=min(len(gpu_raw), n_lamps), replace=False))
    else:
        n_cand = len(O.vantage_candidates(wl["scene"], wl["vantage"])["points"])
        raw = np.sort(rng.choice(n_cand, size=min(n_cand, 6 * n_lamps), replace=False))
    v = O.vantage(wl["scene"], wl["vantage"], idx=raw)
    ok = v["feasible"] & ~v["ambiguous"]
    if gpu_raw is None:
        ok &= np.cumsum(ok) <= n_lamps
    # GPU-feasible candidates the oracle rejects outright (parity failures of a3)
    oracle_setup.rejected = int((~v["feasible"] & ~v["ambiguous"]).sum()) if gpu_raw is not None else 0
    return O, pat, np.ascontiguousarray(v["samples"][ok], np.float32), raw[ok]


class oracle_setup:  # noqa: N801 — a namespace for the last setup's a3 disagreement count
    rejected = 0


def oracle_time(O, pat, lamps, seconds, seed=1, batch=None, keep=False):
    """Oracle entries of uniformly random (patch, lamp) pairs for ~`seconds` of
    wall clock on all host threads; keep=True also returns the pairs and results."""
    rng = np.random.default_rng(seed)
    threads = O.default_threads()
    batch = batch or 64 * threads
    done, t0 = 0, time.perf_counter()
    kept = []
    while True:
        pi = rng.integers(0, pat["N"], batch)
        pj = rng.integers(0, len(lamps), batch)
        r = O.irradiance_pairs(pat, lamps, pi, pj)
        if keep:
            kept.append((pi, pj, r))
        done += batch
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    # each pair is one entry with L lamp samples (the lamps array carries L)
    return done / el, done, el, threads, kept


def gpu_pairs(A, vb, ci, ri, L):
    """GPU values and visibility bits of local (column, row) pairs."""
    import torch
    gA = A[torch.from_numpy(ci).to(A.device), torch.from_numpy(ri).to(A.device)].double().cpu().numpy()
    gvis = np.stack([(vb[ci, l, ri // 32] >> (ri % 32).astype(np.uint32)) & 1 for l in range(L)], 1).astype(bool)
    return gA, gvis


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
    O, pat, lamps, _ = oracle_sample_setup(wl)
    per_step = max(2.0, min(8.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_time(O, pat, lamps, per_step / 4)
    tot_pairs, tot_t = 0, 0.0
    for s in range(args.steps):
        v, n, el, threads, _ = oracle_time(O, pat, lamps, per_step, seed=100 + s)
        tot_pairs += n
        tot_t += el
    value = tot_pairs / tot_t
    sample = (f"{tot_pairs} uniformly random (patch, configuration) pairs of {wl['name']} "
              f"({pat['N']} patches, {len(lamps)} oracle-feasible configurations incl. the reach proxy), "
              f"brute force fp64, {args.steps} steps of ~{per_step:.0f} s")
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
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nRanks) on stderr
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
    lamps, raw0 = scene.vantage(wl["vantage"])
    N, K_all, L = scene.N, lamps.shape[0], lamps.shape[1]
    ld = scene.ld()
    if args.weak:   # per-rank work fixed: K/8 configurations per rank, total K = N_gpus x K/8
        K = min(K_all, ws * ((K_all + 7) // 8))
    else:           # strong: the fixed full problem shared by the ranks
        K = K_all
    cols = shard.block_cyclic(K, ws, rank, 32)
    n_loc = len(cols)
    A = torch.empty((n_loc, ld), dtype=torch.float32, device=dev)
    t_glob = vectors.sparse_plan(K, seed=0)
    t_loc = torch.from_numpy(t_glob[cols]).to(dev)
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

    def step(desc, t_in, i=None, host_out=None):
        """One pass of the whole hot path (a1–a8).  desc: device-resident or
        pinned-host scene input; t_in: this rank's dwell times (device, or
        pinned host: copied in); host_out: pinned buffers for μ, g (read back)."""
        ev = ev_ph[i] if i is not None else None
        if ev:
            ev[0].record(stream)
        # a1, a2: N > 1 builds once on rank 0 and broadcasts the scene image
        sc = uvd.Scene(desc) if ws == 1 or args.no_bcast else shard.broadcast_scene(desc)
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
        t = t_in if t_in.is_cuda else t_in.to(dev, non_blocking=True)
        # a7: μ = A·t, A·𝟙 (ever-visible rows) and g = Aᵀ·y in one pass over A
        mu, rowsum, g = uvd.fluence_multi(A, N, x=t, y=y, rowsum=True)
        shard.reduce_partials(mu, rowsum)                     # NCCL all_reduce (N > 1)
        if ev:
            ev[4].record(stream)
        cov = sc.coverage(mu, configs.MU_MIN, rowsum)         # a8
        sc.sync_status()
        if host_out is not None:
            host_out[0].copy_(mu, non_blocking=True)
            host_out[1].copy_(g, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        sc.close()
        if ev:
            ev[5].record(stream)
        return cov, g

    for _ in range(max(3, args.warmup)):
        step(desc_dev, t_loc)
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
        cov, _ = step(desc_dev, t_loc, i)
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
    lam, raw = sc.vantage(wl["vantage"])
    r = sc.irradiance(lam, cols=cols, out=A, counters=True)
    cnt = r["counters"].cpu().numpy().astype(np.float64)
    cnt = shard.sum_over_ranks(cnt, device=dev).cpu().numpy()
    pairs = float(N) * K * L
    flops = FLOP_PER_PAIR * pairs + FLOP_PER_RAY * cnt[0] + FLOP_PER_BOX * cnt[1] + FLOP_PER_TRI * cnt[2]
    achieved = flops / ws / (k_ms / 1e3) / 1e12
    traffic, traffic_note, ncu_issue = None, None, None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")
    if not os.path.exists(tfile):
        tfile = os.path.join(ROOT, "profiles", "ncu_traffic_r01.json")
    if os.path.exists(tfile) and args.workload == "C5" and not args.weak:
        tr = json.load(open(tfile))
        traffic = tr["bytes_per_col"] * K  # per launch: all columns of the step
        traffic_note = (f"DRAM read+write of {tr['capture']} ({tr['cols']}-column launch), scaled per column "
                        f"to this {K}-column launch")
        ncu_issue = tr.get("ncu_issue")
    roofline = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP32_PEAK_TFLOPS,
                # what bounds it (ncu of the same kernel): issue slots and threads per warp
                "ncu_issue": ncu_issue,
                "frac_vs_measured_ffma": achieved / FFMA_MEASURED_TFLOPS if FFMA_MEASURED_TFLOPS else None,
                "traffic": traffic, "traffic_note": traffic_note,
                "kernel": "k_assemble", "kernel_ms": k_ms, "kernel_ms_median": k_med,
                "kernel_ms_best": k_best, "imbalance": imbalance,
                "kernel_share": k_ms / ms_step,
                "rays_per_s": cnt[0] / (k_ms / 1e3),
                "per_launch": {"rays": cnt[0], "box_tests": cnt[1], "tri_tests": cnt[2],
                               "warp_node_fetches": cnt[3], "fixup_entries": cnt[4], "flops_fp32eq": flops},
                "peak_note": ("guide: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz; frac_vs_measured_ffma against our "
                              f"FFMA microbenchmark ({FFMA_MEASURED_TFLOPS} TFLOP/s, profiles/peaks_r01.json); "
                              "flops per unit: DESIGN.md §6 (reading R1)")}

    # a7 (HBM-bound, one pass) against the measured HBM peak: algorithmic bytes
    # of the step's three products = A once + the vectors (t, y, μ, A·𝟙, g)
    a7_bytes = 4.0 * ld * n_loc + 8.0 * (3 * N + 2 * n_loc)
    a7_ms = phases["fluence"]
    a7 = {"kernels": "k_gemv_multi (A·t, A·𝟙, Aᵀ·y in one pass) + k_gemv_t_reduce", "bytes": a7_bytes, "ms": a7_ms,
          "achieved_gbs": a7_bytes / (a7_ms / 1e3) / 1e9, "peak_gbs": HBM_PEAK_GBS,
          "frac": a7_bytes / (a7_ms / 1e3) / 1e9 / HBM_PEAK_GBS,
          "note": "phase time includes the all_reduce for N > 1"}

    if args.dump:  # per-rank shard dump for offline re-checks (outside the timed region)
        rd = sc.irradiance(lam, cols=cols, out=A, vis_bits=True)
        sc.sync_status()
        hp = shard.dump_shard(args.dump, workload=args.workload, A=A, n_rows=N, cols=cols,
                              raw=raw.cpu().numpy()[np.asarray(cols, np.int64)],
                              lamps=lam[torch.as_tensor(cols, device=lam.device)], orig_id=sc.patches()["orig_id"],
                              power_w=80.0, vis_bits=rd["vis_bits"], rank=rank, world=ws)
        print(f"[bench] rank {rank}: shard dump {hp}", file=sys.stderr, flush=True)
        del rd

    # parity material: the timed kernel (not the instrumented one) once more in
    # the same launch configuration, with visibility bits and the fix-up list
    par_src = None
    if rank == 0 and ws == 1 and not (args.no_cpu_baseline and args.no_parity):
        rp = sc.irradiance(lam, cols=cols, out=A, vis_bits=True, fixups=1 << 24)
        sc.sync_status()
        par_src = dict(vb=rp["vis_bits"].cpu().numpy().view(np.uint32), fixups=rp["fixups"].cpu().numpy(),
                       fixup_count=rp["fixup_count"], raw=raw.cpu().numpy(),
                       orig=sc.patches()["orig_id"].cpu().numpy())
        del rp
    sc.close()

    # end to end through the public API from pinned host buffers: the same step
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(uvd, shard, torch, step, sc_np, is_mesh, t_loc, N, n_loc, K, dev,
                      dist if ws > 1 else None, max(10, args.e2e_steps))

    cpu, parity_blk = None, None
    if par_src is not None:
        cpu, parity_blk = cpu_and_parity(args, wl, A, par_src, cols, L)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": DTYPE,
                "data": "synthetic",
                "config": {"workload": wl["name"], "n_patches": N, "n_tris": int(len(sc_np["tris"])) if is_mesh else 2 * N,
                           "k_configs": K, "k_per_gpu": n_loc, "lamp_samples": L,
                           "columns": "block-cyclic, blocks of 32",
                           "A_bytes": int(K) * ld * 4,
                           "l2": "inputs larger than L2: every step rebuilds the BVH and writes the "
                                 f"{K * ld * 4 / 1e9:.1f} GB dense A",
                           "precision": ("fp32 conservative box tests and fp32 triangle filter with forward "
                                         "error bounds; undecided rays re-traced with exact fp64 triangle tests; "
                                         "fp64 ray setup, front-face test and Eq. 7; A stored fp32"),
                           "step": "scene_create+vantage+irradiance+fluence(A·t, A·1, Aᵀy)+coverage",
                           "scene_build": ("every rank" if ws == 1 or args.no_bcast else
                                           "rank 0, broadcast as a uvd_scene_export image")},
                "phases_ms": phases, "roofline": roofline, "roofline_a7": a7, "cpu_baseline": cpu,
                "parity": parity_blk, "e2e": e2e, "gpu_launches": int(n_launch), "clocks": clk}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_and_parity(args, wl, A, src, cols, L):
    """The oracle on this workload (rank 0, N = 1): timed on random pairs of 48
    of the GPU's configurations (the cpu_baseline), those same pairs compared
    with the GPU's entries, plus entries drawn from the GPU's fix-up list (the
    rays the fp32 pass left undecided) — the parity block."""
    from oracle import parity
    O, pat, olamps, oraw = oracle_sample_setup(wl, gpu_raw=src["raw"][np.asarray(cols)])
    pos = {int(q): k for k, q in enumerate(src["raw"][np.asarray(cols)])}   # grid id -> local column
    lcol = np.array([pos[int(q)] for q in oraw], np.int64)
    inv_orig = np.empty_like(src["orig"])
    inv_orig[src["orig"]] = np.arange(len(src["orig"]))
    cpu = None
    secs = 0.0 if args.no_cpu_baseline else args.cpu_seconds
    v, n, el, threads, kept = oracle_time(O, pat, olamps, max(secs, 0.5), keep=True)
    if not args.no_cpu_baseline:
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": (f"{n} uniformly random (patch, configuration) pairs of the bench workload: "
                          f"{len(olamps)} of the step's configurations (oracle feasibility incl. the reach "
                          f"proxy, oracle lamp samples), brute force fp64, {el:.1f} s on {threads} threads"),
               "extrapolated_full_matrix_s": float(pat["N"]) * len(src["raw"]) / v if v > 0 else None}
    if args.no_parity:
        return cpu, None
    stats = None
    for pi, pj, r in kept:
        ci, ri = lcol[pj], inv_orig[pi]
        gA, gvis = gpu_pairs(A, src["vb"], ci, ri, L)
        st = parity.stats_from(pat, olamps, pi, pj, gA, gvis, r)
        stats = st if stats is None else parity.merge(stats, st)
    stats["degenerate_fraction"] = stats["degenerate_rays"] / max(stats["rays"], 1)
    stats.pop("mismatch_at", None)
    stats.pop("bad_at", None)
    # fix-up entries of the sampled columns (the hard cases)
    fl = src["fixups"].astype(np.uint64)
    fc, fr = (fl >> np.uint64(32)).astype(np.int64), (fl & np.uint64(0xffffffff)).astype(np.int64)
    colset = {int(c): k for k, c in enumerate(lcol)}
    sel = np.nonzero(np.isin(fc, lcol))[0]
    rng = np.random.default_rng(7)
    sel = rng.choice(sel, min(len(sel), 1000), replace=False) if len(sel) else sel
    fix = None
    if len(sel):
        ci, ri = fc[sel], fr[sel]
        gA, gvis = gpu_pairs(A, src["vb"], ci, ri, L)
        fix = parity.compare_pairs(pat, olamps, src["orig"][ri], np.array([colset[int(c)] for c in ci]), gA, gvis)
        fix.pop("mismatch_at", None)
        fix.pop("bad_at", None)
    blk = {"oracle": "fp64 brute force (oracle/), same configurations and patches",
           "vantage_rejected_by_oracle": oracle_setup.rejected,
           "random_pairs": stats, "fixup_entries": fix,
           "fixup_fraction_of_entries": src["fixup_count"] / (float(pat["N"]) * len(cols)),
           "gates": {"mismatches": 0, "degenerate_fraction": 1e-4, "rel_err": 1e-5}}
    return cpu, blk


def run_e2e(uvd, shard, torch, step, sc_np, is_mesh, t_loc, N, n_loc, K, dev, dist, steps):
    """The same step through the public API with HOST inputs: the triangle soup
    and this rank's dwell times come from pinned host memory and μ, g and the
    coverage go back to the host inside the timed region (wall clock, a
    synchronisation at the end of every step, max over ranks)."""
    if is_mesh:
        Vh = torch.from_numpy(np.ascontiguousarray(sc_np["vertices"], np.float32)).pin_memory()
        Fh = torch.from_numpy(np.ascontiguousarray(sc_np["tris"], np.int32)).pin_memory()
        desc = dict(vertices=Vh.numpy(), tris=Fh.numpy())
        h2d_scene = Vh.numel() * 4 + Fh.numel() * 4
    else:
        desc = sc_np
        h2d_scene = 0
    th = t_loc.cpu().pin_memory()
    host_out = (torch.empty(N, dtype=torch.float64).pin_memory(), torch.empty(n_loc, dtype=torch.float64).pin_memory())
    step(desc, th, host_out=host_out)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step(desc, th, host_out=host_out)
    el = time.perf_counter() - t0
    el = shard.max_over_ranks([el], device=dev)[0]
    return {"value": N * K / (el / steps), "unit": UNIT, "steps": steps,
            "h2d_bytes_per_step": int(h2d_scene + th.numel() * 8),
            "d2h_bytes_per_step": int(N * 8 + n_loc * 8 + 3 * 8 + 8),
            "note": "same step as the device-timed one (a1–a8 incl. A·1, Aᵀ·y, sync_status), host scene "
                    "and dwell times copied in, μ, g and coverage read back, wall clock"}


if __name__ == "__main__":
    sys.exit(main())
