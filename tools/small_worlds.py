"""C1/C2 (launch-bound small scenes): entries/s of the assembly
call per world, sequential vs the 25 C2 worlds on 25 concurrent streams, and
with the calls captured in one CUDA graph.  Prints one JSON line.

usage: python tools/small_worlds.py [reps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import configs  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    worlds = [configs.c1()] + [configs.c2(s) for s in range(25)]
    scenes, lamps, outs = [], [], []
    for w in worlds:
        sc = uvd.Scene(w["scene"])
        lam, _ = sc.vantage(w["vantage"])
        scenes.append(sc)
        lamps.append(lam)
        outs.append(torch.empty((lam.shape[0], sc.ld()), dtype=torch.float32, device="cuda"))
    entries = [sc.N * lam.shape[0] for sc, lam in zip(scenes, lamps)]
    res = {}
    # C1 alone
    for _ in range(5):
        scenes[0].irradiance(lamps[0], out=outs[0])
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(reps):
        scenes[0].irradiance(lamps[0], out=outs[0])
    e1.record()
    torch.cuda.synchronize()
    res["c1_us_per_matrix"] = e0.elapsed_time(e1) * 1e3 / reps
    res["c1_entries_per_s"] = entries[0] / (res["c1_us_per_matrix"] * 1e-6)
    # 25 C2 worlds: sequential on one stream
    c2 = list(range(1, 26))
    e0.record()
    for _ in range(reps):
        for k in c2:
            scenes[k].irradiance(lamps[k], out=outs[k])
    e1.record()
    torch.cuda.synchronize()
    t_seq = e0.elapsed_time(e1) * 1e-3 / reps
    tot = sum(entries[k] for k in c2)
    res["c2_sequential_ms"] = t_seq * 1e3
    res["c2_sequential_entries_per_s"] = tot / t_seq
    # 25 concurrent streams
    streams = [torch.cuda.Stream() for _ in c2]
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        for s, k in zip(streams, c2):
            with torch.cuda.stream(s):
                scenes[k].irradiance(lamps[k], out=outs[k], stream=s)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    t_con = e0.elapsed_time(e1) * 1e-3 / reps
    res["c2_25streams_ms"] = t_con * 1e3
    res["c2_25streams_entries_per_s"] = tot / t_con
    # one CUDA graph replaying all 25 assemblies
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for k in c2:
            scenes[k].irradiance(lamps[k], out=outs[k], stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for k in c2:
                scenes[k].irradiance(lamps[k], out=outs[k], stream=s)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    t_g = e0.elapsed_time(e1) * 1e-3 / reps
    res["c2_graph_ms"] = t_g * 1e3
    res["c2_graph_entries_per_s"] = tot / t_g
    res["c2_entries"] = tot
    res["c2_mean_patches"] = float(np.mean([scenes[k].N for k in c2]))
    res["c2_mean_configs"] = float(np.mean([lamps[k].shape[0] for k in c2]))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
