"""C3 workload (BASELINE configs[2]): the A·t / Aᵀ·y iteration loop that a
first-order dwell-time LP solver runs (10 000 iterations of
μ = A·t; y = max(0, μ_min − μ); g = Aᵀ·y; t = max(0, t + η(g − 1)) — the
shape of a PDHG step, not a solver).  Times µs/iteration eagerly and under
CUDA-graph capture and prints one JSON line.

usage: python tools/c3_loop.py [iters]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import configs, vectors  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    out = []
    for seed in range(10):
        c = configs.c3(seed)
        sc = uvd.Scene(c["scene"])
        lam, _ = sc.vantage(c["vantage"])
        A = sc.irradiance(lam)["A"]
        N, K = sc.N, lam.shape[0]
        t = torch.from_numpy(vectors.dense_iterate(K, seed)).cuda()
        eta = 1e-3
        mu = torch.empty(N, dtype=torch.float64, device="cuda")
        y = torch.empty(N, dtype=torch.float64, device="cuda")
        g = torch.empty(K, dtype=torch.float64, device="cuda")

        def it():
            uvd.fluence(A, N, t, out=mu)
            torch.clamp(configs.MU_MIN - mu, min=0.0, out=y)
            uvd.fluence(A, N, y, transpose=True, out=g)
            t.add_(eta * (g - 1.0)).clamp_(min=0.0)

        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                it()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(iters):
                it()
            e1.record(s)
            torch.cuda.synchronize()
            eager_us = e0.elapsed_time(e1) * 1e3 / iters
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                for _ in range(10):
                    it()
            e0.record(s)
            for _ in range(iters // 10):
                graph.replay()
            e1.record(s)
            torch.cuda.synchronize()
            graph_us = e0.elapsed_time(e1) * 1e3 / (iters // 10 * 10)
        out.append(dict(seed=seed, N=N, K=K, eager_us=eager_us, graph_us=graph_us))
        sc.close()
    print(json.dumps({"workload": "C3: 10 random 2.5D rooms, 0.5 m grid, A·t / Aᵀ·y loop",
                      "iters": iters, "median_eager_us_per_iter": float(np.median([o["eager_us"] for o in out])),
                      "median_graph_us_per_iter": float(np.median([o["graph_us"] for o in out])),
                      "rooms": out}))


if __name__ == "__main__":
    main()
