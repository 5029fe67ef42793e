"""World-size-2 gloo test of the multi-GPU host logic on CPU:
block-cyclic column shards partition the columns, per-rank partial fluence
μ_r = A_r·t_r summed by all_reduce equals the single-process μ, coverage on the
reduced μ matches, and timings reduce with MAX."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_14137_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A, t, area, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    K = A.shape[1]
    cols = shard.block_cyclic(K, world, rank)
    mu = torch.from_numpy(O.fluence(A[:, cols], t[cols]))
    ones = torch.from_numpy(O.fluence(A[:, cols], np.ones(len(cols))))
    shard.reduce_partials(mu, ones)
    cov = O.coverage(mu.numpy(), area, 280.0, ones.numpy())
    tmax = shard.max_over_ranks([float(rank + 1), -float(rank)])
    out[rank] = (cols, mu.numpy(), ones.numpy(), cov, tmax)
    dist.barrier()
    dist.destroy_process_group()


def test_block_cyclic_partition():
    for K, W in ((1000, 2), (999, 4), (65, 8), (31, 3)):
        parts = [shard.block_cyclic(K, W, r) for r in range(W)]
        allc = sorted(c for p in parts for c in p)
        assert allc == list(range(K))
        for p in parts:
            assert all(p[i] < p[i + 1] for i in range(len(p) - 1))
    with pytest.raises(ValueError):
        shard.block_cyclic(10, 2, 2)


def test_two_rank_fluence_allreduce_matches_single():
    from oracle import oracle as O
    from synth import configs
    c = configs.c3(2)
    pat = O.extruded_patches(c["scene"])
    v = O.vantage(c["scene"], c["vantage"])
    lam = v["samples"][v["feasible"]]
    A = O.irradiance_matrix(pat, lam, mode="2d")["A"].astype(np.float32)
    K = A.shape[1]
    t = np.random.default_rng(0).uniform(0, 300, K)
    ref_mu = O.fluence(A, t)
    ref_cov = O.coverage(ref_mu, pat["area"], 280.0, O.fluence(A, np.ones(K)))
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, A, t, pat["area"], out), nprocs=2, join=True)
    cols0, mu0, ones0, cov0, t0 = out[0]
    cols1, mu1, ones1, cov1, t1 = out[1]
    assert sorted(cols0 + cols1) == list(range(K))
    assert np.allclose(mu0, ref_mu, rtol=1e-12) and np.array_equal(mu0, mu1)
    assert np.array_equal(ones0, ones1)
    assert np.allclose(cov0, ref_cov, rtol=1e-12) and np.array_equal(cov0, cov1)
    assert t0 == t1 == [2.0, 0.0]
