"""Multi-rank CUDA path: two processes on
cuda:0 (the GPU pool is single-GPU) with a gloo process group, each calling
libuvd on its block-cyclic column shard; the partial μ = A_r·t_r and A_r·𝟙 are
summed by all_reduce; the scene is built once (rank 0) and broadcast as a
uvd_scene_export image (gloo broadcast of a CUDA tensor).  Checks: every rank's A shard and visibility bits equal
the corresponding columns of a single-process assembly bit for bit, the
reduced μ equals the single-process μ within 1e-12 relative (reduction order
only), and coverage agrees.  Plus a torchrun dry run of bench.py's multi-rank
path (gloo, ranks sharing the device) on a small workload.

The ranks never wait on each other inside a kernel: they only meet in the
host-side collective, so sharing one GPU is a functional test of the plumbing,
not a performance stand-in for several GPUs."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2103_14137_b200 import shard, uvd
    from synth import configs, vectors, ward
    desc = ward.ward(seed=2, n_bays=1, e=0.12)
    sc = shard.broadcast_scene(desc)  # rank 0 builds, the other rank imports the broadcast image
    lamps, _ = sc.vantage(configs.FLOAT_OPTS)
    K, N = lamps.shape[0], sc.N
    cols = shard.block_cyclic(K, world, rank, 32)
    r = sc.irradiance(lamps, cols=cols, vis_bits=True)
    t = torch.from_numpy(vectors.sparse_plan(K, seed=3)).cuda()
    mu = uvd.fluence(r["A"], N, t[cols].contiguous())
    rowsum = uvd.fluence(r["A"], N, torch.ones(len(cols), dtype=torch.float64, device="cuda"))
    shard.reduce_partials(mu, rowsum)     # gloo all_reduce on CUDA tensors
    cov = sc.coverage(mu, configs.MU_MIN, rowsum)
    sc.sync_status()
    out[rank] = dict(cols=cols, A=r["A"][:, :N].cpu().numpy(), vb=r["vis_bits"].cpu().numpy(),
                     mu=mu.cpu().numpy(), cov=cov, K=K)
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def uvd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd as U
    return U


def test_two_ranks_on_libuvd_match_single_process(uvd):
    import torch.multiprocessing as mp
    from synth import configs, vectors, ward
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    desc = ward.ward(seed=2, n_bays=1, e=0.12)
    sc = uvd.Scene(desc)
    lamps, _ = sc.vantage(configs.FLOAT_OPTS)
    K, N = lamps.shape[0], sc.N
    full = sc.irradiance(lamps, vis_bits=True)
    A = full["A"][:, :N].cpu().numpy()
    vb = full["vis_bits"].cpu().numpy()
    t = torch.from_numpy(vectors.sparse_plan(K, seed=3)).cuda()
    mu = uvd.fluence(full["A"], N, t).cpu().numpy()
    rowsum = uvd.fluence(full["A"], N, torch.ones(K, dtype=torch.float64, device="cuda"))
    cov = sc.coverage(torch.from_numpy(mu).cuda(), configs.MU_MIN, rowsum)
    seen = []
    for rank in (0, 1):
        o = out[rank]
        assert o["K"] == K
        c = np.asarray(o["cols"])
        seen += list(c)
        assert np.array_equal(o["A"], A[c]), f"rank {rank}: A shard differs from the single-process columns"
        assert np.array_equal(o["vb"], vb[c])
        assert np.allclose(o["mu"], mu, rtol=1e-12, atol=0)
        assert np.allclose(o["cov"], cov, rtol=1e-12)
    assert sorted(seen) == list(range(K))
    assert np.array_equal(out[0]["mu"], out[1]["mu"])


def test_bench_torchrun_gloo_dry_run(uvd, tmp_path):
    """bench.py's multi-rank path end to end under torchrun (2 ranks, gloo,
    one device): one JSON line from rank 0 with n_gpus = 2, max-over-ranks
    timing and the per-rank column shard; each rank's shard dump (--dump)
    re-checks clean against the oracle offline (tools/recheck_dump.py)."""
    env = dict(os.environ, BENCH_BACKEND="gloo")
    prefix = str(tmp_path / "mr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--workload", "C2", "--no-cpu-baseline",
           "--no-e2e", "--no-clocks", "--dump", prefix]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["k_per_gpu"] < d["config"]["k_configs"]
    assert d["roofline"]["imbalance"] >= 1.0
    q = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "recheck_dump.py"), prefix, "--pairs", "2000"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert q.returncode == 0, q.stdout[-2000:] + q.stderr[-2000:]
    st = [json.loads(ln) for ln in q.stdout.splitlines() if ln.startswith("{")]
    assert sorted(x["rank"] for x in st) == [0, 1] and all(x["mismatches"] == 0 for x in st)
