"""Per-rank shard dumps (SURVEY §5 checkpoint: A shards and visibility bits
for offline parity re-checks): the uvd-shard/1 writer and reader round-trip
every section bit for bit (CPU), and on a GPU a bench run's dump re-checks
clean against the oracle with tools/recheck_dump.py."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dump_load_roundtrip(tmp_path):
    from paper_2103_14137_b200 import shard
    rng = np.random.default_rng(0)
    n_cols, ld, N, L = 5, 96, 70, 2
    A = rng.random((n_cols, ld), dtype=np.float32)
    vb = rng.integers(0, 2**32, (n_cols, L, (N + 31) // 32), dtype=np.uint64).astype(np.uint32)
    lamps = rng.random((n_cols, L, 3), dtype=np.float32)
    orig = rng.permutation(N).astype(np.int64)
    cols, raw = [3, 4, 35, 36, 67], np.array([10, 11, 40, 41, 90])
    prefix = str(tmp_path / "shard")
    hp = shard.dump_shard(prefix, workload="C2", A=A, n_rows=N, cols=cols, raw=raw, lamps=lamps, orig_id=orig,
                          power_w=80.0, vis_bits=vb, rank=1, world=2)
    head = json.load(open(hp))
    assert head["format"] == "uvd-shard/1" and head["rank"] == 1 and head["world"] == 2
    h2, sec = shard.load_shard(prefix, 1)
    assert h2 == head and h2["cols"] == cols and h2["raw"] == raw.tolist()
    assert np.array_equal(sec["A"], A[:, :N]) and np.array_equal(sec["vis_bits"], vb)
    assert np.array_equal(sec["lamps"], lamps) and np.array_equal(sec["orig_id"], orig)
    with pytest.raises(FileNotFoundError):
        shard.load_shard(prefix, 0)


@pytest.mark.gpu
def test_bench_dump_rechecks_clean(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    prefix = str(tmp_path / "c2")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "C2", "--steps", "1",
                        "--warmup", "3", "--no-cpu-baseline", "--no-parity", "--no-e2e", "--no-clocks",
                        "--dump", prefix], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    q = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "recheck_dump.py"), prefix, "--pairs", "3000"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert q.returncode == 0, q.stdout[-2000:] + q.stderr[-2000:]
    st = [json.loads(ln) for ln in q.stdout.splitlines() if ln.startswith("{")]
    assert st and all(s["mismatches"] == 0 and s["entries_beyond_tol"] == 0 for s in st)
