"""Multi-GPU plumbing of the hot path: column sharding and the
one exchange step.  Pure host logic (torch.distributed), no CUDA needed here:

* vantage columns are sharded block-cyclically (blocks of 32) so clutter-
  dependent column costs balance across ranks; the scene is replicated;
* assembly needs no exchange (columns are independent);
* the partial fluence μ_r = A_r·t_r and A_r·𝟙 are summed by all_reduce (NCCL on
  GPUs, gloo in the CPU tests);
* timings are reduced with MAX (the slowest rank defines the step);
* the scene can be built once (rank 0) and broadcast as a uvd_scene_export
  image instead of being rebuilt by every rank (`broadcast_scene`).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def block_cyclic(k_total: int, world: int, rank: int, block: int = 32) -> list[int]:
    """Global column ids owned by `rank`: blocks of `block` consecutive
    columns dealt round-robin over `world` ranks."""
    if world < 1 or not 0 <= rank < world or block < 1:
        raise ValueError("bad shard spec")
    return [j for j in range(k_total) if (j // block) % world == rank]


def reduce_partials(*tensors: torch.Tensor) -> None:
    """Sum per-rank partial fluence vectors in place (the path's only exchange)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        for t in tensors:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)


def max_over_ranks(values: list[float], device=None) -> list[float]:
    """Element-wise MAX over ranks of host scalars (step timings)."""
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return list(values)
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def sum_over_ranks(values, device=None):
    """Element-wise SUM over ranks (instrumentation counters)."""
    t = torch.as_tensor(values, dtype=torch.float64, device=device).clone()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def broadcast_scene(desc, device=None, src: int = 0):
    """Rank `src` builds the scene (uvd_scene_create) and broadcasts its
    uvd_scene_export image; every other rank imports it (uvd_scene_import):
    the same scene bit for bit, one build instead of one per rank.
    Single process: a plain build."""
    from . import uvd
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return uvd.Scene(desc, device=device)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if dist.get_rank() == src:
        sc = uvd.Scene(desc, device=dev.index)
        img = sc.export()
        n = torch.tensor([img.numel()], dtype=torch.int64, device=dev)
    else:
        sc = None
        n = torch.zeros(1, dtype=torch.int64, device=dev)
    dist.broadcast(n, src)
    if sc is None:
        img = torch.empty(int(n.item()), dtype=torch.uint8, device=dev)
    dist.broadcast(img, src)
    return sc if sc is not None else uvd.Scene.from_image(img, device=dev.index)
