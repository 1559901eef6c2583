"""Multi-process plumbing for `bench.py --gpus N` (one process per GPU, torch.distributed).

Round 1 runs REPLICAS: every rank simulates the whole circuit (an independent shot, seed ^ rank);
there is no data-path collective.  The only exchanges are the barrier and the max-over-ranks of
the device-measured step time.  Backend: nccl when CUDA is usable, gloo otherwise (CPU tests).
Row sharding of a single tableau would replace `shot_seed` by a slot range
from `slot_range` (stabilizer i and destabilizer i stay on one rank) -- see DESIGN.md section 7.
"""
from __future__ import annotations

import os


def env_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def init(backend: str | None = None):
    """Initialise torch.distributed if WORLD_SIZE > 1.  Returns (rank, local_rank, world)."""
    import torch
    import torch.distributed as dist
    rank, local_rank, world = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {"device_id": torch.device("cuda", local_rank)} if backend == "nccl" else {}
        dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    return rank, local_rank, world


def shot_seed(seed: int, rank: int) -> int:
    """Per-rank seed of the replica (SPEC:333 derives shot seeds as seed XOR shot index)."""
    return seed ^ rank


def slot_range(n: int, rank: int, world: int):
    """Contiguous range of row slots [lo, hi) owned by `rank` under row sharding: slot i is
    stabilizer i together with destabilizer i, so the deterministic branch (destabilizer j selects
    stabilizer j) stays local.  Word aligned (multiples of 64) so that column slices are whole words."""
    words = (n + 63) // 64
    per = (words + world - 1) // world
    lo = min(words, rank * per) * 64
    hi = min(words, (rank + 1) * per) * 64
    return min(lo, n), min(hi, n)


def barrier():
    import torch
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize()


def max_over_ranks(value: float) -> float:
    """Slowest rank's value (device times are reduced this way, never wall clocks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_records(checksum: int):
    """All ranks' record checksums on every rank (replicas with different seeds must differ only
    in the random outcomes)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [int(checksum)]
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    mine = torch.tensor([checksum], dtype=torch.int64, device=dev)
    out = [torch.zeros_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(out, mine)
    return [int(t.item()) for t in out]


def finalize():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
