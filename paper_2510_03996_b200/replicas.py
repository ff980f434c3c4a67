"""Multi-GPU plumbing for the hot path: independent replicas.

The path does not shard: a key switch needs every
limb, so limb-sharding would cost an all-to-all per rotation.  Each rank runs
its own images / ciphertext batches with its own resident keys; the only
collectives are a start/stop barrier and a max-reduction of the timed region
(torch.distributed over NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Tuple


def world() -> Tuple[int, int]:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def barrier(device=None):
    import torch
    import torch.distributed as dist
    if device is not None and device.type == "cuda":
        torch.cuda.synchronize(device)
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (timed-region milliseconds) over all ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(local_ms: float, units_per_rank: int, device=None) -> Tuple[float, float]:
    """Whole-job throughput: all ranks' units over the slowest rank's time.

    Returns (units_per_second, max_ms)."""
    ws, _ = world()
    mx = max_over_ranks(local_ms, device)
    return ws * units_per_rank / (mx / 1e3), mx
