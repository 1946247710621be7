"""Multi-GPU layout of the path: independent replicas, no data-path collective.

Frames and streams are independent: each rank owns whole frames or whole
streams, keeps its own 2-slot memory and weights, and never exchanges activations.  The
only cross-rank operations are control-plane: a barrier around the timed region and a
max-reduction of the per-rank timings (bench.py), plus an optional final gather of
per-frame results.  These helpers are backend-agnostic (NCCL on GPUs, gloo in the CPU
tests).
"""

from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def stream_owner(stream: int, world_size: int) -> int:
    """C3: stream s runs on rank s mod world (8 streams on 8 GPUs = one each)."""
    return stream % world_size


def rank_streams(rank: int, world_size: int, n_streams: int) -> list[int]:
    """Streams owned by `rank` (co-resident streams are batched with per-stream slots)."""
    return [s for s in range(n_streams) if stream_owner(s, world_size) == rank]


def frame_seeds(rank: int, n: int, stride: int = 100003) -> list[int]:
    """C5 weak scaling: rank r's n frames use seeds r*stride + i (disjoint across ranks)."""
    return [rank * stride + i for i in range(n)]


def allreduce_max(value: float, device=None) -> float:
    """Max of a scalar over all ranks (identity without an initialised process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(t, device=None):
    """Final gather of per-rank results (equal shapes) onto rank 0: a list ordered by
    rank on rank 0, None elsewhere (`dist.gather`: NCCL on GPUs over NVLink / NVSwitch,
    gloo on CPU)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [t]
    t = t.contiguous()
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())] \
        if dist.get_rank() == 0 else None
    dist.gather(t, out, dst=0)
    return out
