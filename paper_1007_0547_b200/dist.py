"""Host-side plumbing for running one detection across ranks.

Points of one image are sharded contiguously across ranks: votes are sums over points, so every
rank counts its own lines and libhht adds the per-level vote vectors with an in-place NCCL
allreduce; every rank then takes identical split decisions and compacts only its own lists.
A batch of independent images is sharded by whole images instead (no collective at all).

This module only moves arrays and small values between processes (torch.distributed): the
method's arithmetic stays in libhht. It is backend-agnostic (nccl on the GPU box, gloo in the
CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from .synth import shard


@dataclass
class Shard:
    points: np.ndarray        # int32 [n_local, 2]
    offsets: np.ndarray       # int64 [B_local + 1], local image offsets
    comm_world: int           # ranks that share the detection through NCCL (1 = independent)
    image_lo: int             # first global image index owned (image sharding), else 0
    mode: str                 # "points" or "images"


def make_shard(points: np.ndarray, offsets: np.ndarray, rank: int, world: int) -> Shard:
    """Single image (B = 1): contiguous point shard, NCCL across all ranks.
    Batch (B > 1): whole images, no collective (each rank owns an independent set of trees)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    B = offsets.shape[0] - 1
    if B > 1:
        lo, hi = shard(B, rank, world)
        p = np.ascontiguousarray(points[offsets[lo]:offsets[hi]])
        return Shard(p, offsets[lo:hi + 1] - offsets[lo], 1, lo, "images")
    lo, hi = shard(int(offsets[-1]), rank, world)
    p = np.ascontiguousarray(points[lo:hi])
    return Shard(p, np.array([0, p.shape[0]], dtype=np.int64), world, 0, "points")


def broadcast_bytes(data: Optional[bytes], src: int = 0) -> bytes:
    """Broadcast a small byte string (e.g. the 128-byte ncclUniqueId) from `src`."""
    import torch.distributed as dist
    obj = [data]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def _coll_device():
    """Device for collective tensors: the current CUDA device under NCCL (which rejects CPU tensors),
    the CPU under gloo."""
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def check_consistent(N: int, depth: int, threshold: int, halves: int, images: int) -> None:
    """Raise if ranks disagree on the call arguments (libhht re-checks with NCCL: HHT_EMISMATCH)."""
    import torch
    import torch.distributed as dist
    v = torch.tensor([N, depth, threshold, halves, images], dtype=torch.int64, device=_coll_device())
    lo, hi = v.clone(), v.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    if not torch.equal(lo, hi):
        raise ValueError(f"ranks disagree on (N, depth, threshold, halves, images): min {lo.tolist()} max {hi.tolist()}")


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device if device is not None else _coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device if device is not None else _coll_device())
    dist.all_reduce(t)
    return float(t.item())


def env_rank_world() -> Tuple[int, int, int]:
    import os
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))
