"""Host-side plumbing of the multi-GPU hot path (one process per GPU).

Data parallel, weak scaling: rank g holds records
[g*R, (g+1)*R) of an N*R-record dataset and a full hot-table replica
(P:L298-301).  This module only moves host-side control values through a
torch.distributed process group; every data-path exchange (loggers, the
sampling histograms, the hot-gradient all-gathers) is NCCL inside libfae.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from . import Ctx, fae_comm_init, fae_get_nccl_id


def shard(records_per_rank: int, rank: int) -> tuple:
    """(record_base, n_records) of this rank's contiguous shard."""
    return rank * records_per_rank, records_per_rank


def broadcast_bytes(payload: Optional[bytes], src: int, nbytes: int,
                    device: Optional[torch.device] = None) -> bytes:
    """Broadcast `nbytes` bytes from rank `src` (any backend)."""
    t = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_rank() == src:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(t.device))
    dist.broadcast(t, src)
    return bytes(t.cpu().numpy().tobytes())


def init_comm(ctx: Ctx, device: Optional[torch.device] = None):
    """Create the library's own NCCL communicator: rank 0 draws the id, the
    process group broadcasts it, every rank calls fae_comm_init."""
    rank, world = dist.get_rank(), dist.get_world_size()
    nid = fae_get_nccl_id() if rank == 0 else None
    nid = broadcast_bytes(nid, 0, 128, device)
    fae_comm_init(ctx, nid, rank, world)


def max_over_ranks(v: int, device: Optional[torch.device] = None) -> int:
    """Hot-batch count of the slowest rank: every rank runs that many steps
    (a rank past its last batch contributes an empty gradient)."""
    t = torch.tensor([int(v)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return int(t.item())


def sum_over_ranks(v: float, device: Optional[torch.device] = None) -> float:
    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
