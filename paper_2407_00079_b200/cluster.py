"""Prefill / decode partitioning of one 8xB200 NVSwitch box (one process per
GPU) and the pair handshake.

Ranks [0, N/2) are prefill GPUs, [N/2, N) decode GPUs, pair i = (i, i + N/2)
(SURVEY.md 8(e)).  The reference's cluster is a vector of prefill and decode
instances in one process (proj/src/sim_engine.cpp:681-690); here each instance
is a GPU and the Messenger link between them is NVLink.  NVSwitch gives every
pair the full per-direction bandwidth, so pairing is free of topology cost.
With N = 1 the two instances share one GPU ("local").

The handshake exchanges what the sender must map (CUDA IPC handles of the
decode pool / receive ring / flag words) and the decode block tables -- in the
reference the decode choice and its resources are decided by the Conductor
(proj/src/conductor.cpp:238) before the stream starts.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch.distributed as dist


@dataclass(frozen=True)
class PairRole:
    role: str   # "local" | "prefill" | "decode"
    pair: int
    peer: int   # rank of the other end (== own rank when local)
    pairs: int


def pair_topology(world: int, rank: int) -> PairRole:
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad world/rank {world}/{rank}")
    if world == 1:
        return PairRole("local", 0, 0, 1)
    if world % 2:
        raise ValueError("prefill/decode pairing needs an even number of GPUs")
    half = world // 2
    if rank < half:
        return PairRole("prefill", rank, rank + half, half)
    return PairRole("decode", rank - half, rank - half, half)


def exchange_with_peer(role: PairRole, payload) -> object:
    """All-gather one picklable payload per rank; return the pair peer's."""
    world = dist.get_world_size()
    out = [None] * world
    dist.all_gather_object(out, payload)
    return out[role.peer]


def max_over_ranks(x: float, device=None) -> float:
    """Max of a float over all ranks (timing: the slowest rank defines the step)."""
    import torch
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device=device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device=device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
