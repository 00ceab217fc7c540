"""Host plumbing of the multi-GPU layout: which patch a rank
holds, and the NCCL unique id handshake for ``yy_create_dist``.

One process per GPU.  World 1: both patches on the one GPU (``yy_create``).
World 2: rank r holds patch r (Yin = 0, Yang = 1); the Yin<->Yang fringe
exchange (Alg. 1 steps 1/3/7) and the per-(quantity, patch) norms
(RD24) are swapped pairwise over NCCL inside ``yy_step``.  Radial slabs
(worlds 4 and 8, partitioned r-solve P:L477-480) are not built.

``torch.distributed`` is used only to move the 128-byte id from rank 0 to the
partner (any backend: gloo moves it through host memory, nccl through the GPU).
"""
from __future__ import annotations

SUPPORTED_WORLDS = (1, 2)


def plan(world: int, rank: int) -> dict:
    """{'patches': (...), 'partner': rank or None} for this rank."""
    if world not in SUPPORTED_WORLDS:
        raise ValueError(f"world {world}: only 1 (both patches) or 2 (one patch per rank) is built; "
                         "radial slabs for 4/8 GPUs are not")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if world == 1:
        return {"patches": (0, 1), "partner": None}
    return {"patches": (rank,), "partner": 1 - rank}


def share_unique_id(rank: int, device=None) -> bytes:
    """Rank 0 draws an NCCL unique id (yy_nccl_unique_id), every rank returns it.
    Needs an initialised torch.distributed default group."""
    import torch
    import torch.distributed as td

    from .yy import nccl_unique_id

    buf = torch.zeros(128, dtype=torch.uint8, device=device if device is not None else "cpu")
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    td.broadcast(buf, src=0)
    return bytes(buf.cpu().tolist())
