"""Host plumbing of the multi-GPU layout: which patch a rank
holds, and the NCCL unique id handshake for ``yy_create_dist``.

One process per GPU.  World 1: both patches on the one GPU (``yy_create``).
World 2*nslab: rank r holds radial slab r % nslab of patch r // nslab (Yin on
the first nslab ranks); inside ``yy_step`` the Yin<->Yang fringe (P:L481-483,
Alg. 1 steps 1/3/7) is swapped with the same slab of the other patch, r-halo rows
with the slab neighbours, the boundary rows of the partitioned r-solve
within the patch, and the per-(quantity, patch, slab) norms (RD24) with everyone,
over NCCL point-to-point.

``torch.distributed`` is used only to move the 128-byte id from rank 0 to the
partner (any backend: gloo moves it through host memory, nccl through the GPU).
"""
from __future__ import annotations

SUPPORTED_WORLDS = (1, 2, 4, 8, 16)


def plan(world: int, rank: int, nr: int | None = None) -> dict:
    """This rank's part of the shell: patch, radial slab, and the ranks it talks to
    (fringe partner = same slab of the other patch; slab neighbours below/above).
    world = 1: both patches, no partners.  nr (cells per patch, optional) is
    checked for the slab split."""
    if world not in SUPPORTED_WORLDS:
        raise ValueError(f"world {world}: 1 (both patches) or 2*nslab ranks (nslab = 1, 2, 4, 8)")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if world == 1:
        return {"patches": (0, 1), "patch": None, "slab": 0, "nslab": 1, "partner": None,
                "below": None, "above": None}
    S = world // 2
    if nr is not None and (nr % S or nr // S < 4):
        raise ValueError(f"nr = {nr} does not split into {S} radial slabs of >= 4 rows")
    p, sl = divmod(rank, S)
    return {"patches": (p,), "patch": p, "slab": sl, "nslab": S, "partner": (1 - p) * S + sl,
            "below": rank - 1 if sl > 0 else None, "above": rank + 1 if sl < S - 1 else None}


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
