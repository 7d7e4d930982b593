"""Host side of the row-sharded solve: shard planning and communicator
setup over a torch.distributed process group.

One process per GPU. Rank g owns the contiguous row block ``shard_rows(m, world, g)`` of
the m x n input; ``attach_process_group`` gives the rank's ``Solver`` an NCCL
communicator of its own (rank 0 creates the 128-byte NCCL unique id, the process group
broadcasts it — any backend, gloo included), after which
``Solver.randomized_ksvd_sharded[_device]`` runs collectively. The reference has no
multi-process path; the sharded solve computes the same
``randomized_ksvd`` (rsvd.hpp:58) with the sums over rows all-reduced.
"""
from __future__ import annotations

from .rsvd import ArgumentError, Solver, nccl_unique_id


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Row range [r0, r1) of `rank`: contiguous blocks, the first m % world ranks get one
    extra row (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ArgumentError(f"rank {rank} outside [0, {world})")
    if m < world:
        raise ArgumentError(f"cannot shard {m} rows over {world} ranks")
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def broadcast_unique_id(uid: bytes | None, group=None) -> bytes:
    """Rank 0's 128-byte id to every rank of the torch.distributed group."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    dev = torch.device("cpu")
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    # src is a global rank: the group's rank 0 (not global rank 0) created the id
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast(buf, src=src, group=group)
    return bytes(buf.cpu().tolist())


def attach_process_group(solver: Solver, group=None) -> tuple[int, int]:
    """Give `solver` an NCCL communicator spanning the ranks of `group`."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = nccl_unique_id() if rank == 0 else None
    uid = broadcast_unique_id(uid, group)
    solver.attach_nccl(uid, rank, world)
    return rank, world
