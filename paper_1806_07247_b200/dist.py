"""Host-side multi-GPU plumbing of the lateral-slice partition.

Columns of unfold(B) map 1:1 to columns of unfold(C) (Eq. (9)), so rank r can
compute C(:, J_r, :) = A * B(:, J_r, :) for its own contiguous block J_r of lateral slices with
no exchange.  A is replicated once (setup, NCCL broadcast through the C ABI); the per-call path
has no collective.  These helpers are backend-agnostic so that the same code runs under NCCL on
the GPU box and under gloo in the CPU tests.
"""
from __future__ import annotations


def lateral_shard(n4: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous block [start, stop) of the n4 lateral slices owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n4, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def exchange_uid(make_uid, src: int = 0) -> bytes:
    """Rank `src` creates the 128-byte NCCL unique id (make_uid()), every rank receives it."""
    import torch.distributed as dist
    obj = [make_uid() if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def replicate(t, root: int = 0, handle=None):
    """One-time replication of A from `root` to every rank, in place.

    With a tprod Handle (GPU box) this is the library's ncclBroadcast (tprod_bcast_f32/f64);
    otherwise torch.distributed.broadcast (gloo CPU tests)."""
    flat = t.permute(2, 1, 0) if t.dim() == 3 else t     # Matlab layout -> contiguous view
    if handle is not None:
        handle.bcast_(flat, root=root)
    else:
        import torch.distributed as dist
        dist.broadcast(flat, src=root)
    return t


def max_over_ranks(x: float, device=None) -> float:
    """Timing reduction: the job's time is the slowest rank's."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_lateral(C_local, n4: int, dst: int = 0):
    """Reassemble the full n1 x n4 x n3 result on `dst` from the ranks' shards (verification)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    n1, _, n3 = C_local.shape
    parts = []
    for r in range(world):
        s, e = lateral_shard(n4, world, r)
        buf = C_local.permute(2, 1, 0).contiguous() if r == rank else \
            torch.empty((n3, e - s, n1), dtype=C_local.dtype, device=C_local.device)
        dist.broadcast(buf, src=r)
        parts.append(buf)
    if rank != dst:
        return None
    return torch.cat(parts, dim=1).permute(2, 1, 0)
