"""Multi-GPU plumbing: degree shards and the one collective.

Components (l, m) are independent (transform.cpp:265-287 only reads f, h and the tables), so
ranks compute contiguous degree ranges [l0, l1) with no data-path communication. The only
exchange is a final gather of the per-component results to rank 0: every rank's digest rows
[l0^2, l1^2) (coeff_index(l, m) = l^2 + l + m makes a degree range a contiguous row range).
Rows are copied, never reduced, so the gathered digests are bit-identical to a one-rank run.
"""
from __future__ import annotations

from .configs import shard_degrees  # noqa: F401  (re-exported: balanced l-ranges)


def row_range(l0: int, l1: int) -> tuple[int, int]:
    """Digest/volume rows of degrees [l0, l1)."""
    return l0 * l0, l1 * l1


def gather_digests(local, l0: int, l1: int, lmax: int, group=None, dst: int = 0):
    """Assemble the full digest table on rank `dst`.

    local : torch tensor [coeff_count(lmax), 8] holding this rank's rows (others ignored)
    Returns the full table on `dst` (a new tensor on local's device), None elsewhere.
    Uses all_gather of padded row blocks (works on nccl and gloo).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = row_range(l0, l1)
    bounds = torch.tensor([r0, r1], dtype=torch.int64, device=local.device)
    all_bounds = [torch.zeros_like(bounds) for _ in range(world)]
    dist.all_gather(all_bounds, bounds, group=group)
    spans = [(int(b[0]), int(b[1])) for b in all_bounds]
    width = max(1, max(b - a for a, b in spans))
    block = torch.zeros((width, local.shape[1]), dtype=local.dtype, device=local.device)
    block[: r1 - r0] = local[r0:r1]
    blocks = [torch.zeros_like(block) for _ in range(world)]
    dist.all_gather(blocks, block, group=group)
    if rank != dst:
        return None
    full = torch.full((((lmax + 1) ** 2), local.shape[1]), float("nan"), dtype=local.dtype,
                      device=local.device)
    for (a, b), blk in zip(spans, blocks):
        full[a:b] = blk[: b - a]
    return full
