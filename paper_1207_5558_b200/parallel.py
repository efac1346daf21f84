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


def gather_volumes(local, l0: int, l1: int, lmax: int, group=None, dst: int = 0):
    """Assemble the full distribution on rank `dst` (configs 1-2 gather the
    whole distribution, 70 MB / 6.2 GB).

    local : torch tensor [l1^2 - l0^2, ...] holding the volumes of this rank's degree shard in
            coeff_index order (row i is component l0^2 + i: the layout of a materialized plan's
            device distribution and of Plan.forward_copy with first_index = l0^2)
    Returns the [coeff_count(lmax), ...] distribution on `dst`, None elsewhere. A degree range
    is a contiguous row range, so every shard is received straight into its rows of the
    result (point-to-point send / recv: NCCL P2P over NVLink on devices, gloo on the host);
    nothing is reduced, so the gathered distribution is bitwise the one-rank result.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = row_range(l0, l1)
    if local.shape[0] != r1 - r0:
        raise ValueError("local must hold exactly the rows of degrees [l0, l1)")
    bounds = torch.tensor([r0, r1], dtype=torch.int64, device=local.device)
    all_bounds = [torch.zeros_like(bounds) for _ in range(world)]
    dist.all_gather(all_bounds, bounds, group=group)
    spans = [(int(b[0]), int(b[1])) for b in all_bounds]
    local = local.contiguous()
    if rank != dst:
        if r1 > r0:
            dist.send(local, dst=dst, group=group)
        return None
    full = torch.empty(((lmax + 1) ** 2,) + tuple(local.shape[1:]), dtype=local.dtype,
                       device=local.device)
    covered = torch.zeros((lmax + 1) ** 2, dtype=torch.bool)
    for src, (a, b) in enumerate(spans):
        if b <= a:
            continue
        if src == dst:
            full[a:b] = local
        else:
            dist.recv(full[a:b], src=src, group=group)  # a contiguous view: no staging copy
        covered[a:b] = True
    if not bool(covered.all()):
        raise ValueError("the shards do not cover every degree up to lmax")
    return full


def gather_sampled(local: dict, vol_shape, dtype, device, group=None, dst: int = 0):
    """Gather sampled component volumes {(l, m): tensor} to rank `dst` (configs
    3-5 gather sampled volumes, not the distribution). Every rank passes the sampled components
    of its own shard; returns the merged dict on `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    keys = sorted(local)
    all_keys = [None] * world
    dist.all_gather_object(all_keys, keys, group=group)
    if rank != dst:
        if keys:
            dist.send(torch.stack([local[k].reshape(vol_shape) for k in keys]).contiguous(),
                      dst=dst, group=group)
        return None
    out = {k: local[k].reshape(vol_shape) for k in keys}
    for src, ks in enumerate(all_keys):
        if src == dst or not ks:
            continue
        buf = torch.empty((len(ks),) + tuple(vol_shape), dtype=dtype, device=device)
        dist.recv(buf, src=src, group=group)
        for i, k in enumerate(ks):
            if tuple(k) in out:
                raise ValueError(f"component {k} sampled on two ranks")
            out[tuple(k)] = buf[i]
    return out
