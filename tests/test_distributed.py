"""The multi-rank path on CPU (gloo, world size 2): degree shards laid out by the engine's own
shard rule (slsht_cuda_shard_bounds, the split of a multi-GPU plan) are computed independently
(here by the CPU oracle: this container has no device; tests/test_gpu.py runs the same gather
on engine-computed shards) and gathered to rank 0 with paper_1207_5558_b200.parallel.
gather_digests; the result must reproduce the one-rank table bit for bit (rows are copied,
never reduced)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    import oracle
    import paper_1207_5558_b200 as S
    from paper_1207_5558_b200.parallel import gather_digests

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = oracle.Oracle()
    L_f, L_h = 6, 3
    rng = np.random.default_rng(11)
    f = rng.standard_normal(49) + 1j * rng.standard_normal(49)
    h = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    bounds = S.shard_bounds(0, L_f + L_h + 1, False, world)
    l0, l1 = bounds[rank], bounds[rank + 1]
    local = torch.full(((L_f + L_h + 1) ** 2, 8), float("nan"), dtype=torch.float64)
    lm = [(l, m) for l in range(l0, l1) for m in range(-l, l + 1)]
    vols = O.components(f, L_f, h, L_h, lm)
    for (l, m), v in vols.items():
        local[l * l + l + m] = torch.from_numpy(O.digest(L_h, v))
    full = gather_digests(local, l0, l1, L_f + L_h)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_digests_gather_bitwise(tmp_path, oracle_lib):
    import torch.multiprocessing as mp

    out = tmp_path / "full.npy"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    full = np.load(out)
    rng = np.random.default_rng(11)
    f = rng.standard_normal(49) + 1j * rng.standard_normal(49)
    h = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    ref = np.full_like(full, np.nan)
    vols = oracle_lib.forward_fast(f, 6, False, h, 3, False)
    for (l, m), v in vols.items():
        ref[l * l + l + m] = oracle_lib.digest(3, v)
    assert not np.isnan(full).any()
    assert np.array_equal(full, ref)


def _volume_worker(rank, world, port, out_path):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    import oracle
    import paper_1207_5558_b200 as S
    from paper_1207_5558_b200.parallel import gather_sampled, gather_volumes

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = oracle.Oracle()
    L_f, L_h = 5, 2
    rng = np.random.default_rng(12)
    f = rng.standard_normal(36) + 1j * rng.standard_normal(36)
    h = rng.standard_normal(9) + 1j * rng.standard_normal(9)
    bounds = S.shard_bounds(0, L_f + L_h + 1, False, world)
    l0, l1 = bounds[rank], bounds[rank + 1]
    lm = [(l, m) for l in range(l0, l1) for m in range(-l, l + 1)]
    vols = O.components(f, L_f, h, L_h, lm)
    shape = S.volume_shape(L_h)
    local = torch.from_numpy(np.stack([vols[k].reshape(shape) for k in lm])) if lm else \
        torch.zeros((0,) + shape, dtype=torch.complex128)
    full = gather_volumes(torch.view_as_real(local), l0, l1, L_f + L_h)
    sampled = {k: torch.view_as_real(torch.from_numpy(vols[k].reshape(shape)))
               for k in lm if (k[0] + k[1]) % 3 == 0}
    got = gather_sampled(sampled, shape + (2,), torch.float64, "cpu")
    if rank == 0:
        keys = sorted(got)
        np.savez(out_path, full=torch.view_as_complex(full).numpy(),
                 keys=np.array(keys), sampled=np.stack([torch.view_as_complex(got[k].contiguous()).numpy()
                                                        for k in keys]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_volumes_gather_bitwise(tmp_path, oracle_lib, world):
    """the full distribution (configs 1-2) and sampled volumes (configs 3-5) are
    gathered to rank 0 by point-to-point row-block transfers; bitwise the one-process result."""
    import torch.multiprocessing as mp

    out = tmp_path / "full.npz"
    mp.spawn(_volume_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    got = np.load(out)
    rng = np.random.default_rng(12)
    f = rng.standard_normal(36) + 1j * rng.standard_normal(36)
    h = rng.standard_normal(9) + 1j * rng.standard_normal(9)
    vols = oracle_lib.forward_fast(f, 5, False, h, 2, False)
    import paper_1207_5558_b200 as S
    shape = S.volume_shape(2)
    assert got["full"].shape == (64,) + shape
    for (l, m), v in vols.items():
        assert np.array_equal(got["full"][l * l + l + m], v.reshape(shape)), (l, m)
    want = sorted(k for k in vols if (k[0] + k[1]) % 3 == 0)
    assert [tuple(k) for k in got["keys"]] == want
    for i, k in enumerate(want):
        assert np.array_equal(got["sampled"][i], vols[k].reshape(shape)), k
