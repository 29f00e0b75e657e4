"""Label-sharded merge orchestration on CPU (gloo, world size 2): shard_range + merge_keys_allreduce.

Each rank filters its contiguous label shard with the oracle (the GPU is replaced by the oracle here; the
CUDA kernels' keys are checked bit-exactly against the same packing in tests/test_gpu_parity.py), packs
signed keys, and the int64 allreduce-MIN must reproduce the unsharded WTA.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _signed_keys(cost, labels):
    return (O.pack_keys(cost.astype(np.float32), labels) ^ np.uint64(1 << 63)).view(np.int64)


def _worker(rank, world, port, L, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1803_00005_b200 import merge_keys_allreduce, shard_range
    I, V = synth.iid_volume(20, 14, L, 3, seed=21)
    l0, l1 = shard_range(L, world, rank)
    Z = O.hgf_filter(I, V[l0:l1], 0.05, 2, 2).astype(np.float32)
    lab = l0 + np.argmin(Z, axis=0)
    cost = Z.min(axis=0)
    keys = torch.from_numpy(_signed_keys(cost, lab).copy())
    merge_keys_allreduce(keys)
    if rank == 0:
        np.save(out_path, keys.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("L", [7, 2])
def test_gloo_world2_merge_equals_unsharded(tmp_path, L):
    world = 2
    out = str(tmp_path / "keys.npy")
    mp.spawn(_worker, args=(world, _free_port(), L, out), nprocs=world, join=True)
    merged = np.load(out)
    I, V = synth.iid_volume(20, 14, L, 3, seed=21)
    Z = O.hgf_filter(I, V, 0.05, 2, 2).astype(np.float32)
    full = _signed_keys(Z.min(axis=0), np.argmin(Z, axis=0))
    assert np.array_equal(merged, full)


def test_shard_range_partition():
    from paper_1803_00005_b200 import shard_range
    for L in (1, 7, 60, 256):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(L, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


class _FakeHandle:
    """Stands in for HGF in gather_stats_rows: H rows, a CPU statistics buffer (the real one is on the GPU)."""

    def __init__(self, H, C):
        self.H = H
        self.buf = torch.full((H, C), float("nan"))

    def stats_view(self):
        return self.buf


def _stats_worker(rank, world, port, H, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1803_00005_b200 import gather_stats_rows, shard_range
    h = _FakeHandle(H, 6)
    y0, y1 = shard_range(H, world, rank)
    rows = torch.arange(H, dtype=torch.float32)[:, None] * 10 + torch.arange(6, dtype=torch.float32)[None, :]
    h.buf[y0:y1] = rows[y0:y1]                       # this rank's band only (prepare_rows on the GPU)
    gather_stats_rows(h)
    torch.save(h.buf, out_path + f".{rank}")
    dist.destroy_process_group()


@pytest.mark.parametrize("H", [8, 7])                 # equal bands (all-gather) and unequal (broadcasts)
def test_gloo_world2_row_sharded_statistics(tmp_path, H):
    world = 2
    out = str(tmp_path / "stats")
    mp.spawn(_stats_worker, args=(world, _free_port(), H, out), nprocs=world, join=True)
    rows = torch.arange(H, dtype=torch.float32)[:, None] * 10 + torch.arange(6, dtype=torch.float32)[None, :]
    for r in range(world):
        assert torch.equal(torch.load(out + f".{r}"), rows)
