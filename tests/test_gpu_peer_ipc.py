"""The fused label-sharded WTA merge (hgf_aggregate_wta_peer + PeerKeys/PeerMerge)
end to end across PROCESSES: two ranks (processes) share cuda:0, exchange their owner key buffers with CUDA IPC
(hgf_ipc_get_handle / hgf_ipc_open over a gloo process group), and every step's label shards are merged by
system-scope 64-bit atomic MINs into the owner's rows; five steps with changing volumes through the double-buffered
owner buffers, each rank's rows against the ORACLE's argmin over the whole volume.

The kernels of the two processes never wait on one another (the ordering is the 4-byte all-reduce between
the steps), so sharing one GPU is safe (the profiling guide's rule about spinning kernels does not apply)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W, H, L, STEPS = 96, 61, 20, 5


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import synth
    from paper_1803_00005_b200 import HGF, PeerMerge, shard_range

    scene = synth.make_stereo_scene(W, H, L, seed=17)
    gi = torch.from_numpy(scene.left).cuda()
    base = torch.from_numpy(synth.stereo_cost_volume_np(scene, L)).cuda()
    h = HGF(W, H, 3, 2, 9, 0.05)
    pm = PeerMerge(h)                              # IPC handle exchange over the gloo group
    l0, l1 = shard_range(L, world, rank)
    lab = torch.empty((pm.rows, W), dtype=torch.int32, device="cuda")
    h.prepare_rows(gi, 0, H)                       # replicated statistics (every rank, all rows)
    got = []
    for s in range(STEPS):
        perm = torch.roll(torch.arange(L, device="cuda"), 3 * s)
        vol = (base[perm] + 0.01 * s).contiguous()
        pm.aggregate(vol[l0:l1].contiguous(), lab, label_offset=l0)
        torch.cuda.synchronize()
        got.append(lab[: pm.y1 - pm.y0].cpu().numpy().copy())
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), y0=pm.y0, y1=pm.y1, **{f"s{s}": g for s, g in enumerate(got)})
    pm.close()
    h.close()
    dist.barrier()
    dist.destroy_process_group()


def test_peer_merge_two_processes_ipc(tmp_path):
    import torch.multiprocessing as mp

    import oracle as O
    import synth
    from tests.parity_util import check_labels

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    scene = synth.make_stereo_scene(W, H, L, seed=17)
    base = synth.stereo_cost_volume_np(scene, L)
    rows = {}
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        rows[r] = d
    assert int(rows[0]["y0"]) == 0 and int(rows[world - 1]["y1"]) == H
    for s in range(STEPS):
        perm = np.roll(np.arange(L), 3 * s)
        V = (base[perm] + np.float32(0.01 * s)).astype(np.float32)
        Z = O.hgf_filter(scene.left, V, 0.05, 9, 2)
        lab = np.concatenate([rows[r][f"s{s}"] for r in range(world)], axis=0)
        assert lab.shape == (H, W)
        check_labels(lab, Z, float(np.abs(V).max()))
