"""Out-of-bounds write checks without compute-sanitizer (closed on this pool: profiles/r02_compute_sanitizer_closed.txt).

Every output of the public entry points is handed to the library as a view into a larger device buffer whose
slack before and after is filled with a sentinel bit pattern; after the call the slack must be bit-for-bit
untouched, and the outputs must equal those of a call into exactly-sized buffers.  Ragged geometries exercise
every kernel edge: W % 4 != 0 (the repacked k_coef5 chunk), odd W, partial 16-pixel groups and 128-pixel strips,
label counts that are not multiples of 32 (partial label batches), one row, one pixel, the opt-in k_agg5 and the
degree-3 planar path; the fused-merge entry point writes into guarded owner buffers."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

GUARD = 4096                       # elements of slack on each side
SENT = {torch.float32: 0x7FA5A5A5, torch.int32: 0x5A5A5A5A, torch.int64: 0x5A5A5A5A5A5A5A5A}


def guarded(shape, dtype):
    n = int(np.prod(shape))
    buf = torch.empty(n + 2 * GUARD, dtype=dtype, device="cuda")
    if dtype == torch.float32:
        buf.view(torch.int32).fill_(SENT[dtype] - (1 << 32) if SENT[dtype] >= (1 << 31) else SENT[dtype])
    else:
        buf.fill_(SENT[dtype])
    return buf, buf[GUARD:GUARD + n].view(shape)


def untouched(buf, n):
    v = buf.view(torch.int32) if buf.dtype == torch.float32 else buf
    sent = SENT[buf.dtype]
    if buf.dtype == torch.float32 and sent >= (1 << 31):
        sent -= 1 << 32
    head, tail = v[:GUARD], v[GUARD + n:]
    return bool((head == sent).all()) and bool((tail == sent).all())


CASES = [
    # (W, H, m, d, L, r, env)
    (77, 53, 3, 2, 5, 9, {}),                 # W % 4 != 0: repacked chunk, partial group
    (301, 140, 3, 2, 40, 9, {}),              # odd W, 3 strips, 2 label batches (one partial)
    (300, 140, 3, 2, 33, 7, {"HGF_AGG5": "1"}),
    (45, 70, 3, 3, 4, 9, {}),                 # degree 3, W % 4 != 0: planar k_coef2 -> k_agg3
    (67, 1, 3, 2, 3, 3, {}),                  # one row
    (1, 1, 3, 2, 4, 2, {}),                   # one pixel
]


@pytest.mark.parametrize("W,H,m,d,L,r,env", CASES)
def test_outputs_stay_in_bounds(monkeypatch, W, H, m, d, L, r, env):
    from paper_1803_00005_b200 import HGF
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    scene = synth.make_stereo_scene(max(W, 8), max(H, 8), L, seed=W + H)
    g = torch.from_numpy(np.ascontiguousarray(scene.left[:, :H, :W])).cuda()
    vol = torch.from_numpy(np.ascontiguousarray(synth.stereo_cost_volume_np(scene, L)[:, :H, :W])).cuda()
    h = HGF(W, H, m, d, r, 0.05)
    ref = h.aggregate_wta_ex(g, vol, labels=True, min_cost=True, filtered=True, keys=True)
    torch.cuda.synchronize()
    bl, lab = guarded((H, W), torch.int32)
    bm, mc = guarded((H, W), torch.float32)
    bf, flt = guarded((L, H, W), torch.float32)
    bk, keys = guarded((H, W), torch.int64)
    h.aggregate_wta_ex(g, vol, out={"labels": lab, "min_cost": mc, "filtered": flt, "keys": keys})
    bd, dst = guarded((H, W), torch.float32)
    h.filter(g, vol[0].contiguous(), dst)
    torch.cuda.synchronize()
    for buf, n in ((bl, H * W), (bm, H * W), (bf, L * H * W), (bk, H * W), (bd, H * W)):
        assert untouched(buf, n), "write outside an output buffer"
    assert torch.equal(lab, ref["labels"]) and torch.equal(keys, ref["keys"])
    assert torch.equal(flt, ref["filtered"]) and torch.equal(mc, ref["min_cost"])
    if h.kernel_path.startswith(("coef5", "coef3")):
        # fused merge: two owners of ceil(H/2) rows, each guarded
        R = (H + 1) // 2
        own = [guarded((R, W), torch.int64) for _ in range(2)]
        for _, o in own:
            h.fill_keys(o)
        ptrs = torch.tensor([o.data_ptr() for _, o in own], dtype=torch.int64, device="cuda")
        h.prepare_rows(g, 0, H)
        h.aggregate_wta_peer(vol, ptrs, 2, R)
        torch.cuda.synchronize()
        for b, _ in own:
            assert untouched(b, R * W), "fused merge wrote outside an owner buffer"
        assert torch.equal(torch.cat([o for _, o in own])[:H], ref["keys"])
    h.close()
