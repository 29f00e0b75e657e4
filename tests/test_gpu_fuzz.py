"""Randomised GPU parity sweep: seeded random shapes (ragged widths and heights, 1..70 labels, degrees 1..3,
n up to 9, radii 1..12, both modes, stereo-like and iid costs) through the default entry points -- the
aggregation (whichever slice kernels the shape selects: k_coef5/k_coef3/k_coef2 -> k_agg6 with or without its
label split / k_agg3 / the generic kernels) and the single-slice hgf_filter (its fused pass) -- each against the
float64 oracle under the north_star rules (tests/parity_util.py)."""
import numpy as np
import pytest

import oracle as O
import synth
from tests.parity_util import check_labels, check_z

pytestmark = pytest.mark.gpu


def _cases(n, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        m = int(rng.integers(1, 4))
        d = int(rng.integers(1, 4))
        if m * d > 9:
            d = 9 // m
        W = int(rng.integers(8, 180))
        H = int(rng.integers(8, 120))
        L = int(rng.integers(1, 71))
        r = int(rng.integers(1, 13))
        mode = "gf" if rng.random() < 0.3 else "hgf"
        dist = "iid" if rng.random() < 0.3 else "stereo"
        lam = float(rng.choice([1e-3, 0.01, 0.05, 0.2]))
        out.append((i, W, H, m, d, L, r, lam, mode, dist))
    return out


CASES = _cases(24)


def _inputs(W, H, m, L, dist, seed):
    if dist == "iid":
        return synth.iid_volume(W, H, L, m, seed=seed)
    scene = synth.make_stereo_scene(W, H, max(L, 2), seed=seed)
    I = scene.left if m == 3 else np.ascontiguousarray(synth.smooth_guides(W, H, m, seed=seed))
    return I, np.ascontiguousarray(synth.stereo_cost_volume_np(scene, max(L, 2))[:L])


@pytest.mark.parametrize("i,W,H,m,d,L,r,lam,mode,dist", CASES, ids=[f"fuzz{c[0]}" for c in CASES])
def test_fuzz_aggregate_and_filter(i, W, H, m, d, L, r, lam, mode, dist):
    import torch

    from paper_1803_00005_b200 import HGF
    I, V = _inputs(W, H, m, L, dist, seed=100 + i)
    I, V = np.ascontiguousarray(I, dtype=np.float32), np.ascontiguousarray(V, dtype=np.float32)
    h = HGF(W, H, m, d, r, lam, mode=mode)
    gi, gv = torch.from_numpy(I).cuda(), torch.from_numpy(V).cuda()
    out = h.aggregate_wta_ex(gi, gv, labels=True, min_cost=True, filtered=True, keys=True)
    single = h.filter(gi, gv[0].contiguous())
    torch.cuda.synchronize()
    h.close()
    Z = O.hgf_filter(I, V, lam, r, d, mode=mode)
    s_v = float(np.abs(V).max()) or 1.0
    check_z(out["filtered"].cpu().numpy(), Z, s_v)
    check_labels(out["labels"].cpu().numpy(), Z, s_v)
    lab = out["labels"].cpu().numpy()
    # the WTA outputs are consistent with each other and with the filtered slices of the same run
    assert np.array_equal(out["min_cost"].cpu().numpy(),
                          np.take_along_axis(out["filtered"].cpu().numpy(), lab[None].astype(np.int64), 0)[0])
    ku = O.pack_keys(out["min_cost"].cpu().numpy(), lab) ^ np.uint64(1 << 63)
    assert np.array_equal(out["keys"].cpu().numpy().view(np.uint64), ku)
    check_z(single.cpu().numpy(), Z[0], s_v)
