"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times, on sampled outputs.

Z(q) depends only on inputs within 2r of q (w_p uses Omega_p, Z(q) averages p in Omega_q), so the float64
oracle run on the crop [q - 2r, q + 2r] ∩ image gives Z(q) exactly (the crop edge is either the image edge
or more than r away from every window the output touches).  Sampled pixels: the four corners, edge
midpoints, the centre and seeded random interior points.  All labels are checked at every sample, and the
WTA label against the oracle's argmin over all labels.
"""
import numpy as np
import pytest

import oracle as O
import synth
from tests.parity_util import check_labels, check_z

pytestmark = pytest.mark.gpu


def _samples(W, H, n_rand, seed):
    pts = [(0, 0), (W - 1, 0), (0, H - 1), (W - 1, H - 1), (W // 2, 0), (0, H // 2), (W - 1, H // 2),
           (W // 2, H - 1), (W // 2, H // 2)]
    rng = np.random.default_rng(seed)
    pts += [(int(rng.integers(0, W)), int(rng.integers(0, H))) for _ in range(n_rand)]
    return pts


def _crop(x, y, W, H, R):
    return max(0, y - R), min(H, y + R + 1), max(0, x - R), min(W, x + R + 1)


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_fullsize_sampled_parity(cfg):
    import torch

    from paper_1803_00005_b200 import HGF
    c = synth.config(cfg)
    W, H, L, r, d, lam = c["W"], c["H"], c["L"], c["r"], c["d"], c["lam"]
    scene = synth.make_stereo_scene(W, H, L, c["seed"])
    guide = torch.from_numpy(scene.left).cuda()
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    h = HGF(W, H, c["m"], d, r, lam)
    out = h.aggregate_wta_ex(guide, vol, labels=True, filtered=True)
    torch.cuda.synchronize()
    s_v = float(vol.abs().max())
    for (x, y) in _samples(W, H, 8, seed=c["seed"]):
        y0, y1, x0, x1 = _crop(x, y, W, H, 2 * r)
        I = scene.left[:, y0:y1, x0:x1].astype(np.float64)
        V = vol[:, y0:y1, x0:x1].double().cpu().numpy()
        Z = O.hgf_filter(I, V, lam, r, d)
        zq = Z[:, y - y0, x - x0]
        zg = out["filtered"][:, y, x].cpu().numpy()
        check_z(zg, zq, s_v)
        check_labels(out["labels"][y, x].cpu().numpy().reshape(1, 1), zq.reshape(L, 1, 1), s_v)
    h.close()


@pytest.mark.parametrize("m,d,r", [(3, 3, 4), (10, 2, 16)])
def test_c5_single_slice_sampled(m, d, r):
    """BASELINE config 5: 1920x1080 single-slice hgf_filter; n = 9 (fast path) and n = 20, r = 16 (generic path)."""
    import torch

    from paper_1803_00005_b200 import HGF
    c = synth.config("C5")
    W, H, lam = c["W"], c["H"], c["lam"]
    I = synth.smooth_guides(W, H, m, seed=5)
    scene = synth.make_stereo_scene(W, H, 64, seed=5)
    Y = synth.stereo_cost_volume_np(scene, 64, 20, 21)[0]
    h = HGF(W, H, m, d, r, lam)
    dst = h.filter(torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda())
    torch.cuda.synchronize()
    zg = dst.cpu().numpy()
    s_v = float(np.abs(Y).max())
    for (x, y) in _samples(W, H, 4, seed=5):
        y0, y1, x0, x1 = _crop(x, y, W, H, 2 * r)
        Z = O.hgf_filter(I[:, y0:y1, x0:x1], Y[y0:y1, x0:x1], lam, r, d)
        check_z(np.array([zg[y, x]]), np.array([Z[y - y0, x - x0]]), s_v)
    h.close()
