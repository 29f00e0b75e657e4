"""GPU parity for the post-processing row (readings P1-P4 of DESIGN.md §11d):
the right-view aggregation, the left-right check + row fill (bit-exact) and the weighted median (equal to
the oracle, or a weighted median of the oracle's float64 weights within 1e-4 of the half-weight
threshold where float32 weights order the decision differently), all through the C ABI."""
import numpy as np
import pytest

import oracle as O
import synth
from tests.parity_util import check_labels, check_z

pytestmark = pytest.mark.gpu

WMF_TOL = 1e-4      # relative slack on the half-weight threshold (float32 weights: expf + sums, ~1e-6)
WMF_AGREE = 0.999   # share of inconsistent pixels whose median must equal the oracle's exactly


def _torch():
    import torch
    return torch


def _hgf(W, H, m, d, r, lam, mode="hgf"):
    from paper_1803_00005_b200 import HGF
    return HGF(W, H, m, d, r, lam, mode=mode)


@pytest.mark.parametrize("W,H,L,label_offset,d,r,mode", [(96, 64, 16, 0, 2, 4, "hgf"), (77, 45, 12, 3, 1, 3, "gf"),
                                                          (600, 36, 50, 7, 2, 5, "hgf")])
def test_stereo_wta_right_parity(W, H, L, label_offset, d, r, mode):
    """P1: the right view's slices built on the GPU (match at x + d), filtered with the right view as guide,
    against the oracle's right-view cost filtered by the oracle."""
    torch = _torch()
    scene = synth.make_stereo_scene(W, H, L + label_offset, seed=80 + W)
    h = _hgf(W, H, 3, d, r, 0.05, mode)
    out = h.stereo_wta_right(torch.from_numpy(scene.left).cuda(), torch.from_numpy(scene.right).cuda(), L,
                             label_offset=label_offset, labels=True, filtered=True)
    torch.cuda.synchronize()
    C = O.stereo_cost_right(scene.left, scene.right, L, l0=label_offset)
    Z = O.hgf_filter(scene.right, C, 0.05, r, d, mode=mode)
    s_v = float(np.abs(C).max())
    check_z(out["filtered"].cpu().numpy(), Z, s_v)
    check_labels_near_ties(out["labels"].cpu().numpy() - label_offset, Z, s_v)
    h.close()


def check_labels_near_ties(lab_gpu, Z, s_v):
    """Labels bit-exact wherever the oracle's top-two gap exceeds 1e-4 (parity_util's rule); at the
    near-ties the GPU's label must be one of the near-optimal ones (within 1e-4 of the minimum).  The right
    view's last columns are truncated for every disparity with x + d >= W, so its slices tie there far more
    often than 1 pixel in 10^4 at these small sizes."""
    from tests.parity_util import GAP
    lab_ora = np.argmin(Z, axis=0)
    srt = np.sort(Z, axis=0)
    den = np.maximum(np.abs(srt[0]), 1e-3 * s_v)
    clear = (srt[1] - srt[0]) / den > GAP
    assert not np.any((lab_gpu != lab_ora) & clear)
    zg = np.take_along_axis(Z, lab_gpu[None].astype(np.int64), axis=0)[0]
    assert np.all((zg - srt[0]) / den <= GAP)


def check_wmf(gpu, ora_final, filled, valid, img, radius, ss, sc):
    """Inconsistent pixels: equal to the oracle, or a valid weighted median of the oracle's weights."""
    inv = ~valid
    n_inv = int(inv.sum())
    if n_inv == 0:
        return
    diff = inv & (gpu != ora_final)
    assert 1.0 - diff.sum() / n_inv >= WMF_AGREE, f"{int(diff.sum())} of {n_inv} medians differ"
    for y, x in zip(*np.nonzero(diff)):
        vals, w = O.window_weights(filled, img, y, x, radius, ss, sc)
        dg = int(gpu[y, x])
        assert dg in vals, f"({y},{x}): {dg} is not a window value"
        half = 0.5 * w.sum()
        below = vals[vals < dg]
        assert w[vals <= dg].sum() >= half * (1 - WMF_TOL), f"({y},{x}): below the half weight"
        if below.size:
            assert w[vals <= below.max()].sum() < half * (1 + WMF_TOL), f"({y},{x}): not the smallest median"


@pytest.mark.parametrize("W,H,L,m,tol,radius,ss,sc", [
    (96, 64, 16, 3, 0, 9, 9.0, 0.1),      # the defaults
    (133, 70, 24, 3, 1, 4, 3.0, 0.2),     # ragged width, tolerance 1
    (40, 31, 8, 1, 0, 15, 20.0, 0.05),    # gray image, the largest radius
    (33, 5, 6, 3, 0, 0, 1.0, 1.0),        # radius 0: the fill alone
    (1, 1, 4, 3, 0, 2, 1.0, 1.0),         # one pixel
])
def test_lr_postprocess_parity(W, H, L, m, tol, radius, ss, sc):
    """P2-P4 alone on seeded disparity maps (synth.make_lr_maps): consistency flags and every consistent
    pixel bit-exact, medians as check_wmf."""
    torch = _torch()
    left, dL, dR = synth.make_lr_maps(W, H, L, seed=90 + W)
    img = np.ascontiguousarray(left[:m])
    h = _hgf(W, H, m, 1, 1, 0.05)
    out = h.lr_postprocess(torch.from_numpy(img).cuda(), torch.from_numpy(dL).cuda(), torch.from_numpy(dR).cuda(),
                           tol=tol, radius=radius, sigma_s=ss, sigma_c=sc, valid=True)
    torch.cuda.synchronize()
    gv = out["valid"].cpu().numpy().astype(bool)
    gd = out["disp"].cpu().numpy()
    valid = O.lr_consistency(dL, dR, tol)
    filled = O.occlusion_fill(dL, valid)
    final = O.weighted_median_fill(filled, valid, img, radius, ss, sc)
    assert np.array_equal(gv, valid)
    assert np.array_equal(gd[valid], dL[valid])
    if radius == 0:
        assert np.array_equal(gd, filled)                 # one-pixel window: the median is the fill value
    check_wmf(gd, final, filled, valid, img, radius, ss, sc)
    h.close()


def test_lr_postprocess_rows_without_anchor_and_full_consistency():
    """P3 edge cases on the GPU: a row with no consistent pixel keeps its values; identical constant maps are
    consistent exactly where x >= d; the output equals the input there."""
    torch = _torch()
    W, H = 50, 6
    img = np.random.default_rng(5).random((3, H, W)).astype(np.float32)
    dL = np.full((H, W), 4, np.int32)
    dR = np.full((H, W), 4, np.int32)
    dR[2] = 7                                           # row 2: nothing consistent
    h = _hgf(W, H, 3, 1, 1, 0.05)
    out = h.lr_postprocess(torch.from_numpy(img).cuda(), torch.from_numpy(dL).cuda(), torch.from_numpy(dR).cuda(),
                           radius=0, valid=True)
    torch.cuda.synchronize()
    v = out["valid"].cpu().numpy().astype(bool)
    assert not v[2].any() and not v[:, :4].any() and v[[0, 1, 3, 4, 5], 4:].all()
    assert np.array_equal(out["disp"].cpu().numpy(), dL)
    h.close()


def test_stereo_disparity_pipeline():
    """hgf_stereo_disparity end to end against the oracle's pipeline (oracle left / right maps from the
    oracle's costs, then P2-P4): raw maps as label parity; the final map equal wherever the raw maps of
    the pixel's window rows agree on both sides (the fill runs along rows, the median over 2 rho + 1 rows)."""
    torch = _torch()
    W, H, L, d, r, rho = 80, 56, 12, 1, 4, 4
    scene = synth.make_stereo_scene(W, H, L, seed=95)
    h = _hgf(W, H, 3, d, r, 0.05)
    out = h.stereo_disparity(torch.from_numpy(scene.left).cuda(), torch.from_numpy(scene.right).cuda(), L,
                             radius=rho, sigma_s=4.0, raw=True, valid=True)
    torch.cuda.synchronize()
    CL = O.stereo_cost(scene.left, scene.right, L)
    CR = O.stereo_cost_right(scene.left, scene.right, L)
    ZL = O.hgf_filter(scene.left, CL, 0.05, r, d)
    ZR = O.hgf_filter(scene.right, CR, 0.05, r, d)
    gL, gR = out["disp_left"].cpu().numpy(), out["disp_right"].cpu().numpy()
    check_labels(gL, ZL, float(np.abs(CL).max()))
    check_labels(gR, ZR, float(np.abs(CR).max()))
    oL, oR = O.wta(ZL), O.wta(ZR)
    final, valid = O.lr_postprocess(scene.left, oL, oR, radius=rho, sigma_s=4.0)
    row_ok = np.all(gL == oL, axis=1) & np.all(gR == oR, axis=1)
    win_ok = np.array([row_ok[max(0, y - rho):y + rho + 1].all() for y in range(H)])
    assert win_ok.mean() >= 0.5, "too few comparable rows"
    gd = out["disp"].cpu().numpy()
    assert np.array_equal(out["valid"].cpu().numpy().astype(bool)[row_ok], valid[row_ok])
    filled = O.occlusion_fill(oL, valid)
    sel = win_ok[:, None] & np.ones((1, W), bool)
    mism = sel & (gd != final)
    for y, x in zip(*np.nonzero(mism)):               # only near-threshold medians may differ
        vals, w = O.window_weights(filled, scene.left, y, x, rho, 4.0, 0.1)
        half = 0.5 * w.sum()
        dg = int(gd[y, x])
        assert dg in vals and w[vals <= dg].sum() >= half * (1 - WMF_TOL)
        below = vals[vals < dg]
        assert below.size == 0 or w[vals <= below.max()].sum() < half * (1 + WMF_TOL)
    h.close()


def test_postprocess_invalid_arguments():
    torch = _torch()
    from paper_1803_00005_b200 import HGFError
    W, H = 32, 8
    h = _hgf(W, H, 3, 1, 1, 0.05)
    img = torch.zeros(3, H, W, device="cuda")
    dm = torch.zeros(H, W, dtype=torch.int32, device="cuda")
    for kw in ({"tol": -1}, {"radius": 16}, {"radius": -1}, {"sigma_s": 0.0}, {"sigma_c": float("nan")}):
        with pytest.raises(HGFError):
            h.lr_postprocess(img, dm, dm, **kw)
    with pytest.raises(HGFError):
        h.stereo_disparity(img, img, 4, radius=99)
    h.close()
