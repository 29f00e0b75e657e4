"""Generator "stereo-like v1": seeded synthetic stereo pairs and matching-cost volumes.

Structure follows the paper's workloads: Middlebury-style scenes with piecewise-planar
disparity and textured regions (Fig 5), costs per Hosni's framework that the
paper defers to, written out in SPEC S:400 (truncated colour + gradient terms).
No part of the HGF method is computed here.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# (W, H, L, m, d, r, lambda, seed) — BASELINE.json configs; lambda for C2-C5 is the paper's 0.05.
CONFIGS = {
    "C1": dict(W=64, H=48, L=8, m=3, d=1, r=2, lam=1e-3, seed=1),
    "C2": dict(W=450, H=375, L=60, m=3, d=2, r=9, lam=0.05, seed=2),
    "C2n9": dict(W=450, H=375, L=60, m=3, d=3, r=9, lam=0.05, seed=2),
    "C3": dict(W=1920, H=1080, L=128, m=3, d=2, r=9, lam=0.05, seed=3),
    "C3n9": dict(W=1920, H=1080, L=128, m=3, d=3, r=9, lam=0.05, seed=3),
    "C4": dict(W=3840, H=2160, L=256, m=3, d=2, r=9, lam=0.05, seed=4),
    "C4n9": dict(W=3840, H=2160, L=256, m=3, d=3, r=9, lam=0.05, seed=4),
    "C5": dict(W=1920, H=1080, L=1, m=3, d=2, r=9, lam=0.05, seed=5),
}

ALPHA_COLOUR = np.float32(0.11)
ALPHA_GRAD = np.float32(0.89)
TAU_COLOUR = np.float32(0.028)
TAU_GRAD = np.float32(0.008)


def config(name: str) -> dict:
    c = dict(CONFIGS[name])
    c["n"] = c["m"] * c["d"]
    c["name"] = name
    return c


@dataclass
class StereoScene:
    left: np.ndarray    # (3, H, W) float32 in [0, 1]  (the guide)
    right: np.ndarray   # (3, H, W) float32 in [0, 1]
    disp: np.ndarray    # (H, W) int32 ground-truth disparity in [0, L)


def _smooth_field(rng, H, W, n_waves=3, amp=0.15, base=0.4):
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    f = np.full((H, W), base)
    for _ in range(n_waves):
        fy, fx = rng.uniform(0.5, 3.0, size=2) * 2 * np.pi / np.array([H, W])
        ph = rng.uniform(0, 2 * np.pi)
        f += (amp / n_waves) * np.sin(fy * yy + fx * xx + ph)
    return f


def make_stereo_scene(W: int, H: int, L: int, seed: int) -> StereoScene:
    rng = np.random.Generator(np.random.PCG64(seed))
    left = np.stack([_smooth_field(rng, H, W) for _ in range(3)])
    left += rng.normal(0, 0.04, size=left.shape) * 0.5
    # background: slanted plane over [0.1 L, 0.4 L]
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    a, b = rng.uniform(-1, 1, size=2)
    plane = a * xx / max(W - 1, 1) + b * yy / max(H - 1, 1)
    plane = (plane - plane.min()) / max(np.ptp(plane), 1e-9)
    disp = 0.1 * L + plane * 0.3 * L
    # regions: ~8 per 0.1 MP, painted in increasing disparity order
    K = max(3, int(round(8 * W * H / 1e5)))
    regions = []
    for _ in range(K):
        cy, cx = rng.uniform(0, H), rng.uniform(0, W)
        ry, rx = rng.uniform(0.03, 0.15) * H, rng.uniform(0.03, 0.15) * W
        d0 = rng.uniform(0.3 * L, 0.9 * L)
        slope = rng.uniform(-0.05, 0.05, size=2) * L / max(W, H) * rng.integers(0, 2)
        colour = rng.uniform(0.05, 0.95, size=3)
        ellipse = bool(rng.integers(0, 2))
        regions.append((d0, cy, cx, ry, rx, slope, colour, ellipse))
    regions.sort(key=lambda t: t[0])
    for d0, cy, cx, ry, rx, slope, colour, ellipse in regions:
        y0, y1 = int(max(0, cy - ry)), int(min(H, cy + ry + 1))
        x0, x1 = int(max(0, cx - rx)), int(min(W, cx + rx + 1))
        if y1 <= y0 or x1 <= x0:
            continue
        sy, sx = yy[y0:y1, x0:x1], xx[y0:y1, x0:x1]
        if ellipse:
            mask = ((sy - cy) / ry) ** 2 + ((sx - cx) / rx) ** 2 <= 1.0
        else:
            mask = np.ones(sy.shape, dtype=bool)
        dv = d0 + slope[0] * (sy - cy) + slope[1] * (sx - cx)
        disp[y0:y1, x0:x1] = np.where(mask, dv, disp[y0:y1, x0:x1])
        tex = rng.normal(0, 0.04, size=(3,) + sy.shape)
        for c in range(3):
            left[c, y0:y1, x0:x1] = np.where(mask, colour[c] + tex[c], left[c, y0:y1, x0:x1])
    left += rng.normal(0, 0.01, size=left.shape)
    left = np.clip(left, 0.0, 1.0)
    disp = np.clip(np.rint(disp), 0, L - 1).astype(np.int32)
    # right view: forward warp right(x - d) <- left(x), z-buffer (larger d wins; ties: larger x)
    tx = xx.astype(np.int64) - disp
    valid = tx >= 0
    flat_t = (yy.astype(np.int64) * W + tx)[valid]
    keyv = (disp.astype(np.int64) * W + xx.astype(np.int64))[valid]
    zbuf = np.full(H * W, -1, dtype=np.int64)
    np.maximum.at(zbuf, flat_t, keyv)
    right = np.stack([_smooth_field(rng, H, W) for _ in range(3)])    # hole fill: background texture
    right += rng.normal(0, 0.02, size=right.shape)
    filled = zbuf >= 0
    src_x = (zbuf[filled] % W)
    src_y = np.nonzero(filled)[0] // W
    rflat = right.reshape(3, -1)
    rflat[:, np.nonzero(filled)[0]] = left[:, src_y, src_x]
    right = rflat.reshape(3, H, W) + rng.normal(0, 0.01, size=right.shape)
    right = np.clip(right, 0.0, 1.0)
    return StereoScene(left.astype(np.float32), right.astype(np.float32), disp)


def _grad_x(gray: np.ndarray) -> np.ndarray:
    """Central x-difference of the channel mean, clamped at the borders (float32 arithmetic)."""
    g = np.empty_like(gray)
    g[:, 1:-1] = (gray[:, 2:] - gray[:, :-2]) * np.float32(0.5)
    g[:, 0] = gray[:, 1] - gray[:, 0]
    g[:, -1] = gray[:, -1] - gray[:, -2]
    return g


def _gray(img: np.ndarray) -> np.ndarray:
    return ((img[0] + img[1]) + img[2]) / np.float32(3.0)


def stereo_cost_volume_np(scene: StereoScene, L: int, l0: int = 0, l1: int | None = None) -> np.ndarray:
    """C(x, y, d) = 0.11 min(mean_c |L_c(x,y) - R_c(x-d,y)|, 0.028) + 0.89 min(|dxL - dxR(x-d)|, 0.008).

    Slices d in [l0, l1).  Out-of-range (x - d < 0) takes the truncation values.  float32.
    """
    l1 = L if l1 is None else l1
    Lf, Rf = scene.left, scene.right
    H, W = Lf.shape[1:]
    gl, gr = _grad_x(_gray(Lf)), _grad_x(_gray(Rf))
    out = np.empty((l1 - l0, H, W), dtype=np.float32)
    trunc = ALPHA_COLOUR * TAU_COLOUR + ALPHA_GRAD * TAU_GRAD
    for k, dd in enumerate(range(l0, l1)):
        c = np.full((H, W), trunc, dtype=np.float32)
        if dd < W:
            a = np.abs(Lf[:, :, dd:] - Rf[:, :, :W - dd])
            col = ((a[0] + a[1]) + a[2]) / np.float32(3.0)
            grd = np.abs(gl[:, dd:] - gr[:, :W - dd])
            c[:, dd:] = ALPHA_COLOUR * np.minimum(col, TAU_COLOUR) + ALPHA_GRAD * np.minimum(grd, TAU_GRAD)
        out[k] = c
    return out


def stereo_cost_volume_torch(scene: StereoScene, L: int, device, l0: int = 0, l1: int | None = None, out=None):
    """Same cost as stereo_cost_volume_np, built with torch float32 element-wise ops on `device`.

    Used by bench.py / GPU tests to materialise multi-GB volumes directly in HBM (input generation,
    not the timed hot path).  Returns a contiguous (l1 - l0, H, W) float32 tensor.
    """
    import torch
    l1 = L if l1 is None else l1
    Lt = torch.from_numpy(scene.left).to(device)
    Rt = torch.from_numpy(scene.right).to(device)
    H, W = Lt.shape[1:]
    gl = torch.from_numpy(_grad_x(_gray(scene.left))).to(device)
    gr = torch.from_numpy(_grad_x(_gray(scene.right))).to(device)
    trunc = float(ALPHA_COLOUR * TAU_COLOUR + ALPHA_GRAD * TAU_GRAD)
    if out is None:
        out = torch.empty((l1 - l0, H, W), dtype=torch.float32, device=device)
    ac, ag = float(ALPHA_COLOUR), float(ALPHA_GRAD)
    tc, tg = float(TAU_COLOUR), float(TAU_GRAD)
    for k, dd in enumerate(range(l0, l1)):
        sl = out[k]
        sl.fill_(trunc)
        if dd < W:
            a = (Lt[:, :, dd:] - Rt[:, :, :W - dd]).abs_()
            col = ((a[0] + a[1]) + a[2]) / 3.0
            grd = (gl[:, dd:] - gr[:, :W - dd]).abs_()
            sl[:, dd:] = torch.clamp_max(col, tc) * ac + torch.clamp_max(grd, tg) * ag
    return out


def iid_volume(W: int, H: int, L: int, m: int, seed: int):
    """Stress distribution 'iid': guide ~ U[0,1)^m, V ~ U[0,1)^L (no structure, many near-ties)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    guide = rng.random((m, H, W), dtype=np.float32)
    vol = rng.random((L, H, W), dtype=np.float32)
    return guide, vol


def smooth_guides(W: int, H: int, m: int, seed: int) -> np.ndarray:
    """C5 guides: m independent smooth-plus-edges fields in [0, 1] (float32)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.empty((m, H, W), dtype=np.float32)
    yy, xx = np.mgrid[0:H, 0:W]
    for c in range(m):
        f = _smooth_field(rng, H, W, amp=0.3, base=0.5)
        for _ in range(4):
            a, b, t = rng.normal(size=3)
            f = f + 0.2 * np.sign(a * (xx - W / 2) + b * (yy - H / 2) + t * min(W, H) / 4)
        f += rng.normal(0, 0.01, size=f.shape)
        out[c] = np.clip((f - f.min()) / max(np.ptp(f), 1e-9), 0, 1)
    return out


def make_lr_maps(W: int, H: int, L: int, seed: int, noise: float = 0.05):
    """Inputs for the post-processing step alone (NEXT-3): the scene's left view, a left disparity map (the
    ground truth with a fraction `noise` of pixels replaced by random labels) and a right disparity map
    (the ground truth forward-warped to the right view, larger disparity wins, unmatched pixels 0, with the
    same kind of noise).  Returns (left (3, H, W) float32, dL int32 (H, W), dR int32 (H, W))."""
    scene = make_stereo_scene(W, H, L, seed)
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    gt = scene.disp.astype(np.int64)
    dR = np.zeros((H, W), dtype=np.int64)
    for y in range(H):
        for x in range(W):
            t = x - gt[y, x]
            if t >= 0 and gt[y, x] > dR[y, t]:
                dR[y, t] = gt[y, x]
    dL = gt.copy()
    for m in (dL, dR):
        flip = rng.random((H, W)) < noise
        m[flip] = rng.integers(0, L, size=int(flip.sum()))
    return scene.left, dL.astype(np.int32), dR.astype(np.int32)
