"""Parity rules shared by the GPU tests and smoke().

Filtered costs:  e(p,l) = |Z_gpu - Z_ora| / max(|Z_ora|, 1e-3 s_V) <= 1e-4, s_V = max|V|
                 (BASELINE.json north_star: "max relative error 1e-4 (fp32 against fp64)"; a pure
                 relative error is ill-posed where Z -> 0, hence the 1e-3 s_V floor).
Labels:          bit-exact wherever the oracle's top-two gap (Z_(2)-Z_(1)) / max(|Z_(1)|, 1e-3 s_V)
                 exceeds 1e-4, and agreement >= 99.99 % overall.
"""
import os

import numpy as np

Z_TOL = 1e-4
GAP = 1e-4
AGREE = 0.9999


def z_error(z_gpu, z_ora, s_v):
    z_gpu = np.asarray(z_gpu, dtype=np.float64)
    z_ora = np.asarray(z_ora, dtype=np.float64)
    den = np.maximum(np.abs(z_ora), 1e-3 * s_v)
    return np.abs(z_gpu - z_ora) / den


def check_z(z_gpu, z_ora, s_v, tol=Z_TOL):
    e = z_error(z_gpu, z_ora, s_v)
    assert np.all(np.isfinite(np.asarray(z_gpu))), "non-finite GPU output"
    worst = float(e.max()) if e.size else 0.0
    if os.environ.get("HGF_PARITY_REPORT"):
        print(f"[parity] max normalised error {worst:.3e} (tol {tol:.0e})")
    assert worst <= tol, f"max relative error {worst:.3e} > {tol:.1e}"
    return worst


def check_labels(lab_gpu, Z_ora, s_v):
    """Z_ora: (L, H, W) oracle filtered costs."""
    lab_gpu = np.asarray(lab_gpu)
    lab_ora = np.argmin(Z_ora, axis=0)            # lowest index on ties
    if Z_ora.shape[0] >= 2:
        srt = np.sort(Z_ora, axis=0)
        gap = (srt[1] - srt[0]) / np.maximum(np.abs(srt[0]), 1e-3 * s_v)
        clear = gap > GAP
    else:
        clear = np.ones(lab_ora.shape, dtype=bool)
    mism_clear = int(np.count_nonzero((lab_gpu != lab_ora) & clear))
    agree = float(np.mean(lab_gpu == lab_ora))
    assert mism_clear == 0, f"{mism_clear} label mismatches where the oracle gap > {GAP}"
    assert agree >= AGREE, f"label agreement {agree:.6f} < {AGREE}"
    return agree, float(np.mean(~clear))
