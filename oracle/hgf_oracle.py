"""HGF oracle: a plain, slow, float64 CPU implementation of what the hot path computes.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The product path (``paper_1803_00005_b200``) never imports it, and this module
imports nothing from the product path: the two share no code, headers, tables or
constants.  Inputs come from ``synth`` (seeded generators with none of the
method's arithmetic).

Paper: Dai et al., "Hardware-Efficient Guided Image Filtering for Multi-Label
Problem", CVPR 2018 (arXiv 1803.00005).  ``P:n`` below is line n of
``PAPER.md`` (the LaTeX source); equation numbers follow SURVEY.md's list
(Eq1 P:36 ... Eq16).

Readings of the paper taken here (all listed in DESIGN.md §3):
  F1  alpha^0_00 = -lambda^-1 (lambda + G_00)^-1   (printed: -(lambda+G_00)^-1)
  F2  Eq11 first case carries gamma (gamma F + alpha), as Eq4 does (P:145 vs P:315)
  F3  Eq13 W_k = lambda^-1 G_{k,n+1} + sum_{i,j=0..n} alpha_ij G_ki G_{j,n+1}, k = 0..n
  F4  Eq5's I_{ki} read as G_{ki}
  F5  F^kappa_ij = u_i v_j, u_i = sum_{m<k} alpha_im G_mk, v_j = sum_{m<k} alpha_mj G_km
  F6  windows clipped at the image border, exact counts N_p (A(X) = B(X)/B(G_0))
  F7  B is a box SUM ("equal to the sum of its neighboring pixels"): lambda is against sums
  F9  HGF penalises the intercept w(0) (Eq7); GF (§5.1) does not (Eq15)
  F14 WTA ties resolve to the lowest label index
  P1-P4 post-processing (NEXT-3; P:641 names it only): right-view cost, left-right check, row fill,
      bilateral weighted median -- see the functions at the end and DESIGN.md §11d
  F18 Eq8 reads Z(q) = 1/|Omega_q| sum_{p in Omega_q} (sum_i w_p(i) G_i(q) + w_p(0))

Parity pins for every function live in tests/test_oracle_*.py (run with -m "not gpu").
No function here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "box_sum", "box_count", "box_mean", "box_sum_brute",
    "poly_guidance", "gram_planes", "alpha_recursion", "weights_eq13",
    "hgf_filter", "hgf_filter_brute", "gf_he",
    "wta", "aggregate_wta", "pack_keys", "unpack_keys",
    "stereo_cost", "stereo_cost_brute", "segmentation_cost",
    "stereo_cost_right", "lr_consistency", "occlusion_fill", "window_weights", "weighted_median_fill", "lr_postprocess",
]

MODE_HGF = "hgf"
MODE_GF = "gf"


# --------------------------------------------------------------------------
# Box filter (§4.3; Prop 2)
# --------------------------------------------------------------------------
def _sat(X: np.ndarray) -> np.ndarray:
    """Summed-area table (Crow 1984, cited P:342): S[..., y, x] = sum of X over rows < y, cols < x."""
    X = np.asarray(X, dtype=np.float64)
    H, W = X.shape[-2:]
    S = np.zeros(X.shape[:-2] + (H + 1, W + 1), dtype=np.float64)
    S[..., 1:, 1:] = X.cumsum(axis=-2).cumsum(axis=-1)
    return S


def box_sum(X: np.ndarray, r: int) -> np.ndarray:
    """B(X)(p) = sum_{q in Omega_p} X(q), Omega_p the (2r+1)^2 box clipped to the image (F6, F7).

    Works on any leading shape; the last two axes are (H, W).
    """
    X = np.asarray(X, dtype=np.float64)
    H, W = X.shape[-2:]
    S = _sat(X)
    y0 = np.clip(np.arange(H) - r, 0, H)
    y1 = np.clip(np.arange(H) + r + 1, 0, H)
    x0 = np.clip(np.arange(W) - r, 0, W)
    x1 = np.clip(np.arange(W) + r + 1, 0, W)
    return (S[..., y1[:, None], x1[None, :]] - S[..., y0[:, None], x1[None, :]]
            - S[..., y1[:, None], x0[None, :]] + S[..., y0[:, None], x0[None, :]])


def box_sum_brute(X: np.ndarray, r: int) -> np.ndarray:
    """Explicit double loop over every clipped window (used to pin box_sum; tiny inputs only)."""
    X = np.asarray(X, dtype=np.float64)
    H, W = X.shape[-2:]
    out = np.zeros_like(X)
    for y in range(H):
        for x in range(W):
            out[..., y, x] = X[..., max(0, y - r):min(H, y + r + 1), max(0, x - r):min(W, x + r + 1)].sum(axis=(-2, -1))
    return out


def box_count(H: int, W: int, r: int) -> np.ndarray:
    """N_p = |Omega_p| = B(G_0)(p) with G_0 the ones image."""
    ny = np.minimum(np.arange(H) + r, H - 1) - np.maximum(np.arange(H) - r, 0) + 1
    nx = np.minimum(np.arange(W) + r, W - 1) - np.maximum(np.arange(W) - r, 0) + 1
    return (ny[:, None] * nx[None, :]).astype(np.float64)


def box_mean(X: np.ndarray, r: int) -> np.ndarray:
    """Average operator A(X) = B(X) / B(G_0) (Eq14)."""
    X = np.asarray(X, dtype=np.float64)
    return box_sum(X, r) / box_count(X.shape[-2], X.shape[-1], r)


# --------------------------------------------------------------------------
# Polynomial guidance (§4.2; P:630 uses j <= 2)
# --------------------------------------------------------------------------
def poly_guidance(I: np.ndarray, d: int) -> np.ndarray:
    """G_{(i-1)d+j} = I_i^j, i = 1..m, j = 1..d, stacked channel-major.

    I: (m, H, W).  Returns (m*d, H, W) float64.  Powers by repeated multiplication.
    """
    I = np.asarray(I, dtype=np.float64)
    if I.ndim == 2:
        I = I[None]
    if d < 1:
        raise ValueError("degree d must be >= 1")
    m = I.shape[0]
    G = np.empty((m * d,) + I.shape[1:], dtype=np.float64)
    for i in range(m):
        t = np.ones(I.shape[1:], dtype=np.float64)
        for j in range(d):
            t = t * I[i]
            G[i * d + j] = t
    return G


# --------------------------------------------------------------------------
# Gram planes G_ij = B(G_i G_j) (Prop 2; Eq12)
# --------------------------------------------------------------------------
def gram_planes(G: np.ndarray, r: int, Y: np.ndarray | None = None):
    """Return (Gram, Gy) where, with G_0 = ones:

    Gram[i, j] = B(G_i G_j) for 0 <= i, j <= n   (shape (n+1, n+1, H, W))
    Gy[j]      = B(G_j Y) = G_{j,n+1}            (shape (n+1, H, W)), if Y is given (G_{n+1} = Y)
    """
    G = np.asarray(G, dtype=np.float64)
    n, H, W = G.shape
    ext = np.concatenate([np.ones((1, H, W)), G], axis=0)
    Gram = np.empty((n + 1, n + 1, H, W))
    for i in range(n + 1):
        for j in range(i, n + 1):
            Gram[i, j] = box_sum(ext[i] * ext[j], r)
            Gram[j, i] = Gram[i, j]
    Gy = None
    if Y is not None:
        Y = np.asarray(Y, dtype=np.float64)
        Gy = box_sum(ext * Y[None], r)
    return Gram, Gy


# --------------------------------------------------------------------------
# Proposition 1: the hardware-efficient inverse (Eq4, plane form Eq11)
# --------------------------------------------------------------------------
def alpha_recursion(Gram: np.ndarray, lam: float) -> np.ndarray:
    """alpha such that (lam E + sum_i c_i c_i^T)^-1 = lam^-1 E + sum_ij alpha_ij c_i c_j^T (Eq4).

    Gram: (K, K, ...) with Gram[i, j] = c_i^T c_j (any trailing per-pixel shape: the plane form).
    Runs kappa = 1..K-1 from alpha^0_00 (F1), each step reading only alpha^{kappa-1}.
    """
    Gram = np.asarray(Gram, dtype=np.float64)
    K = Gram.shape[0]
    inv_lam = 1.0 / lam
    alpha = np.zeros_like(Gram)
    # F1: alpha^0_00 = -lambda^-1 (lambda + G_00)^-1
    alpha[0, 0] = -inv_lam / (lam + Gram[0, 0])
    for k in range(1, K):
        prev = alpha[:k, :k].copy()                                          # alpha^{kappa-1}
        u = np.einsum("im...,m...->i...", prev, Gram[:k, k])                # u_i = sum_m alpha_im G_m,kappa
        v = np.einsum("mj...,m...->j...", prev, Gram[k, :k])                # v_j = sum_m alpha_mj G_kappa,m
        quad = np.einsum("mn...,m...,n...->...", prev, Gram[k, :k], Gram[:k, k])
        gamma = -1.0 / (1.0 + inv_lam * Gram[k, k] + quad)                  # gamma^kappa
        alpha[:k, :k] = gamma * u[:, None] * v[None, :] + prev              # i<k, j<k: gamma F + alpha (F2)
        alpha[:k, k] = inv_lam * gamma * u                                   # i<k, j=k
        alpha[k, :k] = inv_lam * gamma * v                                   # i=k, j<k
        alpha[k, k] = inv_lam * inv_lam * gamma                              # i=j=k
    return alpha


def weights_eq13(alpha: np.ndarray, Gram: np.ndarray, Gy: np.ndarray, lam: float) -> np.ndarray:
    """Eq13 / Eq5 (F3, F4): W_k = lam^-1 G_{k,n+1} + sum_{i,j} alpha_ij G_ki G_{j,n+1}, k = 0..n."""
    t = np.einsum("ij...,j...->i...", alpha, Gy)           # sum_j alpha_ij G_{j,n+1}
    return Gy / lam + np.einsum("ki...,i...->k...", Gram, t)


# --------------------------------------------------------------------------
# The filter (Eq6-8, Eq14; GF mode Eq15-16)
# --------------------------------------------------------------------------
def _aggregate(W: np.ndarray, G: np.ndarray, r: int) -> np.ndarray:
    """Eq14: Z = sum_{i=1..n} A(W_i) G_i + A(W_0)  (== Eq8)."""
    AW = box_mean(W, r)
    return AW[0] + np.einsum("i...,i...->...", AW[1:], G)


def _solve_batched(M: np.ndarray, b: np.ndarray) -> np.ndarray:
    """w_p = M_p^-1 b_p for every pixel.  M: (K, K, H, W); b: (K, H, W) or (K, L, H, W)."""
    K = M.shape[0]
    Mp = np.moveaxis(M, (0, 1), (-2, -1))                      # (H, W, K, K)
    if b.ndim == 3:
        bp = np.moveaxis(b, 0, -1)[..., None]                  # (H, W, K, 1)
        return np.moveaxis(np.linalg.solve(Mp, bp)[..., 0], -1, 0)
    bp = np.moveaxis(b, (0, 1), (-2, -1))                      # (H, W, K, L)
    return np.moveaxis(np.linalg.solve(Mp, bp), (-2, -1), (0, 1))


def hgf_weights(G: np.ndarray, Y: np.ndarray, lam: float, r: int, mode: str = MODE_HGF,
                method: str = "solve") -> np.ndarray:
    """Per-pixel coefficients w_p = (w_p(0), ..., w_p(n)) (shape (n+1, H, W) or (n+1, L, H, W)).

    mode "hgf": Eq7 -> Eq2: w = (lam E + X^T X)^-1 X^T c_{n+1}; all n+1 coefficients penalised.
    mode "gf":  Eq15/16: centred slopes (lam E + X'^T X')^-1 X'^T c', w(0) = mean(c) - w^T mean(x).
    method "solve": a dense solve per pixel (the plain definition).
    method "paper": Prop 1 recursion (alpha) + Eq13 / Eq5 weights (the paper's scheme).
    Y may be (H, W) or a stack (L, H, W) of slices.
    """
    G = np.asarray(G, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    n, H, W = G.shape
    Gram, _ = gram_planes(G, r)
    ext = np.concatenate([np.ones((1, H, W)), G], axis=0)
    if Y.ndim == 2:
        Gy = box_sum(ext * Y[None], r)                          # (n+1, H, W)
    else:
        Gy = box_sum(ext[:, None] * Y[None], r)                 # (n+1, L, H, W)
    if mode == MODE_HGF:
        if method == "solve":
            M = Gram + lam * np.eye(n + 1)[:, :, None, None]
            return _solve_batched(M, Gy)
        if method == "paper":
            alpha = alpha_recursion(Gram, lam)
            if Gy.ndim == 3:
                return weights_eq13(alpha, Gram, Gy, lam)
            return np.stack([weights_eq13(alpha, Gram, Gy[:, l], lam) for l in range(Gy.shape[1])], axis=1)
        raise ValueError(method)
    if mode == MODE_GF:
        N = Gram[0, 0]
        mu = Gram[0, 1:] / N                                    # x-bar
        # centred Gram G'_ij = c'_i^T c'_j = G_ij - N mu_i mu_j  (i, j = 1..n)
        Gc = Gram[1:, 1:] - N * mu[:, None] * mu[None, :]
        ybar = Gy[0] / N                                        # c_{n+1} bar
        if Gy.ndim == 3:
            cc = Gy[1:] - N * mu * ybar                         # X'^T c'_{n+1}
        else:
            cc = Gy[1:] - N * mu[:, None] * ybar[None]
        if method == "solve":
            M = Gc + lam * np.eye(n)[:, :, None, None]
            ws = _solve_batched(M, cc)
        elif method == "paper":
            alpha = alpha_recursion(Gc, lam)                    # same technique on Eq16
            if cc.ndim == 3:
                ws = weights_eq13(alpha, Gc, cc, lam)
            else:
                ws = np.stack([weights_eq13(alpha, Gc, cc[:, l], lam) for l in range(cc.shape[1])], axis=1)
        else:
            raise ValueError(method)
        if ws.ndim == 3:
            w0 = ybar - np.einsum("i...,i...->...", ws, mu)
        else:
            w0 = ybar - np.einsum("il...,i...->l...", ws, mu)
        return np.concatenate([w0[None], ws], axis=0)
    raise ValueError(mode)


def hgf_filter(I: np.ndarray, Y: np.ndarray, lam: float, r: int, d: int, mode: str = MODE_HGF,
               method: str = "solve") -> np.ndarray:
    """Z = HGF(Y; guidance synthesised from I) (Fig 2): guidance -> Gram -> w -> Eq14.

    I: (m, H, W) raw guide; Y: (H, W) slice or (L, H, W) stack.  Returns Z with Y's shape.
    """
    G = poly_guidance(I, d)
    w = hgf_weights(G, Y, lam, r, mode=mode, method=method)
    if w.ndim == 3:
        return _aggregate(w, G, r)
    return np.stack([_aggregate(w[:, l], G, r) for l in range(w.shape[1])], axis=0)


def hgf_filter_brute(I: np.ndarray, Y: np.ndarray, lam: float, r: int, d: int,
                     mode: str = MODE_HGF) -> np.ndarray:
    """Explicit per-window regression + explicit Eq8 aggregation (tiny inputs only).

    For each p: gather X_p = [1, G_1..G_n] over the clipped window, solve the ridge normal
    equations by LU (np.linalg.solve); then Z(q) = mean_{p in Omega_q} (w_p(0) + sum_i w_p(i) G_i(q)).
    """
    G = poly_guidance(I, d)
    Y = np.asarray(Y, dtype=np.float64)
    n, H, W = G.shape
    w = np.zeros((n + 1, H, W))
    for y in range(H):
        for x in range(W):
            ys = slice(max(0, y - r), min(H, y + r + 1))
            xs = slice(max(0, x - r), min(W, x + r + 1))
            cols = [np.ones(G[0, ys, xs].size)] + [G[i, ys, xs].ravel() for i in range(n)]
            X = np.stack(cols, axis=1)
            c = Y[ys, xs].ravel()
            if mode == MODE_HGF:
                w[:, y, x] = np.linalg.solve(lam * np.eye(n + 1) + X.T @ X, X.T @ c)
            else:
                Xc = X[:, 1:] - X[:, 1:].mean(axis=0)[None]
                cc = c - c.mean()
                ws = np.linalg.solve(lam * np.eye(n) + Xc.T @ Xc, Xc.T @ cc)
                w[1:, y, x] = ws
                w[0, y, x] = c.mean() - ws @ X[:, 1:].mean(axis=0)
    Z = np.zeros((H, W))
    for y in range(H):
        for x in range(W):
            acc, cnt = 0.0, 0
            for py in range(max(0, y - r), min(H, y + r + 1)):
                for px in range(max(0, x - r), min(W, x + r + 1)):
                    acc += w[0, py, px] + sum(w[i + 1, py, px] * G[i, y, x] for i in range(n))
                    cnt += 1
            Z[y, x] = acc / cnt
    return Z


def gf_he(I: np.ndarray, p: np.ndarray, eps: np.ndarray | float, r: int) -> np.ndarray:
    """He et al.'s guided filter closed form (means; gray or colour guide), used to pin GF mode.

    a = (Sigma_p + eps U)^-1 cov_p(I, p), b = mean(p) - a^T mean(I), q = mean(a)^T I + mean(b).
    eps may be a per-pixel plane (GF mode's lambda against sums gives eps_p = lambda / N_p).
    """
    I = np.asarray(I, dtype=np.float64)
    if I.ndim == 2:
        I = I[None]
    p = np.asarray(p, dtype=np.float64)
    m, H, W = I.shape
    mI = box_mean(I, r)
    mp = box_mean(p, r)
    cov = box_mean(I * p[None], r) - mI * mp[None]
    Sig = np.empty((m, m, H, W))
    for i in range(m):
        for j in range(m):
            Sig[i, j] = box_mean(I[i] * I[j], r) - mI[i] * mI[j]
    eps = np.broadcast_to(np.asarray(eps, dtype=np.float64), (H, W))
    Sig = Sig + np.eye(m)[:, :, None, None] * eps[None, None]
    a = _solve_batched(Sig, cov)
    b = mp - np.einsum("i...,i...->...", a, mI)
    return np.einsum("i...,i...->...", box_mean(a, r), I) + box_mean(b, r)


# --------------------------------------------------------------------------
# Winner-takes-all (§1) and the packed keys of the label-sharded merge
# --------------------------------------------------------------------------
def wta(Z: np.ndarray) -> np.ndarray:
    """label(q) = min{ l : Z_l(q) = min_k Z_k(q) } (F14).  Z: (L, H, W) -> int32 (H, W)."""
    Z = np.asarray(Z)
    L = Z.shape[0]
    best = Z[0].copy()
    lab = np.zeros(Z.shape[1:], dtype=np.int32)
    for l in range(1, L):                       # strict '<' keeps the lowest index on ties
        better = Z[l] < best
        best = np.where(better, Z[l], best)
        lab = np.where(better, l, lab)
    return lab


def aggregate_wta(I, V, lam, r, d, mode=MODE_HGF, method="solve", return_z=False):
    """Multi-label aggregation (filter every slice of V(x, y, l)) followed by WTA."""
    Z = hgf_filter(I, V, lam, r, d, mode=mode, method=method)
    lab = wta(Z)
    if return_z:
        return lab, Z
    return lab


def _orderable_u32(f32: np.ndarray) -> np.ndarray:
    """Monotone map of float32 bit patterns to uint32 (negative: ~bits; non-negative: bits | 2^31)."""
    f = np.asarray(f32, dtype=np.float32) + np.float32(0.0)     # -0.0 -> +0.0
    b = f.view(np.uint32).astype(np.uint64)
    neg = (b >> np.uint64(31)) & np.uint64(1)
    return np.where(neg == 1, (~b) & np.uint64(0xFFFFFFFF), b | np.uint64(0x80000000)).astype(np.uint64)


def pack_keys(cost_f32: np.ndarray, labels: np.ndarray) -> np.ndarray:
    """key = orderable(cost) << 32 | label  (uint64): min over keys = (min cost, lowest label)."""
    return (_orderable_u32(cost_f32) << np.uint64(32)) | np.asarray(labels).astype(np.uint64)


def unpack_keys(keys: np.ndarray):
    """Inverse of pack_keys: returns (cost float32, label int32)."""
    keys = np.asarray(keys, dtype=np.uint64)
    o = (keys >> np.uint64(32)) & np.uint64(0xFFFFFFFF)
    hi = (o >> np.uint64(31)) & np.uint64(1)
    b = np.where(hi == 1, o & np.uint64(0x7FFFFFFF), (~o) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return b.view(np.float32), (keys & np.uint64(0xFFFFFFFF)).astype(np.int32)


# ----------------------------------------------------------------------------- stereo cost
def _gray_grad_x(img: np.ndarray) -> np.ndarray:
    """d/dx of the channel mean: central difference inside, one-sided at the two border columns."""
    g = img.astype(np.float64).mean(axis=0)
    out = np.empty_like(g)
    if g.shape[1] == 1:
        out[:] = 0.0
        return out
    out[:, 1:-1] = 0.5 * (g[:, 2:] - g[:, :-2])
    out[:, 0] = g[:, 1] - g[:, 0]
    out[:, -1] = g[:, -1] - g[:, -2]
    return out


def stereo_cost(left: np.ndarray, right: np.ndarray, L: int, l0: int = 0, alpha: float = 0.11,
                tau_c: float = 0.028, tau_g: float = 0.008) -> np.ndarray:
    """Truncated colour + gradient matching cost of disparity d = l0 .. l0+L-1 (the paper defers the stereo
    cost to Hosni et al.; the form here is SPEC S:400):

        C(x, y, d) = alpha min(mean_c |L_c(x,y) - R_c(x-d,y)|, tau_c) + (1-alpha) min(|dx L~ - dx R~(x-d)|, tau_g)

    with L~ / R~ the channel means and dx the central x-difference (one-sided at the borders); pixels with
    x - d < 0 take the truncation value alpha tau_c + (1-alpha) tau_g.  float64, (L, H, W)."""
    left = left.astype(np.float64)
    right = right.astype(np.float64)
    _, H, W = left.shape
    gl, gr = _gray_grad_x(left), _gray_grad_x(right)
    trunc = alpha * tau_c + (1.0 - alpha) * tau_g
    out = np.full((L, H, W), trunc)
    for k in range(L):
        d = l0 + k
        if d >= W:
            continue
        col = np.abs(left[:, :, d:] - right[:, :, :W - d]).mean(axis=0)
        grd = np.abs(gl[:, d:] - gr[:, :W - d])
        out[k, :, d:] = alpha * np.minimum(col, tau_c) + (1.0 - alpha) * np.minimum(grd, tau_g)
    return out


def stereo_cost_brute(left: np.ndarray, right: np.ndarray, L: int, l0: int = 0, alpha: float = 0.11,
                      tau_c: float = 0.028, tau_g: float = 0.008) -> np.ndarray:
    """stereo_cost by explicit per-pixel loops (tiny inputs only; pins the vectorised form)."""
    m, H, W = left.shape

    def gray(img, y, x):
        return sum(float(img[c, y, x]) for c in range(m)) / m

    def gx(img, y, x):
        if W == 1:
            return 0.0
        if x == 0:
            return gray(img, y, 1) - gray(img, y, 0)
        if x == W - 1:
            return gray(img, y, W - 1) - gray(img, y, W - 2)
        return 0.5 * (gray(img, y, x + 1) - gray(img, y, x - 1))

    out = np.empty((L, H, W))
    for k in range(L):
        d = l0 + k
        for y in range(H):
            for x in range(W):
                if x - d < 0:
                    out[k, y, x] = alpha * tau_c + (1 - alpha) * tau_g
                    continue
                col = sum(abs(float(left[c, y, x]) - float(right[c, y, x - d])) for c in range(m)) / m
                grd = abs(gx(left, y, x) - gx(right, y, x - d))
                out[k, y, x] = alpha * min(col, tau_c) + (1 - alpha) * min(grd, tau_g)
    return out



# ----------------------------------------------------------------------------- segmentation cost
SEG_BINS = 32


def segmentation_cost(image: np.ndarray, fg: np.ndarray, bg: np.ndarray, bins: int = SEG_BINS) -> np.ndarray:
    """Two cost slices (0 = foreground, 1 = background) for the segmentation workload (labels are
    foreground / background, costs as in Hosni et al.; the form is SPEC S:406-409): per class, per-channel
    histograms of the seed pixels' colours with `bins` bins (bin = min(floor(v * bins), bins - 1) of a [0,1]
    intensity), Laplace-smoothed (+1 per bin): p_c(b) = (count_c(b) + 1) / (N + bins).  The colour
    likelihood is the product over channels (readings S1, S2 in DESIGN.md), the cost its negative log
    normalised by its largest possible value m log(N + bins) (a colour no seed has), so each slice lies in
    (0, 1].
    image: (m, H, W); fg, bg: boolean (H, W) seed masks, both non-empty.  float64 (2, H, W)."""
    img = np.asarray(image, dtype=np.float64)
    m = img.shape[0]
    b = np.minimum(np.floor(img * bins), bins - 1).astype(np.int64)
    b = np.maximum(b, 0)
    out = []
    for seeds in (fg, bg):
        seeds = np.asarray(seeds, dtype=bool)
        N = int(seeds.sum())
        if N == 0:
            raise ValueError("empty seed set")
        nll = np.zeros(img.shape[1:])
        for c in range(m):
            counts = np.bincount(b[c][seeds], minlength=bins).astype(np.float64)
            p = (counts + 1.0) / (N + bins)
            nll -= np.log(p[b[c]])
        out.append(nll / (m * np.log(N + bins)))
    return np.stack(out)


# ----------------------------------------------------------------------------- post-processing
# P:641 names the step ("post processing" of Hosni et al.'s framework) and gives nothing else; the
# readings P1-P4 below follow Hosni et al.'s published framework: a right-view disparity
# map from the same aggregation, a left-right consistency check, filling of inconsistent pixels from the
# nearest consistent pixels of the row (the lower disparity: background), then a weighted median with
# bilateral weights over the filled pixels only.

def stereo_cost_right(left: np.ndarray, right: np.ndarray, L: int, l0: int = 0, alpha: float = 0.11,
                      tau_c: float = 0.028, tau_g: float = 0.008) -> np.ndarray:
    """Reading P1: the right view's cost of disparity d = l0 .. l0+L-1 is stereo_cost with the roles of the
    views exchanged and the match searched at x + d:

        C_R(x, y, d) = alpha min(mean_c |R_c(x,y) - L_c(x+d,y)|, tau_c) + (1-alpha) min(|dx R~(x,y) - dx L~(x+d,y)|, tau_g)

    pixels with x + d >= W take the truncation value.  float64, (L, H, W)."""
    left = left.astype(np.float64)
    right = right.astype(np.float64)
    _, H, W = left.shape
    gl, gr = _gray_grad_x(left), _gray_grad_x(right)
    trunc = alpha * tau_c + (1.0 - alpha) * tau_g
    out = np.full((L, H, W), trunc)
    for k in range(L):
        d = l0 + k
        if d >= W:
            continue
        col = np.abs(right[:, :, :W - d] - left[:, :, d:]).mean(axis=0)
        grd = np.abs(gr[:, :W - d] - gl[:, d:])
        out[k, :, :W - d] = alpha * np.minimum(col, tau_c) + (1.0 - alpha) * np.minimum(grd, tau_g)
    return out


def lr_consistency(dL: np.ndarray, dR: np.ndarray, tol: int = 0) -> np.ndarray:
    """Reading P2: pixel (x, y) of the left disparity map is consistent iff its match lies inside the right
    view, x - dL(x,y) >= 0, and the right map agrees there: |dL(x,y) - dR(x - dL(x,y), y)| <= tol.
    dL, dR: int (H, W) disparities; returns bool (H, W)."""
    dL = np.asarray(dL, dtype=np.int64)
    dR = np.asarray(dR, dtype=np.int64)
    H, W = dL.shape
    xr = np.arange(W)[None, :] - dL
    inside = (xr >= 0) & (xr < W)
    rows = np.broadcast_to(np.arange(H)[:, None], (H, W))
    match = dR[rows, np.clip(xr, 0, W - 1)]
    return inside & (np.abs(dL - match) <= tol)


def occlusion_fill(dL: np.ndarray, valid: np.ndarray) -> np.ndarray:
    """Reading P3: an inconsistent pixel takes the disparity of the nearest consistent pixel to its left or
    to its right on the same row, the lower of the two where both exist (occlusions belong to the
    background), the one that exists otherwise; a row without any consistent pixel keeps its values.
    Consistent pixels are unchanged.  int64 (H, W)."""
    dL = np.asarray(dL, dtype=np.int64)
    valid = np.asarray(valid, dtype=bool)
    H, W = dL.shape
    xs = np.broadcast_to(np.arange(W)[None, :], (H, W))
    left_idx = np.maximum.accumulate(np.where(valid, xs, -1), axis=1)            # nearest valid at or left of x
    right_idx = np.minimum.accumulate(np.where(valid, xs, W)[:, ::-1], axis=1)[:, ::-1]   # ... at or right of x
    rows = np.broadcast_to(np.arange(H)[:, None], (H, W))
    has_l, has_r = left_idx >= 0, right_idx < W
    vl = np.where(has_l, dL[rows, np.clip(left_idx, 0, W - 1)], 0)
    vr = np.where(has_r, dL[rows, np.clip(right_idx, 0, W - 1)], 0)
    fill = np.where(has_l & has_r, np.minimum(vl, vr), np.where(has_l, vl, np.where(has_r, vr, dL)))
    return np.where(valid, dL, fill)


def window_weights(D: np.ndarray, image: np.ndarray, y: int, x: int, radius: int, sigma_s: float,
                   sigma_c: float):
    """Reading P4's window at pixel (y, x): the values D(q) and bilateral weights

        w(p, q) = exp(-|q - p|^2 / sigma_s^2 - sum_c (I_c(q) - I_c(p))^2 / sigma_c^2)

    over the (2 radius + 1)^2 window clipped at the image border (I channels first).  Returns
    (values int64 (n,), weights float64 (n,))."""
    img = np.asarray(image, dtype=np.float64)
    H, W = D.shape
    y0, y1, x0, x1 = max(0, y - radius), min(H, y + radius + 1), max(0, x - radius), min(W, x + radius + 1)
    yy, xx = np.mgrid[y0:y1, x0:x1]
    dist2 = ((yy - y) ** 2 + (xx - x) ** 2).astype(np.float64)
    col2 = ((img[:, y0:y1, x0:x1] - img[:, y, x][:, None, None]) ** 2).sum(axis=0)
    w = np.exp(-dist2 / sigma_s ** 2 - col2 / sigma_c ** 2).ravel()
    return np.asarray(D[y0:y1, x0:x1], dtype=np.int64).ravel(), w


def weighted_median_fill(D: np.ndarray, valid: np.ndarray, image: np.ndarray, radius: int, sigma_s: float,
                         sigma_c: float) -> np.ndarray:
    """Reading P4: every inconsistent pixel p takes the weighted median of the filled map D over its window
    (window_weights): the smallest window value d with sum_{q: D(q) <= d} w(p, q) >= 1/2 sum_q w(p, q).
    Consistent pixels are unchanged.  int64 (H, W)."""
    D = np.asarray(D, dtype=np.int64)
    out = D.copy()
    for y, x in zip(*np.nonzero(~np.asarray(valid, dtype=bool))):
        vals, w = window_weights(D, image, y, x, radius, sigma_s, sigma_c)
        half = 0.5 * w.sum()
        for d in np.unique(vals):                                   # ascending
            if w[vals <= d].sum() >= half:
                out[y, x] = d
                break
    return out


def lr_postprocess(image: np.ndarray, dL: np.ndarray, dR: np.ndarray, tol: int = 0, radius: int = 9,
                   sigma_s: float = 9.0, sigma_c: float = 0.1):
    """P2 -> P3 -> P4 in order.  Returns (final disparity int64 (H, W), consistency mask bool (H, W))."""
    valid = lr_consistency(dL, dR, tol)
    filled = occlusion_fill(dL, valid)
    return weighted_median_fill(filled, valid, image, radius, sigma_s, sigma_c), valid
