"""Pins for oracle/ against things other than itself (-m "not gpu").

Each test names the passage it follows.  Pins: brute force, exact integer arithmetic,
independent solvers (LU inverse / least squares / Cramer), closed forms, He et al.'s
textbook closed form, invariants, and SPEC/closed-form fixtures in tests/golden/.
Several tests also show that the plausible *misreadings* of the paper (printed
alpha^0_00, Eq11 without gamma, dropped intercept penalty) FAIL the same pins.
"""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
RNG = np.random.default_rng(12345)


# ---------------------------------------------------------------- box filter (Prop 2)
@pytest.mark.parametrize("shape,r", [((9, 11), 1), ((9, 11), 2), ((5, 3), 3), ((1, 1), 2), ((7, 13), 7), ((16, 4), 1)])
def test_box_sum_exact_on_integers(shape, r):
    X = RNG.integers(0, 2 ** 20, size=shape).astype(np.float64)
    assert np.array_equal(O.box_sum(X, r), O.box_sum_brute(X, r))


def test_box_sum_golden():
    g = GOLD["box_sum_2x2_r1"]
    assert np.array_equal(O.box_sum(np.array(g["plane"], float), g["r"]), np.array(g["expect"], float))
    g = GOLD["box_sum_ones_2x2_r1"]
    assert np.array_equal(O.box_sum(np.array(g["plane"], float), g["r"]), np.array(g["expect"], float))
    g = GOLD["box_sum_ones_5x5_r1"]
    B = O.box_sum(np.ones((g["H"], g["W"])), g["r"])
    assert B[0, 0] == g["corner"] and B[2, 2] == g["centre"]
    assert np.array_equal(O.box_count(g["H"], g["W"], g["r"]), B)
    g = GOLD["box_mean_half"]
    assert np.allclose(O.box_mean(np.array(g["plane"], float), g["r"]), g["expect"], rtol=0, atol=1e-15)


def test_box_linearity_and_count():
    X, Y = RNG.random((2, 12, 17))
    a, b = 0.3, -2.5
    assert np.allclose(O.box_sum(a * X + b * Y, 3), a * O.box_sum(X, 3) + b * O.box_sum(Y, 3), atol=1e-12)
    for H, W, r in [(1, 1, 3), (4, 9, 2), (20, 20, 9)]:
        assert np.array_equal(O.box_count(H, W, r), O.box_sum_brute(np.ones((H, W)), r))


# ---------------------------------------------------------------- polynomial guidance
def test_poly_guidance_golden_and_order():
    g = GOLD["poly_half_d3"]
    G = O.poly_guidance(np.full((1, 2, 2), g["value"]), g["d"])
    assert np.array_equal(G[:, 0, 0], np.array(g["expect"]))
    I = RNG.random((3, 4, 5))
    G = O.poly_guidance(I, 2)
    expect = np.stack([I[0], I[0] ** 2, I[1], I[1] ** 2, I[2], I[2] ** 2])   # channel-major
    assert np.allclose(G, expect, rtol=1e-15, atol=0)
    assert np.array_equal(O.poly_guidance(I, 1), I)


# ---------------------------------------------------------------- Gram (Prop 2, Eq12)
def test_gram_golden():
    g = GOLD["gram_2x2_r1"]
    Gram, _ = O.gram_planes(np.array([g["plane"]], float), g["r"])
    assert np.all(Gram[1, 1] == g["expect_G11"])
    assert np.all(Gram[0, 1] == g["expect_G01"]) and np.all(Gram[0, 0] == g["expect_G00"])


def test_gram_vs_naive_window_dot_products():
    H, W, r, n = 7, 9, 2, 3
    G = RNG.integers(0, 1000, size=(n, H, W)).astype(np.float64)
    Y = RNG.integers(0, 1000, size=(H, W)).astype(np.float64)
    Gram, Gy = O.gram_planes(G, r, Y)
    ext = np.concatenate([np.ones((1, H, W)), G])
    for y in range(H):
        for x in range(W):
            sl = (slice(None), slice(max(0, y - r), y + r + 1), slice(max(0, x - r), x + r + 1))
            C = ext[sl].reshape(n + 1, -1)
            assert np.array_equal(Gram[:, :, y, x], C @ C.T)
            assert np.array_equal(Gy[:, y, x], C @ Y[sl[1:]].ravel())


# ---------------------------------------------------------------- Prop 1 (Eq4)
def _random_windows(N, K, rng):
    C = rng.random((N, K))
    C[:, 0] = 1.0                       # c_0 = ones
    return C


@pytest.mark.parametrize("N", [9, 25, 225])
@pytest.mark.parametrize("K", [1, 2, 4, 7, 10])
@pytest.mark.parametrize("lam", [0.05, 1.0, 2.0])
def test_alpha_inverse_identity(N, K, lam):
    """(lam E + sum c_i c_i^T)(lam^-1 E + sum alpha_ij c_i c_j^T) = E in the |Omega|-dim space (Prop 1)."""
    rng = np.random.default_rng(N * 100 + K)
    C = _random_windows(N, K, rng)
    alpha = O.alpha_recursion(C.T @ C, lam)
    A = lam * np.eye(N) + C @ C.T
    Ainv = np.eye(N) / lam + C @ alpha @ C.T
    assert np.linalg.norm(A @ Ainv - np.eye(N)) <= 1e-8
    # M^-1 = -lam alpha where M = lam E + Gram (Woodbury), vs an LU inverse (np.linalg.inv)
    Minv = np.linalg.inv(lam * np.eye(K) + C.T @ C)
    assert np.abs(-lam * alpha - Minv).max() <= 1e-9 * np.abs(Minv).max()
    assert np.abs(alpha - alpha.T).max() <= 1e-9 * np.abs(alpha).max()


def test_alpha_golden_and_misreadings_fail():
    for key in ("alpha00_lambda1", "alpha00_lambda2"):
        g = GOLD[key]
        a = O.alpha_recursion(np.array([[g["G00"]]]), g["lambda"])
        assert a[0, 0] == pytest.approx(g["expect"], rel=1e-15)
    # printed init -(lambda+G00)^-1 fails the identity at lambda = 2 (reading F1)
    g = GOLD["alpha00_lambda2"]
    assert -1.0 / (g["lambda"] + g["G00"]) == pytest.approx(g["printed_formula_value"])
    N, K, lam = 25, 4, 0.05
    C = _random_windows(N, K, np.random.default_rng(7))
    Gram = C.T @ C

    def recursion(init_printed=False, drop_gamma=False):
        inv = 1 / lam
        al = np.zeros((K, K))
        al[0, 0] = -1 / (lam + Gram[0, 0]) if init_printed else -inv / (lam + Gram[0, 0])
        for k in range(1, K):
            u = al[:k, :k] @ Gram[:k, k]
            gam = -1 / (1 + inv * Gram[k, k] + Gram[k, :k] @ u)
            al[:k, :k] = (1.0 if drop_gamma else gam) * np.outer(u, u) + al[:k, :k]
            al[:k, k] = al[k, :k] = inv * gam * u
            al[k, k] = inv * inv * gam
        return al

    def resid(al):
        return np.linalg.norm((lam * np.eye(N) + C @ C.T) @ (np.eye(N) / lam + C @ al @ C.T) - np.eye(N))

    assert resid(recursion()) < 1e-9
    assert np.allclose(recursion(), O.alpha_recursion(Gram, lam), rtol=1e-12, atol=0)
    assert resid(recursion(init_printed=True)) > 1.0          # F1 misreading fails
    assert resid(recursion(drop_gamma=True)) > 1.0            # F2 misreading fails


def test_gamma_denominator_at_least_one():
    C = _random_windows(49, 8, np.random.default_rng(3))
    Gram = C.T @ C
    lam = 0.05
    al = O.alpha_recursion(Gram, lam)
    # -1/gamma_kappa = 1 + c^T A^-1 c >= 1 ; alpha_kk = lam^-2 gamma  => gamma in [-1, 0)
    gam = np.diag(al)[1:] * lam * lam
    assert np.all(gam < 0) and np.all(gam >= -1)


# ---------------------------------------------------------------- weights (Eq2, Eq5/Eq13)
def test_weights_closed_forms():
    g = GOLD["weights_n0"]
    # n = 0: only c_0 = ones, Y = 1 in a 3x3 window (one pixel at the centre of a 3x3 image, r = 1)
    Gram = np.array([[g["N"]]], float)
    Gy = np.array([g["N"] * g["Y"]])
    al = O.alpha_recursion(Gram, g["lambda"])
    W = O.weights_eq13(al, Gram, Gy, g["lambda"])
    assert W[0] == pytest.approx(g["expect"], rel=1e-14)


@pytest.mark.parametrize("mode", ["hgf", "gf"])
def test_weights_three_solvers_agree(mode):
    """Prop-1 + Eq13 == dense solve == augmented least squares [X; sqrt(lam) D] w = [y; 0] (Eq7 / Eq15)."""
    H, W, r, lam = 6, 7, 2, 0.05
    I = RNG.random((2, H, W))
    Y = RNG.random((H, W))
    G = O.poly_guidance(I, 2)
    w_solve = O.hgf_weights(G, Y, lam, r, mode=mode, method="solve")
    w_paper = O.hgf_weights(G, Y, lam, r, mode=mode, method="paper")
    n = G.shape[0]
    D = np.eye(n + 1) if mode == "hgf" else np.diag([0.0] + [1.0] * n)
    for y in range(H):
        for x in range(W):
            sl = (slice(max(0, y - r), y + r + 1), slice(max(0, x - r), x + r + 1))
            X = np.stack([np.ones(Y[sl].size)] + [G[i][sl].ravel() for i in range(n)], 1)
            A = np.vstack([X, np.sqrt(lam) * D])
            rhs = np.concatenate([Y[sl].ravel(), np.zeros(n + 1)])
            w_ls = np.linalg.lstsq(A, rhs, rcond=None)[0]
            assert np.allclose(w_solve[:, y, x], w_ls, rtol=1e-9, atol=1e-9)
    assert np.allclose(w_paper, w_solve, rtol=1e-7, atol=1e-7)


def test_hgf_n1_cramer():
    """n = 1 (gray, d = 1): 2x2 system [[lam+N, S1],[S1, lam+S11]] w = [Sy, S1y] by Cramer's rule."""
    H, W, r, lam = 8, 9, 2, 0.05
    I = RNG.random((1, H, W))
    Y = RNG.random((H, W))
    N = O.box_count(H, W, r)
    S1 = O.box_sum(I[0], r)
    S11 = O.box_sum(I[0] * I[0], r)
    Sy = O.box_sum(Y, r)
    S1y = O.box_sum(I[0] * Y, r)
    a, b, c, d = lam + N, S1, S1, lam + S11
    det = a * d - b * c
    w0 = (Sy * d - b * S1y) / det
    w1 = (a * S1y - c * Sy) / det
    w = O.hgf_weights(I, Y, lam, r, mode="hgf")
    assert np.allclose(w[0], w0, rtol=1e-10) and np.allclose(w[1], w1, rtol=1e-10)
    Z = (O.box_sum(w0, r) + I[0] * O.box_sum(w1, r)) / N          # Eq14 written out
    assert np.allclose(O.hgf_filter(I, Y, lam, r, 1), Z, rtol=1e-10, atol=1e-12)


# ---------------------------------------------------------------- whole filter (Eq8/Eq14)
@pytest.mark.parametrize("mode", ["hgf", "gf"])
@pytest.mark.parametrize("m,d,r,H,W", [(3, 2, 2, 9, 11), (1, 3, 1, 6, 5), (2, 1, 3, 7, 7), (3, 3, 2, 5, 13)])
def test_filter_definition_vs_brute_vs_paper(mode, m, d, r, H, W):
    rng = np.random.default_rng(m * 31 + d * 7 + r)
    I = rng.random((m, H, W))
    Y = rng.random((H, W))
    lam = 0.05
    z_def = O.hgf_filter(I, Y, lam, r, d, mode=mode)
    z_brute = O.hgf_filter_brute(I, Y, lam, r, d, mode=mode)
    z_paper = O.hgf_filter(I, Y, lam, r, d, mode=mode, method="paper")
    assert np.allclose(z_def, z_brute, rtol=1e-9, atol=1e-10)
    assert np.allclose(z_paper, z_def, rtol=1e-6, atol=1e-8)


@pytest.mark.parametrize("mode", ["hgf", "gf"])
@pytest.mark.parametrize("method", ["solve", "paper"])
@pytest.mark.parametrize("m,d,r,H,W,L", [(3, 2, 2, 8, 10, 3), (1, 3, 1, 6, 5, 2), (2, 1, 3, 7, 9, 4)])
def test_multislice_stack_equals_per_slice_and_brute(mode, method, m, d, r, H, W, L):
    """The stacked (L, H, W) branches of hgf_weights / hgf_filter (the form every GPU parity test compares
    against: the 4-D batched solve of the HGF mode, the GF mode's stacked centring cc = Gy - N mu ybar and
    the w0 = ybar - sum_i w_i mu_i contraction, the per-slice Eq13 loop of method "paper") against
    (a) hgf_filter_brute slice by slice -- explicit window gathers + LU + the explicit Eq8 double loop
    (P:257-262), no box filter, no SAT, no batched solve -- and (b) the single-slice branch."""
    rng = np.random.default_rng(1000 + 97 * m + 13 * d + r + L)
    I = rng.random((m, H, W))
    Y = rng.random((L, H, W))
    lam = 0.05
    z_stack = O.hgf_filter(I, Y, lam, r, d, mode=mode, method=method)
    assert z_stack.shape == (L, H, W)
    G = O.poly_guidance(I, d)
    w_stack = O.hgf_weights(G, Y, lam, r, mode=mode, method=method)
    assert w_stack.shape == (m * d + 1, L, H, W)
    for l in range(L):
        z_brute = O.hgf_filter_brute(I, Y[l], lam, r, d, mode=mode)
        tol = (1e-9, 1e-10) if method == "solve" else (1e-6, 1e-8)
        assert np.allclose(z_stack[l], z_brute, rtol=tol[0], atol=tol[1])
        assert np.allclose(z_stack[l], O.hgf_filter(I, Y[l], lam, r, d, mode=mode, method=method), rtol=1e-12,
                           atol=1e-13)
        assert np.allclose(w_stack[:, l], O.hgf_weights(G, Y[l], lam, r, mode=mode, method=method), rtol=1e-12,
                           atol=1e-13)


def test_multislice_gf_centring_terms_written_out():
    """GF mode's stacked centring (Eq16 P:369 via §5.1's centred regression): the stacked weights
    equal the per-window textbook solve written out with explicit means -- w = (lam E + Xc^T Xc)^-1 Xc^T cc,
    w0 = mean(c) - w^T mean(x) -- for every slice, so a transposed operand or a dropped N mu ybar term in the
    stacked branch fails."""
    rng = np.random.default_rng(77)
    m, d, r, H, W, L, lam = 2, 2, 2, 6, 7, 3, 0.05
    I = rng.random((m, H, W))
    Y = rng.random((L, H, W))
    G = O.poly_guidance(I, d)
    w = O.hgf_weights(G, Y, lam, r, mode="gf")
    n = m * d
    for l in range(L):
        for y in range(H):
            for x in range(W):
                ys = slice(max(0, y - r), min(H, y + r + 1))
                xs = slice(max(0, x - r), min(W, x + r + 1))
                X = np.stack([G[i][ys, xs].ravel() for i in range(n)], 1)
                c = Y[l][ys, xs].ravel()
                Xc, cc = X - X.mean(0), c - c.mean()
                ws = np.linalg.solve(lam * np.eye(n) + Xc.T @ Xc, Xc.T @ cc)
                assert np.allclose(w[1:, l, y, x], ws, rtol=1e-9, atol=1e-11)
                assert np.isclose(w[0, l, y, x], c.mean() - ws @ X.mean(0), rtol=1e-9, atol=1e-11)


def test_intercept_penalty_distinguishes_modes():
    """HGF (Eq7) penalises w(0); GF (Eq15) does not — a dropped/added intercept term changes Z."""
    I = RNG.random((3, 10, 10))
    Y = RNG.random((10, 10))
    zh = O.hgf_filter(I, Y, 0.05, 2, 1, mode="hgf")
    zg = O.hgf_filter(I, Y, 0.05, 2, 1, mode="gf")
    assert np.abs(zh - zg).max() > 1e-4


@pytest.mark.parametrize("m", [1, 3])
def test_gf_mode_equals_he_closed_form(m):
    """GF mode (§5.1) == He et al.'s closed form with eps_p = lambda / N_p (B is a sum, F7)."""
    H, W, r, lam = 12, 15, 3, 0.05
    I = RNG.random((m, H, W))
    Y = RNG.random((H, W))
    eps = lam / O.box_count(H, W, r)
    assert np.allclose(O.hgf_filter(I, Y, lam, r, 1, mode="gf"), O.gf_he(I, Y, eps, r), rtol=1e-10, atol=1e-12)


# ---------------------------------------------------------------- invariants (north-star oracle checks)
def test_gf_constant_in_constant_out_and_large_eps_box_mean():
    I = RNG.random((3, 11, 13))
    c = 0.37
    z = O.hgf_filter(I, np.full((11, 13), c), 0.05, 2, 2, mode="gf")
    assert np.abs(z - c).max() <= 1e-12
    Y = RNG.random((11, 13))
    z = O.hgf_filter(I, Y, 1e9, 2, 2, mode="gf")               # slopes -> 0, Z -> A(A(Y))
    assert np.abs(z - O.box_mean(O.box_mean(Y, 2), 2)).max() <= 1e-7


def test_hgf_linearity_and_large_lambda_limit():
    I = RNG.random((3, 9, 10))
    Y1, Y2 = RNG.random((2, 9, 10))
    f = lambda Y, lam=0.05: O.hgf_filter(I, Y, lam, 2, 2)
    assert np.allclose(f(2 * Y1 - 3 * Y2), 2 * f(Y1) - 3 * f(Y2), atol=1e-11)
    lam = 1e9
    G = O.poly_guidance(I, 2)
    ext = np.concatenate([np.ones((1, 9, 10)), G])
    limit = sum(ext[k] * O.box_mean(O.box_sum(ext[k] * Y1, 2), 2) for k in range(ext.shape[0]))
    assert np.abs(lam * f(Y1, lam) - limit).max() <= 1e-6 * np.abs(limit).max()


def test_wta_golden_and_brute():
    g = GOLD["wta_ties"]
    Z = np.array(g["costs"])[:, None, :]                        # (L, 1, 2)
    assert O.wta(Z)[0].tolist() == g["expect"]
    Z = RNG.integers(0, 4, size=(6, 5, 7)).astype(np.float64)    # many exact ties
    lab = O.wta(Z)
    for y in range(5):
        for x in range(7):
            col = list(Z[:, y, x])
            assert lab[y, x] == col.index(min(col))


def test_label_permutation_and_affine_invariance():
    I = RNG.random((3, 10, 12))
    V = RNG.random((7, 10, 12))
    lab, Z = O.aggregate_wta(I, V, 0.05, 2, 2, return_z=True)
    srt = np.sort(Z, axis=0)
    clear = (srt[1] - srt[0]) > 1e-9
    perm = RNG.permutation(7)
    lab_p = O.aggregate_wta(I, V[perm], 0.05, 2, 2)
    assert np.array_equal(perm[lab_p][clear], lab[clear])          # argmin(V o perm) = perm^-1(argmin V)
    lab_a = O.aggregate_wta(I, 3.0 * V + 0.25, 0.05, 2, 2)
    assert np.array_equal(lab_a[clear], lab[clear])


def test_keys_order_and_roundtrip():
    cost = np.array([0.5, -0.0, 0.0, -1.5, 2.0, np.float32(1e-30), -np.float32(1e-30)], np.float32)
    lab = np.array([3, 7, 1, 2, 9, 4, 5], np.int32)
    k = O.pack_keys(cost, lab)
    c2, l2 = O.unpack_keys(k)
    assert np.array_equal(l2, lab)
    assert np.array_equal(c2, cost + np.float32(0.0))
    order = np.argsort(k, kind="stable")
    lex = sorted(range(len(cost)), key=lambda i: (float(cost[i]), int(lab[i])))
    assert order.tolist() == lex
    # min over per-shard keys == global (min cost, lowest label)
    V = RNG.integers(0, 5, size=(8, 6)).astype(np.float32)   # (L, P) with ties
    full = O.pack_keys(V.min(0), V.argmin(0))
    shards = [O.pack_keys(V[a:b].min(0), a + V[a:b].argmin(0)) for a, b in [(0, 3), (3, 5), (5, 8)]]
    assert np.array_equal(np.minimum.reduce(shards), full)


# ----------------------------------------------------------------------------- stereo cost (NEXT-2)
def test_stereo_cost_matches_brute_force_and_edge_cases():
    rng = np.random.default_rng(3)
    left = rng.random((3, 5, 9))
    right = rng.random((3, 5, 9))
    a = O.stereo_cost(left, right, 6, l0=1)
    b = O.stereo_cost_brute(left, right, 6, l0=1)
    assert np.allclose(a, b, rtol=0, atol=1e-15)
    trunc = 0.11 * 0.028 + 0.89 * 0.008
    assert np.all(a[:, :, 0] == trunc)                     # x - d < 0 for every d >= 1 at x = 0
    assert np.all(a[4] [:, :5] == trunc)                    # d = 5: columns 0..4 out of range
    # identical views at d = 0: zero colour and gradient terms
    z = O.stereo_cost(left, left, 1)
    assert np.all(z == 0.0)
    # a view shifted by exactly s pixels matches at d = s away from the border columns
    s = 2
    shifted = np.zeros_like(left)
    shifted[:, :, :9 - s] = left[:, :, s:]
    c = O.stereo_cost(left, shifted, 4)
    assert np.allclose(c[s][:, s + 1:-1], 0.0, atol=1e-15)


def test_stereo_cost_truncation_bounds_and_weights():
    rng = np.random.default_rng(4)
    left, right = rng.random((3, 6, 11)), rng.random((3, 6, 11))
    c = O.stereo_cost(left, right, 5, alpha=0.3, tau_c=0.1, tau_g=0.05)
    assert c.min() >= 0.0 and c.max() <= 0.3 * 0.1 + 0.7 * 0.05 + 1e-15
    # untruncated regime: huge thresholds give exactly alpha*colour + (1-alpha)*gradient
    big = O.stereo_cost(left, right, 3, alpha=0.25, tau_c=1e9, tau_g=1e9)
    col = np.abs(left[:, :, 2:] - right[:, :, :-2]).mean(axis=0)
    gl, gr = np.gradient(left.mean(axis=0), axis=1), np.gradient(right.mean(axis=0), axis=1)   # same stencil
    g = gl[:, 2:] - gr[:, :-2]
    assert np.allclose(big[2][:, 2:], 0.25 * col + 0.75 * np.abs(g), rtol=0, atol=1e-14)


def test_stereo_cost_agrees_with_the_workload_generator():
    """Two independent implementations of S:400: the oracle (float64) and synth's input generator (float32)."""
    import synth
    scene = synth.make_stereo_scene(40, 24, 12, seed=9)
    gen = synth.stereo_cost_volume_np(scene, 12)
    ora = O.stereo_cost(scene.left, scene.right, 12)
    # the generator works in float32 on [0, 1] intensities: a few ulps (6e-8) of the gradient terms
    assert np.abs(gen - ora).max() < 3e-7


def test_stereo_rectangle_shift_fixture_recovers_disparity():
    """SPEC S:403 [DERIVED]: uniform background, a textured rectangle shifted by 4 px between the views ->
    WTA after HGF filtering recovers disparity 4 inside the rectangle (background: disparity 0)."""
    H, W, L, s = 24, 48, 8, 4
    rng = np.random.default_rng(7)
    left = np.full((3, H, W), 0.3)
    tex = 0.5 + 0.3 * rng.random((3, 10, 14))
    left[:, 7:17, 20:34] = tex
    right = np.full((3, H, W), 0.3)
    right[:, 7:17, 20 - s:34 - s] = tex
    C = O.stereo_cost(left, right, L)
    Z = O.hgf_filter(left, C, 0.05, 2, 1)
    lab = O.wta(Z)
    assert np.all(lab[9:15, 23:31] == s)


# ----------------------------------------------------------------------------- segmentation cost (NEXT-4)
def _two_colour_scene():
    H, W = 20, 30
    img = np.empty((3, H, W))
    img[:] = np.array([0.9, 0.2, 0.1])[:, None, None]          # foreground colour
    img[:, :, 15:] = np.array([0.1, 0.3, 0.8])[:, None, None]  # background colour (right half)
    fg = np.zeros((H, W), bool)
    bg = np.zeros((H, W), bool)
    fg[10, 5] = True
    bg[10, 25] = True
    return img, fg, bg


def test_segmentation_cost_spec_examples():
    img, fg, bg = _two_colour_scene()
    C = O.segmentation_cost(img, fg, bg)
    assert C.shape == (2, 20, 30) and C.min() > 0.0 and C.max() <= 1.0          # 1 = colour never seeded
    # a colour seen only in the fg seeds costs less as fg (S:408 example 1)
    assert np.all(C[0][:, :15] < C[1][:, :15]) and np.all(C[1][:, 15:] < C[0][:, 15:])
    # identical seed distributions -> identical slices (S:408 example 2)
    same = O.segmentation_cost(img, fg, fg)
    assert np.abs(same[0] - same[1]).max() <= 1e-12
    # closed form for one seed pixel: p = 2/33 in its bin, 1/33 elsewhere (Laplace +1, 32 bins)
    assert np.isclose(C[0][10, 5], -3 * np.log(2 / 33) / (3 * np.log(33)), rtol=0, atol=1e-15)
    assert np.isclose(C[1][10, 5], -3 * np.log(1 / 33) / (3 * np.log(33)), rtol=0, atol=1e-15)
    with pytest.raises(ValueError):
        O.segmentation_cost(img, fg, np.zeros_like(bg))


def test_segmentation_two_colour_fixture_labels_regions():
    """S:409 [DERIVED]: two-colour image, one seed pixel per region -> WTA after HGF filtering labels each
    region (0 = fg left, 1 = bg right) away from the boundary."""
    img, fg, bg = _two_colour_scene()
    C = O.segmentation_cost(img, fg, bg)
    lab = O.wta(O.hgf_filter(img, C, 0.05, 2, 1))
    assert np.all(lab[:, :12] == 0) and np.all(lab[:, 18:] == 1)


# ----------------------------------------------------------------------------- post-processing (NEXT-3)
def test_stereo_cost_right_mirror_identities():
    """P1 pinned two ways: C_R(x, d) = C_L(x + d, d) wherever x + d < W (the same pair of pixels), and the
    right cost is the left cost of the x-mirrored views with their roles exchanged (the central difference
    and its one-sided borders both change sign under the mirror; the truncation region maps onto x + d >= W)."""
    rng = np.random.default_rng(21)
    left, right = rng.random((3, 6, 13)), rng.random((3, 6, 13))
    L, l0 = 7, 1
    cr = O.stereo_cost_right(left, right, L, l0=l0, alpha=0.3, tau_c=0.2, tau_g=0.1)
    cl = O.stereo_cost(left, right, L, l0=l0, alpha=0.3, tau_c=0.2, tau_g=0.1)
    trunc = 0.3 * 0.2 + 0.7 * 0.1
    for k in range(L):
        d = l0 + k
        assert np.allclose(cr[k][:, :13 - d], cl[k][:, d:], rtol=0, atol=1e-15)
        assert np.all(cr[k][:, 13 - d:] == trunc)
    mir = O.stereo_cost(right[:, :, ::-1], left[:, :, ::-1], L, l0=l0, alpha=0.3, tau_c=0.2, tau_g=0.1)[:, :, ::-1]
    assert np.allclose(cr, mir, rtol=0, atol=1e-15)


def _lr_brute(dL, dR, tol):
    H, W = dL.shape
    ok = np.zeros((H, W), bool)
    for y in range(H):
        for x in range(W):
            t = x - int(dL[y, x])
            ok[y, x] = 0 <= t < W and abs(int(dL[y, x]) - int(dR[y, t])) <= tol
    return ok


def _fill_brute(dL, valid):
    H, W = dL.shape
    out = np.array(dL, dtype=np.int64)
    for y in range(H):
        for x in range(W):
            if valid[y, x]:
                continue
            lv = next((int(dL[y, t]) for t in range(x - 1, -1, -1) if valid[y, t]), None)
            rv = next((int(dL[y, t]) for t in range(x + 1, W) if valid[y, t]), None)
            if lv is not None and rv is not None:
                out[y, x] = min(lv, rv)
            elif lv is not None or rv is not None:
                out[y, x] = lv if lv is not None else rv
    return out


def test_lr_consistency_cases():
    """P2: brute force on random maps (tolerance 0 and 1); a constant-disparity pair is consistent exactly
    where the match lies inside the right view (x >= d); a disparity pointing left of column 0 never is."""
    rng = np.random.default_rng(22)
    dL, dR = rng.integers(0, 4, (7, 15)), rng.integers(0, 4, (7, 15))
    for tol in (0, 1, 3):
        assert np.array_equal(O.lr_consistency(dL, dR, tol), _lr_brute(dL, dR, tol))
    assert O.lr_consistency(dL, dR, 3)[:, 3:].all()
    d = np.full((4, 10), 3)
    v = O.lr_consistency(d, d)
    assert not v[:, :3].any() and v[:, 3:].all()
    assert not O.lr_consistency(np.array([[5, 5]]), np.array([[5, 5]]), tol=100).any()


def test_occlusion_fill_cases():
    """P3: hand-worked rows and brute force."""
    X = 0
    d = np.array([[7, X, X, 3, 9, X, 5, X]])
    v = np.array([[1, 0, 0, 1, 1, 0, 1, 0]], bool)
    assert O.occlusion_fill(d, v).tolist() == [[7, 3, 3, 3, 9, 5, 5, 5]]
    assert O.occlusion_fill(np.array([[4, 8, 6]]), np.array([[0, 0, 1]], bool)).tolist() == [[6, 6, 6]]
    assert O.occlusion_fill(np.array([[4, 8, 6]]), np.zeros((1, 3), bool)).tolist() == [[4, 8, 6]]   # no anchor
    rng = np.random.default_rng(23)
    dL = rng.integers(0, 30, (9, 21))
    valid = rng.random((9, 21)) < 0.4
    valid[3] = False
    assert np.array_equal(O.occlusion_fill(dL, valid), _fill_brute(dL, valid))


def test_weighted_median_special_cases():
    """P4: with every weight equal (sigma_s, sigma_c -> inf) the weighted median is the lower median of the
    clipped window, sorted(values)[ceil(n/2) - 1]; a dominant colour class decides alone; consistent pixels
    are unchanged."""
    rng = np.random.default_rng(24)
    H, W, r = 9, 12, 2
    D = rng.integers(0, 20, (H, W))
    valid = rng.random((H, W)) < 0.5
    img = rng.random((3, H, W))
    out = O.weighted_median_fill(D, valid, img, r, 1e12, 1e12)
    for y in range(H):
        for x in range(W):
            if valid[y, x]:
                assert out[y, x] == D[y, x]
                continue
            win = np.sort(D[max(0, y - r):y + r + 1, max(0, x - r):x + r + 1].ravel())
            assert out[y, x] == win[(len(win) + 1) // 2 - 1]
    # two colours: the pixels sharing p's colour carry all the weight at small sigma_c
    img2 = np.zeros((1, H, W))
    img2[0, :, 6:] = 1.0
    D2 = np.where(np.arange(W)[None, :] < 6, 3, 11) + 0 * D
    D2[4, 2] = 11                                     # a wrong value inside the dark region
    v2 = np.ones((H, W), bool)
    v2[4, 2] = False
    out2 = O.weighted_median_fill(D2, v2, img2, 3, 1e12, 0.05)
    assert out2[4, 2] == 3


def test_weighted_median_matches_explicit_sum():
    """P4 against an explicit double loop over the window and an explicit threshold search."""
    rng = np.random.default_rng(25)
    H, W, r, ss, sc = 7, 9, 2, 2.5, 0.3
    D = rng.integers(0, 6, (H, W))
    valid = rng.random((H, W)) < 0.6
    img = rng.random((2, H, W))
    out = O.weighted_median_fill(D, valid, img, r, ss, sc)
    for y in range(H):
        for x in range(W):
            if valid[y, x]:
                continue
            acc = {}
            for qy in range(max(0, y - r), min(H, y + r + 1)):
                for qx in range(max(0, x - r), min(W, x + r + 1)):
                    c2 = sum((img[c, qy, qx] - img[c, y, x]) ** 2 for c in range(2))
                    wq = np.exp(-((qy - y) ** 2 + (qx - x) ** 2) / ss ** 2 - c2 / sc ** 2)
                    acc[int(D[qy, qx])] = acc.get(int(D[qy, qx]), 0.0) + wq
            tot, run, med = sum(acc.values()), 0.0, None
            for d in sorted(acc):
                run += acc[d]
                if run >= 0.5 * tot:
                    med = d
                    break
            assert out[y, x] == med


def test_lr_postprocess_improves_synthetic_stereo():
    """End to end on a synthetic scene: the post-processed map has fewer bad pixels than the raw left map,
    consistent pixels keep their raw disparity, and every output is a disparity of the label range."""
    import synth
    W, H, L = 72, 48, 16
    scene = synth.make_stereo_scene(W, H, L, seed=31)
    dL = O.wta(O.hgf_filter(scene.left, O.stereo_cost(scene.left, scene.right, L), 0.05, 4, 1))
    dR = O.wta(O.hgf_filter(scene.right, O.stereo_cost_right(scene.left, scene.right, L), 0.05, 4, 1))
    final, valid = O.lr_postprocess(scene.left, dL, dR, radius=4, sigma_s=4.0)
    assert np.array_equal(final[valid], dL[valid])
    assert final.min() >= 0 and final.max() < L
    bad_raw = np.mean(np.abs(dL - scene.disp) > 1)
    bad_pp = np.mean(np.abs(final - scene.disp) > 1)
    assert 0.0 < valid.mean() < 1.0 and bad_pp < bad_raw
