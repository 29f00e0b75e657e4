"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on the same seeded inputs."""
import os

import numpy as np
import pytest

import oracle as O
import synth
from tests.parity_util import check_labels, check_z

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _hgf(W, H, m, d, r, lam, mode="hgf"):
    from paper_1803_00005_b200 import HGF
    return HGF(W, H, m, d, r, lam, mode=mode)


def _run(I, V, d, r, lam, mode="hgf", label_offset=0):
    torch = _torch()
    m, H, W = I.shape
    h = _hgf(W, H, m, d, r, lam, mode)
    gi = torch.from_numpy(np.ascontiguousarray(I)).cuda()
    gv = torch.from_numpy(np.ascontiguousarray(V)).cuda()
    out = h.aggregate_wta_ex(gi, gv, label_offset=label_offset, labels=True, min_cost=True, filtered=True, keys=True)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["launches"] = h.last_launch_count
    h.close()
    return res


CASES = [
    # (name, W, H, m, d, L, r, lam, mode)
    ("C1-hgf", 64, 48, 3, 1, 8, 2, 1e-3, "hgf"),
    ("C1-gf", 64, 48, 3, 1, 8, 2, 1e-3, "gf"),
    ("ragged-n6", 77, 53, 3, 2, 5, 9, 0.05, "hgf"),
    ("ragged-n9", 45, 70, 3, 3, 4, 9, 0.05, "hgf"),
    ("gray-n1", 40, 33, 1, 1, 3, 4, 0.05, "hgf"),
    ("gray-n3-gf", 40, 33, 1, 3, 3, 3, 0.05, "gf"),
    ("n20", 36, 20, 10, 2, 2, 5, 0.05, "hgf"),
    # k_stats3 with an odd number of Gram pairs (n = 18: 189; n = 15 at r = 16: 135) -- alignment of its buffers
    ("n18-gf", 37, 22, 6, 3, 2, 4, 0.05, "gf"),
    ("n15-r16", 40, 35, 5, 3, 2, 16, 0.05, "hgf"),
    # k_stats3 at the maximum radius (k_stats2's tiles do not fit): odd pair count (n = 11: 77), GF n = 20
    ("n11-r32", 40, 30, 11, 1, 2, 32, 0.05, "hgf"),
    ("n20-r32-gf", 33, 35, 10, 2, 2, 32, 0.05, "gf"),
    ("r16", 50, 41, 3, 2, 3, 16, 0.05, "hgf"),
    ("r32-small-image", 20, 17, 3, 2, 3, 32, 0.05, "hgf"),
    ("one-row", 67, 1, 3, 2, 3, 3, 0.05, "hgf"),
    ("one-pixel", 1, 1, 3, 2, 4, 2, 0.05, "hgf"),
    # degenerate frames on the default kernels: a single column (W % 4 != 0: repacked k_coef5 rows), and 40 labels on
    # one pixel / one column / a 3 x 2 frame (k_agg6's label split over a single tile)
    ("one-column", 1, 67, 3, 2, 3, 3, 0.05, "hgf"),
    ("one-pixel-L40", 1, 1, 3, 2, 40, 9, 0.05, "hgf"),
    ("one-column-L40", 1, 45, 3, 2, 40, 9, 0.05, "gf"),
    ("3x2-L40", 3, 2, 3, 2, 40, 9, 0.05, "hgf"),
    ("L1", 33, 35, 3, 2, 1, 9, 0.05, "hgf"),
    # label-interleaved k_coef3 -> k_agg3 path: two strips + a partial 16-pixel group, a partial 32-label batch
    ("il-n6-L35", 100, 37, 3, 2, 35, 9, 0.05, "hgf"),
    ("il-n6-r4-gf", 132, 29, 3, 2, 33, 4, 0.05, "gf"),
    ("il-n3-r7", 68, 40, 3, 1, 40, 7, 1e-3, "hgf"),
    # k_coef3 with 16-label CTAs and wider statistics records (n = 7..9)
    ("il-n9", 100, 37, 3, 3, 20, 9, 0.05, "hgf"),
    ("il-n8-gf", 132, 29, 4, 2, 17, 4, 0.05, "gf"),
    ("il-n7", 68, 40, 7, 1, 33, 7, 1e-3, "hgf"),
    # raw-guide channels m = 4..6 (degree 1) and m = 4 (degree 2): k_coef3 for L > 2, the planar k_coef2 path for
    # the few-label calls (L <= 2), where round 1 fell back to the generic kernels
    ("m6-d1", 100, 37, 6, 1, 20, 9, 0.05, "hgf"),
    ("m5-d1-L2", 90, 47, 5, 1, 2, 4, 0.05, "gf"),
    ("m4-d2-L1", 77, 41, 4, 2, 1, 7, 0.05, "hgf"),
    ("m4-d2", 68, 40, 4, 2, 33, 7, 0.05, "gf"),
    ("m6-d1-L1-r9", 130, 35, 6, 1, 1, 9, 0.05, "hgf"),
]


@pytest.mark.parametrize("name,W,H,m,d,L,r,lam,mode", CASES, ids=[c[0] for c in CASES])
def test_aggregate_parity(name, W, H, m, d, L, r, lam, mode):
    seed = sum(name.encode()) % 1000                                   # stable across processes
    scene = synth.make_stereo_scene(max(W, 8), max(H, 8), max(L, 2), seed=seed)
    if m == 3:
        I = scene.left[:, :H, :W]
    else:
        I = synth.smooth_guides(W, H, m, seed=7)
    V = synth.stereo_cost_volume_np(scene, max(L, 2))[:L, :H, :W]
    I, V = np.ascontiguousarray(I), np.ascontiguousarray(V)
    res = _run(I, V, d, r, lam, mode)
    Z = O.hgf_filter(I, V, lam, r, d, mode=mode)
    s_v = float(np.abs(V).max())
    check_z(res["filtered"], Z, s_v)
    check_labels(res["labels"], Z, s_v)
    # min cost and keys agree with the filtered slices of the same run (bit-exact)
    lab = res["labels"]
    assert np.array_equal(res["min_cost"], np.take_along_axis(res["filtered"], lab[None].astype(np.int64), 0)[0])
    ku = O.pack_keys(res["min_cost"], lab) ^ np.uint64(1 << 63)
    assert np.array_equal(res["keys"].view(np.uint64), ku)


def test_c2_full_parity():
    """BASELINE config 2 in full: 450x375 Middlebury size, degree-2 RGB (n = 6), 60 labels, r = 9 -- on the
    default k_coef5 -> k_agg6 path (W % 4 != 0: each chunk is repacked into 452-float rows for the TMA)."""
    c = synth.config("C2")
    h = _hgf(c["W"], c["H"], c["m"], c["d"], c["r"], c["lam"])
    assert h.kernel_path == "coef5+agg6", h.kernel_path
    h.close()
    scene = synth.make_stereo_scene(c["W"], c["H"], c["L"], c["seed"])
    V = synth.stereo_cost_volume_np(scene, c["L"])
    res = _run(scene.left, V, c["d"], c["r"], c["lam"])
    Z = O.hgf_filter(scene.left, V, c["lam"], c["r"], c["d"])
    s_v = float(np.abs(V).max())
    check_z(res["filtered"], Z, s_v)
    agree, near = check_labels(res["labels"], Z, s_v)
    assert agree >= 0.9999


def test_iid_stress_parity():
    """'iid' distribution: U[0,1) guide and costs, many near-ties (numerics stress)."""
    I, V = synth.iid_volume(96, 64, 12, 3, seed=11)
    res = _run(I, V, 2, 9, 0.05)
    Z = O.hgf_filter(I, V, 0.05, 9, 2)
    check_z(res["filtered"], Z, 1.0)
    check_labels(res["labels"], Z, 1.0)


def test_filter_entry_point():
    torch = _torch()
    I = synth.smooth_guides(70, 45, 3, seed=3)
    Y = synth.iid_volume(70, 45, 1, 1, seed=4)[1][0]
    h = _hgf(70, 45, 3, 2, 7, 0.05)
    dst = h.filter(torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda())
    torch.cuda.synchronize()
    check_z(dst.cpu().numpy(), O.hgf_filter(I, Y, 0.05, 7, 2), 1.0)
    h.close()


# hgf_filter's fused single-slice pass (k_stats4<n, 1>: the statistics pass also sums the slice's cost products and
# writes its coefficients, then the planar aggregation): ragged frames, degrees 1..3, n up to 9, both modes, against
# the oracle and against the unfused path (HGF_FILTER_FUSED=0: statistics -> k_coef2 -> aggregation).
FILTER1_CASES = [
    # (W, H, m, d, r, mode)
    (133, 71, 3, 2, 9, "hgf"),
    (133, 71, 3, 2, 9, "gf"),
    (96, 50, 1, 1, 4, "hgf"),
    (70, 45, 3, 3, 7, "gf"),
    (64, 97, 2, 2, 1, "hgf"),
    (128, 40, 6, 1, 9, "hgf"),
]


@pytest.mark.parametrize("W,H,m,d,r,mode", FILTER1_CASES)
def test_filter_fused_single_slice(monkeypatch, W, H, m, d, r, mode):
    torch = _torch()
    I = synth.smooth_guides(W, H, m, seed=W + r)
    scene = synth.make_stereo_scene(W, H, 16, seed=H)
    Y = np.ascontiguousarray(synth.stereo_cost_volume_np(scene, 16, 5, 6)[0])
    g, y = torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda()
    out = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("HGF_FILTER_FUSED", fused)
        h = _hgf(W, H, m, d, r, 0.05, mode)
        out[fused] = h.filter(g, y)
        torch.cuda.synchronize()
        launches = h.last_launch_count
        h.close()
        if fused == "1":
            assert launches == 3, launches        # guidance, fused statistics + coefficients, aggregation
    s_v = float(np.abs(Y).max())
    Z = O.hgf_filter(I, Y, 0.05, r, d, mode=mode)
    check_z(out["1"].cpu().numpy(), Z, s_v)
    check_z(out["0"].cpu().numpy(), Z, s_v)


def test_c5_full_frame_fused_filter():
    """BASELINE config 5 at n = 6, r = 9 (RGB, degree 2) in full: every pixel of the 1920x1080 single-slice
    hgf_filter (fused path) against the oracle."""
    torch = _torch()
    c = synth.config("C5")
    W, H, lam = c["W"], c["H"], c["lam"]
    I = synth.smooth_guides(W, H, 3, seed=5)
    scene = synth.make_stereo_scene(W, H, 64, seed=5)
    Y = np.ascontiguousarray(synth.stereo_cost_volume_np(scene, 64, 20, 21)[0])
    h = _hgf(W, H, 3, 2, 9, lam)
    dst = h.filter(torch.from_numpy(I).cuda(), torch.from_numpy(Y).cuda())
    torch.cuda.synchronize()
    assert h.last_launch_count == 3
    h.close()
    check_z(dst.cpu().numpy(), O.hgf_filter(I, Y, lam, 9, 2), float(np.abs(Y).max()))


def test_deterministic_and_label_offset_and_permutation():
    I, V = synth.iid_volume(50, 40, 6, 3, seed=5)
    a = _run(I, V, 2, 4, 0.05)
    b = _run(I, V, 2, 4, 0.05, label_offset=100)
    assert np.array_equal(a["filtered"], b["filtered"])
    assert np.array_equal(a["labels"] + 100, b["labels"])
    perm = np.array([3, 0, 5, 1, 4, 2])
    c = _run(I, np.ascontiguousarray(V[perm]), 2, 4, 0.05)
    assert np.array_equal(c["filtered"], a["filtered"][perm])          # per-slice arithmetic independent of l


@pytest.mark.parametrize("coef3", ["1", "0"])
def test_chunked_equals_single_chunk(monkeypatch, coef3):
    """1 MiB budget: 32-label chunks (the interleaved k_coef3 layout's minimum) or 1-label chunks (planar)."""
    monkeypatch.setenv("HGF_COEF3", coef3)
    I, V = synth.iid_volume(512, 300, 40, 3, seed=6)                   # 4.3 MB of coefficients per label
    a = _run(I, V, 2, 5, 0.05)
    monkeypatch.setenv("HGF_COEF_BUDGET_MB", "1")
    b = _run(I, V, 2, 5, 0.05)
    assert b["launches"] > a["launches"]
    for k in ("filtered", "labels", "min_cost", "keys"):
        assert np.array_equal(a[k], b[k]), k


def test_shard_merge_equals_unsharded():
    """Label sharding: per-shard keys, elementwise int64 MIN == unsharded keys (bit-exact)."""
    torch = _torch()
    from paper_1803_00005_b200 import shard_range
    I, V = synth.iid_volume(48, 36, 11, 3, seed=8)
    full = _run(I, V, 2, 3, 0.05)
    keys = None
    for rank in range(3):
        l0, l1 = shard_range(11, 3, rank)
        part = _run(I, np.ascontiguousarray(V[l0:l1]), 2, 3, 0.05, label_offset=l0)
        keys = part["keys"] if keys is None else np.minimum(keys, part["keys"])
    assert np.array_equal(keys, full["keys"])
    h = _hgf(48, 36, 3, 2, 3, 0.05)
    lab, cost = h.unpack_keys(torch.from_numpy(keys).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(lab.cpu().numpy(), full["labels"])
    assert np.array_equal(cost.cpu().numpy(), full["min_cost"])


@pytest.mark.parametrize("W,H,L", [(40, 30, 7), (160, 90, 100)])
def test_host_entry_point_matches_device(W, H, L):
    """hgf_aggregate_wta_host (pageable host buffers, 32-label staging chunks double-buffered against the compute)
    gives the device path's labels bit for bit, also over several chunks."""
    torch = _torch()
    I, V = synth.iid_volume(W, H, L, 3, seed=9)
    dev = _run(I, V, 2, 3, 0.05)
    h = _hgf(W, H, 3, 2, 3, 0.05)
    lab = h.aggregate_wta_host(torch.from_numpy(I), torch.from_numpy(V))
    assert np.array_equal(lab.numpy(), dev["labels"])


def test_invalid_arguments_fail_loudly():
    torch = _torch()
    from paper_1803_00005_b200 import HGF, HGFError
    with pytest.raises(HGFError):
        HGF(10, 10, 3, 2, 2, 0.0)
    with pytest.raises(HGFError):
        HGF(10, 10, 11, 2, 2, 0.05)          # n = 22 > HGF_MAX_CHANNELS
    h = HGF(10, 10, 3, 2, 2, 0.05)
    with pytest.raises(HGFError):
        h.aggregate_wta(torch.zeros(3, 10, 10, device="cuda"), torch.zeros(2, 10, 11, device="cuda"))


@pytest.mark.parametrize("kernel_env,val", [("HGF_COEF3", "0"), ("HGF_NO_V3", "1"), ("HGF_FORCE_V1", "1"),
                                             ("HGF_COEF4", "1")])
def test_kernel_variants_parity(monkeypatch, kernel_env, val):
    """Every coefficient/aggregation kernel variant against the oracle (k_coef2, v2 flat layout, v1, k_coef4)."""
    monkeypatch.setenv(kernel_env, val)
    c = synth.config("C2")
    scene = synth.make_stereo_scene(c["W"], c["H"], c["L"], c["seed"])
    V = synth.stereo_cost_volume_np(scene, 40)[:, :200, :260].copy()
    I = np.ascontiguousarray(scene.left[:, :200, :260])
    res = _run(I, V, c["d"], c["r"], c["lam"])
    Z = O.hgf_filter(I, V, c["lam"], c["r"], c["d"])
    s_v = float(np.abs(V).max())
    check_z(res["filtered"], Z, s_v)
    check_labels(res["labels"], Z, s_v)


# k_coef4 is an opt-in experiment (slower than the default): two representative cases here, the
# variant sweep above covers it once more at the C2 crop
@pytest.mark.parametrize("r,mode,m,d", [(9, "hgf", 3, 2), (2, "gf", 1, 3)])
def test_coef4_tensor_core_parity(monkeypatch, r, mode, m, d):
    """k_coef4 (tcgen05 horizontal sums): radii 1..9, both modes, n = 1..6, a ragged third strip, 20 labels."""
    monkeypatch.setenv("HGF_COEF4", "1")
    W, H, L = 292, 61, 20
    scene = synth.make_stereo_scene(W, H, L, seed=40 + r)
    I = scene.left if m == 3 else synth.smooth_guides(W, H, m, seed=41)
    V = synth.stereo_cost_volume_np(scene, L)
    res = _run(np.ascontiguousarray(I), V, d, r, 0.05, mode)
    Z = O.hgf_filter(I, V, 0.05, r, d, mode=mode)
    s_v = float(np.abs(V).max())
    check_z(res["filtered"], Z, s_v)
    check_labels(res["labels"], Z, s_v)


@pytest.mark.parametrize("coef4", ["0", "1"])
def test_prepared_row_bands_equal_unsharded(monkeypatch, coef4):
    """Row-sharded statistics (hgf_prepare_rows per band + hgf_aggregate_wta_prepared) == the one-call path,
    bit-exactly; bands of unequal height, as uneven rank counts produce."""
    torch = _torch()
    monkeypatch.setenv("HGF_COEF4", coef4)
    c = synth.config("C2")
    scene = synth.make_stereo_scene(c["W"], c["H"], c["L"], c["seed"])
    V = synth.stereo_cost_volume_np(scene, 40)[:, :200, :260].copy()
    I = np.ascontiguousarray(scene.left[:, :200, :260])
    ref = _run(I, V, c["d"], c["r"], c["lam"])
    h = _hgf(260, 200, 3, c["d"], c["r"], c["lam"], "hgf")
    gi, gv = torch.from_numpy(I).cuda(), torch.from_numpy(V).cuda()
    view = h.stats_view()
    view.fill_(float("nan"))                              # every row must come from some band
    for y0, y1 in ((0, 70), (70, 151), (151, 200)):
        h.prepare_rows(gi, y0, y1)
    out = h.aggregate_wta_prepared(gv, labels=True, min_cost=True, filtered=True, keys=True)
    torch.cuda.synchronize()
    for k in ("filtered", "labels", "min_cost", "keys"):
        assert np.array_equal(out[k].cpu().numpy(), ref[k]), k
    h.close()


def test_prepared_path_unsupported_config_fails_loudly():
    torch = _torch()
    from paper_1803_00005_b200 import HGFError
    h = _hgf(42, 30, 3, 3, 4, 0.05, "hgf")                  # W % 4 != 0, degree 3: planar statistics, no row bands
    assert h.kernel_path == "coef2+agg3"
    with pytest.raises(HGFError):
        h.prepare_rows(torch.zeros(3, 30, 42, device="cuda"), 0, 30)
    with pytest.raises(HGFError):
        h.stats_view()
    h.close()


@pytest.mark.parametrize("W,H,L,label_offset,d,r,mode", [(150, 90, 24, 0, 2, 9, "hgf"), (97, 61, 40, 5, 1, 4, "gf"),
                                                          (64, 48, 8, 0, 1, 2, "hgf"),
                                                          # W % 4 == 0: k_stereo_cost4, two 512-px segments
                                                          (640, 40, 70, 9, 2, 9, "hgf")])
def test_stereo_wta_parity(W, H, L, label_offset, d, r, mode):
    """NEXT-2: cost slices built on the GPU from the two views, then aggregation + WTA, against the
    oracle's own stereo cost filtered by the oracle."""
    torch = _torch()
    scene = synth.make_stereo_scene(W, H, L + label_offset, seed=50 + W)
    h = _hgf(W, H, 3, d, r, 0.05, mode)
    out = h.stereo_wta(torch.from_numpy(scene.left).cuda(), torch.from_numpy(scene.right).cuda(), L,
                       label_offset=label_offset, labels=True, min_cost=True, filtered=True, keys=True)
    torch.cuda.synchronize()
    C = O.stereo_cost(scene.left, scene.right, L, l0=label_offset)
    Z = O.hgf_filter(scene.left, C, 0.05, r, d, mode=mode)
    s_v = float(np.abs(C).max())
    check_z(out["filtered"].cpu().numpy(), Z, s_v)
    lab = out["labels"].cpu().numpy()
    check_labels(lab - label_offset, Z, s_v)
    h.close()


def test_stereo_wta_equals_volume_path():
    """The constructed slices match the workload generator's volume: same labels (off near-ties) and
    filtered costs within fp32 rounding of the cost arithmetic."""
    torch = _torch()
    W, H, L = 200, 120, 48
    scene = synth.make_stereo_scene(W, H, L, seed=61)
    h = _hgf(W, H, 3, 2, 9, 0.05, "hgf")
    gl = torch.from_numpy(scene.left).cuda()
    a = h.stereo_wta(gl, torch.from_numpy(scene.right).cuda(), L, labels=True, filtered=True)
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    b = h.aggregate_wta_ex(gl, vol, labels=True, filtered=True)
    torch.cuda.synchronize()
    fa, fb = a["filtered"].cpu().numpy(), b["filtered"].cpu().numpy()
    s_v = float(vol.abs().max())
    check_z(fa, fb.astype(np.float64), s_v, tol=1e-5)
    assert np.mean(a["labels"].cpu().numpy() == b["labels"].cpu().numpy()) >= 0.9999
    h.close()


def test_stereo_wta_invalid_arguments():
    torch = _torch()
    from paper_1803_00005_b200 import HGFError
    h = _hgf(32, 16, 1, 2, 2, 0.05, "hgf")                 # n_guide = 1: no stereo views
    v = torch.zeros(3, 16, 32, device="cuda")
    with pytest.raises(HGFError):
        h.stereo_wta(v, v, 4)
    h.close()
    h = _hgf(32, 16, 3, 1, 2, 0.05, "hgf")
    with pytest.raises(HGFError):
        h.stereo_wta(v, v, 4, alpha=1.5)
    with pytest.raises(HGFError):
        h.stereo_wta(v, v, 0)
    h.close()


def test_stereo_rectangle_shift_fixture_on_gpu():
    """SPEC S:403 fixture through hgf_stereo_wta: disparity 4 recovered inside the shifted rectangle."""
    torch = _torch()
    H, W, L, s = 24, 48, 8, 4
    rng = np.random.default_rng(7)
    left = np.full((3, H, W), 0.3, dtype=np.float32)
    tex = (0.5 + 0.3 * rng.random((3, 10, 14))).astype(np.float32)
    left[:, 7:17, 20:34] = tex
    right = np.full((3, H, W), 0.3, dtype=np.float32)
    right[:, 7:17, 20 - s:34 - s] = tex
    h = _hgf(W, H, 3, 1, 2, 0.05, "hgf")
    out = h.stereo_wta(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda(), L)
    torch.cuda.synchronize()
    lab = out["labels"].cpu().numpy()
    assert np.all(lab[9:15, 23:31] == s)
    # (no filtered-cost gate here: the exactly uniform background makes the centred Gram vanish, a
    # degenerate guide outside the stereo-like workloads the 1e-4 bound is stated for)
    h.close()


@pytest.mark.parametrize("W,H,d,r,mode", [(96, 64, 2, 5, "hgf"), (61, 47, 1, 3, "gf")])
def test_segment_parity(W, H, d, r, mode):
    """NEXT-4: seed-histogram costs built on the GPU, aggregation + WTA, against the oracle."""
    torch = _torch()
    scene = synth.make_stereo_scene(W, H, 8, seed=70 + W)
    img = np.ascontiguousarray(scene.left)
    rng = np.random.default_rng(W)
    fg = rng.random((H, W)) < 0.02
    bg = rng.random((H, W)) < 0.02
    fg[:, : W // 3] |= rng.random((H, W // 3)) < 0.05               # some structure in the seed colours
    h = _hgf(W, H, 3, d, r, 0.05, mode)
    out = h.segment(torch.from_numpy(img).cuda(), torch.from_numpy(fg).cuda(), torch.from_numpy(bg).cuda(),
                    labels=True, min_cost=True, filtered=True)
    torch.cuda.synchronize()
    C = O.segmentation_cost(img, fg, bg)
    Z = O.hgf_filter(img, C, 0.05, r, d, mode=mode)
    s_v = float(np.abs(C).max())
    check_z(out["filtered"].cpu().numpy(), Z, s_v)
    check_labels(out["labels"].cpu().numpy(), Z, s_v)
    h.close()


def test_segment_two_colour_fixture_and_empty_seeds():
    torch = _torch()
    from paper_1803_00005_b200 import HGFError
    H, W = 20, 30
    img = np.empty((3, H, W), np.float32)
    img[:] = np.array([0.9, 0.2, 0.1], np.float32)[:, None, None]
    img[:, :, 15:] = np.array([0.1, 0.3, 0.8], np.float32)[:, None, None]
    fg = np.zeros((H, W), np.uint8)
    bg = np.zeros((H, W), np.uint8)
    fg[10, 5] = 1
    bg[10, 25] = 1
    h = _hgf(W, H, 3, 1, 2, 0.05, "hgf")
    gi = torch.from_numpy(img).cuda()
    lab = h.segment(gi, torch.from_numpy(fg).cuda(), torch.from_numpy(bg).cuda())["labels"].cpu().numpy()
    assert np.all(lab[:, :12] == 0) and np.all(lab[:, 18:] == 1)
    with pytest.raises(HGFError):
        h.segment(gi, torch.from_numpy(fg).cuda(), torch.zeros(H, W, dtype=torch.uint8, device="cuda"))
    h.close()


def test_peer_merge_equals_allreduce_merge():
    """Fused WTA merge over peer memory (hgf_aggregate_wta_peer): two label shards x two row owners, run in
    one process (the owners are plain device buffers here; across processes they are CUDA-IPC mappings):
    the owners' rows are bit-exactly the unsharded keys, and unpack to the unsharded labels."""
    torch = _torch()
    from paper_1803_00005_b200 import PeerKeys, shard_range
    W, H, L = 180, 77, 30
    scene = synth.make_stereo_scene(W, H, L, seed=91)
    gi = torch.from_numpy(scene.left).cuda()
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    h = _hgf(W, H, 3, 2, 9, 0.05, "hgf")
    ref = h.aggregate_wta_ex(gi, vol, labels=True, keys=True)
    # world = 1 through PeerKeys (no IPC)
    pk = PeerKeys(h)
    pk.reset()
    h.prepare_rows(gi, 0, H)
    h.aggregate_wta_peer(vol, pk.ptrs, 1, pk.rows)
    torch.cuda.synchronize()
    assert torch.equal(pk.keys, ref["keys"])
    lab = torch.empty((H, W), dtype=torch.int32, device="cuda")
    h.unpack_keys_n(pk.keys, lab)
    assert torch.equal(lab, ref["labels"])
    pk.close()
    # two owners (rows split) x two label shards
    R = (H + 1) // 2
    owners = [torch.empty((R, W), dtype=torch.int64, device="cuda") for _ in range(2)]
    for o in owners:
        h.fill_keys(o)
    ptrs = torch.tensor([o.data_ptr() for o in owners], dtype=torch.int64, device="cuda")
    for rank in range(2):
        l0, l1 = shard_range(L, 2, rank)
        h.aggregate_wta_peer(vol[l0:l1].contiguous(), ptrs, 2, R, label_offset=l0)
    torch.cuda.synchronize()
    merged = torch.cat(owners)[:H]
    assert torch.equal(merged, ref["keys"])
    h.close()


def test_peer_merge_with_label_split():
    """The fused merge on a small frame with >= 32 labels, where k_agg6 splits each tile's labels over several CTAs
    (k_keys_finalize then does the system-scope MIN into the owners): the owner rows equal the one-call keys."""
    torch = _torch()
    from paper_1803_00005_b200 import PeerKeys
    W, H, L = 180, 77, 80
    scene = synth.make_stereo_scene(W, H, L, seed=92)
    gi = torch.from_numpy(scene.left).cuda()
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    h = _hgf(W, H, 3, 2, 9, 0.05, "hgf")
    ref = h.aggregate_wta_ex(gi, vol, labels=True, keys=True)
    pk = PeerKeys(h)
    pk.reset()
    h.prepare_rows(gi, 0, H)
    h.aggregate_wta_peer(vol, pk.ptrs, 1, pk.rows)
    torch.cuda.synchronize()
    assert torch.equal(pk.keys, ref["keys"])
    pk.close()
    h.close()


def test_peer_merge_double_buffered_steps():
    """PeerMerge (the bench's N > 1 step): alternating owner buffers over several steps whose volumes differ,
    each step's labels equal to the one-call path's (a stale buffer would leak the previous step's minima)."""
    torch = _torch()
    from paper_1803_00005_b200 import PeerMerge
    W, H, L = 152, 61, 20          # the prepared (per-pixel statistics) path needs W % 4 == 0
    scene = synth.make_stereo_scene(W, H, L, seed=17)
    gi = torch.from_numpy(scene.left).cuda()
    base = synth.stereo_cost_volume_torch(scene, L, "cuda")
    h = _hgf(W, H, 3, 2, 9, 0.05, "hgf")
    pm = PeerMerge(h)
    lab = torch.empty((H, W), dtype=torch.int32, device="cuda")
    h.prepare_rows(gi, 0, H)
    for s in range(5):
        # step s: labels permuted and costs raised, so every step has a different WTA map and larger minima
        perm = torch.roll(torch.arange(L, device="cuda"), s * 3)
        vol = (base[perm] + 0.01 * s).contiguous()
        ref = h.aggregate_wta_ex(gi, vol, labels=True)["labels"]
        h.prepare_rows(gi, 0, H)
        pm.aggregate(vol, lab)
        torch.cuda.synchronize()
        assert torch.equal(lab, ref), s
    assert pm.steps == 5
    pm.close()
    h.close()


@pytest.mark.parametrize("promo", ["none", "64", "256"])
def test_tma_l2_promotion_knob_is_bit_identical(promo, monkeypatch):
    """HGF_TMA_L2PROMO only changes the cache policy of k_agg3's coefficient-tile loads: the filtered costs
    and labels are bit-identical to the default (128-byte promotion) on the interleaved k_coef3 -> k_agg3
    path (W multiple of 16, n = 6, r = 9, 40 labels: two 32-label groups, a ragged one)."""
    torch = _torch()
    W, H, L = 208, 72, 40
    scene = synth.make_stereo_scene(W, H, L, seed=77)
    g = torch.from_numpy(scene.left).cuda()
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    monkeypatch.setenv("HGF_AGG6", "0")        # the knob applies to k_agg3's maps
    monkeypatch.delenv("HGF_TMA_L2PROMO", raising=False)
    h = _hgf(W, H, 3, 2, 9, 0.05, "hgf")
    a = h.aggregate_wta_ex(g, vol, labels=True, filtered=True)
    torch.cuda.synchronize()
    h.close()
    monkeypatch.setenv("HGF_TMA_L2PROMO", promo)
    h = _hgf(W, H, 3, 2, 9, 0.05, "hgf")
    b = h.aggregate_wta_ex(g, vol, labels=True, filtered=True)
    torch.cuda.synchronize()
    h.close()
    assert torch.equal(a["filtered"], b["filtered"])
    assert torch.equal(a["labels"], b["labels"])


# Full frames on the default slice path at the geometry bench.py runs (verdict r01 item 2b): >= 3 strips, >= 3 row
# bands, >= 2 label batches, and the C4 band length (270 rows: the fp32 running window sums of a band march 288
# steps without a restart), with the stereo-like and the iid near-tie distributions; k_coef3 at the same band length.
BAND_CASES = [
    # (name, W, H, L, distribution, env, expected kernel path)
    ("coef5-3strips-3bands-2batches", 300, 560, 40, "stereo", {"HGF_COEF5_BH": "270"}, "coef5+agg6"),
    ("coef5-iid-band270", 260, 560, 34, "iid", {"HGF_COEF5_BH": "270"}, "coef5+agg6"),
    # k_agg3 (HGF_AGG6=0) on the same interleaved layout
    ("coef5-agg3-band270", 300, 560, 40, "stereo", {"HGF_COEF5_BH": "270", "HGF_AGG6": "0"}, "coef5+agg3"),
    # the opt-in row-marching aggregation (k_agg5) at its band length: 3 bands x 2 label groups
    ("coef5-agg5", 300, 560, 40, "stereo", {"HGF_COEF5_BH": "270", "HGF_AGG5": "1", "HGF_AGG5_BH": "270"},
     "coef5+agg5"),
    ("coef3-band270", 300, 560, 40, "stereo", {"HGF_COEF5": "0", "HGF_COEF3_BH": "270"}, "coef3+agg6"),
    # W % 4 != 0 on k_coef5 (repacked rows; odd width: the guide pairs' own pitch), 3 strips
    ("coef5-odd-width", 301, 140, 40, "stereo", {}, "coef5+agg6"),
]


@pytest.mark.parametrize("name,W,H,L,dist,env,path", BAND_CASES, ids=[c[0] for c in BAND_CASES])
def test_full_frame_band_geometry(monkeypatch, name, W, H, L, dist, env, path):
    torch = _torch()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    if dist == "stereo":
        scene = synth.make_stereo_scene(W, H, L, seed=300 + L)
        I, V = scene.left, synth.stereo_cost_volume_np(scene, L)
    else:
        I, V = synth.iid_volume(W, H, L, 3, seed=301)
    I, V = np.ascontiguousarray(I), np.ascontiguousarray(V)
    h = _hgf(W, H, 3, 2, 9, 0.05)
    assert h.kernel_path == path
    out = h.aggregate_wta_ex(torch.from_numpy(I).cuda(), torch.from_numpy(V).cuda(), labels=True, min_cost=True,
                             filtered=True)
    torch.cuda.synchronize()
    h.close()
    Z = O.hgf_filter(I, V, 0.05, 9, 2)
    s_v = float(np.abs(V).max())
    check_z(out["filtered"].cpu().numpy(), Z, s_v)
    check_labels(out["labels"].cpu().numpy(), Z, s_v)


def test_default_kernel_path_is_coef5():
    """The headline configs (RGB degree 2, r = 9, W % 4 == 0 or not) run k_coef5 -> k_agg6 by default."""
    for W, H in ((3840, 2160), (1920, 1080), (452, 375), (450, 375), (451, 77)):
        h = _hgf(W, H, 3, 2, 9, 0.05)
        assert h.kernel_path == "coef5+agg6", (W, H, h.kernel_path)
        h.close()


def test_shard_merge_against_oracle():
    """A9 (label-sharded WTA merge, north_star (4)): three contiguous label shards, each through
    hgf_aggregate_wta_ex(label_offset, keys), merged by elementwise int64 MIN and unpacked -- labels and
    minimum cost against the ORACLE's argmin / min over the whole volume (not only against the unsharded run)."""
    torch = _torch()
    from paper_1803_00005_b200 import shard_range
    W, H, L = 180, 77, 30
    scene = synth.make_stereo_scene(W, H, L, seed=93)
    V = synth.stereo_cost_volume_np(scene, L)
    gi = torch.from_numpy(scene.left).cuda()
    h = _hgf(W, H, 3, 2, 9, 0.05)
    keys = None
    for rank in range(3):
        l0, l1 = shard_range(L, 3, rank)
        part = h.aggregate_wta_ex(gi, torch.from_numpy(np.ascontiguousarray(V[l0:l1])).cuda(), label_offset=l0,
                                  keys=True)["keys"]
        keys = part if keys is None else torch.minimum(keys, part)
    lab, cost = h.unpack_keys(keys)
    # the same merge through the fused peer-memory path (two owners x two shards, one process)
    R = (H + 1) // 2
    owners = [torch.empty((R, W), dtype=torch.int64, device="cuda") for _ in range(2)]
    for o in owners:
        h.fill_keys(o)
    ptrs = torch.tensor([o.data_ptr() for o in owners], dtype=torch.int64, device="cuda")
    h.prepare_rows(gi, 0, H)
    vol = torch.from_numpy(V).cuda()
    for rank in range(2):
        l0, l1 = shard_range(L, 2, rank)
        h.aggregate_wta_peer(vol[l0:l1].contiguous(), ptrs, 2, R, label_offset=l0)
    torch.cuda.synchronize()
    peer_keys = torch.cat(owners)[:H]
    h.close()
    Z = O.hgf_filter(scene.left, V, 0.05, 9, 2)
    s_v = float(np.abs(V).max())
    check_labels(lab.cpu().numpy(), Z, s_v)
    check_z(cost.cpu().numpy(), Z.min(axis=0), s_v)
    assert torch.equal(peer_keys, keys)


def test_two_stream_chunk_pipeline_bit_identical(monkeypatch):
    """HGF_PIPELINE=1 (coefficients of chunk c + 1 on the handle stream while chunk c is aggregated on an aux stream,
    the coefficient buffer split in two halves): bit-identical to the sequential chunk loop, incl. the fused merge."""
    torch = _torch()
    W, H, L = 208, 72, 150
    scene = synth.make_stereo_scene(W, H, L, seed=78)
    g = torch.from_numpy(scene.left).cuda()
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    monkeypatch.setenv("HGF_COEF_BUDGET_MB", str(64 * 7 * 4 * H * W // (1 << 20) + 1))   # 64 labels per chunk
    outs = []
    for pipe in ("0", "1"):
        monkeypatch.setenv("HGF_PIPELINE", pipe)
        h = _hgf(W, H, 3, 2, 9, 0.05)
        o = h.aggregate_wta_ex(g, vol, labels=True, min_cost=True, filtered=True, keys=True)
        torch.cuda.synchronize()
        outs.append(o)
        h.close()
    for k in ("labels", "min_cost", "filtered", "keys"):
        assert torch.equal(outs[0][k], outs[1][k]), k


@pytest.mark.parametrize("m,d,L,path", [(3, 2, 1, "small"), (3, 2, 2, "small"), (3, 2, 3, "main"), (6, 1, 1, "small")])
def test_few_label_path_matches_main_path_and_oracle(monkeypatch, m, d, L, path):
    """Few-label calls (L <= 2: hgf_filter, segmentation) run k_coef2 on planar statistics + the planar k_agg3; the
    result agrees with the oracle and, within fp32 rounding, with the lane-per-label main path (HGF_SMALL_L=0)."""
    W, H = 150, 61
    scene = synth.make_stereo_scene(W, H, max(L, 2), seed=31 * m + L)
    I = scene.left if m == 3 else synth.smooth_guides(W, H, m, seed=8)
    V = synth.stereo_cost_volume_np(scene, max(L, 2))[:L]
    a = _run(np.ascontiguousarray(I), np.ascontiguousarray(V), d, 9, 0.05)
    monkeypatch.setenv("HGF_SMALL_L", "0")
    b = _run(np.ascontiguousarray(I), np.ascontiguousarray(V), d, 9, 0.05)
    Z = O.hgf_filter(I, V, 0.05, 9, d)
    s_v = float(np.abs(V).max())
    check_z(a["filtered"], Z, s_v)
    check_z(b["filtered"], Z, s_v)
    check_labels(a["labels"], Z, s_v)
    assert np.abs(a["filtered"] - b["filtered"]).max() <= 1e-4 * max(s_v, 1e-30)


# k_agg6 (warp-specialised, per-plane pipeline; 8-pixel owners holding the guidance planes or 16-pixel owners
# holding the raw channels) performs k_agg3's arithmetic in the same order: bit-identical filtered costs, labels,
# minimum costs and keys, over ragged tiles, several 32-label groups, multi-chunk WTA carries (small
# HGF_COEF_BUDGET_MB), degrees 1..3 and radii 1..9; k_agg6 also against the oracle on the smaller cases.
AGG6_CASES = [
    # (W, H, L, m, d, r, budget MB, owner width: "16" = raw-channel owners where m <= 3, "8" = HGF_AGG6_KX=8)
    (208, 72, 40, 3, 2, 9, None, "16"),
    (208, 72, 40, 3, 2, 9, None, "8"),
    (301, 101, 70, 3, 2, 9, "1", "16"),
    (77, 53, 5, 3, 2, 9, None, "16"),
    (160, 97, 33, 1, 2, 4, None, "16"),
    (96, 130, 12, 2, 3, 1, None, "16"),
    (112, 80, 7, 3, 1, 6, None, "16"),
    (128, 64, 9, 6, 1, 7, None, "8"),
]


@pytest.mark.parametrize("W,H,L,m,d,r,budget,kx", AGG6_CASES)
def test_agg6_bit_identical_to_agg3(monkeypatch, W, H, L, m, d, r, budget, kx):
    torch = _torch()
    scene = synth.make_stereo_scene(W, H, L, seed=W + L)
    I = np.ascontiguousarray(synth.smooth_guides(W, H, m, seed=W)) if m != 3 else scene.left
    g = torch.from_numpy(I).cuda()
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    if kx == "8":
        monkeypatch.setenv("HGF_AGG6_KX", "8")
    if budget:
        monkeypatch.setenv("HGF_COEF_BUDGET_MB", budget)
    out = {}
    for agg6 in ("1", "0"):
        monkeypatch.setenv("HGF_AGG6", agg6)
        h = _hgf(W, H, m, d, r, 0.05)
        assert h.kernel_path.endswith("+agg6" if agg6 == "1" else "+agg3"), h.kernel_path
        o = h.aggregate_wta_ex(g, vol, labels=True, min_cost=True, keys=True, filtered=True)
        torch.cuda.synchronize()
        out[agg6] = {k: v.cpu().numpy() for k, v in o.items()}
        h.close()
    a, b = out["1"], out["0"]
    for k in ("filtered", "labels", "min_cost", "keys"):
        assert np.array_equal(a[k], b[k]), k
    if W * H * L <= 208 * 72 * 40:
        V = synth.stereo_cost_volume_np(scene, L)
        Z = O.hgf_filter(I, V, 0.05, r, d)
        check_z(a["filtered"], Z, float(np.abs(V).max()))
        check_labels(a["labels"], Z, float(np.abs(V).max()))


@pytest.mark.parametrize("W,H,L,budget", [(300, 140, 40, None), (450, 375, 60, None), (208, 72, 100, "1")])
def test_agg6_label_split_bit_identical(monkeypatch, W, H, L, budget):
    """Small frames (fewer k_agg6 tiles than ~1.5 waves) split each tile's labels over several CTAs merged by 64-bit
    atomic MIN keys: labels, minimum cost, keys and filtered costs equal the unsplit run bit for bit (ties keep the
    lowest label through the key's low word), also across coefficient-buffer chunks."""
    torch = _torch()
    scene = synth.make_stereo_scene(W, H, L, seed=L)
    g = torch.from_numpy(scene.left).cuda()
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    if budget:
        monkeypatch.setenv("HGF_COEF_BUDGET_MB", budget)
    out = {}
    for split in ("1", "0"):
        monkeypatch.setenv("HGF_AGG6_SPLIT", split)
        h = _hgf(W, H, 3, 2, 9, 0.05)
        assert h.kernel_path == "coef5+agg6"
        o = h.aggregate_wta_ex(g, vol, labels=True, min_cost=True, keys=True, filtered=True)
        torch.cuda.synchronize()
        out[split] = {k: v.cpu().numpy() for k, v in o.items()}
        h.close()
    for k in ("filtered", "labels", "min_cost", "keys"):
        assert np.array_equal(out["1"][k], out["0"][k]), k


@pytest.mark.parametrize("W,H,L,m,d,r", [(300, 140, 40, 3, 2, 9), (133, 71, 9, 2, 3, 4), (90, 200, 5, 1, 1, 16)])
def test_stats5_bit_identical_to_stats4(monkeypatch, W, H, L, m, d, r):
    """k_stats5 (warp-specialised statistics pass: vertical / horizontal / recursion warps pipelined through
    mbarriers) performs k_stats4's arithmetic in k_stats4's order: the aggregated results are bit-identical
    (HGF_STATS5=0 runs k_stats4)."""
    torch = _torch()
    scene = synth.make_stereo_scene(W, H, L, seed=W)
    I = np.ascontiguousarray(synth.smooth_guides(W, H, m, seed=W)) if m != 3 else scene.left
    g = torch.from_numpy(I).cuda()
    vol = synth.stereo_cost_volume_torch(scene, L, "cuda")
    out = {}
    for s5 in ("1", "0"):
        monkeypatch.setenv("HGF_STATS5", s5)         # 1: k_stats5 also for the statistics pass
        h = _hgf(W, H, m, d, r, 0.05)
        o = h.aggregate_wta_ex(g, vol, labels=True, filtered=True)
        torch.cuda.synchronize()
        out[s5] = {k: v.cpu().numpy() for k, v in o.items()}
        h.close()
    for k in ("filtered", "labels"):
        assert np.array_equal(out["1"][k], out["0"][k]), k
