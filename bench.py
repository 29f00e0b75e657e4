#!/usr/bin/env python
"""Benchmark of the HGF hot path (BASELINE.json metric): cost-volume voxels/s aggregated + WTA.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl own|reference]
Under torchrun (N > 1): one rank per GPU, labels sharded contiguously, statistics replicated (or row-sharded
with HGF_BENCH_STATS=sharded), keys merged by atomic MIN into the row owners over NVLink (or NCCL
allreduce-MIN with HGF_BENCH_MERGE=nccl).  Rank 0 prints ONE JSON line.  A "step" = one pass of the whole hot path over one
synthetic frame: guidance -> float64 statistics -> every label slice filtered -> WTA (-> merge).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cost-volume voxels/sec aggregated+WTA; achieved HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "voxels/s"
SM_COUNT = 148
FP32_LANES = 128
FP64_LANES = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-rows", type=int, default=64)
    ap.add_argument("--cpu-sample-labels", type=int, default=8, help="labels per host core in the CPU baseline")
    return ap.parse_args()


# ----------------------------------------------------------------------------- algorithmic work
def alg_flops_per_voxel(n):
    """Per voxel (fp32): F(n) = 2n^2 + 17n + 13, split by kernel class --
    coef (steps A5 + A6): n products + 4(n+1) stage-1 box adds + (1 + 2n) for m_p and c' + (2n^2 + 2n) matvec
    and h + (2n + 2) w_0 = 2n^2 + 11n + 7 (145 at n = 6); agg (A7 + A8): 4(n+1) stage-2 box adds + (2n + 1) Z
    + 1 WTA = 6n + 6 (42 at n = 6)."""
    return {"coef": 2 * n * n + 11 * n + 7, "agg": 6 * n + 6}


def alg_flops_stats_per_pixel(n):
    """fp64 per pixel: Gram (1 mul + 4 adds per product plane) + Prop-1 recursion."""
    K = n + 1
    gram = 5 * (K * (K + 1) // 2 - 1)
    rec = sum(2 * k * k + 2 * k + 3 * k * k + 2 * k + 6 for k in range(1, K))
    return gram + rec


def alg_bytes(W, H, L, m):
    """HBM bytes the pass must move: the cost volume once, the guide once, the labels once."""
    return 4 * W * H * L + 4 * m * W * H + 4 * W * H


def workload_name(c):
    return (f"{c['name']}: {c['W']}x{c['H']} stereo-like v1, RGB degree-{c['d']} polynomial guidance (n={c['n']}), "
            f"{c['L']} labels, r={c['r']}, lambda={c['lam']}, HGF mode")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle sample
def oracle_sample(scene_left, vol_band_np, c, y0, rows, halo_top):
    """Time the float64 oracle on a row band (with 2r halos) of the workload; returns (voxels, seconds)."""
    import numpy as np

    import oracle as O
    t = time.perf_counter()
    I = scene_left
    Z = O.hgf_filter(I, vol_band_np, c["lam"], c["r"], c["d"])
    lab = np.argmin(Z, axis=0)
    dt = time.perf_counter() - t
    _ = lab[halo_top:halo_top + rows]
    return rows * vol_band_np.shape[2] * vol_band_np.shape[0], dt


def make_band(scene, c, y0, rows, labels):
    import numpy as np

    import synth
    r2 = 2 * c["r"]
    ya, yb = max(0, y0 - r2), min(c["H"], y0 + rows + r2)
    sub = synth.StereoScene(np.ascontiguousarray(scene.left[:, ya:yb]), np.ascontiguousarray(scene.right[:, ya:yb]),
                            scene.disp[ya:yb])
    V = synth.stereo_cost_volume_np(sub, c["L"], 0, labels)
    return sub.left, V, y0 - ya


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_labels_worker(job):
    """One process of the label-parallel CPU baseline: the oracle on a label sub-range of the band."""
    import numpy as np

    import oracle as O
    I, V, lam, r, d = job
    Z = O.hgf_filter(I, V, lam, r, d)
    return Z.min(axis=0), np.argmin(Z, axis=0)


def cpu_baseline(scene, c, rows, labels_per_core, y0=None):
    """The float64 oracle (as it stands) on a bounded sample of the workload, label-parallel over every host core
    the process may use: one process per core, OPENBLAS_NUM_THREADS=1, labels split contiguously,
    per-pixel minima merged; wall time of the whole sample."""
    import multiprocessing as mp

    import numpy as np
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    y0 = c["H"] // 2 if y0 is None else y0
    rows = min(rows, c["H"])
    y0 = min(y0, c["H"] - rows)
    labels = min(c["L"], labels_per_core * cores)
    I, V, halo = make_band(scene, c, y0, rows, labels)
    bounds = np.linspace(0, labels, min(cores, labels) + 1).astype(int)
    jobs = [(I, np.ascontiguousarray(V[a:b]), c["lam"], c["r"], c["d"]) for a, b in zip(bounds[:-1], bounds[1:])
            if b > a]
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mp.get_context("fork")
    t = time.perf_counter()
    with ctx.Pool(len(jobs)) as pool:
        parts = pool.map(_oracle_labels_worker, jobs)
    best = np.full(parts[0][0].shape, np.inf)
    lab = np.zeros(parts[0][0].shape, dtype=np.int64)
    for (mn, am), a in zip(parts, bounds[:-1]):
        upd = mn < best
        best = np.where(upd, mn, best)
        lab = np.where(upd, am + a, lab)
    dt = time.perf_counter() - t
    vox = rows * c["W"] * labels
    return {"value": vox / dt, "unit": UNIT, "cores": len(jobs), "kind": "oracle", "voxels": vox, "seconds": dt,
            "sample": (f"rows {y0}-{y0 + rows - 1} (+{2 * c['r']}-row halos) x {c['W']} cols x labels 0-{labels - 1} "
                       f"of {c['name']}: {vox} voxels in {dt:.2f} s wall, numpy float64, label-parallel over "
                       f"{len(jobs)} processes x 1 thread ({cores} cores available; CPU: {_cpu_model()})")}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, c):
    """The base contract's reference arm for this tier: the float64 oracle as it stands, on the box's host cores
    (label-parallel, as cpu_baseline), each step a bounded sample of the workload (a 16-row band + halos x W x
    8 labels per core; the band start varies per step).  N > 1: rank 0 alone runs it, the other ranks exit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import synth
    scene = synth.make_stereo_scene(c["W"], c["H"], c["L"], c["seed"])
    rows = 16
    vals, last = [], None
    for i in range(args.warmup + args.steps):
        y0 = (i * 97) % max(1, c["H"] - rows)
        cb = cpu_baseline(scene, c, rows, 8, y0=y0)
        if i >= args.warmup:
            vals.append(cb)
        last = cb
    # value = voxels over the summed wall time of the timed steps
    tot_vox = sum(v["voxels"] for v in vals)
    tot_s = sum(v["seconds"] for v in vals)
    value = tot_vox / tot_s
    sample = (f"per step: a {rows}-row band (+{2 * c['r']}-row halos) x {c['W']} cols x (8 labels per core) of "
              f"{c['name']} (band start varies per step); " + last["sample"].split("numpy float64, ")[1])
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / len(vals),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (stereo-like v1, seeded)", "config": config_json(c, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_json(c, n_gpus):
    return {"workload": workload_name(c), "W": c["W"], "H": c["H"], "labels": c["L"], "n_guide": c["m"],
            "poly_degree": c["d"], "n": c["n"], "radius": c["r"], "lambda": c["lam"],
            "parallelism": (f"labels sharded x{n_gpus} (WTA merged by atomic MIN into the row owners over NVLink, "
                            "fallback NCCL allreduce-MIN), statistics " + ("rows sharded (NCCL all-gather)"
                            if os.environ.get("HGF_BENCH_STATS") == "sharded" else "replicated")
                            if n_gpus > 1 else "single GPU"),
            "l2": "inputs larger than L2 (cost volume > 126 MB); no flush needed"}


def stereo_leg(h, scene, L, W, H, args, torch):
    """NEXT-2 (hgf_stereo_wta): the same voxels aggregated + WTA, with the cost slices built on the GPU from
    the two views; device throughput and end to end from pinned host views (only 2 x 3 x H x W floats in)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    left_h = torch.from_numpy(scene.left).pin_memory()
    right_h = torch.from_numpy(scene.right).pin_memory()
    left, right = left_h.to(dev), right_h.to(dev)
    lab = torch.empty((H, W), dtype=torch.int32, device=dev)
    lab_h = torch.empty((H, W), dtype=torch.int32, pin_memory=True)
    for _ in range(max(1, args.warmup)):
        h.stereo_wta(left, right, L, out={"labels": lab})
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        h.stereo_wta(left, right, L, out={"labels": lab})
    e1.record(st)
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / args.steps
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        left.copy_(left_h, non_blocking=True)
        right.copy_(right_h, non_blocking=True)
        h.stereo_wta(left, right, L, out={"labels": lab})
        lab_h.copy_(lab, non_blocking=True)
        torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.e2e_steps
    post = postprocess_leg(h, left, right, lab, L, W, H, args, torch)
    return {"value": W * H * L / (dev_ms / 1e3), "ms_per_step": dev_ms, "unit": UNIT,
            "e2e": {"value": W * H * L / dt, "unit": UNIT, "h2d_bytes_per_step": 2 * left_h.numel() * 4,
                    "d2h_bytes_per_step": lab_h.numel() * 4},
            "api": "hgf_stereo_wta (SURVEY 8(f) NEXT-2: S:400 cost slices built per chunk on the GPU)",
            "postprocess": post}


def postprocess_leg(h, left, right, lab, L, W, H, args, torch):
    """NEXT-3 (hgf_stereo_disparity = left map + right map + readings P2-P4): device ms of the
    whole pipeline per frame, and of hgf_lr_postprocess alone on this frame's two maps (defaults rho = 9,
    sigma_s = 9, sigma_c = 0.1)."""
    dev = left.device
    disp = torch.empty((H, W), dtype=torch.int32, device=dev)
    dR = h.stereo_wta_right(left, right, L)["labels"]
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"disp": disp, "valid": torch.empty((H, W), dtype=torch.uint8, device=dev)}
    for _ in range(3):
        h.lr_postprocess(left, lab, dR, out=out)
    torch.cuda.synchronize()
    reps = 20
    e0.record(st)
    for _ in range(reps):
        h.lr_postprocess(left, lab, dR, out=out)
    e1.record(st)
    torch.cuda.synchronize()
    pp_ms = e0.elapsed_time(e1) / reps
    invalid = 1.0 - float(out["valid"].float().mean())
    steps = max(1, min(args.steps, 5))
    h.stereo_disparity(left, right, L, out={"disp": disp})
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(steps):
        h.stereo_disparity(left, right, L, out={"disp": disp})
    e1.record(st)
    torch.cuda.synchronize()
    return {"pipeline_ms_per_frame": e0.elapsed_time(e1) / steps, "postprocess_ms": pp_ms,
            "inconsistent_fraction": invalid,
            "api": "hgf_stereo_disparity / hgf_lr_postprocess (SURVEY 8(f) NEXT-3)"}


def segment_leg(args, torch):
    """NEXT-4 (hgf_segment): foreground/background labels of a 1920x1080 frame (L = 2, seed-histogram costs
    built on the GPU), the paper's segmentation workload; device ms per frame."""
    import synth
    from paper_1803_00005_b200 import HGF
    W, H = 1920, 1080
    scene = synth.make_stereo_scene(W, H, 8, 3)
    dev = torch.device("cuda", torch.cuda.current_device())
    img = torch.from_numpy(scene.left).to(dev)
    g = torch.Generator(device="cpu").manual_seed(3)
    fg = (torch.rand((H, W), generator=g) < 0.01).to(torch.uint8)
    fg[:, W // 2:] = 0
    bg = (torch.rand((H, W), generator=g) < 0.01).to(torch.uint8)
    bg[:, :W // 2] = 0
    fg, bg = fg.to(dev), bg.to(dev)
    h = HGF(W, H, 3, 2, 9, 0.05)
    lab = torch.empty((H, W), dtype=torch.int32, device=dev)
    for _ in range(max(1, args.warmup)):
        h.segment(img, fg, bg, out={"labels": lab})
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        h.segment(img, fg, bg, out={"labels": lab})
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / args.steps * 1e3
    h.close()
    return {"ms_per_frame": ms, "workload": "1920x1080, RGB degree-2 guidance (n=6), r=9, L=2 (fg/bg), 1% seeds",
            "timing": "wall clock around synchronised calls (hgf_segment reads the seed counts back once)",
            "api": "hgf_segment (SURVEY 8(f) NEXT-4)"}


# ----------------------------------------------------------------------------- own arm
def main():
    args = parse()
    import synth
    c = synth.config(args.config)
    if args.impl == "reference":
        return run_reference(args, c)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1803_00005_b200 import HGF, HGFError, PeerMerge, gather_stats_rows, merge_keys_allreduce, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    W, H, L, m, d, r, lam = c["W"], c["H"], c["L"], c["m"], c["d"], c["r"], c["lam"]
    n = c["n"]
    l0, l1 = shard_range(L, world, rank)
    Ls = l1 - l0
    scene = synth.make_stereo_scene(W, H, L, c["seed"])
    guide = torch.from_numpy(scene.left).to(dev)
    vol = synth.stereo_cost_volume_torch(scene, L, dev, l0, l1)
    torch.cuda.synchronize()
    h = HGF(W, H, m, d, r, lam)
    labels = torch.empty((H, W), dtype=torch.int32, device=dev)
    keys = torch.empty((H, W), dtype=torch.int64, device=dev)
    mincost = torch.empty((H, W), dtype=torch.float32, device=dev)

    # N > 1: slices label-sharded; the label-independent statistics replicated on every rank by default
    # (k_stats4 takes ~1.1 ms at C4, less than an NCCL all-gather of the other ranks' 0.93 GB of statistics
    # rows) or row-sharded + all-gathered (HGF_BENCH_STATS=sharded); WTA merged by the fused peer-memory
    # merge (default) or the NCCL allreduce-MIN of packed keys (HGF_BENCH_MERGE=nccl) -- DESIGN.md §10
    stats_mode = os.environ.get("HGF_BENCH_STATS", "replicated")
    y0, y1 = (0, H) if stats_mode == "replicated" else shard_range(H, world, rank)
    prepared = False
    if world > 1:
        try:
            h.stats_view()
            prepared = True
        except HGFError:
            prepared = False
    row_sharded = prepared and stats_mode != "replicated"
    # fused merge: the aggregation kernel atomicMin's keys into the row owners' buffers over NVLink (CUDA IPC),
    # two owner buffers used alternately, one 4-byte collective per step (PeerMerge)
    peer = None
    if world > 1 and prepared and os.environ.get("HGF_BENCH_MERGE", "peer") == "peer":
        try:
            peer = PeerMerge(h)
        except Exception as ex:   # no peer mapping on this box: the NCCL merge below
            print(f"[bench] peer merge unavailable ({ex}); using allreduce-MIN", file=sys.stderr)
            peer = None
    band_labels = labels[: (peer.y1 - peer.y0)] if peer is not None else None

    def step():
        if world == 1:
            h.aggregate_wta(guide, vol, labels)
        elif peer is not None:
            h.prepare_rows(guide, y0, y1)
            if row_sharded:
                gather_stats_rows(h)
            peer.aggregate(vol, labels, label_offset=l0)
        elif prepared:
            h.prepare_rows(guide, y0, y1)
            if row_sharded:
                gather_stats_rows(h)
            h.aggregate_wta_prepared(vol, label_offset=l0, labels=False, keys=True, out={"keys": keys})
            merge_keys_allreduce(keys)
            h.unpack_keys(keys, labels, mincost)
        else:
            h.aggregate_wta_ex(guide, vol, label_offset=l0, labels=False, keys=True, out={"keys": keys})
            merge_keys_allreduce(keys)
            h.unpack_keys(keys, labels, mincost)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    h.profile_read()
    h.set_profiling(True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    prof = h.profile_read()
    h.set_profiling(False)
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    launches = sum(cnt for _, cnt in prof.values())
    lt = torch.tensor([launches], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
    voxels = W * H * L * args.steps
    value = voxels / (ms_max / 1e3)

    # roofline of the dominant kernel class (largest device time inside the timed region)
    fl = alg_flops_per_voxel(n)
    dom = max(("coef", "agg", "stats"), key=lambda k: prof[k][0])
    dom_ms, dom_cnt = prof[dom]
    if dom in ("coef", "agg"):
        flops_total = fl[dom] * W * H * Ls * args.steps
        peak = SM_COUNT * FP32_LANES * 2 * 1965e6 / 1e12
    else:
        flops_total = alg_flops_stats_per_pixel(n) * W * H * args.steps
        peak = SM_COUNT * FP64_LANES * 2 * 1965e6 / 1e12
    achieved = flops_total / dom_cnt / (dom_ms / dom_cnt / 1e3) / 1e12 if dom_cnt else 0.0
    # dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel, per launch, from the `ncu --set full`
    # capture committed in profiles/ncu_traffic.json -- used only when it was taken of the kernel this handle runs
    # (the file names the kernel and the commit it was captured at)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            ent = tj.get(c["name"], {}).get(dom)
            path_kernels = {"coef": h.kernel_path.split("+")[0], "agg": h.kernel_path.split("+")[1]}
            if isinstance(ent, dict) and (dom == "stats" or ent.get("kernel", "").startswith("k_" + path_kernels[dom])):
                traffic = ent["bytes_per_launch"]
                traffic_src = f"{ent['kernel']} @ {tj.get('_commit', '?')} ({ent.get('labels_per_launch')} labels/launch)"
        except Exception:
            traffic = None
    roofline = {"bound": "alu", "kernel": {"coef": "k_coef", "agg": "k_agg", "stats": "k_stats"}[dom],
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_source": traffic_src, "kernels": h.kernel_path,
                "flops_per_voxel": fl[dom] if dom in ("coef", "agg") else None,
                "peak_basis": ("148 SMs x 128 FP32 lanes x 2 (FMA) x 1965 MHz (B200_PROFILING.md unit counts/clock)"
                               if dom != "stats" else "148 SMs x 64 FP64 lanes x 2 x 1965 MHz"),
                "share_of_step": dom_ms / (ms_max if world == 1 else ms) if ms else None}
    # the pipe that binds the aggregation kernel in this design: the SM's L1/shared-memory data pipe, one 128-byte
    # wavefront per clock per SM (B200_PROFILING.md); ncu's per-launch shared-memory wavefront counts of each slice
    # kernel (profiles/ncu_traffic.json, used only for the kernels this handle runs) over its live launch time
    smem_pipe = None
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            sj = tj.get(c["name"], {})
            wpeak = SM_COUNT * 1965e6 / 1e9
            smem_pipe = {"unit": "G wavefronts/s (128 B each)", "peak": wpeak, "source": tj.get("_commit"),
                         "basis": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum per launch / live launch time; "
                                  "peak 1 wavefront/clk/SM x 148 SMs x 1965 MHz; TMA writes not counted"}
            path_kernels = {"coef": h.kernel_path.split("+")[0], "agg": h.kernel_path.split("+")[1]}
            for k in ("coef", "agg"):
                kms, kcnt = prof[k]
                ent = sj.get(k)
                if isinstance(ent, dict) and ent.get("kernel", "").startswith("k_" + path_kernels[k]) and kcnt:
                    ach = ent["smem_wavefronts_per_launch"] / (kms / kcnt / 1e3) / 1e9
                    smem_pipe[k] = {"kernel": ent["kernel"], "achieved": ach, "frac": ach / wpeak}
        except Exception:
            smem_pipe = None
    stage_ms = {k: v[0] / args.steps for k, v in prof.items()}
    hbm_peak = 6536.0
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    hbm_ach = alg_bytes(W, H, L, m) * args.steps / (ms_max / 1e3) / 1e9

    # e2e through the public API with host buffers
    e2e = None
    stereo = None
    segmentation = None
    if not args.no_e2e:
        if world == 1:
            vol_h = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
            vol_h.copy_(vol)
            guide_h = torch.from_numpy(scene.left).pin_memory()
            lab_h = torch.empty((H, W), dtype=torch.int32, pin_memory=True)
            h.aggregate_wta_host(guide_h, vol_h, lab_h)          # warm-up (allocates staging)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                h.aggregate_wta_host(guide_h, vol_h, lab_h)
            dt = time.perf_counter() - t0
            e2e = {"value": W * H * L * args.e2e_steps / dt, "unit": UNIT,
                   "h2d_bytes_per_step": vol_h.numel() * 4 + guide_h.numel() * 4, "d2h_bytes_per_step": lab_h.numel() * 4,
                   "api": "hgf_aggregate_wta_host (chunked H2D overlapped with compute)"}
            del vol_h
            stereo = stereo_leg(h, scene, L, W, H, args, torch)
            segmentation = segment_leg(args, torch)
        else:
            vol_h = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
            vol_h.copy_(vol)
            guide_h = torch.from_numpy(scene.left).pin_memory()
            lab_h = torch.empty((H, W), dtype=torch.int32, pin_memory=True)

            def e2e_step():
                vol.copy_(vol_h, non_blocking=True)
                guide.copy_(guide_h, non_blocking=True)
                step()
                if peer is not None:          # every rank holds the labels of its own rows
                    lab_h[: peer.y1 - peer.y0].copy_(band_labels, non_blocking=True)
                elif rank == 0:
                    lab_h.copy_(labels, non_blocking=True)
                torch.cuda.synchronize()

            e2e_step()
            barrier()
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                e2e_step()
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            e2e = {"value": W * H * L * args.e2e_steps / float(dt.item()), "unit": UNIT,
                   "h2d_bytes_per_step": 4 * W * H * L + 4 * m * W * H * world, "d2h_bytes_per_step": 4 * W * H,
                   "api": ("torch H2D copies + HGF.prepare_rows (" + ("row band + NCCL all-gather of the "
                           "statistics rows" if row_sharded else "all rows") + ") + " +
                           ("HGF.aggregate_wta_peer (keys atomicMin'd into the row owners over NVLink) + "
                            "HGF.unpack_keys_n" if peer is not None else
                            "HGF.aggregate_wta_prepared + NCCL allreduce-MIN + HGF.unpack_keys")
                           if prepared else
                           "torch H2D copies + HGF.aggregate_wta_ex + NCCL allreduce-MIN + HGF.unpack_keys")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        cpu = cpu_baseline(scene, c, args.cpu_sample_rows, args.cpu_sample_labels)

    # whole-step bound (SURVEY 8(d) "binding roofline"): max(HBM time, fp32 time + fp64 time) of the
    # algorithmic work at the peaks above, against the measured step (all ranks' work / N for N > 1)
    fp32_peak = SM_COUNT * FP32_LANES * 2 * 1965e6
    fp64_peak = SM_COUNT * FP64_LANES * 2 * 1965e6
    t_hbm = alg_bytes(W, H, L, m) / (hbm_peak * 1e9)
    t_alu = (fl["coef"] + fl["agg"]) * W * H * L / fp32_peak + alg_flops_stats_per_pixel(n) * W * H / fp64_peak
    t_bound = max(t_hbm, t_alu) / world
    binding = {"t_bound_ms": 1e3 * t_bound, "t_step_ms": ms_max / args.steps,
               "frac": 1e3 * t_bound / (ms_max / args.steps), "bound": "alu" if t_alu > t_hbm else "hbm",
               "basis": "max(alg bytes / HBM, alg fp32 flops / 74.4 TF + alg fp64 flops / 37.2 TF) per step"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (stereo-like v1 generator, seeded; cost volume built in HBM before timing)",
                "config": config_json(c, world), "roofline": roofline, "smem_pipe": smem_pipe,
                "hbm": {"achieved_gbs": hbm_ach, "peak_gbs": hbm_peak, "frac": hbm_ach / hbm_peak,
                        "alg_bytes_per_step": alg_bytes(W, H, L, m)},
                "binding_roofline": binding,
                "stage_ms_per_step": stage_ms, "cpu_baseline": cpu, "e2e": e2e, "stereo_cost_on_gpu": stereo,
                "segmentation": segmentation,
                "gpu_launches": int(lt.item()), "clocks": clk}
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    h.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
