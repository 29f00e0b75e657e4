"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This package holds NONE of the method's arithmetic (no box filter, no Gram, no inverse,
no aggregation, no WTA).  It only draws images, disparities and matching costs with the
structure of the paper's workloads (Middlebury-style stereo; cost per
Hosni's framework as written in SPEC S:400).
"""
from .stereo import (  # noqa: F401
    CONFIGS, StereoScene, config, iid_volume, make_lr_maps, make_stereo_scene, stereo_cost_volume_np,
    stereo_cost_volume_torch, smooth_guides,
)
