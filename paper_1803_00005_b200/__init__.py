"""B200-native Hardware-Efficient Guided Filter (HGF) hot path: Python binding of libhgf.so.

Thin ctypes marshalling over the C ABI in ``include/hgf.h`` (same names).  PyTorch supplies
device memory, streams and process groups; every step of the path runs in the library's
CUDA kernels.  There is no CPU fallback: if the shared library is missing or no CUDA device is
present, constructing :class:`HGF` raises.
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["HGF", "HGFError", "lib", "lib_path", "MODE_HGF", "MODE_GF", "EXPORTED_SYMBOLS",
           "merge_keys_allreduce", "shard_range", "gather_stats_rows", "PeerKeys", "PeerMerge"]

MODE_HGF = 0
MODE_GF = 1
_HERE = os.path.dirname(os.path.abspath(__file__))
# HGF_LIB_PATH: an alternate build of the same library (A/B timing builds only; still the CUDA path)
lib_path = os.environ.get("HGF_LIB_PATH") or os.path.join(_HERE, "libhgf.so")

# Every entry point declared in include/hgf.h (tests check the .so exports all of them).
EXPORTED_SYMBOLS = (
    "hgf_create", "hgf_create_ex", "hgf_destroy", "hgf_set_stream", "hgf_filter",
    "hgf_aggregate_wta", "hgf_aggregate_wta_ex", "hgf_unpack_keys", "hgf_aggregate_wta_host",
    "hgf_last_launch_count", "hgf_status_string", "hgf_last_error", "hgf_set_profiling", "hgf_profile_read",
    "hgf_prepare_rows", "hgf_stats_buffer", "hgf_aggregate_wta_prepared", "hgf_stereo_wta", "hgf_segment",
    "hgf_aggregate_wta_peer", "hgf_fill_keys", "hgf_unpack_keys_n", "hgf_alloc", "hgf_free", "hgf_ipc_get_handle",
    "hgf_ipc_open", "hgf_ipc_close", "hgf_stereo_wta_right", "hgf_lr_postprocess", "hgf_stereo_disparity",
    "hgf_kernel_path",
)
KERNEL_CLASSES = ("guidance", "stats", "coef", "agg", "keys", "cost", "post")   # HGF_KC_* order

_lib = None


class HGFError(RuntimeError):
    pass


def lib():
    """Load libhgf.so (built by ``make`` / ``__graft_entry__.build()``); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise ImportError(f"{lib_path} not built: run `make -j8` (or __graft_entry__.build()); no CPU fallback")
    L = ctypes.CDLL(lib_path)
    c_int, c_double, vp = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
    L.hgf_create.argtypes = [ctypes.POINTER(vp), c_int, c_int, c_int, c_int, c_int, c_double]
    L.hgf_create_ex.argtypes = [ctypes.POINTER(vp), c_int, c_int, c_int, c_int, c_int, c_double, c_int, vp]
    L.hgf_destroy.argtypes = [vp]
    L.hgf_set_stream.argtypes = [vp, vp]
    L.hgf_filter.argtypes = [vp, vp, vp, vp]
    L.hgf_aggregate_wta.argtypes = [vp, vp, vp, c_int, vp]
    L.hgf_aggregate_wta_ex.argtypes = [vp, vp, vp, c_int, c_int, vp, vp, vp, vp]
    L.hgf_unpack_keys.argtypes = [vp, vp, vp, vp]
    L.hgf_aggregate_wta_host.argtypes = [vp, vp, vp, c_int, vp]
    L.hgf_last_launch_count.argtypes = [vp]
    L.hgf_last_launch_count.restype = c_int
    L.hgf_kernel_path.argtypes = [vp]
    L.hgf_kernel_path.restype = ctypes.c_char_p
    L.hgf_status_string.argtypes = [c_int]
    L.hgf_status_string.restype = ctypes.c_char_p
    L.hgf_last_error.argtypes = [vp]
    L.hgf_last_error.restype = ctypes.c_char_p
    L.hgf_set_profiling.argtypes = [vp, c_int]
    L.hgf_set_profiling.restype = c_int
    L.hgf_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_int), c_int]
    L.hgf_profile_read.restype = c_int
    L.hgf_prepare_rows.argtypes = [vp, vp, c_int, c_int]
    L.hgf_stats_buffer.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t)]
    L.hgf_aggregate_wta_prepared.argtypes = [vp, vp, c_int, c_int, vp, vp, vp, vp]
    c_float = ctypes.c_float
    L.hgf_stereo_wta.argtypes = [vp, vp, vp, c_int, c_int, c_float, c_float, c_float, vp, vp, vp, vp]
    L.hgf_stereo_wta_right.argtypes = [vp, vp, vp, c_int, c_int, c_float, c_float, c_float, vp, vp, vp, vp]
    L.hgf_lr_postprocess.argtypes = [vp, vp, vp, vp, c_int, c_int, c_float, c_float, vp, vp]
    L.hgf_stereo_disparity.argtypes = [vp, vp, vp, c_int, c_int, c_float, c_float, c_float, c_int, c_int, c_float,
                                       c_float, vp, vp, vp, vp]
    L.hgf_segment.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.hgf_aggregate_wta_peer.argtypes = [vp, vp, c_int, c_int, vp, c_int, c_int]
    L.hgf_fill_keys.argtypes = [vp, vp, ctypes.c_longlong]
    L.hgf_unpack_keys_n.argtypes = [vp, vp, ctypes.c_longlong, vp, vp]
    L.hgf_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(vp)]
    L.hgf_free.argtypes = [vp]
    L.hgf_ipc_get_handle.argtypes = [vp, ctypes.c_char_p]
    L.hgf_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.hgf_ipc_close.argtypes = [vp]
    for name in ("hgf_create", "hgf_create_ex", "hgf_destroy", "hgf_set_stream", "hgf_filter", "hgf_aggregate_wta",
                 "hgf_aggregate_wta_ex", "hgf_unpack_keys", "hgf_aggregate_wta_host", "hgf_prepare_rows",
                 "hgf_stats_buffer", "hgf_aggregate_wta_prepared", "hgf_stereo_wta", "hgf_segment",
                 "hgf_aggregate_wta_peer", "hgf_fill_keys", "hgf_unpack_keys_n", "hgf_alloc", "hgf_free",
                 "hgf_ipc_get_handle", "hgf_ipc_open", "hgf_ipc_close"):
        getattr(L, name).restype = c_int
    _lib = L
    return L


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class HGF:
    """Handle over ``hgf_create_ex``: W x H images, raw guide with ``n_guide`` channels, polynomial
    degree ``poly_degree`` (n = n_guide * poly_degree, §4.2), radius r, eps = lambda,
    mode ``"hgf"`` (Eq7) or ``"gf"`` (§5.1 Eq15/16)."""

    def __init__(self, W, H, n_guide, poly_degree, radius, eps, mode="hgf", device=None):
        import torch
        if not torch.cuda.is_available():
            raise HGFError("HGF needs a CUDA device (no CPU fallback)")
        self._torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.W, self.H, self.m, self.d, self.r, self.eps = W, H, n_guide, poly_degree, radius, eps
        self.n = n_guide * poly_degree
        self.mode = {"hgf": MODE_HGF, "gf": MODE_GF}[mode] if isinstance(mode, str) else int(mode)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            st = lib().hgf_create_ex(ctypes.byref(h), W, H, n_guide, poly_degree, radius, float(eps), self.mode,
                                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        if st != 0:
            raise HGFError(f"hgf_create_ex: {lib().hgf_status_string(st).decode()}")
        self._h = h

    # ------------------------------------------------------------------ helpers
    def _check(self, st, what):
        if st != 0:
            raise HGFError(f"{what}: {lib().hgf_status_string(st).decode()}: {lib().hgf_last_error(self._h).decode()}")

    def _bind_stream(self):
        s = self._torch.cuda.current_stream(self.device).cuda_stream
        self._check(lib().hgf_set_stream(self._h, ctypes.c_void_p(s)), "hgf_set_stream")

    def _dev(self, t, shape, dtype, name):
        torch = self._torch
        if not isinstance(t, torch.Tensor) or t.device != self.device or t.dtype != dtype or not t.is_contiguous():
            raise HGFError(f"{name} must be a contiguous {dtype} tensor on {self.device}")
        if tuple(t.shape) != tuple(shape):
            raise HGFError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
        return t

    def set_profiling(self, enable=True):
        self._check(lib().hgf_set_profiling(self._h, 1 if enable else 0), "hgf_set_profiling")

    def profile_read(self):
        """{class: (ms, launches)} accumulated since the previous read (synchronises the stream)."""
        n = len(KERNEL_CLASSES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int * n)()
        self._bind_stream()
        self._check(lib().hgf_profile_read(self._h, ms, cnt, n), "hgf_profile_read")
        return {k: (ms[i], cnt[i]) for i, k in enumerate(KERNEL_CLASSES)}

    @property
    def last_launch_count(self):
        return lib().hgf_last_launch_count(self._h)

    @property
    def kernel_path(self):
        """The slice kernels this handle runs (hgf_kernel_path), e.g. "coef5+agg6"."""
        return lib().hgf_kernel_path(self._h).decode()

    # ------------------------------------------------------------------ API (names as in hgf.h)
    def filter(self, guide, src, dst=None):
        torch = self._torch
        self._dev(guide, (self.m, self.H, self.W), torch.float32, "guide")
        self._dev(src, (self.H, self.W), torch.float32, "src")
        if dst is None:
            dst = torch.empty((self.H, self.W), dtype=torch.float32, device=self.device)
        self._dev(dst, (self.H, self.W), torch.float32, "dst")
        self._bind_stream()
        self._check(lib().hgf_filter(self._h, _ptr(guide), _ptr(src), _ptr(dst)), "hgf_filter")
        return dst

    def aggregate_wta(self, guide, cost_volume, labels_out=None):
        torch = self._torch
        L = cost_volume.shape[0]
        self._dev(guide, (self.m, self.H, self.W), torch.float32, "guide")
        self._dev(cost_volume, (L, self.H, self.W), torch.float32, "cost_volume")
        if labels_out is None:
            labels_out = torch.empty((self.H, self.W), dtype=torch.int32, device=self.device)
        self._dev(labels_out, (self.H, self.W), torch.int32, "labels_out")
        self._bind_stream()
        self._check(lib().hgf_aggregate_wta(self._h, _ptr(guide), _ptr(cost_volume), L, _ptr(labels_out)),
                    "hgf_aggregate_wta")
        return labels_out

    def _outputs(self, L, labels, min_cost, filtered, keys, out):
        torch = self._torch
        out = dict(out or {})
        dev, HW = self.device, (self.H, self.W)
        if labels and "labels" not in out:
            out["labels"] = torch.empty(HW, dtype=torch.int32, device=dev)
        if min_cost and "min_cost" not in out:
            out["min_cost"] = torch.empty(HW, dtype=torch.float32, device=dev)
        if filtered and "filtered" not in out:
            out["filtered"] = torch.empty((L,) + HW, dtype=torch.float32, device=dev)
        if keys and "keys" not in out:
            out["keys"] = torch.empty(HW, dtype=torch.int64, device=dev)
        if "labels" in out:
            self._dev(out["labels"], HW, torch.int32, "labels")
        if "min_cost" in out:
            self._dev(out["min_cost"], HW, torch.float32, "min_cost")
        if "filtered" in out:
            self._dev(out["filtered"], (L,) + HW, torch.float32, "filtered")
        if "keys" in out:
            self._dev(out["keys"], HW, torch.int64, "keys")
        return out

    def aggregate_wta_ex(self, guide, cost_volume, label_offset=0, labels=True, min_cost=False, filtered=False,
                         keys=False, out=None):
        """Returns a dict with the requested outputs ('labels', 'min_cost', 'filtered', 'keys')."""
        torch = self._torch
        L = cost_volume.shape[0]
        self._dev(guide, (self.m, self.H, self.W), torch.float32, "guide")
        self._dev(cost_volume, (L, self.H, self.W), torch.float32, "cost_volume")
        out = self._outputs(L, labels, min_cost, filtered, keys, out)
        self._bind_stream()
        self._check(lib().hgf_aggregate_wta_ex(self._h, _ptr(guide), _ptr(cost_volume), L, int(label_offset),
                                               _ptr(out.get("labels")), _ptr(out.get("min_cost")),
                                               _ptr(out.get("filtered")), _ptr(out.get("keys"))),
                    "hgf_aggregate_wta_ex")
        return out

    def stereo_wta(self, left, right, L, label_offset=0, alpha=0.11, tau_color=0.028, tau_grad=0.008, labels=True,
                   min_cost=False, filtered=False, keys=False, out=None):
        """hgf_stereo_wta: cost slices of disparities label_offset .. + L - 1 built on the GPU from the two
        views (S:400 cost), then the HGF aggregation + WTA with the left view as guide."""
        torch = self._torch
        self._dev(left, (3, self.H, self.W), torch.float32, "left")
        self._dev(right, (3, self.H, self.W), torch.float32, "right")
        out = self._outputs(int(L), labels, min_cost, filtered, keys, out)
        self._bind_stream()
        self._check(lib().hgf_stereo_wta(self._h, _ptr(left), _ptr(right), int(L), int(label_offset), float(alpha),
                                         float(tau_color), float(tau_grad), _ptr(out.get("labels")),
                                         _ptr(out.get("min_cost")), _ptr(out.get("filtered")), _ptr(out.get("keys"))),
                    "hgf_stereo_wta")
        return out

    def stereo_wta_right(self, left, right, L, label_offset=0, alpha=0.11, tau_color=0.028, tau_grad=0.008,
                         labels=True, min_cost=False, filtered=False, keys=False, out=None):
        """hgf_stereo_wta_right: the right view's disparity map (reading P1: right view as guide, match at
        x + d).  Views are passed left, right as for stereo_wta."""
        torch = self._torch
        self._dev(left, (3, self.H, self.W), torch.float32, "left")
        self._dev(right, (3, self.H, self.W), torch.float32, "right")
        out = self._outputs(int(L), labels, min_cost, filtered, keys, out)
        self._bind_stream()
        self._check(lib().hgf_stereo_wta_right(self._h, _ptr(left), _ptr(right), int(L), int(label_offset),
                                               float(alpha), float(tau_color), float(tau_grad),
                                               _ptr(out.get("labels")), _ptr(out.get("min_cost")),
                                               _ptr(out.get("filtered")), _ptr(out.get("keys"))),
                    "hgf_stereo_wta_right")
        return out

    def lr_postprocess(self, image, disp_left, disp_right, tol=0, radius=9, sigma_s=9.0, sigma_c=0.1,
                       valid=False, out=None):
        """hgf_lr_postprocess (readings P2-P4): returns {"disp": int32 (H, W)[, "valid": uint8 (H, W)]}."""
        torch = self._torch
        self._dev(image, (self.m, self.H, self.W), torch.float32, "image")
        self._dev(disp_left, (self.H, self.W), torch.int32, "disp_left")
        self._dev(disp_right, (self.H, self.W), torch.int32, "disp_right")
        out = dict(out or {})
        dev = image.device
        if "disp" not in out:
            out["disp"] = torch.empty((self.H, self.W), dtype=torch.int32, device=dev)
        if valid and "valid" not in out:
            out["valid"] = torch.empty((self.H, self.W), dtype=torch.uint8, device=dev)
        self._bind_stream()
        self._check(lib().hgf_lr_postprocess(self._h, _ptr(image), _ptr(disp_left), _ptr(disp_right), int(tol),
                                             int(radius), float(sigma_s), float(sigma_c), _ptr(out.get("valid")),
                                             _ptr(out["disp"])), "hgf_lr_postprocess")
        return out

    def stereo_disparity(self, left, right, L, label_offset=0, alpha=0.11, tau_color=0.028, tau_grad=0.008, tol=0,
                         radius=9, sigma_s=9.0, sigma_c=0.1, raw=False, valid=False, out=None):
        """hgf_stereo_disparity: left map, right map, post-processing.  Returns {"disp"[, "disp_left",
        "disp_right"][, "valid"]} (int32 / uint8 (H, W) CUDA tensors)."""
        torch = self._torch
        self._dev(left, (3, self.H, self.W), torch.float32, "left")
        self._dev(right, (3, self.H, self.W), torch.float32, "right")
        out = dict(out or {})
        dev = left.device
        names = ["disp"] + (["disp_left", "disp_right"] if raw else [])
        for k in names:
            if k not in out:
                out[k] = torch.empty((self.H, self.W), dtype=torch.int32, device=dev)
        if valid and "valid" not in out:
            out["valid"] = torch.empty((self.H, self.W), dtype=torch.uint8, device=dev)
        self._bind_stream()
        self._check(lib().hgf_stereo_disparity(self._h, _ptr(left), _ptr(right), int(L), int(label_offset),
                                               float(alpha), float(tau_color), float(tau_grad), int(tol), int(radius),
                                               float(sigma_s), float(sigma_c), _ptr(out.get("disp_left")),
                                               _ptr(out.get("disp_right")), _ptr(out.get("valid")),
                                               _ptr(out["disp"])), "hgf_stereo_disparity")
        return out

    def segment(self, image, fg_seeds, bg_seeds, labels=True, min_cost=False, filtered=False, out=None):
        """hgf_segment: foreground (0) / background (1) labels from seed masks (uint8 or bool CUDA tensors)."""
        torch = self._torch
        self._dev(image, (self.m, self.H, self.W), torch.float32, "image")
        fg = fg_seeds.to(torch.uint8).contiguous() if fg_seeds.dtype != torch.uint8 else fg_seeds
        bg = bg_seeds.to(torch.uint8).contiguous() if bg_seeds.dtype != torch.uint8 else bg_seeds
        self._dev(fg, (self.H, self.W), torch.uint8, "fg_seeds")
        self._dev(bg, (self.H, self.W), torch.uint8, "bg_seeds")
        out = self._outputs(2, labels, min_cost, filtered, False, out)
        self._bind_stream()
        self._check(lib().hgf_segment(self._h, _ptr(image), _ptr(fg), _ptr(bg), _ptr(out.get("labels")),
                                      _ptr(out.get("min_cost")), _ptr(out.get("filtered"))), "hgf_segment")
        return out

    def aggregate_wta_peer(self, cost_volume, peer_ptrs, world, rows_per_owner, label_offset=0):
        """hgf_aggregate_wta_peer: the slices' keys merged by atomic MIN into the owners' buffers
        (peer_ptrs: int64 CUDA tensor of `world` device addresses, e.g. PeerKeys.ptrs)."""
        torch = self._torch
        L = cost_volume.shape[0]
        self._dev(cost_volume, (L, self.H, self.W), torch.float32, "cost_volume")
        self._dev(peer_ptrs, (world,), torch.int64, "peer_ptrs")
        self._bind_stream()
        self._check(lib().hgf_aggregate_wta_peer(self._h, _ptr(cost_volume), L, int(label_offset), _ptr(peer_ptrs),
                                                 int(world), int(rows_per_owner)), "hgf_aggregate_wta_peer")

    def fill_keys(self, keys):
        self._bind_stream()
        self._check(lib().hgf_fill_keys(self._h, _ptr(keys), keys.numel()), "hgf_fill_keys")

    def unpack_keys_n(self, keys, labels_out, min_cost_out=None):
        self._bind_stream()
        self._check(lib().hgf_unpack_keys_n(self._h, _ptr(keys), keys.numel(), _ptr(labels_out), _ptr(min_cost_out)),
                    "hgf_unpack_keys_n")

    def prepare_rows(self, guide, y0, y1):
        """hgf_prepare_rows: guidance for the frame + statistics of rows [y0, y1)."""
        self._dev(guide, (self.m, self.H, self.W), self._torch.float32, "guide")
        self._bind_stream()
        self._check(lib().hgf_prepare_rows(self._h, _ptr(guide), int(y0), int(y1)), "hgf_prepare_rows")

    def stats_view(self):
        """hgf_stats_buffer as a float32 tensor view (H, bytes_per_row / 4) on the handle's device (no copy;
        valid while the handle lives)."""
        p, bpr = ctypes.c_void_p(), ctypes.c_size_t()
        self._check(lib().hgf_stats_buffer(self._h, ctypes.byref(p), ctypes.byref(bpr)), "hgf_stats_buffer")

        class _View:
            __cuda_array_interface__ = {"shape": (self.H, bpr.value // 4), "typestr": "<f4",
                                        "data": (p.value, False), "version": 3, "strides": None}
        return self._torch.as_tensor(_View(), device=self.device)

    def aggregate_wta_prepared(self, cost_volume, label_offset=0, labels=True, min_cost=False, filtered=False,
                               keys=False, out=None):
        """hgf_aggregate_wta_prepared (statistics from prepare_rows); returns the requested outputs."""
        torch = self._torch
        L = cost_volume.shape[0]
        self._dev(cost_volume, (L, self.H, self.W), torch.float32, "cost_volume")
        out = self._outputs(L, labels, min_cost, filtered, keys, out)
        self._bind_stream()
        self._check(lib().hgf_aggregate_wta_prepared(self._h, _ptr(cost_volume), L, int(label_offset),
                                                     _ptr(out.get("labels")), _ptr(out.get("min_cost")),
                                                     _ptr(out.get("filtered")), _ptr(out.get("keys"))),
                    "hgf_aggregate_wta_prepared")
        return out

    def unpack_keys(self, keys, labels_out=None, min_cost_out=None):
        torch = self._torch
        HW = (self.H, self.W)
        self._dev(keys, HW, torch.int64, "keys")
        if labels_out is None:
            labels_out = torch.empty(HW, dtype=torch.int32, device=self.device)
        if min_cost_out is None:
            min_cost_out = torch.empty(HW, dtype=torch.float32, device=self.device)
        self._bind_stream()
        self._check(lib().hgf_unpack_keys(self._h, _ptr(keys), _ptr(labels_out), _ptr(min_cost_out)),
                    "hgf_unpack_keys")
        return labels_out, min_cost_out

    def aggregate_wta_host(self, guide_host, cost_host, labels_host=None):
        """Host tensors (CPU float32; pinned for overlap) in, host int32 labels out; synchronous."""
        torch = self._torch
        L = cost_host.shape[0]
        for t, nm in ((guide_host, "guide_host"), (cost_host, "cost_host")):
            if t.device.type != "cpu" or t.dtype != torch.float32 or not t.is_contiguous():
                raise HGFError(f"{nm} must be a contiguous float32 CPU tensor")
        if labels_host is None:
            labels_host = torch.empty((self.H, self.W), dtype=torch.int32, pin_memory=True)
        self._bind_stream()
        self._check(lib().hgf_aggregate_wta_host(self._h, _ptr(guide_host), _ptr(cost_host), L, _ptr(labels_host)),
                    "hgf_aggregate_wta_host")
        return labels_host

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().hgf_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_range(L, world, rank):
    """Contiguous label range [l0, l1) of `rank` (first L mod world ranks get one extra label)."""
    base, extra = divmod(L, world)
    l0 = rank * base + min(rank, extra)
    return l0, l0 + base + (1 if rank < extra else 0)


def merge_keys_allreduce(keys, group=None):
    """Label-sharded WTA merge: in-place int64 allreduce-MIN of the signed packed keys (hgf.h)."""
    import torch.distributed as dist
    dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
    return keys


def gather_stats_rows(h, group=None):
    """Row-sharded statistics: every rank computes the statistics of its band of rows
    (shard_range over H) with ``h.prepare_rows`` beforehand; this all-gathers the bands into every rank's
    statistics buffer (in place; NCCL all-gather when the bands are equal, else one broadcast per rank)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    view = h.stats_view()
    bands = [shard_range(h.H, world, r) for r in range(world)]
    if h.H % world == 0:
        y0, y1 = bands[rank]
        dist.all_gather_into_tensor(view, view[y0:y1], group=group)
    else:
        for src, (y0, y1) in enumerate(bands):
            g_src = src if group is None else dist.get_global_rank(group, src)
            dist.broadcast(view[y0:y1].contiguous() if not view[y0:y1].is_contiguous() else view[y0:y1], src=g_src,
                           group=group)
    return view


def _device_view(ptr, shape, typestr, device):
    import torch

    class _V:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_V(), device=device)


class PeerKeys:
    """Owner-partitioned key buffers for hgf_aggregate_wta_peer (the fused merge): rank k owns
    rows [k R, min(H, (k+1) R)), R = ceil(H / world), in a cudaMalloc'd int64 [R][W] buffer; the buffers
    are exchanged once with CUDA IPC (handles all-gathered over the process group) so that every rank's
    aggregation kernel can atomicMin into every owner's rows over NVLink.  With world == 1 no IPC is used."""

    def __init__(self, h, group=None):
        import torch
        import torch.distributed as dist
        self.h, self.group = h, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rows = -(-h.H // self.world)
        # ranks past the last row (world > ceil(H / rows)) own an empty range, never a negative one
        self.y0 = min(h.H, self.rank * self.rows)
        self.y1 = max(self.y0, min(h.H, self.y0 + self.rows))
        nbytes = 8 * self.rows * h.W
        p = ctypes.c_void_p()
        st = lib().hgf_alloc(nbytes, ctypes.byref(p))
        if st != 0:
            raise HGFError(f"hgf_alloc: {lib().hgf_status_string(st).decode()}")
        self._own = p.value
        self._opened = []
        ptrs = [0] * self.world
        ptrs[self.rank] = self._own
        if self.world > 1:
            hd = ctypes.create_string_buffer(64)
            st = lib().hgf_ipc_get_handle(ctypes.c_void_p(self._own), hd)
            if st != 0:
                self.close()
                raise HGFError("hgf_ipc_get_handle failed")
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(hd.raw), group=group)
            for k, raw in enumerate(handles):
                if k == self.rank:
                    continue
                q = ctypes.c_void_p()
                if lib().hgf_ipc_open(raw, ctypes.byref(q)) != 0:
                    self.close()
                    raise HGFError(f"hgf_ipc_open of rank {k}'s key buffer failed (no peer access?)")
                self._opened.append(q.value)
                ptrs[k] = q.value
        self.ptrs = torch.tensor(ptrs, dtype=torch.int64, device=h.device)
        self.keys = _device_view(self._own, (self.rows, h.W), "<i8", h.device)   # this rank's rows

    def reset(self):
        """Fill this rank's rows with the MIN identity (every rank, then a barrier, before the merge)."""
        self.h.fill_keys(self.keys)

    def close(self):
        for q in self._opened:
            lib().hgf_ipc_close(ctypes.c_void_p(q))
        self._opened = []
        if getattr(self, "_own", None):
            lib().hgf_free(ctypes.c_void_p(self._own))
            self._own = None


class PeerMerge:
    """The fused WTA merge step by step: two PeerKeys owner buffers used alternately.  Step s
    resets the buffer of step s + 1, runs hgf_aggregate_wta_peer into the buffer of step s, all-reduces a
    4-byte flag (every rank's atomics of step s have landed; it also orders every owner's reset of the next
    buffer before any rank's atomics of step s + 1) and unpacks this rank's rows.  One collective per step and
    no host synchronisation; the statistics must be prepared (``h.prepare_rows`` / ``gather_stats_rows``)."""

    def __init__(self, h, group=None):
        import torch
        import torch.distributed as dist
        self.h, self.group = h, group
        self.bufs = []
        try:
            self.bufs = [PeerKeys(h, group), PeerKeys(h, group)]
        except Exception:
            self.close()
            raise
        self.world, self.rows = self.bufs[0].world, self.bufs[0].rows
        self.y0, self.y1 = self.bufs[0].y0, self.bufs[0].y1
        for b in self.bufs:
            b.reset()
        torch.cuda.synchronize(h.device)
        if self.world > 1:
            dist.barrier(group=group)
        self.flag = torch.zeros(1, dtype=torch.int32, device=h.device)
        self.steps = 0

    def aggregate(self, cost_volume, labels_out, label_offset=0):
        """One step: labels of this rank's rows [y0, y1) into labels_out[: y1 - y0] (int32, W columns)."""
        import torch.distributed as dist
        cur, nxt = self.bufs[self.steps % 2], self.bufs[(self.steps + 1) % 2]
        self.steps += 1
        nxt.reset()
        self.h.aggregate_wta_peer(cost_volume, cur.ptrs, self.world, cur.rows, label_offset=label_offset)
        if self.world > 1:
            dist.all_reduce(self.flag, group=self.group)
        self.h.unpack_keys_n(cur.keys[: self.y1 - self.y0], labels_out[: self.y1 - self.y0])

    def close(self):
        """Unmap the peers' buffers, wait for every rank to have done so, then free this rank's own."""
        import torch.distributed as dist
        for b in self.bufs:
            for q in b._opened:
                lib().hgf_ipc_close(ctypes.c_void_p(q))
            b._opened = []
        if self.bufs and getattr(self, "world", 1) > 1 and dist.is_initialized():
            dist.barrier(group=self.group)
        for b in self.bufs:
            b.close()
        self.bufs = []
