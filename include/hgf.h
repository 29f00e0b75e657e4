/*
 * hgf.h — C ABI of the B200-native Hardware-Efficient Guided Filter (HGF) hot path.
 *
 * Paper: Dai et al., "Hardware-Efficient Guided Image Filtering for Multi-Label Problem",
 * CVPR 2018, arXiv 1803.00005.  "P:n" = line n of the paper's LaTeX source.
 *
 * The path (BASELINE.json north_star):
 *   1. polynomial guidance  G_{(i-1)d+j} = I_i^j               (§4.2; P:630 uses d = 2)
 *   2. label-independent statistics: Gram planes G_ij = B(G_i G_j) (Prop 2; Eq12)
 *      and the regularised inverse by the paper's recursion (Prop 1 / Eq4; Eq11),
 *      computed ONCE per frame in float64
 *   3. per cost slice (label) l: box sums of p and G_k p, coefficients w (Eq13, reassociated),
 *      box sums of w, output Z (Eq14 P:328-333 == Eq8)
 *   4. winner-takes-all argmin over labels, ties -> lowest label
 *
 * Conventions for every entry point below
 *   - B(.) is a box SUM over the (2r+1)x(2r+1) window clipped to the image; eps is the
 *     paper's lambda against those sums (Eq7).  N_p = clipped window pixel count.
 *   - All image arrays are dense, row-major float32 planes; a stack of planes is plane-major:
 *       guide        [n_guide][H][W]   raw guidance I, values expected in [0, 1]
 *       cost_volume  [L][H][W]         slice l is label (label_offset + l)
 *       labels_out   [H][W] int32      argmin label
 *   - Pointers passed to hgf_filter / hgf_aggregate_wta* / hgf_unpack_keys are CUDA DEVICE
 *     pointers owned by the caller.  These calls allocate nothing, copy nothing host<->device and
 *     are asynchronous on the handle's stream: results are valid after that stream synchronises.
 *     (hgf_aggregate_wta_host is the one entry point that takes host pointers; see there.)
 *   - The library owns only its scratch (guidance planes, statistics planes, coefficient buffer),
 *     allocated by hgf_create* and freed by hgf_destroy.
 *   - A handle is bound to the CUDA device current at create time and is not thread-safe:
 *     use one handle per host thread / stream.
 *   - Errors: every call returns an hgf_status; HGF_ERR_CUDA reports a CUDA failure (including
 *     an asynchronous fault from earlier work on the stream); hgf_last_error() gives detail.
 *     No call falls back to a CPU implementation.
 */
#ifndef HGF_H_
#define HGF_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HGF_API __attribute__((visibility("default")))
#else
#define HGF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hgf_ctx* hgf_handle;

typedef enum {
  HGF_OK = 0,
  HGF_ERR_INVALID_ARGUMENT = 1, /* bad size, null pointer, eps <= 0 or non-finite, ...          */
  HGF_ERR_UNSUPPORTED = 2,      /* n = n_guide*poly_degree > HGF_MAX_CHANNELS, radius > HGF_MAX_RADIUS */
  HGF_ERR_OUT_OF_MEMORY = 3,    /* scratch allocation failed                                    */
  HGF_ERR_CUDA = 4              /* a CUDA runtime error (launch failure or asynchronous fault)  */
} hgf_status;

/* Regression modes.
 * HGF_MODE_HGF: the paper's HGF, Eq7: lambda ||w||^2 penalises ALL n+1 coefficients,
 *               including the intercept w(0).
 * HGF_MODE_GF : the paper's §5.1 guided filter, Eq15/16: slopes penalised, intercept
 *               free (He et al.'s GF with eps_p = lambda / N_p). */
enum { HGF_MODE_HGF = 0, HGF_MODE_GF = 1 };

#define HGF_MAX_CHANNELS 20 /* n = n_guide * poly_degree  (BASELINE config 5 sweeps n = 1..20) */
#define HGF_MAX_RADIUS 32

/* Create a handle for W x H images with an n_guide-channel raw guide, polynomial degree
 * poly_degree (n = n_guide * poly_degree synthesised channels, §4.2), window radius `radius`
 * (side 2r+1) and regulariser eps = lambda > 0 (P:151 needs lambda^-1).  HGF mode, legacy
 * default stream.  Allocates the per-frame scratch on the current device.
 * Errors: INVALID_ARGUMENT (W,H,n_guide,poly_degree,radius < 1, eps <= 0 or non-finite, out==NULL),
 *         UNSUPPORTED (n > HGF_MAX_CHANNELS or radius > HGF_MAX_RADIUS), OUT_OF_MEMORY, CUDA. */
HGF_API hgf_status hgf_create(hgf_handle* out, int W, int H, int n_guide, int poly_degree, int radius, double eps);

/* As hgf_create, with mode (HGF_MODE_HGF | HGF_MODE_GF) and a cudaStream_t (NULL = legacy default). */
HGF_API hgf_status hgf_create_ex(hgf_handle* out, int W, int H, int n_guide, int poly_degree, int radius,
                         double eps, int mode, void* cuda_stream);

/* Free the handle and its scratch (synchronises the handle's stream first).  NULL is accepted. */
HGF_API hgf_status hgf_destroy(hgf_handle h);

/* Re-bind the handle to another cudaStream_t (NULL = legacy default stream). */
HGF_API hgf_status hgf_set_stream(hgf_handle h, void* cuda_stream);

/* Filter one slice (Fig 2 flowchart): dst = HGF(src; guide).
 * guide [n_guide][H][W], src [H][W], dst [H][W] (device, float32; dst must not alias guide/src).
 * Runs steps 1-3 of the path with L = 1. */
HGF_API hgf_status hgf_filter(hgf_handle h, const float* guide, const float* src, float* dst);

/* Multi-label aggregation + WTA: filter every slice of cost_volume [L][H][W] with the
 * guidance synthesised from guide, write labels_out[p] = argmin_l Z_l(p) (ties -> lowest l).
 * L >= 1.  Equivalent to hgf_aggregate_wta_ex(h, guide, cost_volume, L, 0, labels_out, NULL, NULL, NULL). */
HGF_API hgf_status hgf_aggregate_wta(hgf_handle h, const float* guide, const float* cost_volume, int L,
                             int32_t* labels_out);

/* Extended form for label shards and debugging.  Label index reported = label_offset + l.
 * Outputs (each may be NULL; at least one must be non-NULL):
 *   labels_out    int32  [H][W]     argmin label
 *   min_cost_out  float  [H][W]     min_l Z_l
 *   filtered_out  float  [L][H][W]  every filtered slice Z_l (same arithmetic as the WTA path)
 *   keys_out      int64  [H][W]     packed key = (orderable(min cost) << 32 | label) XOR 2^63, where
 *                 orderable(f) = bits(f) | 2^31 for f >= +0 (-0.0 is canonicalised to +0.0),
 *                 ~bits(f) for f < 0.  The unsigned key orders (cost, label) lexicographically;
 *                 the XOR with 2^63 makes the SIGNED int64 order identical, so the label-sharded
 *                 merge is an int64 allreduce-MIN (NCCL ncclInt64/ncclMin, or gloo) over shards.
 * label_offset >= 0 and label_offset + L <= 2^31 - 1. */
HGF_API hgf_status hgf_aggregate_wta_ex(hgf_handle h, const float* guide, const float* cost_volume, int L,
                                int label_offset, int32_t* labels_out, float* min_cost_out,
                                float* filtered_out, int64_t* keys_out);

/* Stereo aggregation with the cost volume built on the GPU.  The label slices are the
 * matching costs of disparities d = label_offset .. label_offset + L - 1 between the two views (the paper
 * defers the cost to Hosni et al.; the form is SPEC S:400):
 *   C(x,y,d) = alpha min(mean_c |L_c(x,y) - R_c(x-d,y)|, tau_color)
 *            + (1 - alpha) min(|dx Lbar(x,y) - dx Rbar(x-d,y)|, tau_grad),
 * Lbar/Rbar the channel means, dx the central x-difference (one-sided at the border columns), x - d < 0 ->
 * alpha tau_color + (1 - alpha) tau_grad; then steps 1-4 exactly as hgf_aggregate_wta_ex with the left view
 * as the guide.  left, right: device [3][H][W] f32 (the handle must have n_guide = 3).  Only the chunk being
 * filtered is materialised (library scratch, allocated on first use).  Outputs as hgf_aggregate_wta_ex;
 * HGF_ERR_INVALID_ARGUMENT for null views, n_guide != 3, alpha outside [0,1] or negative/non-finite
 * thresholds. */
HGF_API hgf_status hgf_stereo_wta(hgf_handle h, const float* left, const float* right, int L, int label_offset,
                                  float alpha, float tau_color, float tau_grad, int32_t* labels_out,
                                  float* min_cost_out, float* filtered_out, int64_t* keys_out);

/* Right-view stereo aggregation (reading P1 of DESIGN.md §11d; P:641 names the
 * post-processing of Hosni et al.'s framework, which needs the right view's disparity map): as
 * hgf_stereo_wta with the right view as the guide and the views' roles exchanged, the match searched at
 * x + d:  C_R(x,y,d) = alpha min(mean_c |R_c(x,y) - L_c(x+d,y)|, tau_color)
 *                    + (1 - alpha) min(|dx Rbar(x,y) - dx Lbar(x+d,y)|, tau_grad),  x + d >= W -> truncation.
 * Arguments, outputs and errors as hgf_stereo_wta (the views are still passed left, right). */
HGF_API hgf_status hgf_stereo_wta_right(hgf_handle h, const float* left, const float* right, int L,
                                        int label_offset, float alpha, float tau_color, float tau_grad,
                                        int32_t* labels_out, float* min_cost_out, float* filtered_out,
                                        int64_t* keys_out);

/* Post-processing of a left disparity map (readings P2-P4 of DESIGN.md §11d, the
 * paper only names the step):
 *   P2  (x,y) is consistent iff x - dL >= 0 and |dL(x,y) - dR(x - dL(x,y), y)| <= tol;
 *   P3  an inconsistent pixel takes the lower disparity of the nearest consistent pixels to its left and
 *       right on its row (the one that exists at a border; unchanged on a row without any);
 *   P4  then the weighted median of the filled map over its (2 radius + 1)^2 window (clipped at the border):
 *       the smallest window value d with sum_{D(q) <= d} w >= 1/2 sum w,
 *       w = exp(-|q - p|^2 / sigma_s^2 - |I(q) - I(p)|^2 / sigma_c^2), float32 weights.
 * Consistent pixels keep dL.  image: device [n_guide][H][W] f32 (the handle's n_guide channels; the left
 * view for stereo); disp_left, disp_right: device int32 [H][W] disparities; valid_out: device u8 [H][W]
 * (1 = consistent) or NULL; disp_out: device int32 [H][W] (must not alias disp_right).  Library scratch
 * (12 bytes per pixel) is allocated on first use.  HGF_ERR_INVALID_ARGUMENT for null pointers, tol < 0,
 * radius outside [0, 15], non-positive or non-finite sigmas. */
HGF_API hgf_status hgf_lr_postprocess(hgf_handle h, const float* image, const int32_t* disp_left,
                                      const int32_t* disp_right, int tol, int radius, float sigma_s,
                                      float sigma_c, uint8_t* valid_out, int32_t* disp_out);

/* The whole stereo disparity pipeline of Hosni et al.'s framework on the GPU: hgf_stereo_wta
 * (left map), hgf_stereo_wta_right (right map), hgf_lr_postprocess (left view as the image).  Cost and
 * post-processing arguments as there; disparities are label_offset + label.  disp_left_out,
 * disp_right_out (raw maps) and valid_out may be NULL; disp_out (the final map) may not.  Launches run on
 * the handle's stream; nothing is read back. */
HGF_API hgf_status hgf_stereo_disparity(hgf_handle h, const float* left, const float* right, int L,
                                        int label_offset, float alpha, float tau_color, float tau_grad, int tol,
                                        int radius, float sigma_s, float sigma_c, int32_t* disp_left_out,
                                        int32_t* disp_right_out, uint8_t* valid_out, int32_t* disp_out);

/* Foreground / background segmentation (cost form of SPEC S:406-409):
 * two cost slices (label 0 = foreground, 1 = background) from per-class, per-channel 32-bin histograms of
 * the seed pixels' colours, Laplace-smoothed: p_c(b) = (count_c(b) + 1) / (N_c + 32), cost
 * C_c(x) = -sum_ch log p_c(bin(I_ch(x))) / (m log(N_c + 32)) in (0, 1], bin(v) = min(floor(32 v), 31);
 * then steps 1-4 with the image as the guide (L = 2).  image: device [n_guide][H][W] f32 in [0,1];
 * fg_seeds, bg_seeds: device [H][W] u8 masks (non-zero = seed).  Outputs as hgf_aggregate_wta_ex
 * (labels are 0 / 1; at least one non-null).  HGF_ERR_INVALID_ARGUMENT for an empty seed set (checked
 * with one small device-to-host read, which synchronises the handle's stream). */
HGF_API hgf_status hgf_segment(hgf_handle h, const float* image, const uint8_t* fg_seeds, const uint8_t* bg_seeds,
                               int32_t* labels_out, float* min_cost_out, float* filtered_out);

/* Fused WTA merge over peer memory (the compute + collective in one kernel): as
 * hgf_aggregate_wta_prepared (statistics from hgf_prepare_rows + the caller's all-gather), but the last
 * aggregation pass combines each pixel's packed key (hgf_aggregate_wta_ex's keys_out encoding) with a
 * 64-bit atomic MIN directly into the key buffer of the rank that owns the pixel's row, over NVLink for a
 * peer GPU.  peer_keys_dev: DEVICE array of `world` device pointers; peer_keys_dev[k] holds rows
 * [k R, min(H, (k+1) R)) as int64 [R][W], R = rows_per_owner, world * R >= H (mapped with hgf_ipc_open for
 * other processes' buffers).  Every owner buffer must hold INT64_MAX (hgf_fill_keys) before any rank starts,
 * and is complete once every rank's call has finished on its stream (the caller synchronises, e.g. stream
 * sync + a process-group barrier); the owner then unpacks its rows with hgf_unpack_keys_n.  Errors as
 * hgf_aggregate_wta_prepared; HGF_ERR_UNSUPPORTED outside the k_coef3/4 + k_agg3 path. */
HGF_API hgf_status hgf_aggregate_wta_peer(hgf_handle h, const float* cost_volume, int L, int label_offset,
                                          int64_t* const* peer_keys_dev, int world, int rows_per_owner);
/* keys[0 .. n) = INT64_MAX (the identity of the MIN merge), on the handle's stream. */
HGF_API hgf_status hgf_fill_keys(hgf_handle h, int64_t* keys, long long n);
/* hgf_unpack_keys over n contiguous keys (e.g. an owner's band of rows). */
HGF_API hgf_status hgf_unpack_keys_n(hgf_handle h, const int64_t* keys, long long n, int32_t* labels_out,
                                     float* min_cost_out);
/* Device memory that can be shared with other processes (cudaMalloc) and CUDA IPC around it: handle64 is
 * a 64-byte cudaIpcMemHandle_t; hgf_ipc_open maps another process's allocation on the current device
 * (peer access enabled lazily), hgf_ipc_close unmaps it.  HGF_ERR_CUDA when the runtime refuses. */
HGF_API hgf_status hgf_alloc(size_t bytes, void** dev_ptr);
HGF_API hgf_status hgf_free(void* dev_ptr);
HGF_API hgf_status hgf_ipc_get_handle(void* dev_ptr, unsigned char* handle64);
HGF_API hgf_status hgf_ipc_open(const unsigned char* handle64, void** dev_ptr);
HGF_API hgf_status hgf_ipc_close(void* dev_ptr);

/* Row-sharded frame preparation.  Steps 1-2 of the path for a row band:
 * the polynomial guidance for the whole frame (cheap, needed by every slice kernel) and the
 * label-independent statistics (Prop 1 recursion, Eq4 P:143-151 with readings F1/F2) of image rows
 * [y0, y1) only, 0 <= y0 <= y1 <= H.  Rows outside the band keep the buffer's previous contents: the caller
 * fills them, e.g. by an all-gather of every rank's band (hgf_stats_buffer), before
 * hgf_aggregate_wta_prepared.  guide: device, [n_guide][H][W] f32.  HGF_ERR_UNSUPPORTED unless the
 * configuration uses the per-pixel statistics layout of the k_coef3/k_coef4 path (n <= 6, W % 4 == 0,
 * r <= 9 and a TMA-capable device); the unsharded entry points always work. */
HGF_API hgf_status hgf_prepare_rows(hgf_handle h, const float* guide, int y0, int y1);

/* The device statistics buffer written by hgf_prepare_rows: H rows of *bytes_per_row bytes each, row y at
 * dev_ptr + y * bytes_per_row (owned by the handle; valid until hgf_destroy).  HGF_ERR_UNSUPPORTED as
 * above. */
HGF_API hgf_status hgf_stats_buffer(hgf_handle h, void** dev_ptr, size_t* bytes_per_row);

/* hgf_aggregate_wta_ex without steps 1-2: the slices use the guidance and statistics already in the
 * handle (from hgf_prepare_rows; every row must be filled).  Arguments, outputs and errors as
 * hgf_aggregate_wta_ex. */
HGF_API hgf_status hgf_aggregate_wta_prepared(hgf_handle h, const float* cost_volume, int L, int label_offset,
                                              int32_t* labels_out, float* min_cost_out, float* filtered_out,
                                              int64_t* keys_out);

/* Unpack merged (signed) keys [H][W] into labels_out (int32, may be NULL) and min_cost_out (float, may be NULL). */
HGF_API hgf_status hgf_unpack_keys(hgf_handle h, const int64_t* keys, int32_t* labels_out, float* min_cost_out);

/* End-to-end form with HOST buffers: guide_host [n_guide][H][W], cost_host [L][H][W] (float32,
 * preferably pinned), labels_host [H][W] int32.  Copies the inputs host->device in label chunks on
 * the handle's stream, overlapped with the aggregation of the previous chunk, then copies the labels
 * back and synchronises the stream before returning.  Device staging buffers are owned by the handle
 * (allocated on first use, sized by the chunk).  Errors as hgf_aggregate_wta_ex. */
HGF_API hgf_status hgf_aggregate_wta_host(hgf_handle h, const float* guide_host, const float* cost_host, int L,
                                  int32_t* labels_host);

/* Kernel classes reported by the tracing calls below. */
enum {
  HGF_KC_GUIDANCE = 0, /* K1 polynomial guidance                 */
  HGF_KC_STATS = 1,    /* K3 float64 Gram + Prop-1 statistics    */
  HGF_KC_COEF = 2,     /* K4a per-slice coefficients w           */
  HGF_KC_AGG = 3,      /* K4b per-slice aggregation Z + WTA      */
  HGF_KC_KEYS = 4,     /* key unpacking                          */
  HGF_KC_COST = 5,     /* stereo cost construction (hgf_stereo_wta) */
  HGF_KC_POST = 6,     /* post-processing (hgf_lr_postprocess)   */
  HGF_KC_COUNT = 7
};

/* Tracing: when enable != 0, every kernel launch of this handle is bracketed by CUDA events recorded
 * on the handle's stream (a few microseconds of host overhead per launch; no device synchronisation). */
HGF_API hgf_status hgf_set_profiling(hgf_handle h, int enable);

/* Synchronise the handle's stream, then write the device time (ms) and launch count accumulated per
 * kernel class since the previous read into ms[0..n) and counts[0..n) (either may be NULL; n <=
 * HGF_KC_COUNT), and reset the accumulators. */
HGF_API hgf_status hgf_profile_read(hgf_handle h, double* ms, int* counts, int n);

/* Number of kernel launches the last hgf_filter / hgf_aggregate_wta* call enqueued. */
HGF_API int hgf_last_launch_count(hgf_handle h);

/* The slice-kernel pair this handle runs, fixed at create time from (W, H, n_guide, poly_degree, radius)
 * and the HGF_* selection variables: "coef5+agg6" (default for m <= 3, d <= 3, n <= 6, r <= 9, W % 4 == 0 or
 * d == 2), "coef3+agg6" (n <= 6 otherwise, W % 4 == 0), "coef5+agg3" / "coef3+agg3" (HGF_AGG6=0), "coef5+agg5"
 * (opt-in), "coef4+agg3", "coef2+agg3", "coef2+agg2", "coef1+agg1".  Few-label calls (L <= 2, hgf_filter) run
 * planar paths whatever this reports (hgf_filter: the fused single-slice pass).  Static string; NULL handle -> "". */
HGF_API const char* hgf_kernel_path(hgf_handle h);

/* Static description of a status code. */
HGF_API const char* hgf_status_string(hgf_status s);

/* Detail for the last failure on this handle ("" if none).  Valid until the next call on h. */
HGF_API const char* hgf_last_error(hgf_handle h);

#ifdef __cplusplus
}
#endif

#endif /* HGF_H_ */
