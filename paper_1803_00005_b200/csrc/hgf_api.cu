// C ABI of the HGF hot path (declared in include/hgf.h).  Validation, scratch ownership, stream
// handling and launch sequencing; every step of the path runs in the kernels of hgf_kernels.cu.
#include <algorithm>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "../../include/hgf.h"
#include "hgf_common.cuh"
#include "hgf_launch.h"

struct hgf_ctx {
  int W = 0, H = 0, m = 0, d = 0, n = 0, r = 0, mode = 0;
  double eps = 0.0;
  int device = 0;
  cudaStream_t stream = nullptr;
  float* G = nullptr;          // [n][H][W]     polynomial guidance (K1)
  float* Gp = nullptr;         // [H][m][gp_pitch][2]  (I_i, I_i^2) pairs for k_coef5 when d = 2 (K1)
  int gp_pitch = 0;            // Gp row pitch in pairs (W rounded up to even)
  float* vpad = nullptr;       // W % 4 != 0: one chunk of the cost volume in rows of ceil4(W) floats (k_coef5 TMA)
  float* stats = nullptr;      // [NS][H][W]    P' upper triangle + nu (K3)
  float* wbuf = nullptr;       // [lcap][n+1][H][W] per-slice coefficients w (K4a -> K4b)
  int lcap = 0;                // labels per coefficient chunk
  float* best_cost = nullptr;  // [H][W] running WTA state across chunks
  int32_t* best_label = nullptr;
  // host-buffer path staging (lazily allocated)
  float* st_guide = nullptr;
  float* sv_grad = nullptr;    // hgf_stereo_wta: dx of the channel mean of the left / right views [2][H][W]
  float* sv_cost = nullptr;    // hgf_stereo_wta: one chunk of constructed cost slices [lcap][H][W]
  float* sg_cost = nullptr;    // hgf_segment: the two cost slices [2][H][W]
  int* sg_counts = nullptr;    // hgf_segment: seed histograms [2][m][32] then seed counts [2]
  int* pp_int = nullptr;       // post-processing: filled map [H][W], then left / right disparity maps [2][H][W]
  uint8_t* pp_valid = nullptr; // post-processing: consistency flags [H][W] (when the caller passes none)
  double* st3_scratch = nullptr;   // k_stats3 (n >= kStats3MinN): Gram planes + one batch of row sums
  long long* const* peer_keys = nullptr;   // hgf_aggregate_wta_peer: set for the duration of the call
  int rows_per_owner = 0;
  float* st_vol[2] = {nullptr, nullptr};
  int32_t* st_labels = nullptr;
  int st_chunk = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_used[2] = {nullptr, nullptr};
  int launches = 0;
  bool fast = false;           // v2 fast-path kernels usable for (m, d, r)
  bool v3agg = false;          // TMA-fed v3 aggregation usable (n <= 9, r <= 9, W % 4 == 0)
  CUtensorMap tm_w[2];         // TMA descriptors over wbuf for k_agg3's two plane groups
  // two-stream chunk pipeline (interleaved layout): the coefficient buffer as two halves of `half` labels; the
  // coefficients of chunk c + 1 (handle stream) overlap the aggregation of chunk c (aux stream)
  int half = 0;                // labels per half (multiple of 32), 0 = no pipeline
  CUtensorMap tm_wh[2][2];     // k_agg3 maps over half b, plane groups A / B
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_coef[2] = {nullptr, nullptr}, ev_agg[2] = {nullptr, nullptr}, ev_join = nullptr;
  hgf::WLayout wlay{};         // coefficient-buffer layout (rows pitched to 16 bytes when v3agg)
  // few-label calls (L <= kSmallL, e.g. hgf_filter): the tile kernel k_coef2 on planar statistics and the planar
  // k_agg3 instead of the lane-per-label k_coef5, which would keep 31 of its 32 lanes idle
  bool small_ok = false;       // the planar maps below exist
  bool planar_now = false;     // set by an entry point for the duration of a few-label call
  hgf::WLayout wlay_planar{};
  CUtensorMap tm_wp[2];
  bool v3coef = false;         // label-batched marching coefficient kernel (needs v3agg's layout, n <= 6)
  bool v4coef = false;         // tensor-core coefficient kernel (planar layout for k_agg3, n <= 6, r <= 9)
  bool v5coef = false;         // horizontal-first coefficient kernel (interleaved layout, n <= 6, r <= 9): default
  CUtensorMap tm_g5;           // TMA descriptor over the raw guide planes of G for k_coef5 (box 164 x 1 x m)
  bool v5agg = false;          // row-marching aggregation k_agg5 (default after k_coef5, n <= 6, r <= 9)
  int nsm = 148;                // SMs of the handle's device
  int lmodel = 0;               // labels of the current call (k_coef5's band height is chosen for it)
  bool v6agg = false;          // warp-specialised aggregation k_agg6 (default on the interleaved layout, n <= 6)
  CUtensorMap tm_w6;           // k_agg6: rank-5 map over wbuf, one-plane box, 64-byte swizzle
  CUtensorMap tm_w5;           // k_agg5: rank-5 map over wbuf, box (16, 4, 6, 1, n + 1), 64-byte swizzle
  CUtensorMap tm_ga5;          // k_agg5: map over G (W, H, n), box (64, 1, n)
  int64_t* fkeys = nullptr;    // k_agg5: the frame's per-pixel minimum keys [H][W] (signed order, hgf.h)
  CUtensorMap tm_g4;           // TMA descriptor over G for k_coef4 (box kCoef4BoxX x 1 x n)
  CUtensorMap tm_g;            // TMA descriptor over G (dims W, H, n; box 88 x 1 x n) for k_coef3
  std::string err;
  // tracing (hgf_set_profiling / hgf_profile_read)
  bool profiling = false;
  struct Rec { int cls; cudaEvent_t a, b; };
  std::vector<Rec> recs;        // recorded since the last read
  std::vector<cudaEvent_t> pool;
};

namespace {

// Every entry point that takes a handle runs on the handle's device (hgf.h: "bound to the CUDA device current
// at create time"): switch to it for the call and restore the caller's current device on return.
// Few-label mode for one call (see hgf_ctx::planar_now): on while the guard lives.
constexpr int kSmallL = 2;
struct SmallLMode {
  hgf_ctx* h;
  SmallLMode(hgf_ctx* hh, int L) : h(hh) {
    const char* e = std::getenv("HGF_SMALL_L");
    if (h) h->planar_now = h->small_ok && L <= kSmallL && !(e && e[0] == '0');
  }
  ~SmallLMode() {
    if (h) h->planar_now = false;
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const hgf_ctx* h) {
    if (h && cudaGetDevice(&prev) == cudaSuccess && prev != h->device) {
      if (cudaSetDevice(h->device) != cudaSuccess) prev = -1;
    } else {
      prev = -1;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

hgf_status fail(hgf_ctx* h, hgf_status s, const std::string& msg) {
  if (h) h->err = msg;
  return s;
}

hgf_status cuda_fail(hgf_ctx* h, cudaError_t e, const char* where) {
  return fail(h, HGF_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

cudaEvent_t take_event(hgf_ctx* h) {
  if (!h->pool.empty()) {
    cudaEvent_t e = h->pool.back();
    h->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Launch wrapper: counts launches and, when tracing, brackets the launch with events.
template <class F>
cudaError_t traced(hgf_ctx* h, int cls, cudaStream_t st, F&& f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (h->profiling) {
    a = take_event(h);
    b = take_event(h);
    cudaEventRecord(a, st);
  }
  cudaError_t e = f();
  if (h->profiling) {
    cudaEventRecord(b, st);
    h->recs.push_back({cls, a, b});
  }
  if (e == cudaSuccess) h->launches++;
  return e;
}

// Coefficient-buffer budget: HGF_COEF_BUDGET_MB, else min(16 GiB, 40% of the free device memory).  The
// v3 coefficient kernel processes labels in batches of 32, so large frames want >= 32 labels per chunk.
size_t coef_budget_bytes() {
  const char* s = std::getenv("HGF_COEF_BUDGET_MB");
  if (s) {
    long long mb = std::atoll(s);
    return (size_t)(mb < 1 ? 1 : mb) << 20;
  }
  size_t fr = 0, tot = 0;
  size_t budget = (size_t)32 << 30;   // <= 40 % of free memory; fewer, larger chunks shorten kernel tails
  if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr / 10 * 4 < budget) budget = fr / 10 * 4;
  return budget < ((size_t)64 << 20) ? ((size_t)64 << 20) : budget;
}

void release(hgf_ctx* h) {
  for (auto& r : h->recs) { h->pool.push_back(r.a); h->pool.push_back(r.b); }
  h->recs.clear();
  for (cudaEvent_t e : h->pool) cudaEventDestroy(e);
  h->pool.clear();
  cudaFree(h->G);
  cudaFree(h->Gp);
  cudaFree(h->vpad);
  cudaFree(h->fkeys);
  cudaFree(h->stats);
  cudaFree(h->wbuf);
  cudaFree(h->best_cost);
  cudaFree(h->best_label);
  cudaFree(h->st_guide);
  cudaFree(h->sv_grad);
  cudaFree(h->sv_cost);
  cudaFree(h->sg_cost);
  cudaFree(h->sg_counts);
  cudaFree(h->pp_int);
  cudaFree(h->pp_valid);
  cudaFree(h->st3_scratch);
  cudaFree(h->st_vol[0]);
  cudaFree(h->st_vol[1]);
  cudaFree(h->st_labels);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->aux) cudaStreamDestroy(h->aux);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_coef[i]) cudaEventDestroy(h->ev_coef[i]);
    if (h->ev_agg[i]) cudaEventDestroy(h->ev_agg[i]);
  }
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_copied[i]) cudaEventDestroy(h->ev_copied[i]);
    if (h->ev_used[i]) cudaEventDestroy(h->ev_used[i]);
  }
}

// Check for an asynchronous fault left by earlier work before enqueueing more.
hgf_status check_async(hgf_ctx* h) {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(h, e, "pending CUDA error");
  }
  return HGF_OK;
}

// Steps 1-2: guidance + label-independent statistics (once per frame).
// Steps 1-2: polynomial guidance (all rows) and the statistics of rows [y0, y1).
hgf_status frame_stats(hgf_ctx* h, const float* guide, int y0, int y1) {
  cudaError_t e = traced(h, HGF_KC_GUIDANCE, h->stream, [&] {
    return hgf::launch_poly_guidance(guide, h->G, h->Gp, h->gp_pitch, h->m, h->d, h->W, h->H, h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "poly_guidance");
  e = traced(h, HGF_KC_STATS, h->stream, [&] {
    const float lam0 = (h->mode == HGF_MODE_HGF) ? (float)h->eps : 0.0f;
    return hgf::launch_stats(h->n, h->G, h->stats, h->W, h->H, h->r, h->eps, h->mode,
                             ((h->v3coef || h->v4coef || h->v5coef) && !h->planar_now) ? 1 : 0, lam0, y0, y1,
                             h->st3_scratch, h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "stats");
  return HGF_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the library does not link libcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D float32 tensor map (x fastest), element strides 1, zero fill out of bounds, no swizzle.
bool encode_map_3d(CUtensorMap* tm, const void* base, long long dx, long long dy, long long dz, long long pitch,
                   long long plane, int bx, int by, int bz) {
  auto encode = tensor_map_encoder();
  if (!encode || ((uintptr_t)base & 15) || ((pitch * 4) & 15) || ((plane * 4) & 15)) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)dx, (cuuint64_t)dy, (cuuint64_t)dz};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)plane * 4};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
  const cuuint32_t es[3] = {1, 1, 1};
  return encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D tensor map over 8-byte elements (the (I, I^2) guide pairs of k_coef5): dims (dx, dy, dz), row pitch and
// plane stride in ELEMENTS, zero fill out of bounds.
bool encode_map_3d_u64(CUtensorMap* tm, const void* base, long long dx, long long dy, long long dz, long long pitch,
                       long long plane, int bx, int by, int bz) {
  auto encode = tensor_map_encoder();
  if (!encode || ((uintptr_t)base & 15) || ((pitch * 8) & 15) || ((plane * 8) & 15)) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)dx, (cuuint64_t)dy, (cuuint64_t)dz};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)plane * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
  const cuuint32_t es[3] = {1, 1, 1};
  return encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K4a for one chunk of Lc slices: the v2 fast path when (m, d, r) allow it, else the generic v1 kernel.
cudaError_t launch_coef_chunk(hgf_ctx* h, const float* guide, const float* vol_chunk, int Lc, float* wdst = nullptr) {
  const float lam0 = (h->mode == HGF_MODE_HGF) ? (float)h->eps : 0.0f;
  if (!wdst) wdst = h->wbuf;
  return traced(h, HGF_KC_COEF, h->stream, [&] {
    if (h->planar_now)
      return hgf::launch_coef_fast(h->m, h->d, guide, h->stats, vol_chunk, h->wbuf, h->wlay_planar, h->W, h->H, h->r,
                                   Lc, lam0, h->stream);
    if (h->v4coef) {
      CUtensorMap tm_vol;
      if (!encode_map_3d(&tm_vol, vol_chunk, h->W, h->H, Lc, (long long)h->W, (long long)h->W * h->H,
                         hgf::kCoef4BoxX, 1, hgf::kCoef4LB))
        return cudaErrorInvalidValue;
      return hgf::launch_coef_v4(h->n, &tm_vol, &h->tm_g4, h->stats, h->wbuf, h->wlay, h->W, h->H, h->r, Lc,
                                 h->stream);
    }
    if (h->v5coef) {
      // TMA descriptor over this chunk's cost slices: dims (W, H, Lc), box 164 x 1 x 32 (k_coef5); rows must be
      // 16-byte multiples, so for W % 4 != 0 the chunk is first copied into rows of ceil4(W) floats (the TMA
      // still reads columns >= W as zero: the tensor's x extent stays W)
      long long pitch = h->W;
      if (h->W % 4) {
        pitch = (h->W + 3) / 4 * 4;
        if (!h->vpad) {
          cudaError_t e = cudaMalloc(&h->vpad, sizeof(float) * (size_t)h->lcap * h->H * pitch);
          if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaMemcpy2DAsync(h->vpad, sizeof(float) * pitch, vol_chunk, sizeof(float) * h->W,
                                          sizeof(float) * h->W, (size_t)h->H * Lc, cudaMemcpyDeviceToDevice, h->stream);
        if (e != cudaSuccess) return e;
        vol_chunk = h->vpad;
      }
      CUtensorMap tm_vol;
      if (!encode_map_3d(&tm_vol, vol_chunk, h->W, h->H, Lc, pitch, pitch * h->H, hgf::kCoef5BoxX, 1,
                         hgf::kCoef5LB))
        return cudaErrorInvalidValue;
      return hgf::launch_coef_v5(h->m, h->d, &tm_vol, &h->tm_g5, h->stats, wdst, h->wlay, h->W, h->H, h->r, Lc,
                                 h->lmodel,
                                 h->stream);
    }
    if (h->v3coef) {
      // TMA descriptor over this chunk's cost slices: dims (W, H, Lc), box 88 x 1 x 32 (k_coef3)
      CUtensorMap tm_vol;
      if (!encode_map_3d(&tm_vol, vol_chunk, h->W, h->H, Lc, (long long)h->W, (long long)h->W * h->H, 88, 1,
                         hgf::coef3_labels(h->n)))
        return cudaErrorInvalidValue;
      return hgf::launch_coef_v3(h->n, &tm_vol, &h->tm_g, h->stats, wdst, h->wlay, h->W, h->H, h->r, Lc, lam0,
                                 h->stream);
    }
    if (h->fast)
      return hgf::launch_coef_fast(h->m, h->d, guide, h->stats, vol_chunk, h->wbuf, h->wlay, h->W, h->H, h->r, Lc, lam0,
                                   h->stream);
    return hgf::launch_coef(h->n, h->G, h->stats, vol_chunk, h->wbuf, h->W, h->H, h->r, Lc, lam0, h->stream);
  });
}

cudaError_t launch_agg_chunk(hgf_ctx* h, const hgf::AggArgs& a, const void* tmaps = nullptr,
                             cudaStream_t st = nullptr) {
  if (h->planar_now)
    return traced(h, HGF_KC_AGG, h->stream, [&] { return hgf::launch_agg_v3(h->n, h->r, h->tm_wp, a, h->stream); });
  if (!tmaps) tmaps = h->planar_now ? h->tm_wp : h->tm_w;
  if (!st) st = h->stream;
  if (st != h->stream) {
    return traced(h, HGF_KC_AGG, st, [&] { return hgf::launch_agg_v3(h->n, h->r, tmaps, a, st); });
  }
  return traced(h, HGF_KC_AGG, h->stream, [&] {
    if (h->v5agg)
      return hgf::launch_agg_v5(h->n, &h->tm_w5, &h->tm_ga5, h->W, h->H, h->r, a.L, a.label_base,
                                hgf::kWGroupLabels, reinterpret_cast<unsigned long long*>(h->fkeys), a.filtered_out,
                                h->stream);
    if (h->v6agg) return hgf::launch_agg_v6(h->m, h->d, h->r, &h->tm_w6, a, h->stream);
    if (h->v3agg) return hgf::launch_agg_v3(h->n, h->r, h->tm_w, a, h->stream);
    return h->fast ? hgf::launch_agg_fast(h->n, a, h->stream) : hgf::launch_agg(h->n, a, h->stream);
  });
}

// TMA descriptor over the coefficient buffer for the v3 aggregation kernel (driver entry point via the
// runtime, so the library does not link libcuda directly).
bool make_wbuf_maps_layout(hgf_ctx* h, float* base, long long labels, const hgf::WLayout& wl, CUtensorMap* out);
bool make_wbuf_maps(hgf_ctx* h, float* base, long long labels, CUtensorMap* out) {
  return make_wbuf_maps_layout(h, base, labels, h->wlay, out);
}
bool make_wbuf_tensor_map(hgf_ctx* h) { return make_wbuf_maps(h, h->wbuf, h->lcap, h->tm_w); }

bool make_wbuf_maps_layout(hgf_ctx* h, float* base, long long labels, const hgf::WLayout& wl, CUtensorMap* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      !fn || q != cudaDriverEntryPointSuccess)
    return false;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  // HGF_TMA_L2PROMO = none | 64 | 128 (default) | 256: L2 sector promotion of the coefficient-tile loads
  // (tuning knob for the interleaved layouts, whose inner runs are 32 or 64 bytes)
  auto wmap_l2_promotion = [] {
    const char* e = std::getenv("HGF_TMA_L2PROMO");
    if (e && !strcmp(e, "none")) return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    if (e && !strcmp(e, "64")) return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    if (e && !strcmp(e, "256")) return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  };
  int bx = 0, by = 0;
  hgf::agg3_box(h->n, h->r, wl.il, &bx, &by);
  const int K = h->n + 1, KA = hgf::agg3_ka(K);
  for (int grp = 0; grp < 2; ++grp) {
    const cuuint32_t planes = (cuuint32_t)(grp == 0 ? KA : K - KA);
    CUresult r;
    if (wl.il) {
      // rank 5 over the label-interleaved layout: (G px, 32 labels, x groups, y, label-batch planes); one
      // box = one label's planes of a BX x BY tile, 4G-byte inner runs, 64-byte swizzle (k_agg3's swz)
      const cuuint64_t G = hgf::kWGroupPx, NL = hgf::kWGroupLabels;
      const cuuint64_t dims[5] = {G, NL, (cuuint64_t)wl.xg, (cuuint64_t)h->H,
                                  (cuuint64_t)(labels / hgf::kWGroupLabels) * K};
      const cuuint64_t strides[4] = {G * 4, G * NL * 4, G * NL * 4 * wl.xg, G * NL * 4 * wl.xg * h->H};
      const cuuint32_t box[5] = {(cuuint32_t)G, 1, (cuuint32_t)(bx / G), (cuuint32_t)by, planes};
      const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
      r = encode(&out[grp], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, base, dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE,
                 hgf::kWGroupPx == 8 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B, wmap_l2_promotion(),
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      const cuuint64_t dims[3] = {(cuuint64_t)(h->W + wl.pad), (cuuint64_t)(h->H + wl.pad),
                                  (cuuint64_t)labels * K};
      const cuuint64_t strides[2] = {(cuuint64_t)wl.pitch * 4, (cuuint64_t)wl.plane * 4};
      const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, planes};
      const cuuint32_t estr[3] = {1, 1, 1};
      r = encode(&out[grp], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return false;
  }
  return true;
}

// Steps 3-4 over labels [0, L) of vol, chunked by the coefficient buffer capacity.  build_chunk (optional)
// constructs the chunk's slices [c0, c0 + Lc) and returns their device pointer instead of vol + c0 HW.
template <class BuildChunk>
hgf_status slices_impl(hgf_ctx* h, const float* guide, const float* vol, int L, int label_offset, float* filtered_out,
                       int do_wta, int32_t* labels_out, float* min_cost_out, int64_t* keys_out, BuildChunk build_chunk) {
  const long long HW = (long long)h->W * h->H;
  h->lmodel = L;
  // opt-in (HGF_PIPELINE=1): measured slower at C4 (36.3 vs 35.2 ms: the overlapped kernels slow each other down
  // -- coef 14.8 -> 20.5 ms, agg 19.2 -> 27.3 ms of device time -- on top of 4 chunks' tails instead of 2)
  const bool pipe_env = std::getenv("HGF_PIPELINE") && std::getenv("HGF_PIPELINE")[0] == '1';
  if (h->half > 0 && !h->v5agg && !h->planar_now && L > h->half && pipe_env) {
    // ---- two-stream chunk pipeline: chunk c's coefficients go to half c % 2 of the buffer on the handle's
    // stream while chunk c - 1 is aggregated on the aux stream (the coefficient kernel is DRAM-bound, the
    // aggregation shared-memory-bound: running them side by side overlaps the two limits)
    cudaError_t e = cudaSuccess;
    if (!h->aux) {
      if ((e = cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(h, e, "aux stream");
      for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&h->ev_coef[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_agg[i], cudaEventDisableTiming);
      }
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(h, e, "pipeline events");
    }
    const int K = h->n + 1;
    const long long half_floats =
        (long long)(h->half / hgf::kWGroupLabels) * K * h->H * h->wlay.xg * (hgf::kWGroupPx * hgf::kWGroupLabels);
    const int nchunks = (L + h->half - 1) / h->half;
    int step = (L + nchunks - 1) / nchunks;
    step = (step + hgf::kWGroupLabels - 1) / hgf::kWGroupLabels * hgf::kWGroupLabels;
    if (step > h->half) step = h->half;
    int ci = 0;
    for (int c0 = 0; c0 < L; c0 += step, ++ci) {
      const int Lc = (L - c0 < step) ? (L - c0) : step;
      const int b = ci & 1;
      const float* chunk = vol ? vol + (long long)c0 * HW : nullptr;
      e = build_chunk(c0, Lc, &chunk);
      if (e != cudaSuccess) return cuda_fail(h, e, "cost construction");
      if (ci >= 2 && (e = cudaStreamWaitEvent(h->stream, h->ev_agg[b], 0)) != cudaSuccess)
        return cuda_fail(h, e, "wait half free");
      e = launch_coef_chunk(h, guide, chunk, Lc, h->wbuf + b * half_floats);
      if (e != cudaSuccess) return cuda_fail(h, e, "coef");
      if ((e = cudaEventRecord(h->ev_coef[b], h->stream)) != cudaSuccess ||
          (e = cudaStreamWaitEvent(h->aux, h->ev_coef[b], 0)) != cudaSuccess)
        return cuda_fail(h, e, "coef -> agg");
      hgf::AggArgs a{};
      a.G = h->G;
      a.wbuf = h->wbuf + b * half_floats;
      a.W = h->W; a.H = h->H; a.r = h->r; a.L = Lc; a.pad = h->wlay.pad; a.il = h->wlay.il;
      a.label_base = label_offset + c0;
      a.filtered_out = filtered_out ? filtered_out + (long long)c0 * HW : nullptr;
      a.do_wta = do_wta;
      a.first = (c0 == 0);
      a.last = (c0 + Lc >= L);
      a.best_cost = h->best_cost;
      a.best_label = h->best_label;
      a.labels_out = labels_out;
      a.min_cost_out = min_cost_out;
      a.keys_out = keys_out;
      a.peer_keys = h->peer_keys;
      a.rows_per_owner = h->rows_per_owner;
      e = launch_agg_chunk(h, a, h->tm_wh[b], h->aux);
      if (e != cudaSuccess) return cuda_fail(h, e, "agg");
      if ((e = cudaEventRecord(h->ev_agg[b], h->aux)) != cudaSuccess) return cuda_fail(h, e, "record agg");
    }
    if ((e = cudaEventRecord(h->ev_join, h->aux)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(h->stream, h->ev_join, 0)) != cudaSuccess)
      return cuda_fail(h, e, "join");
    return HGF_OK;
  }
  // balanced chunks (e.g. 256 labels with a 147-label capacity -> 2 x 128, not 128 + 128 + ... tails)
  const int nchunks = (L + h->lcap - 1) / h->lcap;
  int step = (L + nchunks - 1) / nchunks;
  step = (step + hgf::kWGroupLabels - 1) / hgf::kWGroupLabels * hgf::kWGroupLabels;
  if (step > h->lcap) step = h->lcap;
  // small frames on k_agg6 (fewer tiles than ~1.5 waves): split each tile's labels over several CTAs, merged by
  // 64-bit atomic MIN into the frame's key buffer (HGF_AGG6_SPLIT=0: off)
  const char* se = std::getenv("HGF_AGG6_SPLIT");
  const bool split6 = h->v6agg && !h->planar_now && do_wta && !(se && se[0] == '0') &&
                      hgf::agg6_split(h->W, h->H, h->r, step < L ? step : L, h->nsm) > 1;
  if (split6 && !h->fkeys) {
    cudaError_t e = cudaMalloc(&h->fkeys, sizeof(int64_t) * HW);
    if (e != cudaSuccess) {
      cudaGetLastError();
      h->fkeys = nullptr;
      return cuda_fail(h, e, "key buffer");
    }
  }
  const bool keyed = (h->v5agg || split6) && !h->planar_now && do_wta;
  if (keyed) {
    // k_agg5 / split k_agg6 merge every CTA's minima into the frame's key buffer: start from the MIN identity
    cudaError_t e = traced(h, HGF_KC_KEYS, h->stream,
                           [&] { return hgf::launch_fill_i64(h->fkeys, HW, 0x7fffffffffffffffLL, h->stream); });
    if (e != cudaSuccess) return cuda_fail(h, e, "keys fill");
  }
  for (int c0 = 0; c0 < L; c0 += step) {
    const int Lc = (L - c0 < step) ? (L - c0) : step;
    const float* chunk = vol ? vol + (long long)c0 * HW : nullptr;
    cudaError_t e = build_chunk(c0, Lc, &chunk);
    if (e != cudaSuccess) return cuda_fail(h, e, "cost construction");
    e = launch_coef_chunk(h, guide, chunk, Lc);
    if (e != cudaSuccess) return cuda_fail(h, e, "coef");
    hgf::AggArgs a{};
    const hgf::WLayout& wl = h->planar_now ? h->wlay_planar : h->wlay;
    a.G = h->G;
    a.wbuf = h->wbuf;
    a.W = h->W; a.H = h->H; a.r = h->r; a.L = Lc; a.pad = wl.pad; a.il = wl.il;
    a.label_base = label_offset + c0;
    a.filtered_out = filtered_out ? filtered_out + (long long)c0 * HW : nullptr;
    a.do_wta = do_wta;
    a.first = (c0 == 0);
    a.last = (c0 + Lc >= L);
    a.best_cost = h->best_cost;
    a.best_label = h->best_label;
    a.labels_out = labels_out;
    a.min_cost_out = min_cost_out;
    a.keys_out = keys_out;
    a.peer_keys = h->peer_keys;
    a.rows_per_owner = h->rows_per_owner;
    if (split6) {
      a.fkeys = reinterpret_cast<long long*>(h->fkeys);
      a.nsplit = hgf::agg6_split(h->W, h->H, h->r, Lc, h->nsm);
    }
    e = launch_agg_chunk(h, a);
    if (e != cudaSuccess) return cuda_fail(h, e, "agg");
  }
  if (keyed && (labels_out || min_cost_out || keys_out || h->peer_keys)) {
    cudaError_t e = traced(h, HGF_KC_KEYS, h->stream, [&] {
      return hgf::launch_keys_finalize(h->fkeys, h->W, h->H, labels_out, min_cost_out, keys_out, h->peer_keys,
                                       h->rows_per_owner, h->stream);
    });
    if (e != cudaSuccess) return cuda_fail(h, e, "keys finalize");
  }
  return HGF_OK;
}

hgf_status slices(hgf_ctx* h, const float* guide, const float* vol, int L, int label_offset, float* filtered_out,
                  int do_wta, int32_t* labels_out, float* min_cost_out, int64_t* keys_out) {
  return slices_impl(h, guide, vol, L, label_offset, filtered_out, do_wta, labels_out, min_cost_out, keys_out,
                     [](int, int, const float**) { return cudaSuccess; });
}

// The fused single-slice pass (one slice, few-label mode on): guidance, then the statistics pass that also sums the
// slice's cost products and writes its coefficients (no statistics in HBM, no coefficient kernel), then the planar
// aggregation with the requested outputs.  Returns false (nothing enqueued) where it does not apply.
bool fused_single_ok(hgf_ctx* h) {
  const char* fe = std::getenv("HGF_FILTER_FUSED");
  const hgf::WLayout& wl = h->planar_now ? h->wlay_planar : h->wlay;
  return !wl.il && !(fe && fe[0] == '0') && h->n <= hgf::kStats4MaxN && 64 + 2 * h->r <= 128 &&
         hgf::stats4_smem(h->n, h->r, 1) <= 200 * 1024;
}

hgf_status fused_single(hgf_ctx* h, const float* guide, const float* src, int label_offset, float* filtered_out,
                        int do_wta, int32_t* labels_out, float* min_cost_out, int64_t* keys_out) {
  const hgf::WLayout& wl = h->planar_now ? h->wlay_planar : h->wlay;
  cudaError_t e = traced(h, HGF_KC_GUIDANCE, h->stream, [&] {
    return hgf::launch_poly_guidance(guide, h->G, h->Gp, h->gp_pitch, h->m, h->d, h->W, h->H, h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "poly_guidance");
  e = traced(h, HGF_KC_STATS, h->stream, [&] {
    const float lam0 = (h->mode == HGF_MODE_HGF) ? (float)h->eps : 0.0f;
    return hgf::launch_filter1(h->n, h->G, src, h->wbuf, wl, h->W, h->H, h->r, h->eps, h->mode, lam0, h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "fused statistics + coefficients");
  hgf::AggArgs a{};
  a.G = h->G;
  a.wbuf = h->wbuf;
  a.W = h->W; a.H = h->H; a.r = h->r; a.L = 1; a.pad = wl.pad; a.il = 0;
  a.label_base = label_offset;
  a.filtered_out = filtered_out;
  a.do_wta = do_wta;
  a.first = 1;
  a.last = 1;
  a.best_cost = h->best_cost;
  a.best_label = h->best_label;
  a.labels_out = labels_out;
  a.min_cost_out = min_cost_out;
  a.keys_out = keys_out;
  a.peer_keys = h->peer_keys;
  a.rows_per_owner = h->rows_per_owner;
  e = launch_agg_chunk(h, a);
  if (e != cudaSuccess) return cuda_fail(h, e, "agg");
  return HGF_OK;
}

}  // namespace

extern "C" {

const char* hgf_status_string(hgf_status s) {
  switch (s) {
    case HGF_OK: return "HGF_OK";
    case HGF_ERR_INVALID_ARGUMENT: return "HGF_ERR_INVALID_ARGUMENT";
    case HGF_ERR_UNSUPPORTED: return "HGF_ERR_UNSUPPORTED";
    case HGF_ERR_OUT_OF_MEMORY: return "HGF_ERR_OUT_OF_MEMORY";
    case HGF_ERR_CUDA: return "HGF_ERR_CUDA";
  }
  return "HGF_ERR_UNKNOWN";
}

const char* hgf_last_error(hgf_handle h) { return h ? h->err.c_str() : "null handle"; }

int hgf_last_launch_count(hgf_handle h) { return h ? h->launches : 0; }

const char* hgf_kernel_path(hgf_handle h) {
  if (!h) return "";
  if (h->v3agg) {
    if (h->v5agg) return "coef5+agg5";
    if (h->v5coef) return h->v6agg ? "coef5+agg6" : "coef5+agg3";
    if (h->v4coef) return "coef4+agg3";
    if (h->v3coef) return h->v6agg ? "coef3+agg6" : "coef3+agg3";
    return "coef2+agg3";
  }
  return h->fast ? "coef2+agg2" : "coef1+agg1";
}

hgf_status hgf_create_ex(hgf_handle* out, int W, int H, int n_guide, int poly_degree, int radius, double eps,
                         int mode, void* cuda_stream) {
  if (!out) return HGF_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (W < 1 || H < 1 || n_guide < 1 || poly_degree < 1 || radius < 1) return HGF_ERR_INVALID_ARGUMENT;
  if (!(eps > 0.0) || !std::isfinite(eps)) return HGF_ERR_INVALID_ARGUMENT;
  if (mode != HGF_MODE_HGF && mode != HGF_MODE_GF) return HGF_ERR_INVALID_ARGUMENT;
  if ((long long)W * H > (1LL << 31)) return HGF_ERR_UNSUPPORTED;
  if ((long long)n_guide * poly_degree > HGF_MAX_CHANNELS || radius > HGF_MAX_RADIUS) return HGF_ERR_UNSUPPORTED;
  hgf_ctx* h = new hgf_ctx();
  h->W = W; h->H = H; h->m = n_guide; h->d = poly_degree; h->n = n_guide * poly_degree;
  h->r = radius; h->eps = eps; h->mode = mode;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  cudaGetDevice(&h->device);
  cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->device);
  const size_t HW = (size_t)W * H;
  const int K = h->n + 1;
  {
    const char* f = std::getenv("HGF_FORCE_V1");
    h->fast = hgf::fast_path_ok(h->m, h->d, h->r) && !(f && f[0] == '1');
    const char* g = std::getenv("HGF_NO_V3");
    h->v3agg = h->fast && h->n <= 9 && !(g && g[0] == '1');     // confirmed below once the TMA map exists
  }
  cudaError_t e = cudaSuccess;
  if ((e = cudaMalloc(&h->G, sizeof(float) * h->n * HW)) != cudaSuccess ||
      (e = cudaMalloc(&h->stats, sizeof(float) * std::max(hgf::stats_planes(h->n), hgf::stats_aos_floats(h->n)) * HW)) !=
          cudaSuccess) {
    cudaGetLastError();
    release(h);
    delete h;
    return e == cudaErrorMemoryAllocation ? HGF_ERR_OUT_OF_MEMORY : HGF_ERR_CUDA;
  }
  {
    // default: k_coef3; HGF_COEF4=1 selects k_coef4 (tensor cores), HGF_COEF3=0 k_coef2
    const char* f4 = std::getenv("HGF_COEF4");
    h->v4coef = h->v3agg && h->n <= 6 && (W % 4) == 0 && h->r <= 9 && (f4 && f4[0] == '1') &&
                encode_map_3d(&h->tm_g4, h->G, W, H, h->n, W, (long long)W * H, hgf::kCoef4BoxX, 1, h->n);
    const char* f = std::getenv("HGF_COEF3");
    h->v3coef = !h->v4coef && h->v3agg && h->n <= hgf::kCoef3MaxN && (W % 4) == 0 && !(f && f[0] == '0') &&
                encode_map_3d(&h->tm_g, h->G, W, H, h->n, W, (long long)W * H, 88, 1, h->n);
    // k_coef5 (default where it applies; HGF_COEF5=0 keeps k_coef3): same interleaved layout as k_coef3
    const char* f5 = std::getenv("HGF_COEF5");
    // tm_g5: d = 2: the (I_i, I_i^2) pairs [H][m][W] as 8-byte elements, dims (W, m, H); other degrees: the raw
    // guide channels I_i = G_{(i-1)d+1} (every d-th plane of the guidance buffer), dims (W, H, m)
    // W % 4 != 0 (the paper's 450-column Middlebury frames, BASELINE config 2): each chunk of the cost volume is
    // first copied into a pitched scratch (rows of ceil4(W) floats, the TMA stride rule) -- degree 2 only, whose
    // guide pairs have their own pitched buffer
    h->v5coef = h->v3agg && !h->v4coef && hgf::coef5_ok(h->m, h->d, h->r) && !(f5 && f5[0] == '0') &&
                !(f && f[0] == '0') && ((W % 4) == 0 || h->d == 2);
    h->gp_pitch = W + (W & 1);                 // guide pairs: 8-byte elements, rows of 16-byte multiples
    if (h->v5coef && h->d == 2) {
      if (cudaMalloc(&h->Gp, sizeof(float) * 2 * h->m * (size_t)h->gp_pitch * H) != cudaSuccess) {
        cudaGetLastError();
        h->Gp = nullptr;
      }
      h->v5coef = h->Gp && encode_map_3d_u64(&h->tm_g5, h->Gp, W, h->m, H, h->gp_pitch, (long long)h->gp_pitch * h->m,
                                             hgf::kCoef5BoxX, h->m, 1);
    } else if (h->v5coef) {
      h->v5coef = encode_map_3d(&h->tm_g5, h->G, W, H, h->m, W, (long long)W * H * h->d, hgf::kCoef5BoxX, 1, h->m);
    }
  }
  // coefficient buffer layout: label-interleaved for k_coef3 -> k_agg3, else rows pitched to a multiple of
  // 4 floats for the TMA aggregation, else flat
  const hgf::WLayout flat{0, (long long)HW, W, 0, 0, 0};
  hgf::WLayout padded{};
  padded.pad = 0;
  padded.pitch = (W + 3) / 4 * 4;       // 16-byte rows: TMA global strides
  padded.plane = (long long)H * padded.pitch;
  padded.origin = 0;
  hgf::WLayout inter{};
  inter.il = 1;
  inter.xg = (W + hgf::kWGroupPx - 1) / hgf::kWGroupPx;
  inter.plane = (long long)H * inter.xg * hgf::kWGroupPx;   // floats per (label, plane) slot
  inter.pitch = inter.xg * hgf::kWGroupPx;
  hgf::WLayout lines = padded;          // k_coef4: rows start on 128-byte lines (one line per warp store)
  lines.pitch = (W + 31) / 32 * 32;
  lines.plane = (long long)H * lines.pitch;
  h->wlay = (h->v3coef || h->v5coef) ? inter : (h->v4coef ? lines : (h->v3agg ? padded : flat));
  const size_t per_label = (size_t)K * (size_t)h->wlay.plane * sizeof(float);
  size_t cap = coef_budget_bytes() / per_label;
  cap = cap < 1 ? 1 : (cap > 4096 ? 4096 : cap);
  if (h->wlay.il) cap = cap < (size_t)hgf::kWGroupLabels ? hgf::kWGroupLabels : cap / hgf::kWGroupLabels * hgf::kWGroupLabels;
  h->lcap = (int)cap;
  if ((e = cudaMalloc(&h->wbuf, per_label * h->lcap)) != cudaSuccess ||
      (e = cudaMalloc(&h->best_cost, sizeof(float) * HW)) != cudaSuccess ||
      (e = cudaMalloc(&h->best_label, sizeof(int32_t) * HW)) != cudaSuccess ||
      (e = cudaMemset(h->wbuf, 0, per_label * h->lcap)) != cudaSuccess) {
    cudaGetLastError();
    release(h);
    delete h;
    return e == cudaErrorMemoryAllocation ? HGF_ERR_OUT_OF_MEMORY : HGF_ERR_CUDA;
  }
  if (h->n >= 7) {
    // optional: without it the statistics fall back to k_stats2 / k_stats (register-spilling at large n)
    if (cudaMalloc(&h->st3_scratch, sizeof(double) * hgf::stats3_scratch_planes(h->n) * HW) != cudaSuccess) {
      cudaGetLastError();
      h->st3_scratch = nullptr;
    }
  }
  if (h->v3agg && !((long long)h->lcap * K <= (1LL << 31) && make_wbuf_tensor_map(h))) {
    // no TMA descriptor: v2 coefficients + aggregation on the flat layout (fits the allocation)
    h->v3agg = false;
    h->v3coef = false;
    h->v4coef = false;
    h->v5coef = false;
    h->wlay = flat;
  }
  if (h->v3agg && h->wlay.il && h->fast) {
    // the planar layout in the same buffer (pitch ceil4(W) <= 16 ceil(W/16): fits every interleaved slot)
    h->wlay_planar = padded;
    h->small_ok = make_wbuf_maps_layout(h, h->wbuf, h->lcap, h->wlay_planar, h->tm_wp);
  }
  if (h->v3agg && h->wlay.il && h->lcap >= 2 * hgf::kWGroupLabels) {
    // the two halves of the coefficient buffer for the two-stream chunk pipeline (slices_impl)
    h->half = (h->lcap / 2) / hgf::kWGroupLabels * hgf::kWGroupLabels;
    const long long half_floats =
        (long long)(h->half / hgf::kWGroupLabels) * K * H * h->wlay.xg * (hgf::kWGroupPx * hgf::kWGroupLabels);
    if (!(make_wbuf_maps(h, h->wbuf, h->half, h->tm_wh[0]) &&
          make_wbuf_maps(h, h->wbuf + half_floats, h->half, h->tm_wh[1])))
      h->half = 0;
  }
  {
    // k_agg5 (opt-in, HGF_AGG5=1: parity-green but slower than k_agg3 at C4 -- 32 vs 19 ms)
    const char* f = std::getenv("HGF_AGG5");
    h->v5agg = h->v5coef && h->v3agg && h->n <= hgf::kAgg5MaxN && h->r <= 9 && (f && f[0] == '1');
    if (h->v5agg) {
      auto encode = tensor_map_encoder();
      const cuuint64_t G = hgf::kWGroupPx, NL = hgf::kWGroupLabels;
      const cuuint64_t dims[5] = {G, NL, (cuuint64_t)h->wlay.xg, (cuuint64_t)H,
                                  (cuuint64_t)(h->lcap / hgf::kWGroupLabels) * K};
      const cuuint64_t strides[4] = {G * 4, G * NL * 4, G * NL * 4 * h->wlay.xg, G * NL * 4 * h->wlay.xg * H};
      const cuuint32_t box[5] = {(cuuint32_t)G, (cuuint32_t)hgf::kAgg5LB, 6, 1, (cuuint32_t)K};
      const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
      h->v5agg = encode &&
                 encode(&h->tm_w5, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, h->wbuf, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
                 encode_map_3d(&h->tm_ga5, h->G, W, H, h->n, W, (long long)W * H, 64, 1, h->n);
      if (h->v5agg && cudaMalloc(&h->fkeys, sizeof(int64_t) * HW) != cudaSuccess) {
        cudaGetLastError();
        h->fkeys = nullptr;
        h->v5agg = false;
      }
    }
  }
  if (h->v3agg && h->wlay.il && !h->v5agg && h->n <= hgf::kAgg6MaxN && h->r <= 9 && hgf::kWGroupPx == 16) {
    // k_agg6 (default; HGF_AGG6=0 keeps k_agg3): the same tile with one TMA box per coefficient plane
    const char* f = std::getenv("HGF_AGG6");
    auto encode = tensor_map_encoder();
    const cuuint64_t G = hgf::kWGroupPx, NL = hgf::kWGroupLabels;
    const cuuint64_t dims[5] = {G, NL, (cuuint64_t)h->wlay.xg, (cuuint64_t)H,
                                (cuuint64_t)(h->lcap / hgf::kWGroupLabels) * K};
    const cuuint64_t strides[4] = {G * 4, G * NL * 4, G * NL * 4 * h->wlay.xg, G * NL * 4 * h->wlay.xg * H};
    const cuuint32_t box[5] = {(cuuint32_t)G, 1, (cuuint32_t)((64 + 2 * h->r + 31) / 32 * 32 / G),
                               (cuuint32_t)(hgf::kAgg6TY + 2 * h->r), 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    h->v6agg = !(f && f[0] == '0') && encode &&
               encode(&h->tm_w6, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, h->wbuf, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  *out = h;
  return HGF_OK;
}

hgf_status hgf_create(hgf_handle* out, int W, int H, int n_guide, int poly_degree, int radius, double eps) {
  return hgf_create_ex(out, W, H, n_guide, poly_degree, radius, eps, HGF_MODE_HGF, nullptr);
}

hgf_status hgf_destroy(hgf_handle h) {
  DeviceGuard dg(h);
  if (!h) return HGF_OK;
  cudaStreamSynchronize(h->stream);
  if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
  release(h);
  delete h;
  return HGF_OK;
}

hgf_status hgf_set_stream(hgf_handle h, void* cuda_stream) {
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  return HGF_OK;
}

hgf_status hgf_filter(hgf_handle h, const float* guide, const float* src, float* dst) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!guide || !src || !dst) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null pointer");
  if (dst == src || dst == guide) return fail(h, HGF_ERR_INVALID_ARGUMENT, "dst aliases an input");
  hgf_status s = check_async(h);
  if (s != HGF_OK) return s;
  SmallLMode sm(h, 1);
  if (fused_single_ok(h)) return fused_single(h, guide, src, 0, dst, 0, nullptr, nullptr, nullptr);
  if ((s = frame_stats(h, guide, 0, h->H)) != HGF_OK) return s;
  return slices(h, guide, src, 1, 0, dst, 0, nullptr, nullptr, nullptr);
}

hgf_status hgf_aggregate_wta_ex(hgf_handle h, const float* guide, const float* cost_volume, int L, int label_offset,
                                int32_t* labels_out, float* min_cost_out, float* filtered_out, int64_t* keys_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!guide || !cost_volume) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null input pointer");
  if (L < 1) return fail(h, HGF_ERR_INVALID_ARGUMENT, "L must be >= 1");
  if (label_offset < 0 || (long long)label_offset + L > 2147483647LL)
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "label_offset out of range");
  if (!labels_out && !min_cost_out && !filtered_out && !keys_out)
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "no output requested");
  hgf_status s = check_async(h);
  if (s != HGF_OK) return s;
  SmallLMode sm(h, L);
  const int do_wta = (labels_out || min_cost_out || keys_out) ? 1 : 0;
  // one slice: the fused single-slice pass (as hgf_filter), the WTA over the one label in its aggregation
  if (L == 1 && fused_single_ok(h))
    return fused_single(h, guide, cost_volume, label_offset, filtered_out, do_wta, labels_out, min_cost_out, keys_out);
  if ((s = frame_stats(h, guide, 0, h->H)) != HGF_OK) return s;
  return slices(h, guide, cost_volume, L, label_offset, filtered_out, do_wta, labels_out, min_cost_out, keys_out);
}

hgf_status hgf_prepare_rows(hgf_handle h, const float* guide, int y0, int y1) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!guide) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null guide");
  if (y0 < 0 || y1 > h->H || y0 > y1) return fail(h, HGF_ERR_INVALID_ARGUMENT, "row band out of range");
  if (!(h->v3coef || h->v4coef || h->v5coef))
    return fail(h, HGF_ERR_UNSUPPORTED, "row-band statistics need the per-pixel statistics layout (n <= 6, W % 4 == 0)");
  hgf_status s = check_async(h);
  if (s != HGF_OK) return s;
  return frame_stats(h, guide, y0, y1);
}

hgf_status hgf_stats_buffer(hgf_handle h, void** dev_ptr, size_t* bytes_per_row) {
  DeviceGuard dg(h);
  if (!h || !dev_ptr || !bytes_per_row) return HGF_ERR_INVALID_ARGUMENT;
  if (!(h->v3coef || h->v4coef || h->v5coef))
    return fail(h, HGF_ERR_UNSUPPORTED, "statistics are not stored row-contiguously in this configuration");
  *dev_ptr = h->stats;
  *bytes_per_row = sizeof(float) * (size_t)hgf::stats_aos_floats(h->n) * h->W;
  return HGF_OK;
}

hgf_status hgf_aggregate_wta_prepared(hgf_handle h, const float* cost_volume, int L, int label_offset,
                                      int32_t* labels_out, float* min_cost_out, float* filtered_out,
                                      int64_t* keys_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!cost_volume) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null input pointer");
  if (L < 1) return fail(h, HGF_ERR_INVALID_ARGUMENT, "L must be >= 1");
  if (label_offset < 0 || (long long)label_offset + L > 2147483647LL)
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "label_offset out of range");
  if (!labels_out && !min_cost_out && !filtered_out && !keys_out)
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "no output requested");
  if (!(h->v3coef || h->v4coef || h->v5coef))
    return fail(h, HGF_ERR_UNSUPPORTED, "prepared statistics need the k_coef3/4/5 path");
  hgf_status s = check_async(h);
  if (s != HGF_OK) return s;
  const int do_wta = (labels_out || min_cost_out || keys_out) ? 1 : 0;
  return slices(h, nullptr, cost_volume, L, label_offset, filtered_out, do_wta, labels_out, min_cost_out, keys_out);
}

}  // extern "C"

namespace {

// hgf_stereo_wta (dir = +1: guide = left view, match at x - d) and hgf_stereo_wta_right (dir = -1: guide =
// right view, match at x + d, reading P1).  `base` is the guide view, `other` the searched one.
hgf_status stereo_impl(hgf_ctx* h, const float* base, const float* other, int dir, int L, int label_offset,
                       float alpha, float tau_color, float tau_grad, int32_t* labels_out, float* min_cost_out,
                       float* filtered_out, int64_t* keys_out) {
  if (!base || !other) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null view pointer");
  if (h->m != 3) return fail(h, HGF_ERR_INVALID_ARGUMENT, "stereo needs a 3-channel guide (n_guide = 3)");
  if (L < 1) return fail(h, HGF_ERR_INVALID_ARGUMENT, "L must be >= 1");
  if (label_offset < 0 || (long long)label_offset + L > 2147483647LL)
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "label_offset out of range");
  if (!(alpha >= 0.0f && alpha <= 1.0f) || !(tau_color >= 0.0f) || !(tau_grad >= 0.0f) || !std::isfinite(tau_color) ||
      !std::isfinite(tau_grad))
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "cost parameters: 0 <= alpha <= 1, finite non-negative thresholds");
  if (!labels_out && !min_cost_out && !filtered_out && !keys_out)
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "no output requested");
  const size_t HW = (size_t)h->W * h->H;
  cudaError_t e;
  if (!h->sv_grad) {
    if ((e = cudaMalloc(&h->sv_grad, sizeof(float) * 2 * HW)) != cudaSuccess ||
        (e = cudaMalloc(&h->sv_cost, sizeof(float) * HW * (size_t)h->lcap)) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(h->sv_grad);
      h->sv_grad = nullptr;
      return fail(h, e == cudaErrorMemoryAllocation ? HGF_ERR_OUT_OF_MEMORY : HGF_ERR_CUDA, "cost scratch allocation");
    }
  }
  hgf_status s = check_async(h);
  if (s != HGF_OK) return s;
  if ((s = frame_stats(h, base, 0, h->H)) != HGF_OK) return s;
  e = traced(h, HGF_KC_COST, h->stream, [&] {
    cudaError_t e2 = hgf::launch_stereo_grad(base, h->sv_grad, h->W, h->H, h->stream);
    return e2 != cudaSuccess ? e2 : hgf::launch_stereo_grad(other, h->sv_grad + HW, h->W, h->H, h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "stereo gradients");
  const int do_wta = (labels_out || min_cost_out || keys_out) ? 1 : 0;
  return slices_impl(h, base, nullptr, L, label_offset, filtered_out, do_wta, labels_out, min_cost_out, keys_out,
                     [&](int c0, int Lc, const float** chunk) {
                       *chunk = h->sv_cost;
                       return traced(h, HGF_KC_COST, h->stream, [&] {
                         return hgf::launch_stereo_cost(base, other, h->sv_grad, h->sv_grad + HW, h->sv_cost, h->W,
                                                        h->H, label_offset + c0, Lc, dir, alpha, tau_color, tau_grad,
                                                        h->stream);
                       });
                     });
}

hgf_status pp_scratch(hgf_ctx* h) {
  const size_t HW = (size_t)h->W * h->H;
  cudaError_t e;
  if (!h->pp_int) {
    if ((e = cudaMalloc(&h->pp_int, sizeof(int32_t) * 3 * HW)) != cudaSuccess ||
        (e = cudaMalloc(&h->pp_valid, HW)) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(h->pp_int);
      h->pp_int = nullptr;
      return fail(h, e == cudaErrorMemoryAllocation ? HGF_ERR_OUT_OF_MEMORY : HGF_ERR_CUDA,
                  "post-processing scratch allocation");
    }
  }
  return HGF_OK;
}

// Readings P2-P4 on device maps (the caller has checked the arguments).
hgf_status postprocess_impl(hgf_ctx* h, const float* image, const int32_t* dL, const int32_t* dR, int tol, int radius,
                            float sigma_s, float sigma_c, uint8_t* valid_out, int32_t* disp_out) {
  hgf_status s = pp_scratch(h);
  if (s != HGF_OK) return s;
  cudaError_t e;
  uint8_t* valid = valid_out ? valid_out : h->pp_valid;
  int* fill = h->pp_int;
  e = traced(h, HGF_KC_POST, h->stream, [&] {
    cudaError_t e2 = hgf::launch_lr_fill(dL, dR, h->W, h->H, tol, valid, fill, h->stream);
    return e2 != cudaSuccess ? e2
                             : hgf::launch_wmf(fill, valid, image, h->m, h->W, h->H, radius, sigma_s, sigma_c, disp_out,
                                               h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "post-processing");
  return HGF_OK;
}

hgf_status check_pp_args(hgf_ctx* h, int tol, int radius, float sigma_s, float sigma_c) {
  if (tol < 0) return fail(h, HGF_ERR_INVALID_ARGUMENT, "tol must be >= 0");
  if (radius < 0 || radius > hgf::lr_wmf_max_radius())
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "weighted-median radius must be in [0, 15]");
  if (!(sigma_s > 0.0f) || !(sigma_c > 0.0f) || !std::isfinite(sigma_s) || !std::isfinite(sigma_c))
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "sigma_s and sigma_c must be finite and > 0");
  return HGF_OK;
}

}  // namespace

extern "C" {

hgf_status hgf_stereo_wta(hgf_handle h, const float* left, const float* right, int L, int label_offset,
                          float alpha, float tau_color, float tau_grad, int32_t* labels_out, float* min_cost_out,
                          float* filtered_out, int64_t* keys_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  return stereo_impl(h, left, right, +1, L, label_offset, alpha, tau_color, tau_grad, labels_out, min_cost_out,
                     filtered_out, keys_out);
}

hgf_status hgf_stereo_wta_right(hgf_handle h, const float* left, const float* right, int L, int label_offset,
                                float alpha, float tau_color, float tau_grad, int32_t* labels_out,
                                float* min_cost_out, float* filtered_out, int64_t* keys_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  return stereo_impl(h, right, left, -1, L, label_offset, alpha, tau_color, tau_grad, labels_out, min_cost_out,
                     filtered_out, keys_out);
}

hgf_status hgf_lr_postprocess(hgf_handle h, const float* image, const int32_t* disp_left, const int32_t* disp_right,
                              int tol, int radius, float sigma_s, float sigma_c, uint8_t* valid_out,
                              int32_t* disp_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!image || !disp_left || !disp_right || !disp_out) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null pointer");
  hgf_status s = check_pp_args(h, tol, radius, sigma_s, sigma_c);
  if (s != HGF_OK) return s;
  if ((s = check_async(h)) != HGF_OK) return s;
  return postprocess_impl(h, image, disp_left, disp_right, tol, radius, sigma_s, sigma_c, valid_out, disp_out);
}

hgf_status hgf_stereo_disparity(hgf_handle h, const float* left, const float* right, int L, int label_offset,
                                float alpha, float tau_color, float tau_grad, int tol, int radius, float sigma_s,
                                float sigma_c, int32_t* disp_left_out, int32_t* disp_right_out, uint8_t* valid_out,
                                int32_t* disp_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!disp_out) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null disp_out");
  hgf_status s = check_pp_args(h, tol, radius, sigma_s, sigma_c);
  if (s != HGF_OK) return s;
  const size_t HW = (size_t)h->W * h->H;
  if ((s = pp_scratch(h)) != HGF_OK) return s;
  int32_t* dL = disp_left_out ? disp_left_out : h->pp_int + HW;
  int32_t* dR = disp_right_out ? disp_right_out : h->pp_int + 2 * HW;
  if ((s = stereo_impl(h, left, right, +1, L, label_offset, alpha, tau_color, tau_grad, dL, nullptr, nullptr,
                       nullptr)) != HGF_OK)
    return s;
  if ((s = stereo_impl(h, right, left, -1, L, label_offset, alpha, tau_color, tau_grad, dR, nullptr, nullptr,
                       nullptr)) != HGF_OK)
    return s;
  return postprocess_impl(h, left, dL, dR, tol, radius, sigma_s, sigma_c, valid_out, disp_out);
}

hgf_status hgf_segment(hgf_handle h, const float* image, const uint8_t* fg_seeds, const uint8_t* bg_seeds,
                       int32_t* labels_out, float* min_cost_out, float* filtered_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!image || !fg_seeds || !bg_seeds) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null pointer");
  if (!labels_out && !min_cost_out && !filtered_out) return fail(h, HGF_ERR_INVALID_ARGUMENT, "no output requested");
  const size_t HW = (size_t)h->W * h->H;
  const int nbins = 2 * h->m * 32;
  cudaError_t e;
  if (!h->sg_cost) {
    if ((e = cudaMalloc(&h->sg_cost, sizeof(float) * 2 * HW)) != cudaSuccess ||
        (e = cudaMalloc(&h->sg_counts, sizeof(int) * (nbins + 2))) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(h->sg_cost);
      h->sg_cost = nullptr;
      return fail(h, e == cudaErrorMemoryAllocation ? HGF_ERR_OUT_OF_MEMORY : HGF_ERR_CUDA, "segmentation scratch");
    }
  }
  hgf_status s = check_async(h);
  if (s != HGF_OK) return s;
  int* seeds = h->sg_counts + nbins;
  e = traced(h, HGF_KC_COST, h->stream, [&] {
    cudaError_t e2 = cudaMemsetAsync(h->sg_counts, 0, sizeof(int) * (nbins + 2), h->stream);
    return e2 != cudaSuccess ? e2
                             : hgf::launch_seg_hist(image, fg_seeds, bg_seeds, h->m, h->W, h->H, h->sg_counts, seeds,
                                                    h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "seed histograms");
  // empty seed sets are an argument error: the one host read of this entry point
  int nseeds[2] = {0, 0};
  if ((e = cudaMemcpyAsync(nseeds, seeds, sizeof(nseeds), cudaMemcpyDeviceToHost, h->stream)) != cudaSuccess ||
      (e = cudaStreamSynchronize(h->stream)) != cudaSuccess)
    return cuda_fail(h, e, "seed count read");
  if (nseeds[0] == 0 || nseeds[1] == 0) return fail(h, HGF_ERR_INVALID_ARGUMENT, "empty foreground or background seed set");
  e = traced(h, HGF_KC_COST, h->stream, [&] {
    return hgf::launch_seg_cost(image, h->sg_counts, seeds, h->m, h->W, h->H, h->sg_cost, h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "segmentation cost");
  SmallLMode sm(h, 2);
  if ((s = frame_stats(h, image, 0, h->H)) != HGF_OK) return s;
  const int do_wta = (labels_out || min_cost_out) ? 1 : 0;
  return slices(h, image, h->sg_cost, 2, 0, filtered_out, do_wta, labels_out, min_cost_out, nullptr);
}

hgf_status hgf_aggregate_wta_peer(hgf_handle h, const float* cost_volume, int L, int label_offset,
                                  int64_t* const* peer_keys_dev, int world, int rows_per_owner) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!cost_volume || !peer_keys_dev) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null pointer");
  if (L < 1) return fail(h, HGF_ERR_INVALID_ARGUMENT, "L must be >= 1");
  if (label_offset < 0 || (long long)label_offset + L > 2147483647LL)
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "label_offset out of range");
  if (world < 1 || rows_per_owner < 1 || (long long)rows_per_owner * world < h->H)
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "owners must cover every row: world * rows_per_owner >= H");
  if (!h->v3agg || !(h->v3coef || h->v4coef || h->v5coef))
    return fail(h, HGF_ERR_UNSUPPORTED, "the fused merge needs the k_coef3/4/5 + k_agg3 path");
  hgf_status s = check_async(h);
  if (s != HGF_OK) return s;
  h->peer_keys = reinterpret_cast<long long* const*>(peer_keys_dev);
  h->rows_per_owner = rows_per_owner;
  s = slices(h, nullptr, cost_volume, L, label_offset, nullptr, 1, nullptr, nullptr, nullptr);
  h->peer_keys = nullptr;
  h->rows_per_owner = 0;
  return s;
}

hgf_status hgf_fill_keys(hgf_handle h, int64_t* keys, long long n) {
  DeviceGuard dg(h);
  if (!h || !keys || n < 0) return HGF_ERR_INVALID_ARGUMENT;
  cudaError_t e = hgf::launch_fill_i64(keys, n, (long long)0x7FFFFFFFFFFFFFFFLL, h->stream);
  return e == cudaSuccess ? HGF_OK : cuda_fail(h, e, "fill_keys");
}

hgf_status hgf_unpack_keys_n(hgf_handle h, const int64_t* keys, long long n, int32_t* labels_out,
                             float* min_cost_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!keys || n < 0 || n > (1LL << 31) || (!labels_out && !min_cost_out))
    return fail(h, HGF_ERR_INVALID_ARGUMENT, "null pointer or bad count");
  cudaError_t e = traced(h, HGF_KC_KEYS, h->stream, [&] {
    return hgf::launch_unpack_keys(keys, labels_out, min_cost_out, (int)n, 1, h->stream);
  });
  return e == cudaSuccess ? HGF_OK : cuda_fail(h, e, "unpack_keys");
}

hgf_status hgf_alloc(size_t bytes, void** dev_ptr) {
  if (!dev_ptr || bytes == 0) return HGF_ERR_INVALID_ARGUMENT;
  cudaError_t e = cudaMalloc(dev_ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *dev_ptr = nullptr;
    return e == cudaErrorMemoryAllocation ? HGF_ERR_OUT_OF_MEMORY : HGF_ERR_CUDA;
  }
  return HGF_OK;
}

hgf_status hgf_free(void* dev_ptr) { return cudaFree(dev_ptr) == cudaSuccess ? HGF_OK : HGF_ERR_CUDA; }

hgf_status hgf_ipc_get_handle(void* dev_ptr, unsigned char* handle64) {
  if (!dev_ptr || !handle64) return HGF_ERR_INVALID_ARGUMENT;
  cudaIpcMemHandle_t hd;
  if (cudaIpcGetMemHandle(&hd, dev_ptr) != cudaSuccess) {
    cudaGetLastError();
    return HGF_ERR_CUDA;
  }
  static_assert(sizeof(hd) == 64, "CUDA IPC handle size");
  std::memcpy(handle64, &hd, 64);
  return HGF_OK;
}

hgf_status hgf_ipc_open(const unsigned char* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return HGF_ERR_INVALID_ARGUMENT;
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle64, 64);
  if (cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    *dev_ptr = nullptr;
    return HGF_ERR_CUDA;
  }
  return HGF_OK;
}

hgf_status hgf_ipc_close(void* dev_ptr) {
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? HGF_OK : HGF_ERR_CUDA;
}

hgf_status hgf_aggregate_wta(hgf_handle h, const float* guide, const float* cost_volume, int L, int32_t* labels_out) {
  DeviceGuard dg(h);
  if (!labels_out) return h ? fail(h, HGF_ERR_INVALID_ARGUMENT, "labels_out is null") : HGF_ERR_INVALID_ARGUMENT;
  return hgf_aggregate_wta_ex(h, guide, cost_volume, L, 0, labels_out, nullptr, nullptr, nullptr);
}

hgf_status hgf_unpack_keys(hgf_handle h, const int64_t* keys, int32_t* labels_out, float* min_cost_out) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!keys || (!labels_out && !min_cost_out)) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null pointer");
  cudaError_t e = traced(h, HGF_KC_KEYS, h->stream, [&] {
    return hgf::launch_unpack_keys(keys, labels_out, min_cost_out, h->W, h->H, h->stream);
  });
  if (e != cudaSuccess) return cuda_fail(h, e, "unpack_keys");
  return HGF_OK;
}

hgf_status hgf_aggregate_wta_host(hgf_handle h, const float* guide_host, const float* cost_host, int L,
                                  int32_t* labels_host) {
  DeviceGuard dg(h);
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->launches = 0;
  h->err.clear();
  if (!guide_host || !cost_host || !labels_host) return fail(h, HGF_ERR_INVALID_ARGUMENT, "null pointer");
  if (L < 1) return fail(h, HGF_ERR_INVALID_ARGUMENT, "L must be >= 1");
  const size_t HW = (size_t)h->W * h->H;
  cudaError_t e;
  if (!h->st_guide) {
    // 32-label staging chunks (one label batch of the slice kernels): the H2D copy of chunk c + 1 overlaps the
    // aggregation of chunk c (with whole-call chunks the copy and the compute ran back to back); the band heights
    // are chosen for the whole call (lmodel), so the result is the device path's bit for bit
    h->st_chunk = h->lcap < hgf::kWGroupLabels ? h->lcap : hgf::kWGroupLabels;
    if ((e = cudaMalloc(&h->st_guide, sizeof(float) * h->m * HW)) != cudaSuccess ||
        (e = cudaMalloc(&h->st_vol[0], sizeof(float) * HW * h->st_chunk)) != cudaSuccess ||
        (e = cudaMalloc(&h->st_vol[1], sizeof(float) * HW * h->st_chunk)) != cudaSuccess ||
        (e = cudaMalloc(&h->st_labels, sizeof(int32_t) * HW)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(h, e, "staging allocation");
    for (int i = 0; i < 2; ++i) {
      if ((e = cudaEventCreateWithFlags(&h->ev_copied[i], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&h->ev_used[i], cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(h, e, "event creation");
    }
  }
  hgf_status s = check_async(h);
  if (s != HGF_OK) return s;
  if ((e = cudaMemcpyAsync(h->st_guide, guide_host, sizeof(float) * h->m * HW, cudaMemcpyHostToDevice, h->stream)) !=
      cudaSuccess)
    return cuda_fail(h, e, "guide H2D");
  if ((s = frame_stats(h, h->st_guide, 0, h->H)) != HGF_OK) return s;
  const long long lcap = h->st_chunk;
  const int nchunks = (int)((L + lcap - 1) / lcap);
  h->lmodel = L;
  if (h->v5agg) {
    e = traced(h, HGF_KC_KEYS, h->stream,
               [&] { return hgf::launch_fill_i64(h->fkeys, (long long)HW, 0x7fffffffffffffffLL, h->stream); });
    if (e != cudaSuccess) return cuda_fail(h, e, "keys fill");
  }
  // double-buffered: copy chunk c+1 on copy_stream while chunk c is aggregated on the handle's stream
  for (int c = 0; c < nchunks; ++c) {
    const int b = c & 1;
    const int l0 = (int)(c * lcap);
    const int Lc = (int)((L - l0 < lcap) ? (L - l0) : lcap);
    if (c >= 2 && (e = cudaStreamWaitEvent(h->copy_stream, h->ev_used[b], 0)) != cudaSuccess)
      return cuda_fail(h, e, "wait used");
    if ((e = cudaMemcpyAsync(h->st_vol[b], cost_host + (size_t)l0 * HW, sizeof(float) * HW * Lc,
                             cudaMemcpyHostToDevice, h->copy_stream)) != cudaSuccess)
      return cuda_fail(h, e, "volume H2D");
    if ((e = cudaEventRecord(h->ev_copied[b], h->copy_stream)) != cudaSuccess) return cuda_fail(h, e, "record");
    if ((e = cudaStreamWaitEvent(h->stream, h->ev_copied[b], 0)) != cudaSuccess) return cuda_fail(h, e, "wait copied");
    e = launch_coef_chunk(h, h->st_guide, h->st_vol[b], Lc);
    if (e != cudaSuccess) return cuda_fail(h, e, "coef");
    hgf::AggArgs a{};
    a.G = h->G; a.wbuf = h->wbuf; a.W = h->W; a.H = h->H; a.r = h->r; a.L = Lc; a.label_base = l0;
    a.pad = h->wlay.pad;
    a.il = h->wlay.il;
    a.filtered_out = nullptr; a.do_wta = 1; a.first = (c == 0); a.last = (c == nchunks - 1);
    a.best_cost = h->best_cost; a.best_label = h->best_label; a.labels_out = h->st_labels;
    a.min_cost_out = nullptr; a.keys_out = nullptr;
    e = launch_agg_chunk(h, a);
    if (e != cudaSuccess) return cuda_fail(h, e, "agg");
    if ((e = cudaEventRecord(h->ev_used[b], h->stream)) != cudaSuccess) return cuda_fail(h, e, "record used");
  }
  if (h->v5agg) {
    e = traced(h, HGF_KC_KEYS, h->stream, [&] {
      return hgf::launch_keys_finalize(h->fkeys, h->W, h->H, h->st_labels, nullptr, nullptr, nullptr, 0, h->stream);
    });
    if (e != cudaSuccess) return cuda_fail(h, e, "keys finalize");
  }
  if ((e = cudaMemcpyAsync(labels_host, h->st_labels, sizeof(int32_t) * HW, cudaMemcpyDeviceToHost, h->stream)) !=
      cudaSuccess)
    return cuda_fail(h, e, "labels D2H");
  if ((e = cudaStreamSynchronize(h->stream)) != cudaSuccess) return cuda_fail(h, e, "sync");
  return HGF_OK;
}

hgf_status hgf_set_profiling(hgf_handle h, int enable) {
  if (!h) return HGF_ERR_INVALID_ARGUMENT;
  h->profiling = enable != 0;
  return HGF_OK;
}

hgf_status hgf_profile_read(hgf_handle h, double* ms, int* counts, int n) {
  DeviceGuard dg(h);
  if (!h || n < 0 || n > HGF_KC_COUNT) return HGF_ERR_INVALID_ARGUMENT;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "profile sync");
  double acc[HGF_KC_COUNT] = {0};
  int cnt[HGF_KC_COUNT] = {0};
  for (auto& r : h->recs) {
    float t = 0.0f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
      acc[r.cls] += t;
      cnt[r.cls] += 1;
    }
    h->pool.push_back(r.a);
    h->pool.push_back(r.b);
  }
  h->recs.clear();
  for (int i = 0; i < n; ++i) {
    if (ms) ms[i] = acc[i];
    if (counts) counts[i] = cnt[i];
  }
  return HGF_OK;
}

}  // extern "C"
