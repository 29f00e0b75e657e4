// Internal launcher interface between the C ABI (hgf_api.cu) and the kernels (hgf_kernels.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "hgf_common.cuh"

namespace hgf {

struct AggArgs {
  const float* G;
  const float* wbuf;
  int W, H, r, L, label_base;
  int pad;   // zero margin of the coefficient layout (v3 aggregation)
  int il;    // label-interleaved coefficient layout (WLayout::il)
  float* filtered_out;
  int do_wta, first, last;
  float* best_cost;
  int32_t* best_label;
  int32_t* labels_out;
  float* min_cost_out;
  int64_t* keys_out;
  // fused WTA merge over peer memory (k_agg3 only): the last pass atomicMin's each pixel's key into the key
  // buffer of the rank owning its row: peer_keys[gy / rows_per_owner][(gy % rows_per_owner) * W + gx]
  long long* const* peer_keys;
  int rows_per_owner;
  // k_agg6 label split (small frames): nsplit CTAs per tile over disjoint label ranges, each atomic-MINing its
  // minimum keys (pack_key_signed) into fkeys[H][W]; the caller fills fkeys with the MIN identity before the first
  // chunk and runs launch_keys_finalize after the last (best_cost / best_label / first / last are not used)
  int nsplit;
  long long* fkeys;
};

// Gp (nullable; used when d == 2): (I_i, I_i^2) pairs, layout [H][m][gp_pitch][2], for k_coef5.
cudaError_t launch_poly_guidance(const float* I, float* G, float* Gp, int gp_pitch, int m, int d, int W, int H,
                                 cudaStream_t st);
// aos = 1: per-pixel records of kStatsAos floats (statistics, then kappa = 1/(lam0f + N)) for k_coef3;
// needs the k_stats2 path (else cudaErrorInvalidValue).
// Rows [y0, y1) of the statistics (the k_stats2 path; the v1 kernel only supports the full image).
// scratch3: (stats3_scratch_planes(n)) * H * W doubles, or null (k_stats3 is used for n >= kStats3MinN).
constexpr int kStats4MaxN = 9;      // k_stats4 (row-marching) up to here, when its rows fit SMEM
inline size_t stats4_smem(int n, int r, int lp = 0) {   // = st4::smem_bytes
  return (size_t)2 * ((n + 1) * (n + 2) / 2 - 1 + lp * (n + 1)) * (((64 + 2 * r) | 1) + 65) * sizeof(double);
}
// hgf_filter's fused single-slice pass (k_stats4<n, 1>): guidance G + cost slice P -> the slice's coefficients w
// in the planar layout wo, the statistics never stored; n <= kStats4MaxN, 64 + 2r <= 128, stats4_smem(n, r, 1)
// within 200 KB (else cudaErrorInvalidValue).
cudaError_t launch_filter1(int n, const float* G, const float* P, float* wout, WLayout wo, int W, int H, int r,
                           double lam, int mode, float lam0f, cudaStream_t st);
constexpr int kStats3MinN = 18;     // always k_stats3 from here; below only when k_stats2 does not fit
inline long long stats3_scratch_planes(int n) { return (long long)(n + 1) * (n + 2) / 2 - 1 + 32; }
cudaError_t launch_stats(int n, const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos,
                         float lam0f, int y0, int y1, double* scratch3, cudaStream_t st);
cudaError_t launch_coef(int n, const float* G, const float* stats, const float* vol, float* wbuf, int W, int H,
                        int r, int L, float lam0, cudaStream_t st);
cudaError_t launch_agg(int n, const AggArgs& a, cudaStream_t st);
cudaError_t launch_fill_i64(int64_t* p, long long n, long long v, cudaStream_t st);
cudaError_t launch_unpack_keys(const int64_t* keys, int32_t* labels, float* cost, int W, int H, cudaStream_t st);

}  // namespace hgf

namespace hgf {
// Per-n implementations (defined in hgf_kernels.cuh, instantiated by hgf_inst.cu for n = 1..20).
template <int NC>
cudaError_t stats_impl(const float* G, float* stats, int W, int H, int r, double lam, int mode, cudaStream_t st);
template <int NC>
cudaError_t coef_impl(const float* G, const float* stats, const float* vol, float* wbuf, int W, int H, int r, int L,
                      float lam0, cudaStream_t st);
template <int NC>
cudaError_t agg_impl(const AggArgs& a, cudaStream_t st);
}  // namespace hgf

namespace hgf {
namespace v2 {
// Fast path (n_guide <= 3, degree <= 3, radius <= 9): hgf_slice_v2.cuh, instantiated by hgf_inst.cu / hgf_inst2.cu.
template <int M, int D>
cudaError_t coef2_impl(const float* guide, const float* stats, const float* vol, float* wbuf, WLayout wo, int W, int H, int r,
                       int L, float lam0, cudaStream_t st);
template <int NC>
cudaError_t agg2_impl(const AggArgs& a, cudaStream_t st);
}  // namespace v2
bool fast_path_ok(int m, int d, int r);
cudaError_t launch_coef_fast(int m, int d, const float* guide, const float* stats, const float* vol, float* wbuf, WLayout wo,
                             int W, int H, int r, int L, float lam0, cudaStream_t st);
cudaError_t launch_agg_fast(int n, const AggArgs& a, cudaStream_t st);
// Stereo cost construction (hgf_stereo.cu): dx of the channel mean of a 3-channel view; cost slices of
// disparities [d0, d0 + Lc) of view `base` against view `other` into cost [Lc][H][W], the match at x - d
// (dir = +1, the left view's cost) or x + d (dir = -1, the right view's, reading P1).
cudaError_t launch_stereo_grad(const float* img, float* grad, int W, int H, cudaStream_t st);
cudaError_t launch_stereo_cost(const float* base, const float* other, const float* gb, const float* go, float* cost,
                               int W, int H, int d0, int Lc, int dir, float a, float tc, float tg, cudaStream_t st);
// Post-processing (hgf_stereo.cu, readings P2-P4): consistency flags + row fill, then the weighted median
// over the inconsistent pixels (radius <= lr_wmf_max_radius()).
int lr_wmf_max_radius();
cudaError_t launch_lr_fill(const int* dL, const int* dR, int W, int H, int tol, uint8_t* valid, int* fill,
                           cudaStream_t st);
cudaError_t launch_wmf(const int* fill, const uint8_t* valid, const float* img, int m, int W, int H, int radius,
                       float sigma_s, float sigma_c, int* out, cudaStream_t st);
// Segmentation costs (hgf_stereo.cu): seed histograms counts [2][m][32], seeds [2] (zeroed by the caller),
// then the two cost slices [2][H][W].
cudaError_t launch_seg_hist(const float* img, const uint8_t* fg, const uint8_t* bg, int m, int W, int H, int* counts,
                            int* seeds, cudaStream_t st);
cudaError_t launch_seg_cost(const float* img, const int* counts, const int* seeds, int m, int W, int H, float* cost,
                            cudaStream_t st);
}  // namespace hgf

namespace hgf {
namespace v3 {
// TMA-fed aggregation (hgf_agg_v3.cuh), n <= 9, R <= 9, W % 4 == 0; tmap points to a CUtensorMap over
// the coefficient buffer (dims W, H, planes; box = agg3_box(n, R)).
template <int NC, int R>
cudaError_t agg3_impl(const void* tmap, const AggArgs& a, cudaStream_t st);
}  // namespace v3
// Box of the v3 aggregation TMA for radius R: {BX, BY} (x extent, y extent); z extent = n + 1.
// k_agg3 fetches each slice's K planes as two TMA groups: [0, agg3_ka(K)) and [agg3_ka(K), K).
__host__ __device__ constexpr int agg3_ka(int K) { return (K + 1) / 2; }
// il = 1: label-interleaved layout (BX a multiple of 32 pixels; tensor-map box {16, 1, BX/16, BY, n+1}).
void agg3_box(int n, int R, int il, int* bx, int* by);
cudaError_t launch_agg_v3(int n, int r, const void* tmap, const AggArgs& a, cudaStream_t st);
namespace v3 {
template <int NC>
cudaError_t coef3_impl(const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo, int W,
                       int H, int r, int L, float lam0, cudaStream_t st);
}  // namespace v3
// Label-batched marching coefficient kernel (hgf_coef_v3.cuh): n <= 6, r <= 9, padded layout.
// tm_vol: CUtensorMap over the chunk's cost slices (dims W, H, L; box 88 x 1 x 32); tm_g over G (box 88 x 1 x n).
cudaError_t launch_coef_v3(int n, const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo,
                           int W, int H, int r, int L, float lam0, cudaStream_t st);
// Tensor-core coefficient kernel (hgf_coef_v4.cuh): n <= 6, r <= 9, planar layout (pitch a multiple of 32),
// per-pixel statistics records.  tm_vol: box kCoef4BoxX x 1 x kCoef4LB; tm_g: box kCoef4BoxX x 1 x n.
constexpr int kCoef4BoxX = 152, kCoef4LB = 16;
namespace v4 {
template <int NC>
cudaError_t coef4_impl(const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo, int W,
                       int H, int r, int L, cudaStream_t st);
}  // namespace v4
cudaError_t launch_coef_v4(int n, const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo,
                           int W, int H, int r, int L, cudaStream_t st);
// Horizontal-first coefficient kernel (hgf_coef_v5.cuh, instantiated in hgf_coef5.cu): raw guide channels
// m <= 3, degree d <= 3, n = m d <= 6, r <= 9, label-interleaved layout, per-pixel statistics records.
// tm_vol: box kCoef5BoxX x 1 x kCoef5LB over the chunk's slices; tm_i: box kCoef5BoxX x 1 x m over the raw
// guide channels (the planes G_{(i-1)d+1} = I_i of the guidance buffer).
constexpr int kCoef5BoxX = 164, kCoef5LB = 32, kCoef5MaxN = 6;
// Row-marching aggregation (hgf_agg_v5.cuh, instantiated in hgf_agg5.cu): n <= 6, r <= 9, the label-interleaved
// layout.  tm_w: rank-5 map over the coefficient buffer (16 px, 32 labels, x groups, H, planes), box
// (16, kAgg5LB, 6, 1, n + 1), 64-byte swizzle; tm_g: over G (W, H, n), box (64, 1, n).  Each CTA marches a band
// for labels_per_cta labels (a multiple of kAgg5LB dividing 32) of the chunk's L and atomic-MINs the band's
// minimum keys (signed order, hgf.h) into keys[H][W]; filtered_out (nullable) = the chunk's Z slices.
constexpr int kAgg5LB = 4, kAgg5MaxN = 6;
cudaError_t launch_agg_v5(int n, const void* tm_w, const void* tm_g, int W, int H, int r, int L, int label_base,
                          int labels_per_cta, unsigned long long* keys, float* filtered_out, cudaStream_t st);
// Warp-specialised aggregation (hgf_agg_v6.cuh, instantiated in hgf_agg6.cu): 64 x kAgg6TY tiles on the
// label-interleaved layout, n <= 6, r <= 9; tm: rank-5 map over the coefficient buffer with a one-plane box
// (16, 1, ceil32(64 + 2r) / 16, kAgg6TY + 2r, 1), 64-byte swizzle.  Same AggArgs contract as k_agg3 (a.il == 1).
constexpr int kAgg6MaxN = 6, kAgg6TY = 48;
// k_agg6's label split for a frame of W x H (1 = none): frames of fewer than ~1.5 waves of tiles take the part count
// s minimising waves(tiles * s) x (L / s + 2), the 2 standing for a CTA's fixed cost (prologue, pipeline fill and
// drain) in slice-times; >= 4 labels per part
inline int agg6_split(int W, int H, int r, int L, int nsm) {
  const long long tiles = (long long)((W + (16 - r % 16) % 16 + 63) / 64) * ((H + kAgg6TY - 1) / kAgg6TY);
  // (fewer than 32 labels: the key fill + finalize launches cost more than the split saves)
  if (tiles * 2 >= 3LL * nsm || L < 32) return 1;
  const int smax = L / 4 > 1 ? L / 4 : 1;
  int best_s = 1;
  double best = 1e300;
  for (int s = 1; s <= smax; ++s) {
    const double cost = (double)((tiles * s + nsm - 1) / nsm) * ((double)L / s + 2.0);
    if (cost < best) { best = cost; best_s = s; }
  }
  return best_s;
}
// m, d: guide channels and degree (the owners of m <= 3 hold the raw channels; HGF_AGG6_KX=8 forces the planes).
cudaError_t launch_agg_v6(int m, int d, int r, const void* tm, const AggArgs& a, cudaStream_t st);
// keys[H][W] -> labels_out / min_cost_out / keys_out (each nullable) and, when peer_keys != null, a system-scope
// 64-bit atomic MIN of every pixel's key into the row owner's buffer (the fused label-sharded merge).
cudaError_t launch_keys_finalize(const int64_t* keys, int W, int H, int32_t* labels_out, float* min_cost_out,
                                 int64_t* keys_out, long long* const* peer_keys, int rows_per_owner, cudaStream_t st);
bool coef5_ok(int m, int d, int r);
// Lmodel: the label count the band height is chosen for (the whole call's, so every chunk of a call -- and a call
// whatever its chunking -- marches the same bands and gives the same bits); L: this chunk's labels.
cudaError_t launch_coef_v5(int m, int d, const void* tm_vol, const void* tm_i, const float* stats, float* wbuf,
                           WLayout wo, int W, int H, int r, int L, int Lmodel, cudaStream_t st);
}  // namespace hgf

namespace hgf {
namespace st3 {
template <int NC>
cudaError_t stats3_impl(const float* G, float* stats, double* scratch, int W, int H, int r, double lam, int mode,
                        cudaStream_t st);
}  // namespace st3
namespace st2 {
template <int NC>
cudaError_t stats2_impl(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos, float lam0f,
                        int y0, int y1, cudaStream_t st);
}  // namespace st2
namespace st4 {
template <int NC>
cudaError_t stats4_impl(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos, float lam0f,
                        int y0, int y1, cudaStream_t st);
template <int NC>
cudaError_t filter1_impl(const float* G, const float* P, float* wout, WLayout wo, int W, int H, int r, double lam,
                         int mode, float lam0f, cudaStream_t st);
}  // namespace st4
namespace st5 {
template <int NC>
cudaError_t stats_sel(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos, float lam0f,
                      int y0, int y1, cudaStream_t st);
template <int NC>
cudaError_t filter1_sel(const float* G, const float* P, float* wout, WLayout wo, int W, int H, int r, double lam,
                        int mode, float lam0f, cudaStream_t st);
}  // namespace st5
}  // namespace hgf
