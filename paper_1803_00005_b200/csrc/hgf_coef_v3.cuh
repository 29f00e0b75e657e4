// HGF per-slice coefficients, version 3 (k_coef3<n>): label-batched row marching, warp-specialised.
//
// For each slice l and pixel p (Eq12 with G_{n+1} = p; Eq13 P:304 reassociated):
//     S_0 = B(p),  S_k = B(G_k p)  (k = 1..n),   w = P'(S - nu S_0),   w_0 = S_0/(lambda_0 + N) - nu^T w
//
// A CTA owns a strip of TX = 64 columns x a band of BH rows x a batch of LB = 32 labels, and marches
// down the band one row at a time:
//   * V warps (producers): thread = (column c of the strip plus an r halo, group of 8 labels).  It keeps
//     the vertical running sums V_k(c) = sum_{|dy|<=r} G_k p over the window for its 8 labels in registers
//     (7 x 8 values at n = 6), adding the entering row and subtracting the leaving row (both read straight
//     from global memory: coalesced across columns; the leaving row is an L2 hit).  G_k is label-invariant
//     and is loaded once per row for all 8 labels.  The row of V for the 32 labels goes to SMEM.
//   * H warps (consumers): thread = (label, 16-pixel segment).  It slides the horizontal 2r+1 window over
//     the row of V (S for one pixel at a time, all planes), reads that pixel's statistics from SMEM (the
//     same address for 16 lanes: a broadcast, so the 27 floats per pixel cost ~1 word per voxel), does the
//     n x n matvec and stores w 8 pixels at a time (32-byte runs).
//   * V and H warps run one row apart through a double-buffered SMEM row (named barriers FULL/FREE).
// Label-invariant data (G, statistics) thus never costs per-label shared-memory traffic, which was the
// dominant cost of the tile version (profiles/r01_ncu_v2_coef2_sass_mix.txt).
#pragma once
#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace v3 {

constexpr int C_TX = 64;                    // owned columns per strip
constexpr int C_LB = 32;                    // labels per CTA batch
constexpr int C_LG = 8;                     // labels per V thread
constexpr int C_NG = C_LB / C_LG;           // V label groups
constexpr int C_HSEG = 16;                  // pixels per H thread
constexpr int C_NHW = 4;                    // H warps: 16 labels x 2 segments each
constexpr int C_RMAX = 9;

template <int NC>
struct CoefGeom {
  static constexpr int K = NC + 1, NP = NC * (NC + 1) / 2, NS = NP + NC;
  static constexpr int CXMAX = C_TX + 2 * C_RMAX;         // V columns (strip + halo), max 82
  static constexpr int CP = CXMAX | 1;                      // SMEM column pitch (odd)
  static constexpr int LSTRIDE = K * CP + ((K * CP) % 2 == 0 ? 1 : 0);  // floats per label: odd -> the
                                                            // 16 labels x 2 segments of an H warp hit 32 banks
  static constexpr int VROW = C_LB * LSTRIDE;               // floats per V row buffer
  static constexpr int SROW = NS * C_TX;                    // statistics row [NS][64]
  static constexpr int NVW = (CXMAX * C_NG + 31) / 32;      // V warps
  static constexpr int THREADS = (NVW + C_NHW) * 32;
  static constexpr size_t SMEM = sizeof(float) * (2 * (size_t)VROW + 2 * (size_t)SROW);
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int NC>
__global__ void __launch_bounds__(CoefGeom<NC>::THREADS, 1)
    k_coef3(const float* __restrict__ G, const float* __restrict__ stats, const float* __restrict__ vol,
            float* __restrict__ wbuf, WLayout wo, int W, int H, int r, int L, int BH, float lam0) {
  using Gm = CoefGeom<NC>;
  constexpr int K = Gm::K, NP = Gm::NP, NS = Gm::NS, CP = Gm::CP, LSTRIDE = Gm::LSTRIDE;
  constexpr int NV = Gm::NVW * 32, NH = C_NHW * 32, NALL = NV + NH;
  extern __shared__ __align__(16) float sm[];
  float* vrow = sm;                       // [2][LB][K][CP]
  float* srow = sm + 2 * Gm::VROW;        // [2][NS][TX]
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * C_TX;
  const int Y0 = blockIdx.y * BH, Y1 = min(H, Y0 + BH);
  const int lb0 = blockIdx.z * C_LB;
  const long long HW = (long long)H * W;
  const int CX = C_TX + 2 * r;            // V columns used: image x = x0 - r + c

  if (tid < NV) {
    // ============================ V warps (producers) ============================
    const int g = tid / CX, c = tid % CX;
    const bool active = g < C_NG;
    const int xx = x0 - r + c;
    const bool xin = active && xx >= 0 && xx < W;
    int nl = 0;                            // labels of this thread inside [0, L)
    const float* pv[C_LG];
#pragma unroll
    for (int j = 0; j < C_LG; ++j) {
      const int l = lb0 + g * C_LG + j;
      const bool ok = active && l < L;
      nl += ok ? 1 : 0;
      pv[j] = vol + (ok ? (long long)l : 0) * HW + (xin ? xx : 0);
    }
    float acc[C_LG][K];
#pragma unroll
    for (int j = 0; j < C_LG; ++j)
#pragma unroll
      for (int k = 0; k < K; ++k) acc[j][k] = 0.0f;
    // add (sgn = +1) or subtract (sgn = -1) image row yy's contribution
    auto update = [&](int yy, float sgn) {
      if (!xin || yy < 0 || yy >= H) return;
      const long long ro = (long long)yy * W;
      float gk[NC > 0 ? NC : 1];
#pragma unroll
      for (int k = 0; k < NC; ++k) gk[k] = __ldg(G + k * HW + ro + xx);
#pragma unroll
      for (int j = 0; j < C_LG; ++j) {
        if (j < nl) {
          const float p = __ldg(pv[j] + ro) * sgn;
          acc[j][0] += p;
#pragma unroll
          for (int k = 0; k < NC; ++k) acc[j][k + 1] = fmaf(gk[k], p, acc[j][k + 1]);
        }
      }
    };
    // warm-up window of the band's first output row: rows [Y0 - r, Y0 + r - 1]
    for (int yy = Y0 - r; yy < Y0 + r; ++yy) update(yy, 1.0f);
    for (int y = Y0; y < Y1; ++y) {
      const int b = (y - Y0) & 1;
      if (y - Y0 >= 2) named_sync(3 + b, NALL);   // H warps released buffer b
      update(y + r, 1.0f);
      if (y > Y0) update(y - r - 1, -1.0f);
      if (active) {
        float* dst = vrow + b * Gm::VROW + (g * C_LG) * LSTRIDE + c;
#pragma unroll
        for (int j = 0; j < C_LG; ++j)
#pragma unroll
          for (int k = 0; k < K; ++k) dst[j * LSTRIDE + k * CP] = acc[j][k];
      }
      // statistics row y for the strip's 64 owned pixels (consumed by the H warps with this V row)
      float* sdst = srow + b * Gm::SROW;
      for (int e = tid; e < NS * C_TX; e += NV) {
        const int s = e / C_TX, x = e % C_TX;
        sdst[e] = (x0 + x < W) ? __ldg(stats + s * HW + (long long)y * W + x0 + x) : 0.0f;
      }
      named_arrive(1 + b, NALL);                   // row y ready in buffer b
    }
  } else {
    // ============================ H warps (consumers) ============================
    const int h = tid - NV, hw = h >> 5, ln = h & 31;
    const int lab = (hw & 1) * 16 + (ln & 15);        // label within the batch
    const int seg = 2 * (hw >> 1) + (ln >> 4);        // 16-pixel segment 0..3
    const int l = lb0 + lab;
    const bool lok = l < L;
    const int xs = seg * C_HSEG;                      // first owned pixel (strip-relative)
    for (int y = Y0; y < Y1; ++y) {
      const int b = (y - Y0) & 1;
      named_sync(1 + b, NALL);
      const float* vr = vrow + b * Gm::VROW + lab * LSTRIDE;
      const float* st = srow + b * Gm::SROW;
      float S[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        float a = 0.0f;
        for (int j = 0; j <= 2 * r; ++j) a += vr[k * CP + xs + j];
        S[k] = a;
      }
      float wv[K][8];
      float* wrow = wbuf + wo.origin + (long long)l * K * wo.plane + (long long)y * wo.pitch + x0 + xs;
#pragma unroll 1
      for (int q = 0; q < C_HSEG; q += 8) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int x = xs + q + i;                 // strip-relative pixel
          if (q + i > 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) S[k] += vr[k * CP + x + 2 * r] - vr[k * CP + x - 1];
          }
          // statistics of pixel (y, x0 + x): P' (upper triangle) then nu  -- broadcast reads
          float sp[NS];
#pragma unroll
          for (int s = 0; s < NS; ++s) sp[s] = st[s * C_TX + x];
          const int gx = x0 + x;
          const float kap = 1.0f / (lam0 + (float)window_count(y, gx < W ? gx : W - 1, H, W, r));
          float cc[NC > 0 ? NC : 1];
#pragma unroll
          for (int k = 0; k < NC; ++k) cc[k] = fmaf(-sp[NP + k], S[0], S[k + 1]);
          float w0 = kap * S[0];
#pragma unroll
          for (int a = 0; a < NC; ++a) {
            float t = 0.0f;
#pragma unroll
            for (int bq = 0; bq < NC; ++bq) {
              const int lo = a < bq ? a : bq, hi = a < bq ? bq : a;
              t = fmaf(sp[lo * NC - lo * (lo - 1) / 2 + (hi - lo)], cc[bq], t);
            }
            wv[a + 1][i] = t;
            w0 = fmaf(-sp[NP + a], t, w0);
          }
          wv[0][i] = w0;
        }
        if (lok) {
          const int gx0 = x0 + xs + q;
          if (gx0 + 8 <= W) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
              float4* d4 = reinterpret_cast<float4*>(wrow + k * wo.plane + q);
              d4[0] = make_float4(wv[k][0], wv[k][1], wv[k][2], wv[k][3]);
              d4[1] = make_float4(wv[k][4], wv[k][5], wv[k][6], wv[k][7]);
            }
          } else {
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
              for (int i = 0; i < 8; ++i)
                if (gx0 + i < W) wrow[k * wo.plane + q + i] = wv[k][i];
          }
        }
      }
      named_arrive(3 + b, NALL);                   // buffer b free again
    }
  }
}

template <int NC>
cudaError_t coef3_impl(const float* G, const float* stats, const float* vol, float* wbuf, WLayout wo, int W, int H,
                       int r, int L, float lam0, cudaStream_t st) {
  using Gm = CoefGeom<NC>;
  cudaError_t e = cudaFuncSetAttribute(k_coef3<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::SMEM);
  if (e != cudaSuccess) return e;
  // band height: enough CTAs to fill 148 SMs at least ~4 times, but long enough to amortise the warm-up
  const int strips = (W + C_TX - 1) / C_TX, batches = (L + C_LB - 1) / C_LB;
  int BH = 128;
  while (BH > 32 && (long long)strips * ((H + BH - 1) / BH) * batches < 4 * 148) BH /= 2;
  dim3 grid(strips, (H + BH - 1) / BH, batches);
  k_coef3<NC><<<grid, Gm::THREADS, Gm::SMEM, st>>>(G, stats, vol, wbuf, wo, W, H, r, L, BH, lam0);
  return cudaGetLastError();
}

}  // namespace v3
}  // namespace hgf
