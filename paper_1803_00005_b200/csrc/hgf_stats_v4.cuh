// Label-independent statistics, version 4 (k_stats4<n>): row-marching float64 Gram sums.
//
//   G_ab = B(G_a G_b), 0 <= a <= b <= n, G_0 = ones inside the image (Prop 2; Eq12), then
//   per pixel the Prop-1 recursion (Eq4, readings F1/F2; stats_finish, shared with k_stats2).
//
// k_stats2 box-filters 16x16 tiles with a 2r halo on both axes (4.5x the products at r = 9) and runs its
// recursion on 1/4.5 of the staged pixels.  Here a CTA owns a strip of TX = 64 output columns and a band
// of BH rows and marches down it RB = 2 output rows per iteration:
//   * V phase (thread = strip column c of the TX + 2r columns, image x = x0 - r + c): vertical running
//     sums of the NPAIR products, float64, updated by the entering row y + r and the leaving row y - r - 1
//     (channel values read straight from global memory, coalesced across the warp); the sums of each of
//     the RB rows are written to vs[rb][pair][c], the last one is the next iteration's start.  Rows and
//     columns outside the image read as zero (G_0 included): the clipped windows (F6).
//   * H phase (item = (rb, 16-column segment, pair), pairs fastest): horizontal sliding window of 2r + 1
//     V columns -> hs[rb][pair][x].
//   * R phase (thread = (rb, x)): the pixel's NPAIR Gram sums from hs (lanes = consecutive x,
//     conflict-free), the recursion and the record, in registers.
// Pitches are odd in doubles so that the H phase's pair-strided accesses spread over the banks.
// fp32 x fp32 products are exact in float64; a running sum accumulates at most BH + 2r + 1 row updates.
#pragma once
#include <cstdlib>
#include "hgf_common.cuh"
#include "hgf_launch.h"
#include "hgf_stats_finish.cuh"

#ifndef HGF_ST4_EXP
#define HGF_ST4_EXP 0   // timing experiments only: 1 = no R phase, 2 = no H phase, 3 = neither (wrong results)
#endif

namespace hgf {
namespace st4 {

constexpr int TX = 64;             // output columns per strip
constexpr int RB = 2;              // output rows per iteration
constexpr int THREADS = RB * TX;   // one R item per thread; TX + 2r <= THREADS for r <= 32
constexpr int HSEG = 16;           // pixels per H item
constexpr int NSEG = TX / HSEG;
constexpr int TXP = TX + 1;        // hs row pitch (doubles, odd)

__host__ __device__ constexpr int npair(int n) { return (n + 1) * (n + 2) / 2 - 1; }
// sums per pixel: the Gram pairs, plus (LP = 1, the fused single-slice variant) the cost sums B(G_a p), a = 0..n
__host__ __device__ constexpr int nsums(int n, int lp) { return npair(n) + lp * (n + 1); }
__host__ __device__ inline int vx_pitch(int r) { return (TX + 2 * r) | 1; }
__host__ __device__ inline size_t smem_bytes(int NC, int r, int lp = 0) {
  return (size_t)RB * nsums(NC, lp) * (vx_pitch(r) + TXP) * sizeof(double);
}

// Band height from (W, H) only (row-sharded statistics stay bit-identical, also between k_stats4 and k_stats5):
// >= ~6 CTAs per SM over the whole image where it allows, bands of at most 64 rows (measured at C4: 64 -> 0.89 ms,
// 128 -> 0.95 ms; a waves x (band + warm-up) model picked badly for the fused single-slice pass at r = 4;
// HGF_STATS4_BH sweeps).
inline int band_height(int W, int H) {
  const int strips = (W + TX - 1) / TX;
  int BH = 64;
  while (BH > 16 && (long long)strips * ((H + BH - 1) / BH) < 6 * 148) BH /= 2;
  const char* e = std::getenv("HGF_STATS4_BH");     // tuning runs only
  if (e && std::atoi(e) >= 8) BH = std::atoi(e);
  return BH;
}

// Rows [yb0, yb1).  CTA (bx, by) owns columns [bx*TX, +TX) and the absolute band of rows
// [(yb0/BH + by)*BH, +BH), BH a function of (W, H) only: every row's running sums have the same history
// whichever row range is requested, so row-sharded statistics are bit-identical to the full pass.
// LP = 1 (hgf_filter, one slice p): the cost is an extra channel whose products with G_0..G_n are summed with the
// Gram pairs, and the R phase writes the slice's coefficients w (planar, wl) instead of the statistics
// (filter_finish_m): the statistics never reach HBM and no coefficient kernel runs.
// RT > 0: the radius as a compile-time constant (the H phase's window loops unroll and their shared loads issue
// ahead of the dependent adds); RT = 0: r at run time.
template <int NC, int LP, int RT>
__global__ void __launch_bounds__(THREADS) k_stats4(const float* __restrict__ G, float* __restrict__ stats, int W,
                                                    int H, int r_arg, double lam, int mode, int aos, float lam0f,
                                                    int yb0, int yb1, int BH, const float* __restrict__ P,
                                                    float* __restrict__ wout, WLayout wo) {
  const int r = RT > 0 ? RT : r_arg;
  constexpr int K = NC + 1;
  constexpr int NG = npair(NC);                 // Gram pairs
  constexpr int NPAIR = nsums(NC, LP);          // all running sums
  extern __shared__ __align__(16) double sd[];
  const int VXP = vx_pitch(r);
  double* vs = sd;                             // [RB][NPAIR][VXP]
  double* hs = sd + RB * NPAIR * VXP;          // [RB][NPAIR][TXP]
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TX;
  const int Y0 = (yb0 / BH + (int)blockIdx.y) * BH, Y1 = min(H, Y0 + BH);
  const int Z0 = max(Y0, yb0), Z1 = min(Y1, yb1);      // rows written
  const int CX = TX + 2 * r;
  const long long HW = (long long)H * W;

  // channel values of image row yy at this thread's V column (zero outside the image)
  const int vx = x0 - r + tid;
  const bool vcol = tid < CX;
  const bool xin = vcol && vx >= 0 && vx < W;
  auto load_row = [&](int yy, float (&v)[K + LP]) {
    const bool in = xin && yy >= 0 && yy < H;
    v[0] = in ? 1.0f : 0.0f;
    const float* src = G + (long long)yy * W + vx;
#pragma unroll
    for (int k = 1; k < K; ++k) v[k] = in ? __ldg(src + (k - 1) * HW) : 0.0f;
    if (LP) v[K] = in ? __ldg(P + (long long)yy * W + vx) : 0.0f;
  };

  // warm-up: the window of output row Y0 - 1 (rows Y0 - 1 - r .. Y0 - 1 + r), kept in vs[RB - 1]
  if (vcol) {
    double acc[NPAIR];
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) acc[q] = 0.0;
    for (int yy = Y0 - 1 - r; yy <= Y0 - 1 + r; ++yy) {
      float e[K + LP];
      load_row(yy, e);
      int q = 0;
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = a; b < K; ++b) {
          if (a == 0 && b == 0) continue;
          acc[q] = fma((double)e[a], (double)e[b], acc[q]);
          ++q;
        }
      if constexpr (LP == 1) {
#pragma unroll
        for (int a = 0; a < K; ++a) acc[NG + a] = fma((double)e[a], (double)e[K], acc[NG + a]);
      }
    }
    double* dst = vs + (RB - 1) * NPAIR * VXP + tid;
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) dst[q * VXP] = acc[q];
  }

  for (int yb = Y0; yb < Z1; yb += RB) {
    // ---- V phase: rows yb .. yb + RB - 1
    if (vcol) {
      float e[RB][K + LP], l[RB][K + LP];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        load_row(yb + rb + r, e[rb]);
        load_row(yb + rb - r - 1, l[rb]);
      }
      double acc[NPAIR];
      const double* src = vs + (RB - 1) * NPAIR * VXP + tid;
#pragma unroll
      for (int q = 0; q < NPAIR; ++q) acc[q] = src[q * VXP];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        int q = 0;
#pragma unroll
        for (int a = 0; a < K; ++a)
#pragma unroll
          for (int b = a; b < K; ++b) {
            if (a == 0 && b == 0) continue;
            acc[q] = fma((double)e[rb][a], (double)e[rb][b], fma(-(double)l[rb][a], (double)l[rb][b], acc[q]));
            ++q;
          }
        if constexpr (LP == 1) {
#pragma unroll
          for (int a = 0; a < K; ++a)
            acc[NG + a] = fma((double)e[rb][a], (double)e[rb][K], fma(-(double)l[rb][a], (double)l[rb][K], acc[NG + a]));
        }
        double* dst = vs + rb * NPAIR * VXP + tid;
#pragma unroll
        for (int q2 = 0; q2 < NPAIR; ++q2) dst[q2 * VXP] = acc[q2];
      }
    }
    if (yb + RB <= Z0) continue;                 // rows before the requested range: V only (same thread)
    __syncthreads();
    // ---- H phase: sliding 2r+1-column window sums per (rb, segment, pair); 32-pixel segments when all the items
    // then fit one pass of the CTA (fewer window re-reads: 2.5 instead of 3 loads per output; C4 -6 %), else 16
    constexpr int HS = RB * (TX / 32) * NPAIR <= THREADS ? 32 : HSEG;
    constexpr int NS = TX / HS;
    for (int item = tid; item < ((HGF_ST4_EXP & 2) ? 0 : RB * NS * NPAIR); item += THREADS) {
      const int q = item % NPAIR, sg = (item / NPAIR) % NS, rb = item / (NPAIR * NS);
      const double* v = vs + (rb * NPAIR + q) * VXP + sg * HS;
      double* o = hs + (rb * NPAIR + q) * TXP + sg * HS;
      double a = 0.0;
      for (int j = 0; j <= 2 * r; ++j) a += v[j];
      o[0] = a;
#pragma unroll
      for (int i = 1; i < HS; ++i) {
        a += v[i + 2 * r] - v[i - 1];
        o[i] = a;
      }
    }
    __syncthreads();
    // ---- R phase: one pixel per thread
    {
      const int rb = tid / TX, x = tid % TX;
      const int gy = yb + rb, gx = x0 + x;
      if (!(HGF_ST4_EXP & 1) && gy >= Z0 && gy < Z1 && gx < W) {
        double g[NPAIR];
        const double* src = hs + rb * NPAIR * TXP + x;
#pragma unroll
        for (int q = 0; q < NPAIR; ++q) g[q] = src[q * TXP];
        const double N = (double)window_count(gy, gx, H, W, r);
        if constexpr (LP == 1) {
          float* wl = wout + wo.origin + (long long)gy * wo.pitch + gx;
          if (mode == 0) filter_finish_m<NC, 0>(g, N, lam, lam0f, wl, wo.plane);
          else filter_finish_m<NC, 1>(g, N, lam, lam0f, wl, wo.plane);
        } else {
          stats_finish<NC>(g, N, lam, mode, aos, lam0f, stats, (long long)gy * W + gx, HW);
        }
      }
    }
    // the next V phase overwrites vs only (hs is rewritten after the next barrier)
  }
}

template <int NC, int LP, int RT>
cudaError_t stats4_launch_r(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos,
                          float lam0f, int y0, int y1, const float* P, float* wout, WLayout wo, cudaStream_t st) {
  if (aos && NC > kCoef3MaxN) return cudaErrorInvalidValue;
  if (TX + 2 * r > THREADS) return cudaErrorInvalidValue;
  const size_t smem = smem_bytes(NC, r, LP);
  cudaError_t e = cudaFuncSetAttribute(k_stats4<NC, LP, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (y0 >= y1) return cudaSuccess;
  const int strips = (W + TX - 1) / TX;
  const int BH = band_height(W, H);
  dim3 grid(strips, (y1 + BH - 1) / BH - y0 / BH);
  k_stats4<NC, LP, RT><<<grid, THREADS, smem, st>>>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, BH, P, wout, wo);
  return cudaGetLastError();
}

template <int NC, int LP>
cudaError_t stats4_launch(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos,
                          float lam0f, int y0, int y1, const float* P, float* wout, WLayout wo, cudaStream_t st) {
  if (r == 9)   // the paper's / BASELINE's radius
    return stats4_launch_r<NC, LP, 9>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, P, wout, wo, st);
  return stats4_launch_r<NC, LP, 0>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, P, wout, wo, st);
}

template <int NC>
cudaError_t stats4_impl(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos, float lam0f,
                        int y0, int y1, cudaStream_t st) {
  return stats4_launch<NC, 0>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, nullptr, nullptr, WLayout{}, st);
}

// hgf_filter's fused single-slice pass: guidance G, cost slice P -> coefficients w (planar layout wo) of all rows.
template <int NC>
cudaError_t filter1_impl(const float* G, const float* P, float* wout, WLayout wo, int W, int H, int r, double lam,
                         int mode, float lam0f, cudaStream_t st) {
  return stats4_launch<NC, 1>(G, nullptr, W, H, r, lam, mode, 0, lam0f, 0, H, P, wout, wo, st);
}

}  // namespace st4
}  // namespace hgf
