// Stereo cost construction on the GPU: the label slices of the cost volume are built
// per coefficient chunk from the two views instead of being read from a caller-supplied volume, so only the
// images cross PCIe.  Cost (the paper defers it to Hosni et al.; form of SPEC S:400):
//
//   C(x, y, d) = a min(mean_c |L_c(x,y) - R_c(x-d,y)|, t_c) + (1-a) min(|dx Lbar(x,y) - dx Rbar(x-d,y)|, t_g)
//
// Lbar / Rbar channel means, dx the central x-difference (one-sided at the two border columns); x - d < 0
// takes the truncation value a t_c + (1-a) t_g.
//
// k_stereo_grad: dx of the channel mean, once per frame per view.
// k_stereo_cost: one CTA per 256-pixel row segment; the right-view segment the CTA's disparities touch
// (256 + Lc - 1 pixels x 4 planes) is staged in SMEM once and reused by every label; one coalesced store
// per (label, pixel).  HBM traffic: the 4-byte cost write per voxel (re-read by k_coef via TMA).
#include <cstdint>

#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace {

__global__ void k_stereo_grad(const float* __restrict__ img, float* __restrict__ grad, int W, int H) {
  const long long HW = (long long)W * H;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < HW; p += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(p % W);
    const long long row = p - x;
    auto gray = [&](int xx) {
      const long long q = row + xx;
      return ((img[q] + img[HW + q]) + img[2 * HW + q]) / 3.0f;
    };
    float g = 0.0f;
    if (W > 1) {
      if (x == 0) g = gray(1) - gray(0);
      else if (x == W - 1) g = gray(W - 1) - gray(W - 2);
      else g = (gray(x + 1) - gray(x - 1)) * 0.5f;
    }
    grad[p] = g;
  }
}

constexpr int SEG = 256;

__global__ void __launch_bounds__(SEG) k_stereo_cost(const float* __restrict__ left, const float* __restrict__ right,
                                                     const float* __restrict__ gl, const float* __restrict__ gr,
                                                     float* __restrict__ cost, int W, int H, int d0, int Lc,
                                                     float a, float tc, float tg) {
  extern __shared__ float rs[];                    // [4][SEG + Lc - 1]: right r, g, b, dx Rbar
  const int y = blockIdx.y, x0 = blockIdx.x * SEG, x = x0 + threadIdx.x;
  const long long HW = (long long)W * H, row = (long long)y * W;
  const int span = SEG + Lc - 1;
  const int xr0 = x0 - (d0 + Lc - 1);             // image column of rs[.][0]
  for (int i = threadIdx.x; i < span; i += SEG) {
    const int xr = xr0 + i;
    const bool in = xr >= 0 && xr < W;
    rs[i] = in ? __ldg(right + row + xr) : 0.0f;
    rs[span + i] = in ? __ldg(right + HW + row + xr) : 0.0f;
    rs[2 * span + i] = in ? __ldg(right + 2 * HW + row + xr) : 0.0f;
    rs[3 * span + i] = in ? __ldg(gr + row + xr) : 0.0f;
  }
  __syncthreads();
  if (x >= W) return;
  const float lr = __ldg(left + row + x), lg = __ldg(left + HW + row + x), lb = __ldg(left + 2 * HW + row + x);
  const float lgr = __ldg(gl + row + x);
  const float trunc = a * tc + (1.0f - a) * tg;
  float* out = cost + row + x;
#pragma unroll 4
  for (int k = 0; k < Lc; ++k) {
    const int d = d0 + k;
    float c = trunc;
    if (x - d >= 0) {
      const int i = x - d - xr0;
      const float col = ((fabsf(lr - rs[i]) + fabsf(lg - rs[span + i])) + fabsf(lb - rs[2 * span + i])) / 3.0f;
      const float grd = fabsf(lgr - rs[3 * span + i]);
      c = a * fminf(col, tc) + (1.0f - a) * fminf(grd, tg);
    }
    out[(long long)k * HW] = c;
  }
}

}  // namespace

cudaError_t launch_stereo_grad(const float* img, float* grad, int W, int H, cudaStream_t st) {
  const long long HW = (long long)W * H;
  const int blocks = (int)((HW + 255) / 256 < 148 * 16 ? (HW + 255) / 256 : 148 * 16);
  k_stereo_grad<<<blocks, 256, 0, st>>>(img, grad, W, H);
  return cudaGetLastError();
}

cudaError_t launch_stereo_cost(const float* left, const float* right, const float* gl, const float* gr, float* cost,
                               int W, int H, int d0, int Lc, float a, float tc, float tg, cudaStream_t st) {
  if (Lc < 1) return cudaSuccess;
  const size_t smem = sizeof(float) * 4 * (size_t)(SEG + Lc - 1);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_stereo_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((W + SEG - 1) / SEG, H);
  k_stereo_cost<<<grid, SEG, smem, st>>>(left, right, gl, gr, cost, W, H, d0, Lc, a, tc, tg);
  return cudaGetLastError();
}

}  // namespace hgf

// ----------------------------------------------------------------------------- segmentation (NEXT-4)
// Cost of the two labels (0 = foreground, 1 = background) from per-class per-channel colour histograms of
// the seed pixels (P:648-649 defers to Hosni et al.; form of SPEC S:406-409, readings S1/S2 in DESIGN.md):
//   bin(v) = min(floor(32 v), 31), p_c(b) = (count_c(b) + 1) / (N_c + 32),
//   C_c(x) = -sum_ch log p_c(bin(I_ch(x))) / (m log(N_c + 32))   in (0, 1].
namespace hgf {
namespace {

constexpr int SEG_BINS = 32;

__device__ __forceinline__ int seg_bin(float v) {
  const float f = floorf(v * (float)SEG_BINS);
  return f < 0.0f ? 0 : (f > (float)(SEG_BINS - 1) ? SEG_BINS - 1 : (int)f);
}

// counts: [2][m][32] int, seeds: [2] int (zeroed by the caller)
__global__ void k_seg_hist(const float* __restrict__ img, const uint8_t* __restrict__ fg,
                           const uint8_t* __restrict__ bg, int m, int W, int H, int* __restrict__ counts,
                           int* __restrict__ seeds) {
  extern __shared__ int sh[];                      // [2][m][32] + [2]
  const int nb = 2 * m * SEG_BINS;
  for (int i = threadIdx.x; i < nb + 2; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const long long HW = (long long)W * H;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < HW; p += (long long)gridDim.x * blockDim.x) {
    const bool f = fg[p] != 0, b = bg[p] != 0;
    if (!f && !b) continue;
    for (int c = 0; c < m; ++c) {
      const int bin = seg_bin(img[c * HW + p]);
      if (f) atomicAdd(&sh[(0 * m + c) * SEG_BINS + bin], 1);
      if (b) atomicAdd(&sh[(1 * m + c) * SEG_BINS + bin], 1);
    }
    if (f) atomicAdd(&sh[nb], 1);
    if (b) atomicAdd(&sh[nb + 1], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (sh[i]) atomicAdd(&counts[i], sh[i]);
  if (threadIdx.x < 2 && sh[nb + threadIdx.x]) atomicAdd(&seeds[threadIdx.x], sh[nb + threadIdx.x]);
}

__global__ void k_seg_cost(const float* __restrict__ img, const int* __restrict__ counts,
                           const int* __restrict__ seeds, int m, int W, int H, float* __restrict__ cost) {
  const long long HW = (long long)W * H;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < HW; p += (long long)gridDim.x * blockDim.x) {
    for (int k = 0; k < 2; ++k) {
      const float den = (float)seeds[k] + (float)SEG_BINS;
      float nll = 0.0f;
      for (int c = 0; c < m; ++c) {
        const int bin = seg_bin(img[c * HW + p]);
        nll -= logf(((float)counts[(k * m + c) * SEG_BINS + bin] + 1.0f) / den);
      }
      cost[k * HW + p] = nll / ((float)m * logf(den));
    }
  }
}

}  // namespace

cudaError_t launch_seg_hist(const float* img, const uint8_t* fg, const uint8_t* bg, int m, int W, int H, int* counts,
                            int* seeds, cudaStream_t st) {
  const long long HW = (long long)W * H;
  const int blocks = (int)((HW + 255) / 256 < 148 * 4 ? (HW + 255) / 256 : 148 * 4);
  const size_t smem = sizeof(int) * (2 * (size_t)m * SEG_BINS + 2);
  k_seg_hist<<<blocks, 256, smem, st>>>(img, fg, bg, m, W, H, counts, seeds);
  return cudaGetLastError();
}

cudaError_t launch_seg_cost(const float* img, const int* counts, const int* seeds, int m, int W, int H, float* cost,
                            cudaStream_t st) {
  const long long HW = (long long)W * H;
  const int blocks = (int)((HW + 255) / 256 < 148 * 16 ? (HW + 255) / 256 : 148 * 16);
  k_seg_cost<<<blocks, 256, 0, st>>>(img, counts, seeds, m, W, H, cost);
  return cudaGetLastError();
}

}  // namespace hgf
