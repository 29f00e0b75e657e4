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
#include <climits>
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

// dir = +1: the left view's cost (match at x - d in the other view); dir = -1: the right view's cost
// (reading P1, match at x + d).  `base` is the view whose pixels the slices index, `other` the searched one.
__global__ void __launch_bounds__(SEG) k_stereo_cost(const float* __restrict__ base, const float* __restrict__ other,
                                                     const float* __restrict__ gb, const float* __restrict__ go,
                                                     float* __restrict__ cost, int W, int H, int d0, int Lc, int dir,
                                                     float a, float tc, float tg) {
  extern __shared__ float rs[];                    // [4][SEG + Lc - 1]: other view r, g, b, dx of its mean
  const int y = blockIdx.y, x0 = blockIdx.x * SEG, x = x0 + threadIdx.x;
  const long long HW = (long long)W * H, row = (long long)y * W;
  const int span = SEG + Lc - 1;
  // image column of rs[.][0]: the smallest column any (pixel, disparity) of the CTA reads
  const long long xr0 = dir > 0 ? (long long)x0 - d0 - (Lc - 1) : (long long)x0 + d0;
  for (int i = threadIdx.x; i < span; i += SEG) {
    const long long xr = xr0 + i;
    const bool in = xr >= 0 && xr < W;
    rs[i] = in ? __ldg(other + row + xr) : 0.0f;
    rs[span + i] = in ? __ldg(other + HW + row + xr) : 0.0f;
    rs[2 * span + i] = in ? __ldg(other + 2 * HW + row + xr) : 0.0f;
    rs[3 * span + i] = in ? __ldg(go + row + xr) : 0.0f;
  }
  __syncthreads();
  if (x >= W) return;
  const float lr = __ldg(base + row + x), lg = __ldg(base + HW + row + x), lb = __ldg(base + 2 * HW + row + x);
  const float lgr = __ldg(gb + row + x);
  const float trunc = a * tc + (1.0f - a) * tg;
  float* out = cost + row + x;
#pragma unroll 4
  for (int k = 0; k < Lc; ++k) {
    const long long xo = (long long)x - (long long)dir * (d0 + k);
    float c = trunc;
    if (xo >= 0 && xo < W) {
      const int i = (int)(xo - xr0);
      const float col = ((fabsf(lr - rs[i]) + fabsf(lg - rs[span + i])) + fabsf(lb - rs[2 * span + i])) / 3.0f;
      const float grd = fabsf(lgr - rs[3 * span + i]);
      c = a * fminf(col, tc) + (1.0f - a) * fminf(grd, tg);
    }
    out[(long long)k * HW] = c;
  }
}

// k_stereo_cost4: the same cost, 4 consecutive pixels per thread (512-pixel row segments, 128 threads).  Per
// label a thread loads one new column of the other view per plane and slides the other three in registers
// (the 4 pixels' matches at disparity d + 1 are their matches at d shifted by one column), and writes the 4
// costs with one 16-byte store: 1 shared load per plane and 1/4 store per voxel instead of 4 loads and 1 store
// (k_stereo_cost).  Requires W % 4 == 0 (16-byte aligned rows); the arithmetic per voxel is k_stereo_cost's.
constexpr int SEG4 = 512, T4 = SEG4 / 4;

// The label loop of k_stereo_cost4.  The colour term a min(mean_c |.|, t_c) is evaluated as
// (a/3) min(sum_c |.|, 3 t_c) (one multiply instead of a division; within an ulp of the literal form).
template <int DIR, bool CHECK>
__device__ __forceinline__ void cost4_labels(float (&w)[4][4], const float (&lr)[4], const float (&lg)[4],
                                             const float (&lb)[4], const float (&lgr)[4], const float* rs, int span,
                                             int ib, int xb, int d0, int Lc, int W, long long HW, float a, float tc,
                                             float tg, float* out) {
  const float trunc = a * tc + (1.0f - a) * tg;
  const float a3 = a / 3.0f, tc3 = 3.0f * tc, ag = 1.0f - a;
#pragma unroll 2
  for (int k = 0; k < Lc; ++k) {
    if (k > 0) {
      if (DIR > 0) {
        const int i = ib - k;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          w[c][3] = w[c][2]; w[c][2] = w[c][1]; w[c][1] = w[c][0];
          w[c][0] = rs[c * span + i];
        }
      } else {
        const int i = ib + k + 3;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          w[c][0] = w[c][1]; w[c][1] = w[c][2]; w[c][2] = w[c][3];
          w[c][3] = rs[c * span + i];
        }
      }
    }
    float cv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float col = (fabsf(lr[j] - w[0][j]) + fabsf(lg[j] - w[1][j])) + fabsf(lb[j] - w[2][j]);
      const float grd = fabsf(lgr[j] - w[3][j]);
      float c = fmaf(a3, fminf(col, tc3), ag * fminf(grd, tg));
      if (CHECK) {
        const int xo = xb + j - DIR * (d0 + k);
        if (xo < 0 || xo >= W) c = trunc;
      }
      cv[j] = c;
    }
    *reinterpret_cast<float4*>(out) = make_float4(cv[0], cv[1], cv[2], cv[3]);
    out += HW;
  }
}

template <int DIR>
__global__ void __launch_bounds__(T4) k_stereo_cost4(const float* __restrict__ base, const float* __restrict__ other,
                                                     const float* __restrict__ gb, const float* __restrict__ go,
                                                     float* __restrict__ cost, int W, int H, int d0, int Lc,
                                                     float a, float tc, float tg) {
  extern __shared__ float rs[];                    // [4][SEG4 + Lc + 3]: other view r, g, b, dx of its mean
  const int y = blockIdx.y, x0 = blockIdx.x * SEG4, xb = x0 + 4 * threadIdx.x;
  const long long HW = (long long)W * H, row = (long long)y * W;
  const int span = SEG4 + Lc + 3;
  // image column of rs[.][0]: the smallest column any (pixel, disparity) of the CTA reads, minus one slack column
  const int xr0 = DIR > 0 ? x0 - d0 - Lc : x0 + d0 - 1;
  for (int i = threadIdx.x; i < span; i += T4) {
    const int xr = xr0 + i;
    const bool in = xr >= 0 && xr < W;
    rs[i] = in ? __ldg(other + row + xr) : 0.0f;
    rs[span + i] = in ? __ldg(other + HW + row + xr) : 0.0f;
    rs[2 * span + i] = in ? __ldg(other + 2 * HW + row + xr) : 0.0f;
    rs[3 * span + i] = in ? __ldg(go + row + xr) : 0.0f;
  }
  __syncthreads();
  if (xb >= W) return;
  const float4 r4 = __ldg(reinterpret_cast<const float4*>(base + row + xb));
  const float4 g4 = __ldg(reinterpret_cast<const float4*>(base + HW + row + xb));
  const float4 b4 = __ldg(reinterpret_cast<const float4*>(base + 2 * HW + row + xb));
  const float4 d4 = __ldg(reinterpret_cast<const float4*>(gb + row + xb));
  const float lr[4] = {r4.x, r4.y, r4.z, r4.w}, lg[4] = {g4.x, g4.y, g4.z, g4.w};
  const float lb[4] = {b4.x, b4.y, b4.z, b4.w}, lgr[4] = {d4.x, d4.y, d4.z, d4.w};
  // window w[.][j] = other-view column of pixel xb + j at the current disparity d0 + k:
  // DIR > 0: xb + j - d (index ib + j - k), DIR < 0: xb + j + d (index ib + j + k)
  const int ib = DIR > 0 ? xb - d0 - xr0 : xb + d0 - xr0;
  float w[4][4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int j = 0; j < 4; ++j) w[c][j] = rs[c * span + ib + j];
  float* out = cost + row + xb;
  // interior CTAs (every match column inside the image for every label) skip the per-voxel bounds test
  const bool interior = DIR > 0 ? x0 - d0 - (Lc - 1) >= 0 : x0 + SEG4 - 1 + d0 + Lc - 1 < W;
  if (interior)
    cost4_labels<DIR, false>(w, lr, lg, lb, lgr, rs, span, ib, xb, d0, Lc, W, HW, a, tc, tg, out);
  else
    cost4_labels<DIR, true>(w, lr, lg, lb, lgr, rs, span, ib, xb, d0, Lc, W, HW, a, tc, tg, out);
}

}  // namespace

cudaError_t launch_stereo_grad(const float* img, float* grad, int W, int H, cudaStream_t st) {
  const long long HW = (long long)W * H;
  const int blocks = (int)((HW + 255) / 256 < 148 * 16 ? (HW + 255) / 256 : 148 * 16);
  k_stereo_grad<<<blocks, 256, 0, st>>>(img, grad, W, H);
  return cudaGetLastError();
}

cudaError_t launch_stereo_cost(const float* base, const float* other, const float* gb, const float* go, float* cost,
                               int W, int H, int d0, int Lc, int dir, float a, float tc, float tg, cudaStream_t st) {
  if (Lc < 1) return cudaSuccess;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  // k_stereo_cost4 indexes columns x0 -+ d0 -+ Lc in 32-bit int: only when d0 + Lc stays within W + 2 segments
  // (larger disparities all read as out of range, which the generic kernel handles in 64-bit arithmetic)
  if (W % 4 == 0 && Lc <= 4096 && (long long)d0 + Lc <= (long long)W + 2 * SEG4 && al16(base) && al16(gb) &&
      al16(cost)) {
    const size_t smem4 = sizeof(float) * 4 * (size_t)(SEG4 + Lc + 3);
    if (smem4 <= 200 * 1024) {
      auto kern = dir > 0 ? k_stereo_cost4<1> : k_stereo_cost4<-1>;
      if (smem4 > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem4);
        if (e != cudaSuccess) return e;
      }
      dim3 grid4((W + SEG4 - 1) / SEG4, H);
      kern<<<grid4, T4, smem4, st>>>(base, other, gb, go, cost, W, H, d0, Lc, a, tc, tg);
      return cudaGetLastError();
    }
  }
  const size_t smem = sizeof(float) * 4 * (size_t)(SEG + Lc - 1);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_stereo_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((W + SEG - 1) / SEG, H);
  k_stereo_cost<<<grid, SEG, smem, st>>>(base, other, gb, go, cost, W, H, d0, Lc, dir, a, tc, tg);
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

// ----------------------------------------------------------------------------- post-processing (NEXT-3)
// Readings P2-P4 (P:641 names the step only).
namespace hgf {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// One warp per row.  Pass 1 (left to right, 32 columns at a time): the consistency flag of every pixel and
// the index of the nearest consistent pixel at or left of it (inclusive max-scan of "x if consistent else
// -1" across the warp, carried between chunks), kept in `fill`.  Pass 2 (right to left): the nearest
// consistent pixel at or right of it (suffix min-scan), then the fill value of P3.
__global__ void k_lr_fill(const int* __restrict__ dL, const int* __restrict__ dR, int W, int H, int tol,
                          uint8_t* __restrict__ valid, int* __restrict__ fill) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int y = blockIdx.x * wpb + (threadIdx.x >> 5); y < H; y += gridDim.x * wpb) {
    const long long row = (long long)y * W;
    int carry = -1;
    for (int c0 = 0; c0 < W; c0 += 32) {
      const int x = c0 + lane;
      int idx = -1;
      if (x < W) {
        const int d = dL[row + x];
        const long long t = (long long)x - d;
        bool ok = false;
        if (t >= 0 && t < W) {
          const long long diff = (long long)d - dR[row + t];
          ok = (diff < 0 ? -diff : diff) <= tol;
        }
        valid[row + x] = ok ? 1 : 0;
        idx = ok ? x : -1;
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(kFull, idx, off);
        if (lane >= off) idx = max(idx, v);
      }
      idx = max(idx, carry);
      carry = __shfl_sync(kFull, idx, 31);
      if (x < W) fill[row + x] = idx;
    }
    __syncwarp();
    carry = W;
    for (int c0 = ((W - 1) / 32) * 32; c0 >= 0; c0 -= 32) {
      const int x = c0 + lane;
      int idx = W;
      bool ok = true;
      if (x < W) {
        ok = valid[row + x] != 0;
        idx = ok ? x : W;
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_down_sync(kFull, idx, off);
        if (lane + off < 32) idx = min(idx, v);
      }
      idx = min(idx, carry);
      carry = __shfl_sync(kFull, idx, 0);
      if (x < W && !ok) {
        const int li = fill[row + x];
        const bool hl = li >= 0, hr = idx < W;
        const int vl = hl ? dL[row + li] : 0, vr = hr ? dL[row + idx] : 0;
        fill[row + x] = (hl && hr) ? min(vl, vr) : (hl ? vl : (hr ? vr : dL[row + x]));
      } else if (x < W) {
        fill[row + x] = dL[row + x];
      }
    }
  }
}

// One warp per 32-pixel run of a row.  Consistent pixels copy the filled map; for each inconsistent pixel
// (ballot) the whole warp stages the window's values and bilateral weights in SMEM, sums the weights
// (lane partials in a fixed order, then a shfl_down tree and a broadcast, so every lane holds the same
// float), and bisects on the disparity: s(d) = sum_{D(q) <= d} w is non-decreasing in d in that fixed
// order, s(max) equals the total bit for bit, so the smallest d with s(d) >= total / 2 is a window value.
__device__ __forceinline__ float warp_sum_bcast(float v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
  return __shfl_sync(kFull, v, 0);
}

__global__ void k_wmf(const int* __restrict__ fill, const uint8_t* __restrict__ valid, const float* __restrict__ img,
                      int m, int W, int H, int radius, float inv_ss2, float inv_sc2, int* __restrict__ out) {
  extern __shared__ float wsm[];                   // per warp: [n] weights then [n] values (as int)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int side = 2 * radius + 1, nwin = side * side;
  float* ws = wsm + (size_t)wib * 2 * nwin;
  int* vs = reinterpret_cast<int*>(ws + nwin);
  const long long HW = (long long)W * H;
  const int runs = (W + 31) / 32;
  const long long nrun = (long long)runs * H;
  for (long long rn = (long long)blockIdx.x * wpb + wib; rn < nrun; rn += (long long)gridDim.x * wpb) {
    const int y = (int)(rn / runs), x = (int)(rn % runs) * 32 + lane;
    const long long p = (long long)y * W + x;
    bool todo = false;
    if (x < W) {
      todo = valid[p] == 0;
      if (!todo) out[p] = fill[p];
    }
    unsigned pend = __ballot_sync(kFull, todo);
    while (pend) {
      const int src = __ffs(pend) - 1;
      pend &= pend - 1;
      const int px = (int)(rn % runs) * 32 + src;
      const int y0 = max(0, y - radius), y1 = min(H, y + radius + 1);
      const int x0 = max(0, px - radius), x1 = min(W, px + radius + 1);
      const int ww = x1 - x0, n = (y1 - y0) * ww;
      const long long pc = (long long)y * W + px;
      float part = 0.0f;
      int dmin = INT_MAX, dmax = INT_MIN;
      for (int e = lane; e < n; e += 32) {
        const int qy = y0 + e / ww, qx = x0 + e % ww;
        const long long q = (long long)qy * W + qx;
        float c2 = 0.0f;
        for (int c = 0; c < m; ++c) {
          const float dc = __ldg(img + c * HW + q) - __ldg(img + c * HW + pc);
          c2 = fmaf(dc, dc, c2);
        }
        const float dy = (float)(qy - y), dx = (float)(qx - px);
        const float w = expf(-(dy * dy + dx * dx) * inv_ss2 - c2 * inv_sc2);
        const int v = fill[q];
        ws[e] = w;
        vs[e] = v;
        part += w;
        dmin = min(dmin, v);
        dmax = max(dmax, v);
      }
      const float half = 0.5f * warp_sum_bcast(part);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        dmin = min(dmin, __shfl_xor_sync(kFull, dmin, off));
        dmax = max(dmax, __shfl_xor_sync(kFull, dmax, off));
      }
      __syncwarp();
      long long lo = dmin, hi = dmax;
      while (lo < hi) {
        const long long mid = lo + (hi - lo) / 2;
        float s = 0.0f;
        for (int e = lane; e < n; e += 32) s += vs[e] <= mid ? ws[e] : 0.0f;
        if (warp_sum_bcast(s) >= half) hi = mid; else lo = mid + 1;
      }
      if (lane == 0) out[pc] = (int)lo;
      __syncwarp();
    }
  }
}

}  // namespace

int lr_wmf_max_radius() { return 15; }

cudaError_t launch_lr_fill(const int* dL, const int* dR, int W, int H, int tol, uint8_t* valid, int* fill,
                           cudaStream_t st) {
  const int wpb = 4;
  const int blocks = (H + wpb - 1) / wpb;
  k_lr_fill<<<blocks, wpb * 32, 0, st>>>(dL, dR, W, H, tol, valid, fill);
  return cudaGetLastError();
}

cudaError_t launch_wmf(const int* fill, const uint8_t* valid, const float* img, int m, int W, int H, int radius,
                       float sigma_s, float sigma_c, int* out, cudaStream_t st) {
  const int wpb = 8;
  const int nwin = (2 * radius + 1) * (2 * radius + 1);
  const size_t smem = sizeof(float) * 2 * (size_t)nwin * wpb;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_wmf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long nrun = (long long)((W + 31) / 32) * H;
  const long long need = (nrun + wpb - 1) / wpb;
  const int blocks = (int)(need < 148 * 16 ? need : 148 * 16);
  k_wmf<<<blocks, wpb * 32, smem, st>>>(fill, valid, img, m, W, H, radius, 1.0f / (sigma_s * sigma_s),
                                       1.0f / (sigma_c * sigma_c), out);
  return cudaGetLastError();
}

}  // namespace hgf
