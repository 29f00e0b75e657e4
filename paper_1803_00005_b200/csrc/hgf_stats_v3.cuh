// Label-independent statistics for many channels, version 3 (n >= 7; BASELINE config 5 sweeps n up to 20).
//
// Same quantities as k_stats / k_stats2 (Gram G_ij = B(G_i G_j) in float64, Prop 2; the Prop-1
// recursion P:134-153 with readings F1/F2; P' = -lambda alpha_{1..n,1..n}, nu_k = B(G_k)/(lambda_0 + N)),
// organised so that nothing per pixel has to live in one thread's registers: at n = 20 the Gram has 230
// entries and alpha 441, which k_stats2 spilled to local memory (20-70 ms per 1080p frame).
//
//   k_gram_h3  : horizontal window sums of every product plane G_i G_j (i <= j, (0,0) excluded) in float64,
//                one thread per output pixel, the row segment staged in SMEM -> hs[p][y][x]
//   k_gram_v3  : vertical sliding sums of hs -> the box-summed Gram planes gram[p][y][x] (float64)
//   k_recur3   : a CTA takes 32 consecutive pixels: their Gram entries are staged in SMEM with coalesced
//                loads (lane = pixel), then one warp per pixel runs the recursion with lane i holding row i
//                of alpha in registers (u_i: a dot product per lane; the quadratic form: a warp reduction;
//                the rank-one update: per lane, with u broadcast from SMEM); the outputs are staged in SMEM
//                and written plane by plane (lane = pixel).
#pragma once
#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace st3 {

constexpr int HX = 128;          // k_gram_h3 / k_gram_v3: pixels per CTA along x
constexpr int VROWS = 32;        // k_gram_v3: output rows per CTA (vertical sliding restarts per CTA)
constexpr int PIX = 16;          // k_recur3: pixels per CTA
constexpr int RW = 8;            // k_recur3: warps per CTA
constexpr int PB = 32;           // product planes per horizontal/vertical batch (bounds the scratch)

__host__ __device__ constexpr int npairs(int NC) { return (NC + 1) * (NC + 2) / 2 - 1; }

// pair index p of (i, j), 0 <= i <= j <= n, (0,0) excluded: row-major over the upper triangle
__device__ __forceinline__ int pair_index(int i, int j, int K) { return i * K - i * (i - 1) / 2 + (j - i) - 1; }

// One CTA per (row, 128-pixel segment): all K channel rows staged once (row pitch = 1 mod 32 floats, so
// lanes reading different channels hit different banks), then items (pair z of the batch, 16-pixel
// sub-segment s), pairs fastest across the lanes: each slides the 2r+1 window over its 16 pixels in float64
// (2r+1 products to start, 2 per further pixel: O(1) in r); the sums are staged in SMEM and written out
// coalesced, one plane row at a time.
constexpr int HSUB = 16;
__host__ __device__ inline int gram_h3_span(int r) { return (HX + 2 * r + 31) / 32 * 32 + 1; }
__host__ __device__ inline size_t gram_h3_smem(int NC, int r) {
  return ((size_t)(NC + 1) * gram_h3_span(r) * sizeof(float) + 15) / 16 * 16 + (size_t)PB * (HX + 1) * sizeof(double);
}
template <int NC>
__global__ void __launch_bounds__(HX) k_gram_h3(const float* __restrict__ G, double* __restrict__ hs, int W, int H,
                                                 int r, int p0, int pb) {
  constexpr int K = NC + 1;
  extern __shared__ __align__(16) unsigned char h3_raw[];
  float* row = reinterpret_cast<float*>(h3_raw);    // [K][span]: the channel rows (channel 0 = ones)
  const int span = gram_h3_span(r);
  double* ob = reinterpret_cast<double*>(h3_raw + ((size_t)K * span * sizeof(float) + 15) / 16 * 16);  // [PB][HX+1]
  const int y = blockIdx.y, x0 = blockIdx.x * HX;
  const int wrow = HX + 2 * r;
  const long long HW = (long long)H * W;
  for (int e = threadIdx.x; e < K * wrow; e += HX) {
    const int c = e / wrow, xx = x0 - r + (e % wrow);
    const bool in = xx >= 0 && xx < W;
    row[c * span + e % wrow] = in ? (c == 0 ? 1.0f : __ldg(G + (c - 1) * HW + (long long)y * W + xx)) : 0.0f;
  }
  __syncthreads();
  for (int item = threadIdx.x; item < pb * (HX / HSUB); item += HX) {
    const int z = item % pb, sub = item / pb;
    int i = 0, q = p0 + z + 1;
    while (q >= K - i) { q -= K - i; ++i; }
    const int j = i + q;
    const float* ri = row + i * span + sub * HSUB;
    const float* rj = row + j * span + sub * HSUB;
    double* o = ob + z * (HX + 1) + sub * HSUB;
    double acc = 0.0;
    for (int dx = 0; dx <= 2 * r; ++dx) acc = fma((double)ri[dx], (double)rj[dx], acc);
    o[0] = acc;
#pragma unroll
    for (int t = 1; t < HSUB; ++t) {
      acc = fma((double)ri[t + 2 * r], (double)rj[t + 2 * r], fma(-(double)ri[t - 1], (double)rj[t - 1], acc));
      o[t] = acc;
    }
  }
  __syncthreads();
  const int x = x0 + threadIdx.x;
  if (x >= W) return;
  for (int z = 0; z < pb; ++z) hs[(long long)z * HW + (long long)y * W + x] = ob[z * (HX + 1) + threadIdx.x];
}

template <int NC>   // (templated only so that every per-n translation unit owns its instance)
__global__ void __launch_bounds__(HX) k_gram_v3(const double* __restrict__ hs, double* __restrict__ gram, int W,
                                                 int H, int r, int p0) {
  const int x = blockIdx.x * HX + threadIdx.x, y0 = blockIdx.y * VROWS;
  if (x >= W) return;
  const long long HW = (long long)H * W;
  const double* col = hs + (long long)blockIdx.z * HW + x;
  double* out = gram + (long long)(p0 + blockIdx.z) * HW + x;
  const int y1 = min(H, y0 + VROWS);
  double acc = 0.0;
  for (int yy = max(0, y0 - r); yy <= min(H - 1, y0 + r); ++yy) acc += col[(long long)yy * W];
  out[(long long)y0 * W] = acc;
  for (int y = y0 + 1; y < y1; ++y) {
    if (y + r < H) acc += col[(long long)(y + r) * W];
    if (y - r - 1 >= 0) acc -= col[(long long)(y - r - 1) * W];
    out[(long long)y * W] = acc;
  }
}

// Per-warp dense Gram row pitch (doubles): >= K, even (16-byte aligned rows for the 128-bit broadcasts).
__host__ __device__ constexpr int gs_pitch(int K) { return (K + 1) / 2 * 2; }
__host__ __device__ constexpr size_t recur3_smem(int NC) {
  return sizeof(double) * (((size_t)npairs(NC) * (PIX + 1) + 1) / 2 * 2 + (size_t)RW * (NC + 1) * gs_pitch(NC + 1) +
                           RW * 32) +
         sizeof(float) * (size_t)(NC * (NC + 1) / 2 + NC) * PIX;
}

// One pixel's recursion on one warp (C0 = 0: HGF mode, all n+1 coefficients penalised; C0 = 1: GF mode,
// centred Gram, alpha from index 1 on -- compile-time, so the unrolled steps carry no runtime mode tests).
template <int NC, int C0>
__device__ __forceinline__ void recur3_pixel(const double* __restrict__ g, double* __restrict__ gs,
                                             double* __restrict__ u_s, float* __restrict__ outs, int k, int lane,
                                             double N, double lam) {
  constexpr int K = NC + 1, NP = NC * (NC + 1) / 2;
  constexpr int GP = PIX + 1, KP = gs_pitch(K);
  const double inv_lam = 1.0 / lam;
  // dense symmetric Gram of this pixel, centred over channels 1..n in GF mode (§5.1), built once
  for (int e = lane; e < K * K; e += 32) {
    const int ea = e / K, eb = e % K;
    const int lo = ea < eb ? ea : eb, hi = ea < eb ? eb : ea;
    double v = (lo == 0 && hi == 0) ? N : g[pair_index(lo, hi, K) * GP + k];
    if (C0 != 0 && lo > 0) v -= g[pair_index(0, lo, K) * GP + k] * g[pair_index(0, hi, K) * GP + k] / N;
    gs[ea * KP + eb] = v;
  }
  __syncwarp();
  // lane i holds row i of alpha (a[j] = alpha_ij), rows / columns c0 .. kappa filled so far
  double a[K];
#pragma unroll
  for (int j = 0; j < K; ++j) a[j] = 0.0;
  // F1 (compile-time indices keep a[] in registers)
  if (C0 == 0) {
    if (lane == 0) a[0] = -inv_lam / (lam + gs[0]);
  } else if (lane == 1) {
    a[1] = -inv_lam / (lam + gs[KP + 1]);
  }
#pragma unroll
  for (int kap = 1; kap < K; ++kap) {
    if (kap <= C0) continue;
    // column kappa of the Gram (= row kappa), entries 0..kappa: broadcast 128-bit loads
    double gk[K];
    const double2* row2 = reinterpret_cast<const double2*>(gs + kap * KP);
#pragma unroll
    for (int m = 0; m <= kap; m += 2) {
      const double2 t = row2[m / 2];
      gk[m] = t.x;
      if (m + 1 < K) gk[m + 1] = t.y;
    }
    // u_i = sum_{m < kap} alpha_im G_m,kap  (meaningful in lanes c0 .. kap-1; zero rows elsewhere)
    double u0 = 0.0, u1 = 0.0;
#pragma unroll
    for (int m = 0; m < kap; ++m)
      if (m >= C0) {
        if (m & 1) u1 = fma(a[m], gk[m], u1);
        else u0 = fma(a[m], gk[m], u0);
      }
    const double u = u0 + u1;
    u_s[lane] = u;
    __syncwarp();
    double uj[K];
    const double2* u2 = reinterpret_cast<const double2*>(u_s);
#pragma unroll
    for (int j = 0; j < kap; j += 2) {
      const double2 t = u2[j / 2];
      uj[j] = t.x;
      if (j + 1 < K) uj[j + 1] = t.y;
    }
    // quad = sum_i G_kap,i u_i, formed by every lane from the broadcast values (no reduction)
    double q0 = 0.0, q1 = 0.0;
#pragma unroll
    for (int j = 0; j < kap; ++j)
      if (j >= C0) {
        if (j & 1) q1 = fma(gk[j], uj[j], q1);
        else q0 = fma(gk[j], uj[j], q0);
      }
    const double gam = -1.0 / (1.0 + inv_lam * gk[kap] + (q0 + q1));             // gamma^kappa
    if (lane >= C0 && lane < kap) {
      const double gu = gam * u;
#pragma unroll
      for (int j = 0; j < kap; ++j)
        if (j >= C0) a[j] = fma(gu, uj[j], a[j]);                                  // gamma F + alpha (F2)
      a[kap] = inv_lam * gu;
    } else if (lane == kap) {
#pragma unroll
      for (int j = 0; j < kap; ++j)
        if (j >= C0) a[j] = inv_lam * gam * uj[j];
      a[kap] = inv_lam * inv_lam * gam;
    }
    __syncwarp();                                 // u_s is rewritten by the next step
  }
  // outputs: P' = -lambda alpha_{1..n,1..n} (upper triangle, row-major), then nu_k = G_0k / den
  if (lane >= 1 && lane < K) {
    const int ai = lane;
    int s = (ai - 1) * NC - (ai - 1) * (ai - 2) / 2;     // first upper-triangle slot of row ai
#pragma unroll
    for (int b = 1; b < K; ++b)
      if (b >= ai) outs[(s + (b - ai)) * PIX + k] = (float)(-lam * a[b]);
    const double den = (C0 == 0) ? (lam + N) : N;
    outs[(NP + ai - 1) * PIX + k] = (float)(g[pair_index(0, ai, K) * GP + k] / den);
  }
}

template <int NC>
__global__ void __launch_bounds__(RW * 32) k_recur3(const double* __restrict__ gram, float* __restrict__ stats, int W,
                                                    int H, int r, double lam, int mode) {
  constexpr int K = NC + 1, NPAIR = npairs(NC), NP = NC * (NC + 1) / 2, NS = NP + NC;
  constexpr int GP = PIX + 1;                       // staging pitch: lanes walking pairs spread over the banks
  constexpr int KP = gs_pitch(K);
  static_assert(K <= 32, "one lane per row of alpha");
  extern __shared__ __align__(16) double sm3[];
  double* gs_all = sm3;                             // [RW][K][KP]: each warp's pixel, dense (centred) Gram
  double* g = gs_all + RW * K * KP;                 // [NPAIR][GP]: Gram entries of the CTA's pixels
  double* ubuf = g + (NPAIR * GP + 1) / 2 * 2;      // [RW][32]: u of each warp's current step (16-B aligned)
  float* outs = reinterpret_cast<float*>(ubuf + RW * 32);   // [NS][PIX]: staged outputs
  const long long HW = (long long)H * W;
  const long long pix0 = (long long)blockIdx.x * PIX;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // staging by asynchronous 8-byte copies (cp.async): every load of the CTA is in flight at once instead of
  // one dependent global load per loop trip (the staging was latency-bound)
  for (int e = tid; e < NPAIR * PIX; e += RW * 32) {
    const int p = e / PIX, k = e % PIX;
    const long long pix = pix0 + k;
    double* dst = g + p * GP + k;
    if (pix < HW) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gram + (long long)p * HW + pix)
                   : "memory");
    } else {
      *dst = 0.0;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  double* u_s = ubuf + warp * 32;
  double* gs = gs_all + warp * K * KP;
  for (int k = warp; k < PIX; k += RW) {
    const long long pix = pix0 + k;
    if (pix >= HW) break;
    const int y = (int)(pix / W), x = (int)(pix % W);
    const double N = (double)window_count(y, x, H, W, r);
    if (mode == 0) recur3_pixel<NC, 0>(g, gs, u_s, outs, k, lane, N, lam);
    else recur3_pixel<NC, 1>(g, gs, u_s, outs, k, lane, N, lam);
    __syncwarp();                                   // gs is rebuilt for the warp's next pixel
  }
  __syncthreads();
  for (int e = tid; e < NS * PIX; e += RW * 32) {
    const int s = e / PIX, k = e % PIX;
    const long long pix = pix0 + k;
    if (pix < HW) stats[(long long)s * HW + pix] = outs[e];
  }
}

// scratch: (npairs(NC) + PB) * H * W doubles (the Gram planes, then one batch of horizontal sums)
template <int NC>
cudaError_t stats3_impl(const float* G, float* stats, double* scratch, int W, int H, int r, double lam, int mode,
                        cudaStream_t st) {
  constexpr int NPAIR = npairs(NC);
  const long long HW = (long long)H * W;
  double* gram = scratch;
  double* hs = scratch + (long long)NPAIR * HW;
  cudaError_t e = cudaFuncSetAttribute(k_gram_h3<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)gram_h3_smem(NC, r));
  if (e != cudaSuccess) return e;
  for (int p0 = 0; p0 < NPAIR; p0 += PB) {
    const int pb = NPAIR - p0 < PB ? NPAIR - p0 : PB;
    dim3 gh((W + HX - 1) / HX, H);
    k_gram_h3<NC><<<gh, HX, gram_h3_smem(NC, r), st>>>(G, hs, W, H, r, p0, pb);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    dim3 gv((W + HX - 1) / HX, (H + VROWS - 1) / VROWS, pb);
    k_gram_v3<NC><<<gv, HX, 0, st>>>(hs, gram, W, H, r, p0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  const size_t smem = recur3_smem(NC);
  if ((e = cudaFuncSetAttribute(k_recur3<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return e;
  k_recur3<NC><<<(unsigned)((HW + PIX - 1) / PIX), RW * 32, smem, st>>>(gram, stats, W, H, r, lam, mode);
  return cudaGetLastError();
}

}  // namespace st3
}  // namespace hgf
