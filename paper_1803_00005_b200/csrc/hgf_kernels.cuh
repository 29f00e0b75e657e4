// HGF hot-path kernels for B200 (sm_100a), version 1 (correctness-first tile kernels).
//
//   k_poly_guidance : G_{(i-1)d+j} = I_i^j                              (§4.2)
//   k_stats<n>      : Gram G_ij = B(G_i G_j) in float64 (Prop 2), the Prop-1 recursion
//                     (readings F1/F2), then P' = -lambda alpha_{1..n,1..n} and
//                     nu_k = B(G_k)/(lambda_0 + N) stored as float32 planes (label-independent)
//   k_coef<n>       : per slice: S_0 = B(p), S_k = B(G_k p) (Eq12 with G_{n+1} = p),
//                     w = P'(S - nu S_0), w_0 = S_0/(lambda_0 + N) - nu^T w   (Eq13 P:304 reassociated;
//                     DESIGN.md §4 derives it from Eq2 by the Schur complement of M_00)
//   k_agg<n>        : per slice: Z = (B(w_0) + sum_k G_k B(w_k)) / N   (Eq14), running WTA
//   k_unpack_keys   : merged keys -> labels / min cost
//
// B is a box SUM over the clipped window (F6/F7).  Clipping = zero fill outside the image
// (products with p = 0 or w = 0 vanish); the count N is analytic.
#pragma once
#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {

constexpr int kTX = 32;    // tile width (pixels) of k_coef / k_agg
constexpr int kTY = 16;    // tile height
constexpr int kSegH = 8;   // horizontal sliding-sum segment (restart every 8 outputs: fp32 accuracy)
constexpr int kSegV = 8;   // vertical sliding-sum segment
constexpr int kThreads = kTX * kTY;

// ------------------------------------------------------------------ K3: statistics (float64)
constexpr int kStatT = 16;   // 16x16 output pixels per CTA

template <int NC>
__global__ __launch_bounds__(kStatT * kStatT) void k_stats(const float* __restrict__ G, float* __restrict__ stats,
                                                           int W, int H, int r, double lam, int mode) {
  constexpr int K = NC + 1;                 // channels 0..n (0 = ones inside the image)
  constexpr int NP = K * (K + 1) / 2;       // packed Gram entries (i <= j)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int TS = kStatT + 2 * r;
  float* ti = reinterpret_cast<float*>(smem_raw);          // [TS][TS] channel i tile
  float* tj = ti + TS * TS;                                // [TS][TS] channel j tile
  double* hb = reinterpret_cast<double*>(tj + TS * TS + ((TS * TS) & 1));  // [TS][kStatT]
  const int tid = threadIdx.x;
  const int tx = tid % kStatT, ty = tid / kStatT;
  const int x0 = blockIdx.x * kStatT, y0 = blockIdx.y * kStatT;
  const int gx = x0 + tx, gy = y0 + ty;
  const long long HW = (long long)H * W;

  double g[NP];
  auto load_tile = [&](float* t, int c) {
    for (int e = tid; e < TS * TS; e += blockDim.x) {
      const int yy = y0 - r + e / TS, xx = x0 - r + e % TS;
      const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
      t[e] = in ? (c == 0 ? 1.0f : G[(c - 1) * HW + (long long)yy * W + xx]) : 0.0f;
    }
  };
  int idx = 0;
#pragma unroll 1
  for (int i = 0; i < K; ++i) {
    __syncthreads();
    load_tile(ti, i);
#pragma unroll 1
    for (int j = i; j < K; ++j, ++idx) {
      if (i == 0 && j == 0) { g[0] = 0.0; continue; }     // N_p, analytic below
      __syncthreads();
      if (j != i) load_tile(tj, j);
      __syncthreads();
      const float* tb = (j == i) ? ti : tj;
      // horizontal box sums of the product plane G_i G_j (fp32*fp32 is exact in fp64)
      for (int e = tid; e < TS * kStatT; e += blockDim.x) {
        const int row = e / kStatT, col = e % kStatT;
        double s = 0.0;
        for (int dx = 0; dx <= 2 * r; ++dx) s += (double)ti[row * TS + col + dx] * (double)tb[row * TS + col + dx];
        hb[row * kStatT + col] = s;
      }
      __syncthreads();
      double s = 0.0;
      for (int dy = 0; dy <= 2 * r; ++dy) s += hb[(ty + dy) * kStatT + tx];
      g[idx] = s;
    }
  }
  if (gx >= W || gy >= H) return;
  const double N = (double)window_count(gy, gx, H, W, r);
  // unpack into a dense symmetric matrix (registers for small n, local memory otherwise)
  double Gm[K][K];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = a; b < K; ++b) {
      const int q = a * K - a * (a - 1) / 2 + (b - a);
      const double v = (a == 0 && b == 0) ? N : g[q];
      Gm[a][b] = v;
      Gm[b][a] = v;
    }
  const double inv_lam = 1.0 / lam;
  // Prop 1 recursion over channels c0..K-1 of the matrix A (HGF: A = Gram over 0..n;
  // GF: A = centred Gram over 1..n, the §5.1 form Eq16).  alpha^{c0}_{c0 c0} = -lam^-1 (lam + A_00)^-1 (F1).
  double al[K][K];
  const int c0 = (mode == 0) ? 0 : 1;
  if (mode != 0) {
#pragma unroll
    for (int a = 1; a < K; ++a)
#pragma unroll
      for (int b = 1; b < K; ++b) Gm[a][b] = Gm[a][b] - Gm[0][a] * Gm[0][b] / N;   // G'_ab
  }
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) al[a][b] = 0.0;
  al[c0][c0] = -inv_lam / (lam + Gm[c0][c0]);
#pragma unroll
  for (int k = 1; k < K; ++k) {
    if (k <= c0) continue;
    double u[K];
    double quad = 0.0;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      double s = 0.0;
#pragma unroll
      for (int mm = 0; mm < k; ++mm) s += al[i][mm] * Gm[mm][k];   // u_i = sum_m alpha_im G_mk
      u[i] = s;
    }
#pragma unroll
    for (int i = 0; i < k; ++i) quad += Gm[k][i] * u[i];
    const double gam = -1.0 / (1.0 + inv_lam * Gm[k][k] + quad);    // gamma^kappa
#pragma unroll
    for (int i = 0; i < k; ++i)
#pragma unroll
      for (int j = 0; j < k; ++j) al[i][j] += gam * u[i] * u[j];     // gamma F + alpha (F2)
#pragma unroll
    for (int i = 0; i < k; ++i) { al[i][k] = inv_lam * gam * u[i]; al[k][i] = al[i][k]; }
    al[k][k] = inv_lam * inv_lam * gam;
  }
  // P' = [M^-1]_{1..n,1..n} = -lambda alpha_{1..n,1..n};  nu_k = B(G_k) / (lambda_0 + N)
  const long long p = (long long)gy * W + gx;
  int s = 0;
#pragma unroll
  for (int a = 1; a < K; ++a)
#pragma unroll
    for (int b = a; b < K; ++b) stats[(long long)(s++) * HW + p] = (float)(-lam * al[a][b]);
  const double den = (mode == 0) ? (lam + N) : N;
#pragma unroll
  for (int a = 1; a < K; ++a) stats[(long long)(s++) * HW + p] = (float)(Gm[0][a] / den);
}

// ------------------------------------------------------------------ box passes shared by A and B
// Horizontal sliding sums of a (TY+2r) x (TX+2r) tile `src` (row pitch TXH) into hb[(TY+2r)][TX]:
// hb[row][c] = sum_{dx=0..2r} v(row, c+dx), where v(row, col) = src[row][col] * (gk ? G_k : 1).
template <bool kMulG>
__device__ __forceinline__ void hpass(const float* __restrict__ src, float* __restrict__ hb, int TXH, int TYH, int r,
                                      const float* __restrict__ Gk, int W, int H, int x0, int y0) {
  constexpr int nseg = kTX / kSegH;
  for (int item = threadIdx.x; item < TYH * nseg; item += blockDim.x) {
    const int row = item / nseg, c0 = (item % nseg) * kSegH;
    const int yy = y0 - r + row;
    auto v = [&](int col) -> float {
      float a = src[row * TXH + col];
      if (kMulG) {
        const int xx = x0 - r + col;
        const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
        a = in ? a * __ldg(Gk + (long long)yy * W + xx) : 0.0f;
      }
      return a;
    };
    float acc = 0.0f;
    for (int dx = 0; dx <= 2 * r; ++dx) acc += v(c0 + dx);
    hb[row * kTX + c0] = acc;
#pragma unroll
    for (int s = 1; s < kSegH; ++s) {
      acc += v(c0 + s + 2 * r) - v(c0 + s - 1);
      hb[row * kTX + c0 + s] = acc;
    }
  }
}

// Vertical sliding sums: vs[row][c] = sum_{dy=0..2r} hb[row+dy][c], row in [0, TY).
__device__ __forceinline__ void vpass(const float* __restrict__ hb, float* __restrict__ vs, int r) {
  constexpr int nseg = kTY / kSegV;
  for (int item = threadIdx.x; item < kTX * nseg; item += blockDim.x) {
    const int col = item % kTX, r0 = (item / kTX) * kSegV;
    float acc = 0.0f;
    for (int dy = 0; dy <= 2 * r; ++dy) acc += hb[(r0 + dy) * kTX + col];
    vs[r0 * kTX + col] = acc;
#pragma unroll
    for (int s = 1; s < kSegV; ++s) {
      acc += hb[(r0 + s + 2 * r) * kTX + col] - hb[(r0 + s - 1) * kTX + col];
      vs[(r0 + s) * kTX + col] = acc;
    }
  }
}

__device__ __forceinline__ void load_tile(const float* __restrict__ src, float* __restrict__ t, int TXH, int TYH,
                                          int W, int H, int x0, int y0, int r) {
  for (int e = threadIdx.x; e < TXH * TYH; e += blockDim.x) {
    const int yy = y0 - r + e / TXH, xx = x0 - r + e % TXH;
    const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
    t[e] = in ? __ldg(src + (long long)yy * W + xx) : 0.0f;
  }
}

// ------------------------------------------------------------------ K4a: per-slice coefficients w
template <int NC, bool FEW = false>
__global__ __launch_bounds__(kThreads) void k_coef(const float* __restrict__ G, const float* __restrict__ stats,
                                                   const float* __restrict__ vol, float* __restrict__ wbuf,
                                                   int W, int H, int r, int L, float lam0) {
  constexpr int K = NC + 1;
  constexpr int NP = NC * (NC + 1) / 2;
  constexpr int NS = NP + NC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int TXH = kTX + 2 * r, TYH = kTY + 2 * r;
  float* pt = reinterpret_cast<float*>(smem_raw);   // [TYH][TXH]
  float* hb = pt + TXH * TYH;                        // [TYH][kTX]
  float* vs = hb + TYH * kTX;                        // [kTY][kTX]
  const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool own = gx < W && gy < H;
  const long long HW = (long long)H * W;
  const long long p = own ? (long long)gy * W + gx : 0;

  // FEW (n >= 10, i.e. NS > 64 statistics per pixel, and <= 4 slices, e.g. hgf_filter): the per-pixel arrays spilled
  // to local memory (ncu: GBs of local traffic per slice at n = 20), so the window sums and c'' live in shared memory
  // (each thread its own column) and the statistics are read where used -- same arithmetic, same order; C5 n = 20:
  // 3.75 -> 1.65 ms.  Many slices keep the preloaded (spilling) statistics, which amortise over the labels (n = 12,
  // 40 labels: 5.1 vs 5.6 ms)
  if constexpr (FEW) {
    float* sb = vs + kTY * kTX;                      // [K][kThreads]: S_k, then c''_i in place
    const float kapL = own ? 1.0f / (lam0 + (float)window_count(gy, gx, H, W, r)) : 0.0f;
    auto stat = [&](int q) -> float { return __ldg(stats + (long long)q * HW + p); };
#pragma unroll 1
    for (int l = 0; l < L; ++l) {
      const float* pl = vol + (long long)l * HW;
      __syncthreads();
      load_tile(pl, pt, TXH, TYH, W, H, x0, y0, r);
      __syncthreads();
#pragma unroll 1
      for (int k = 0; k < K; ++k) {
        if (k == 0) hpass<false>(pt, hb, TXH, TYH, r, nullptr, W, H, x0, y0);
        else hpass<true>(pt, hb, TXH, TYH, r, G + (long long)(k - 1) * HW, W, H, x0, y0);
        __syncthreads();
        vpass(hb, vs, r);
        __syncthreads();
        sb[k * kThreads + threadIdx.x] = vs[ty * kTX + tx];
      }
      if (own) {
        const float S0 = sb[threadIdx.x];
#pragma unroll 1
        for (int i = 0; i < NC; ++i)
          sb[(i + 1) * kThreads + threadIdx.x] = fmaf(-stat(NP + i), S0, sb[(i + 1) * kThreads + threadIdx.x]);
        float w0 = kapL * S0;
        float* wl = wbuf + (long long)l * K * HW + p;
#pragma unroll 1
        for (int i = 0; i < NC; ++i) {
          float acc = 0.0f;
#pragma unroll 4
          for (int j = 0; j < NC; ++j) {
            const int a = i < j ? i : j, b = i < j ? j : i;
            acc = fmaf(stat(a * NC - a * (a - 1) / 2 + (b - a)), sb[(j + 1) * kThreads + threadIdx.x], acc);
          }
          w0 = fmaf(-stat(NP + i), acc, w0);
          wl[(i + 1) * HW] = acc;
        }
        wl[0] = w0;
      }
    }
  } else {
  float st[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) st[s] = own ? stats[s * HW + p] : 0.0f;
  const float kap = own ? 1.0f / (lam0 + (float)window_count(gy, gx, H, W, r)) : 0.0f;

#pragma unroll 1
  for (int l = 0; l < L; ++l) {
    const float* pl = vol + (long long)l * HW;
    __syncthreads();
    load_tile(pl, pt, TXH, TYH, W, H, x0, y0, r);
    __syncthreads();
    float S[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k == 0) hpass<false>(pt, hb, TXH, TYH, r, nullptr, W, H, x0, y0);
      else hpass<true>(pt, hb, TXH, TYH, r, G + (long long)(k - 1) * HW, W, H, x0, y0);
      __syncthreads();
      vpass(hb, vs, r);
      __syncthreads();
      S[k] = vs[ty * kTX + tx];
    }
    if (own) {
      // c''_i = S_i - nu_i S_0 ; w = P' c'' ; w_0 = S_0/(lambda_0+N) - nu^T w
      float c[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) c[i] = fmaf(-st[NP + i], S[0], S[i + 1]);
      float w0 = kap * S[0];
      float* wl = wbuf + (long long)l * K * HW + p;
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const int a = i < j ? i : j, b = i < j ? j : i;
          acc = fmaf(st[a * NC - a * (a - 1) / 2 + (b - a)], c[j], acc);
        }
        w0 = fmaf(-st[NP + i], acc, w0);
        wl[(i + 1) * HW] = acc;
      }
      wl[0] = w0;
    }
  }
  }
}

// ------------------------------------------------------------------ K4b: aggregation + WTA
template <int NC>
__global__ __launch_bounds__(kThreads) void k_agg(const float* __restrict__ G, const float* __restrict__ wbuf,
                                                  int W, int H, int r, int L, int label_base,
                                                  float* __restrict__ filtered_out, int do_wta, int first, int last,
                                                  float* __restrict__ best_cost, int32_t* __restrict__ best_label,
                                                  int32_t* __restrict__ labels_out, float* __restrict__ min_cost_out,
                                                  int64_t* __restrict__ keys_out) {
  constexpr int K = NC + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int TXH = kTX + 2 * r, TYH = kTY + 2 * r;
  float* wt = reinterpret_cast<float*>(smem_raw);   // [TYH][TXH]
  float* hb = wt + TXH * TYH;                        // [TYH][kTX]
  float* vs = hb + TYH * kTX;                        // [kTY][kTX]
  const int tx = threadIdx.x % kTX, ty = threadIdx.x / kTX;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const int gx = x0 + tx, gy = y0 + ty;
  const bool own = gx < W && gy < H;
  const long long HW = (long long)H * W;
  const long long p = own ? (long long)gy * W + gx : 0;
  float g[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) g[k] = own ? G[k * HW + p] : 0.0f;
  const float invN = own ? 1.0f / (float)window_count(gy, gx, H, W, r) : 0.0f;
  float best = INFINITY;
  int32_t bl = 0;
  if (do_wta && !first && own) { best = best_cost[p]; bl = best_label[p]; }

#pragma unroll 1
  for (int l = 0; l < L; ++l) {
    float z = 0.0f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      __syncthreads();
      load_tile(wbuf + ((long long)l * K + k) * HW, wt, TXH, TYH, W, H, x0, y0, r);
      __syncthreads();
      hpass<false>(wt, hb, TXH, TYH, r, nullptr, W, H, x0, y0);
      __syncthreads();
      vpass(hb, vs, r);
      __syncthreads();
      const float bw = vs[ty * kTX + tx];
      z = (k == 0) ? bw : fmaf(g[k - 1], bw, z);
    }
    z = z * invN;
    if (own) {
      if (filtered_out) filtered_out[(long long)l * HW + p] = z;
      if (do_wta && z < best) { best = z; bl = label_base + l; }
    }
  }
  if (!do_wta || !own) return;
  if (last) {
    if (labels_out) labels_out[p] = bl;
    if (min_cost_out) min_cost_out[p] = best;
    if (keys_out) keys_out[p] = pack_key_signed(best, bl);
  } else {
    best_cost[p] = best;
    best_label[p] = bl;
  }
}

template <int NC>
cudaError_t stats_impl(const float* G, float* stats, int W, int H, int r, double lam, int mode, cudaStream_t st) {
  const int TS = kStatT + 2 * r;
  const size_t smem = sizeof(float) * (2 * TS * TS + 1) + sizeof(double) * TS * kStatT + 16;
  cudaError_t e = cudaFuncSetAttribute(k_stats<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((W + kStatT - 1) / kStatT, (H + kStatT - 1) / kStatT);
  k_stats<NC><<<grid, kStatT * kStatT, smem, st>>>(G, stats, W, H, r, lam, mode);
  return cudaGetLastError();
}

template <int NC>
inline size_t slice_smem(int r, bool few = false) {
  const int TXH = kTX + 2 * r, TYH = kTY + 2 * r;
  return sizeof(float) * ((size_t)TXH * TYH + (size_t)TYH * kTX + (size_t)kTY * kTX +
                          (few ? (size_t)(NC + 1) * kThreads : 0));   // k_coef<NC, true>'s window-sum buffer
}

template <int NC>
cudaError_t coef_impl(const float* G, const float* stats, const float* vol, float* wbuf, int W, int H, int r,
                             int L, float lam0, cudaStream_t st) {
  constexpr bool LARGE = NC * (NC + 1) / 2 + NC > 64;
  dim3 grid((W + kTX - 1) / kTX, (H + kTY - 1) / kTY);
  if (LARGE && L <= 4) {
    const size_t smem = slice_smem<NC>(r, true);
    cudaError_t e = cudaFuncSetAttribute(k_coef<NC, LARGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_coef<NC, LARGE><<<grid, kThreads, smem, st>>>(G, stats, vol, wbuf, W, H, r, L, lam0);
    return cudaGetLastError();
  }
  const size_t smem = slice_smem<NC>(r);
  cudaError_t e = cudaFuncSetAttribute(k_coef<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_coef<NC><<<grid, kThreads, smem, st>>>(G, stats, vol, wbuf, W, H, r, L, lam0);
  return cudaGetLastError();
}

template <int NC>
cudaError_t agg_impl(const AggArgs& a, cudaStream_t st) {
  const size_t smem = slice_smem<NC>(a.r);
  cudaError_t e = cudaFuncSetAttribute(k_agg<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.W + kTX - 1) / kTX, (a.H + kTY - 1) / kTY);
  k_agg<NC><<<grid, kThreads, smem, st>>>(a.G, a.wbuf, a.W, a.H, a.r, a.L, a.label_base, a.filtered_out, a.do_wta,
                                         a.first, a.last, a.best_cost, a.best_label, a.labels_out, a.min_cost_out,
                                         a.keys_out);
  return cudaGetLastError();
}

}  // namespace hgf
