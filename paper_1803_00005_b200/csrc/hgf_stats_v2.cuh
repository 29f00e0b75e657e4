// Label-independent statistics, version 2 (k_stats2<n>): float64 Gram planes by sliding-window sums.
//
//   G_ij = B(G_i G_j), 0 <= i <= j <= n, G_0 = ones inside the image (Prop 2; Eq12),
//   then per pixel the Prop-1 recursion (Eq4 P:143-151 with readings F1/F2, as in k_stats) giving
//   P' = -lambda alpha_{1..n,1..n} and nu = B(G_k)/(lambda_0 + N), stored as float32 planes.
//
// All n+1 channel tiles (16x16 outputs + r halo, float32) are staged in SMEM once; the product planes
// are box-filtered 8 pairs at a time: horizontal sliding sums (one thread per (pair, row), float64)
// then vertical sliding sums (one thread per (pair, column)), so each product costs O(1) adds per
// output instead of the 2r+1 taps of k_stats.  fp32 x fp32 products are exact in float64.
//
// aos = 1 (for k_coef3): per-pixel records of kStatsAos floats instead of planes: the NS statistics, then
// kappa = 1 / (lambda_0 + N) in float32 (the factor of w_0 in the reassociated Eq13, F10).
#pragma once
#include "hgf_common.cuh"
#include "hgf_launch.h"
#include "hgf_stats_finish.cuh"

namespace hgf {
namespace st2 {

constexpr int T = 16;        // output tile side
constexpr int PB = 7;        // product planes per batch (7 x 34 rows <= 256 threads at r = 9: one H round)
constexpr int THREADS = T * T;

constexpr int HP = T + 1;     // row pitch (doubles) of the horizontal sums: lanes walk rows conflict-free
// Channel tiles: TS rows of pitch TSP = TS rounded up to odd (lanes walk rows in the horizontal pass).
__host__ __device__ inline int tile_pitch(int r) { return (T + 2 * r) | 1; }
__host__ __device__ inline size_t smem_bytes(int NC, int r) {
  const int TS = T + 2 * r;
  return ((size_t)(NC + 1) * TS * tile_pitch(r) * 4 + 15) / 16 * 16 + (size_t)PB * TS * HP * 8 +
         (size_t)PB * T * T * 8 + 16;
}

// Rows [yb0, yb1) only (tiles from row yb0 & ~15; rows outside the band are not written).
template <int NC>
__global__ void __launch_bounds__(THREADS) k_stats2(const float* __restrict__ G, float* __restrict__ stats, int W,
                                                    int H, int r, double lam, int mode, int aos, float lam0f,
                                                    int yb0, int yb1) {
  constexpr int K = NC + 1;
  constexpr int NPAIR = K * (K + 1) / 2 - 1;     // (0,0) is N_p, analytic
  constexpr int NB = (NPAIR + PB - 1) / PB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int TS = T + 2 * r, TSP = tile_pitch(r);
  float* tiles = reinterpret_cast<float*>(smem_raw);                              // [K][TS][TSP]
  double* hb = reinterpret_cast<double*>(smem_raw + (((size_t)K * TS * TSP * 4 + 15) & ~(size_t)15));  // [PB][TS][HP]
  double* vb = hb + PB * TS * HP;                                                 // [PB][T][T]
  const int tid = threadIdx.x;
  const int tx = tid % T, ty = tid / T;
  const int x0 = blockIdx.x * T, y0 = (yb0 / T + (int)blockIdx.y) * T;
  const long long HW = (long long)H * W;

  for (int e = tid; e < K * TS * TS; e += THREADS) {
    const int c = e / (TS * TS), rem = e % (TS * TS);
    const int yy = y0 - r + rem / TS, xx = x0 - r + rem % TS;
    const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
    tiles[(c * TS + rem / TS) * TSP + rem % TS] =
        in ? (c == 0 ? 1.0f : __ldg(G + (c - 1) * HW + (long long)yy * W + xx)) : 0.0f;
  }

  double g[NPAIR];
#pragma unroll
  for (int bt = 0; bt < NB; ++bt) {
    __syncthreads();   // tiles ready (first batch) / vb consumed (later batches)
    // horizontal sliding sums of the products of this batch's pairs
    for (int item = tid; item < PB * TS; item += THREADS) {
      const int pb = item / TS, row = item % TS;
      const int p = bt * PB + pb;
      if (p >= NPAIR) continue;
      // pair index p -> (i, j), i <= j, enumerated row-major over the upper triangle, skipping (0,0)
      int i = 0, q = p + 1;
      while (q >= K - i) { q -= K - i; ++i; }
      const int j = i + q;
      const float* ti = tiles + (i * TS + row) * TSP;
      const float* tj = tiles + (j * TS + row) * TSP;
      double acc = 0.0;
      for (int dx = 0; dx <= 2 * r; ++dx) acc += (double)ti[dx] * (double)tj[dx];
      double* ho = hb + (pb * TS + row) * HP;
      ho[0] = acc;
#pragma unroll
      for (int c = 1; c < T; ++c) {
        acc += (double)ti[c + 2 * r] * (double)tj[c + 2 * r] - (double)ti[c - 1] * (double)tj[c - 1];
        ho[c] = acc;
      }
    }
    __syncthreads();
    // vertical sums: two threads per (pair, column), 8 output rows each (twice the parallelism of one
    // 16-row slide for 19 extra loads)
    for (int item = tid; item < PB * T * 2; item += THREADS) {
      const int pb = item / (2 * T), col = (item / 2) % T, half = item & 1;
      if (bt * PB + pb >= NPAIR) continue;
      const double* hc = hb + pb * TS * HP + col + half * (T / 2) * HP;
      double acc = 0.0;
      for (int dy = 0; dy <= 2 * r; ++dy) acc += hc[dy * HP];
      double* vo = vb + pb * T * T + col + half * (T / 2) * T;
      vo[0] = acc;
#pragma unroll
      for (int y = 1; y < T / 2; ++y) {
        acc += hc[(y + 2 * r) * HP] - hc[(y - 1) * HP];
        vo[y * T] = acc;
      }
    }
    __syncthreads();
#pragma unroll
    for (int pb = 0; pb < PB; ++pb)
      if (bt * PB + pb < NPAIR) g[bt * PB + pb] = vb[(pb * T + ty) * T + tx];
  }
  const int gx = x0 + tx, gy = y0 + ty;
  if (gx >= W || gy >= H || gy < yb0 || gy >= yb1) return;
  const double N = (double)window_count(gy, gx, H, W, r);
  stats_finish<NC>(g, N, lam, mode, aos, lam0f, stats, (long long)gy * W + gx, HW);
}

template <int NC>
cudaError_t stats2_impl(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos, float lam0f,
                        int y0, int y1, cudaStream_t st) {
  if (aos && NC > kCoef3MaxN) return cudaErrorInvalidValue;
  const size_t smem = smem_bytes(NC, r);
  cudaError_t e = cudaFuncSetAttribute(k_stats2<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (y0 >= y1) return cudaSuccess;
  dim3 grid((W + T - 1) / T, (y1 + T - 1) / T - y0 / T);
  k_stats2<NC><<<grid, THREADS, smem, st>>>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1);
  return cudaGetLastError();
}

}  // namespace st2
}  // namespace hgf
