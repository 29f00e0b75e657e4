// Per-pixel end of the statistics pass, shared by k_stats2 and k_stats4: from the float64 Gram sums of one
// pixel to its stored statistics.
//
//   Gram G_ab = B(G_a G_b) (Prop 2, Eq12; G_0 = ones, so G_00 = N analytic), then the
//   Prop-1 recursion (Eq4 P:143-151 with readings F1/F2) giving alpha; stored: P' = -lambda alpha_{1..n,1..n}
//   (upper triangle) and nu = B(G_k)/(lambda_0 + N); aos = 1 adds kappa = 1/(lambda_0 + N) (F10).
//   mode != 0 (GF, paper §5.1): the centred Gram, alpha from index 1 on.
#pragma once
#include "hgf_common.cuh"

namespace hgf {

// g: the Gram sums of pixel p, pairs (a, b), a <= b, enumerated row-major over the upper triangle with (0, 0)
// skipped (the first (n+1)(n+2)/2 - 1 entries; NG may be larger: k_stats4's fused single-slice variant appends the
// cost sums).  Gm = the (centred, GF) Gram matrix, al = alpha of the Prop-1 recursion.
template <int NC, int MODE, int NG>
__device__ __forceinline__ void gram_alpha(const double (&g)[NG], double N, double lam, double (&Gm)[NC + 1][NC + 1],
                                           double (&al)[NC + 1][NC + 1]) {
  constexpr int mode = MODE;   // compile-time: no runtime mode tests in the unrolled recursion
  constexpr int K = NC + 1;
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = a; b < K; ++b) {
      const int idx = a * K - a * (a - 1) / 2 + (b - a) - 1;   // position in g (pair (a,b), (0,0) removed)
      const double v = (a == 0 && b == 0) ? N : g[idx];
      Gm[a][b] = v;
      Gm[b][a] = v;
    }
  const double inv_lam = 1.0 / lam;
  constexpr int c0 = (mode == 0) ? 0 : 1;
  if (mode != 0) {
    const double invN = 1.0 / N;
#pragma unroll
    for (int a = 1; a < K; ++a)
#pragma unroll
      for (int b = a; b < K; ++b) {
        Gm[a][b] = Gm[a][b] - Gm[0][a] * Gm[0][b] * invN;                          // centred Gram (§5.1)
        Gm[b][a] = Gm[a][b];
      }
  }
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) al[a][b] = 0.0;
  // F1 (compile-time indices keep Gm / al in registers)
  if (c0 == 0) al[0][0] = -inv_lam / (lam + Gm[0][0]);
  else if (K > 1) al[1][1] = -inv_lam / (lam + Gm[1][1]);
#pragma unroll
  for (int k = 1; k < K; ++k) {
    if (k <= c0) continue;
    double u[K];
    double quad = 0.0;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < k; ++m) s += al[i][m] * Gm[m][k];               // u_i
      u[i] = s;
    }
#pragma unroll
    for (int i = 0; i < k; ++i) quad += Gm[k][i] * u[i];
    const double gam = -1.0 / (1.0 + inv_lam * Gm[k][k] + quad);          // gamma^kappa
#pragma unroll
    for (int i = 0; i < k; ++i)
#pragma unroll
      for (int j = 0; j < k; ++j) al[i][j] += gam * u[i] * u[j];          // gamma F + alpha (F2)
#pragma unroll
    for (int i = 0; i < k; ++i) {
      al[i][k] = inv_lam * gam * u[i];
      al[k][i] = al[i][k];
    }
    al[k][k] = inv_lam * inv_lam * gam;
  }
}

// Writes the record (aos) or the planar statistics of pixel p.
template <int NC, int MODE>
__device__ __forceinline__ void stats_finish_m(const double (&g)[(NC + 1) * (NC + 2) / 2 - 1], double N, double lam,
                                               int aos, float lam0f, float* __restrict__ stats, long long p,
                                               long long HW) {
  constexpr int mode = MODE;
  constexpr int K = NC + 1;
  double Gm[K][K], al[K][K];
  gram_alpha<NC, MODE>(g, N, lam, Gm, al);
  const double inv_den = 1.0 / ((mode == 0) ? (lam + N) : N);   // one division, then products
  if (aos) {
    constexpr int REC = stats_aos_floats(NC);
    float rec[REC];
    int s = 0;
#pragma unroll
    for (int a = 1; a < K; ++a)
#pragma unroll
      for (int b = a; b < K; ++b) rec[s++] = (float)(-lam * al[a][b]);
#pragma unroll
    for (int a = 1; a < K; ++a) rec[s++] = (float)(Gm[0][a] * inv_den);
    rec[s++] = 1.0f / (lam0f + (float)N);
#pragma unroll
    for (; s < REC; ++s) rec[s] = 0.0f;
    float4* o = reinterpret_cast<float4*>(stats + p * REC);
#pragma unroll
    for (int q = 0; q < REC / 4; ++q) o[q] = make_float4(rec[4 * q], rec[4 * q + 1], rec[4 * q + 2], rec[4 * q + 3]);
    return;
  }
  int s = 0;
#pragma unroll
  for (int a = 1; a < K; ++a)
#pragma unroll
    for (int b = a; b < K; ++b) stats[(long long)(s++) * HW + p] = (float)(-lam * al[a][b]);
#pragma unroll
  for (int a = 1; a < K; ++a) stats[(long long)(s++) * HW + p] = (float)(Gm[0][a] * inv_den);
}

// Single-slice end (k_stats4's fused variant, hgf_filter): g additionally holds, after the Gram pairs, the cost sums
// S_a = B(G_a p) for a = 0..n (G_0 = ones, so S_0 = B(p)).  The coefficients of the slice are those k_coef* form
// from the stored statistics (w = P'(S - nu S_0), w_0 = kappa S_0 - nu^T w, P' = -lambda alpha,
// nu = B(G)/(lambda_0 + N) (HGF) or B(G)/N (GF), kappa = 1/(lambda_0 + N)), here in float64 straight from the
// float64 sums, written as float32 planes w_0..w_n at wl[k * plane].
template <int NC, int MODE, int NG>
__device__ __forceinline__ void filter_finish_m(const double (&g)[NG], double N, double lam, float lam0f,
                                                float* __restrict__ wl, long long plane) {
  constexpr int K = NC + 1;
  constexpr int NPAIR = K * (K + 1) / 2 - 1;
  static_assert(NG == NPAIR + K, "Gram pairs + cost sums");
  double Gm[K][K], al[K][K];
  gram_alpha<NC, MODE>(g, N, lam, Gm, al);
  const double inv_den = 1.0 / ((MODE == 0) ? (lam + N) : N);
  const double S0 = g[NPAIR];
  double c[K];
#pragma unroll
  for (int a = 1; a < K; ++a) c[a] = g[NPAIR + a] - Gm[0][a] * inv_den * S0;
  double w0 = S0 / ((double)lam0f + N);
#pragma unroll
  for (int a = 1; a < K; ++a) {
    double t = 0.0;
#pragma unroll
    for (int b = 1; b < K; ++b) t += (-lam * al[a][b]) * c[b];
    w0 -= Gm[0][a] * inv_den * t;
    wl[a * plane] = (float)t;
  }
  wl[0] = (float)w0;
}

template <int NC>
__device__ __forceinline__ void stats_finish(const double (&g)[(NC + 1) * (NC + 2) / 2 - 1], double N, double lam,
                                             int mode, int aos, float lam0f, float* __restrict__ stats, long long p,
                                             long long HW) {
  if (mode == 0) stats_finish_m<NC, 0>(g, N, lam, aos, lam0f, stats, p, HW);
  else stats_finish_m<NC, 1>(g, N, lam, aos, lam0f, stats, p, HW);
}

}  // namespace hgf
