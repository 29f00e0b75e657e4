// HGF per-slice kernels, version 2 (fast path: n_guide <= 3, degree <= 3, radius <= 9).
//
// k_coef2<M,D>: per slice l, for the CTA's 32x16 owned pixels
//     S_0 = B(p), S_k = B(G_k p)        (Eq12 with G_{n+1} = p; G_{(i-1)d+j} p = p I_i^j)
//     w   = P'(S - nu S_0),  w_0 = S_0/(lambda_0+N) - nu^T w      (Eq13 reassociated)
//   Structure: raw guide tile I (label-invariant) + double-buffered p tile in SMEM (cp.async with
//   zero-fill = clipped windows), horizontal sliding sums over 8-column segments -> H1, vertical
//   sliding sums -> S, owners (stats in registers for all labels) do the matvec and store w.
// k_agg2<N>: per slice l, for the CTA's 64x32 output pixels
//     Z = (B(w_0) + sum_k G_k B(w_k)) / N   (Eq14), running WTA (ties -> lowest label)
//   Structure: vertical sliding sums straight from global (each column of the w tile loaded once
//   into registers), horizontal sliding sums by owner threads that keep G, 1/N and the running
//   (min, argmin) of 8 pixels in registers.
#pragma once
#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace v2 {

constexpr int RMAX = 9;  // fast-path radius limit (register arrays are sized by it)

__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gsrc, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int sz = valid ? 4 : 0;  // src-size 0 -> zero fill (clipped window)
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gsrc), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

__host__ __device__ constexpr int odd_pitch(int x) { return x | 1; }

// ------------------------------------------------------------------------------------------ coef
constexpr int A_TX = 32, A_TY = 16, A_KX = 8, A_NSEG = A_TX / A_KX;

template <int M, int D>
struct CoefCfg {
  static constexpr int NC = M * D, K = NC + 1, NP = NC * (NC + 1) / 2, NS = NP + NC;
  static constexpr int PPT = (NC <= 6) ? 2 : 1;          // owned pixels per thread
  static constexpr int THREADS = 512 / PPT;               // 256 or 512
};

__host__ __device__ inline size_t coef2_smem_floats(int M, int D, int r) {
  const int K = M * D + 1;
  const int IX = odd_pitch(A_TX + 2 * r), IY = A_TY + 2 * r;
  return (size_t)M * IY * IX + 2 * (size_t)IY * IX + (size_t)K * IY * (A_TX + 1) + (size_t)K * A_TY * A_TX;
}

// R > 0: compile-time radius (tile geometry and every window offset fold into immediates); R = 0: runtime r.
template <int M, int D, int R>
__global__ void __launch_bounds__(CoefCfg<M, D>::THREADS)
    k_coef2(const float* __restrict__ guide, const float* __restrict__ stats, const float* __restrict__ vol,
            float* __restrict__ wbuf, WLayout wo, int W, int H, int r_arg, int L, float lam0) {
  const int r = (R > 0) ? R : r_arg;
  using C = CoefCfg<M, D>;
  constexpr int NC = C::NC, K = C::K, NP = C::NP, NS = C::NS, PPT = C::PPT, T = C::THREADS;
  extern __shared__ __align__(16) float sm[];
  const int IX = odd_pitch(A_TX + 2 * r), IY = A_TY + 2 * r, HP = A_TX + 1;
  float* It = sm;                       // [M][IY][IX]
  float* Pt = It + M * IY * IX;         // [2][IY][IX]
  float* H1 = Pt + 2 * IY * IX;         // [K][IY][HP]
  float* Sb = H1 + K * IY * HP;         // [K][A_TY][A_TX]
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * A_TX, y0 = blockIdx.y * A_TY;
  const long long HW = (long long)H * W;

  // label-invariant: raw guide tile (zero outside the image)
  for (int e = tid; e < M * IY * (A_TX + 2 * r); e += T) {
    const int i = e / (IY * (A_TX + 2 * r)), rem = e % (IY * (A_TX + 2 * r));
    const int row = rem / (A_TX + 2 * r), col = rem % (A_TX + 2 * r);
    const int yy = y0 - r + row, xx = x0 - r + col;
    const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
    It[(i * IY + row) * IX + col] = in ? __ldg(guide + i * HW + (long long)yy * W + xx) : 0.0f;
  }
  // owners: stats in registers for all labels
  const int ox = tid % A_TX, oy0 = tid / A_TX;
  float st[PPT][NS];
  float kap[PPT];
  bool own[PPT];
  long long opix[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int gy = y0 + oy0 + j * (T / A_TX), gx = x0 + ox;
    own[j] = gy < H && gx < W;
    opix[j] = own[j] ? (long long)gy * W + gx : 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) st[j][s] = own[j] ? __ldg(stats + s * HW + opix[j]) : 0.0f;
    kap[j] = own[j] ? 1.0f / (lam0 + (float)window_count(gy, gx, H, W, r)) : 0.0f;
  }
  auto load_p = [&](int l, int buf) {
    const float* pl = vol + (long long)l * HW;
    float* dst = Pt + buf * IY * IX;
    const int wid = A_TX + 2 * r;
    for (int e = tid; e < IY * wid; e += T) {
      const int row = e / wid, col = e % wid;
      const int yy = y0 - r + row, xx = x0 - r + col;
      const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
      cp_async4(dst + row * IX + col, in ? pl + (long long)yy * W + xx : pl, in);
    }
    cp_async_commit();
  };
  if (L > 0) load_p(0, 0);

#pragma unroll 1
  for (int l = 0; l < L; ++l) {
    cp_async_wait_all();
    __syncthreads();                                  // p tile of label l visible; H1/S free
    if (l + 1 < L) load_p(l + 1, (l + 1) & 1);        // prefetch overlaps this label's passes
    const float* P = Pt + (l & 1) * IY * IX;
    // ---- horizontal sliding sums of p and p*I_i^j over 8-column segments
    for (int item = tid; item < IY * A_NSEG; item += T) {
      const int row = item / A_NSEG, c0 = (item % A_NSEG) * A_KX;
      const float* Prow = P + row * IX;
      float acc[K];
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = 0.0f;
      auto prod = [&](int col, float (&v)[K]) {
        const float p = Prow[col];
        v[0] = p;
#pragma unroll
        for (int i = 0; i < M; ++i) {
          const float g = It[(i * IY + row) * IX + col];
          float t = p;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            t *= g;
            v[1 + i * D + j] = t;
          }
        }
      };
      for (int dx = 0; dx <= 2 * r; ++dx) {
        float v[K];
        prod(c0 + dx, v);
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] += v[k];
      }
#pragma unroll
      for (int k = 0; k < K; ++k) H1[(k * IY + row) * HP + c0] = acc[k];
#pragma unroll
      for (int s = 1; s < A_KX; ++s) {
        float vin[K], vout[K];
        prod(c0 + s + 2 * r, vin);
        prod(c0 + s - 1, vout);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          acc[k] += vin[k] - vout[k];
          H1[(k * IY + row) * HP + c0 + s] = acc[k];
        }
      }
    }
    __syncthreads();
    // ---- vertical sliding sums -> S[k][y][x]
    for (int item = tid; item < K * A_TX; item += T) {
      const int k = item / A_TX, c = item % A_TX;
      const float* col = H1 + k * IY * HP + c;
      float acc = 0.0f;
      for (int dy = 0; dy <= 2 * r; ++dy) acc += col[dy * HP];
      float* so = Sb + k * A_TY * A_TX + c;
      so[0] = acc;
#pragma unroll
      for (int y = 1; y < A_TY; ++y) {
        acc += col[(y + 2 * r) * HP] - col[(y - 1) * HP];
        so[y * A_TX] = acc;
      }
    }
    __syncthreads();
    // ---- owners: w = P'(S - nu S_0), w_0 = kappa S_0 - nu^T w
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (!own[j]) continue;
      const int oy = oy0 + j * (T / A_TX);
      float S[K];
#pragma unroll
      for (int k = 0; k < K; ++k) S[k] = Sb[(k * A_TY + oy) * A_TX + ox];
      float c[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) c[i] = fmaf(-st[j][NP + i], S[0], S[i + 1]);
      float w0 = kap[j] * S[0];
      float* wl = wbuf + wo.origin + (long long)l * K * wo.plane + (long long)(y0 + oy) * wo.pitch + (x0 + ox);
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const int a = i < q ? i : q, b = i < q ? q : i;
          acc = fmaf(st[j][a * NC - a * (a - 1) / 2 + (b - a)], c[q], acc);
        }
        w0 = fmaf(-st[j][NP + i], acc, w0);
        wl[(i + 1) * wo.plane] = acc;
      }
      wl[0] = w0;
    }
  }
}

// ------------------------------------------------------------------------------------------ agg
constexpr int B_TX = 64, B_TY = 32, B_KX = 8, B_NSEG = B_TX / B_KX, B_THREADS = 256;

__host__ __device__ inline size_t agg2_smem_floats(int NC, int r) {
  return (size_t)(NC + 1) * B_TY * odd_pitch(B_TX + 2 * r);
}

// Vertical sliding sums of the K planes of one slice's w over rows [y0-R, y0+B_TY+R): each column is
// loaded once from global into registers (coalesced across threads), V2[k][y][c] = sum_{dy} w_k(y0+y-R+dy).
template <int R>
__device__ __forceinline__ void agg_vpass(const float* __restrict__ wl, float* __restrict__ V2, int VP, int W, int H,
                                          int x0, int y0, int K, long long HW) {
  constexpr int IY = B_TY + 2 * R;
  const int WX = B_TX + 2 * R;
  for (int item = threadIdx.x; item < K * WX; item += B_THREADS) {
    const int k = item / WX, c = item % WX;
    const int xx = x0 - R + c;
    const bool xin = xx >= 0 && xx < W;
    const float* src = wl + k * HW + xx;
    float col[IY];
#pragma unroll
    for (int y = 0; y < IY; ++y) {
      const int yy = y0 - R + y;
      col[y] = (xin && yy >= 0 && yy < H) ? __ldg(src + (long long)yy * W) : 0.0f;
    }
    float acc = 0.0f;
#pragma unroll
    for (int dy = 0; dy <= 2 * R; ++dy) acc += col[dy];
    float* vo = V2 + k * B_TY * VP + c;
    vo[0] = acc;
#pragma unroll
    for (int y = 1; y < B_TY; ++y) {
      acc += col[y + 2 * R] - col[y - 1];
      vo[y * VP] = acc;
    }
  }
}

template <int NC>
__global__ void __launch_bounds__(B_THREADS, 1)
    k_agg2(const float* __restrict__ G, const float* __restrict__ wbuf, int W, int H, int r, int L, int label_base,
           float* __restrict__ filtered_out, int do_wta, int first, int last, float* __restrict__ best_cost,
           int32_t* __restrict__ best_label, int32_t* __restrict__ labels_out, float* __restrict__ min_cost_out,
           int64_t* __restrict__ keys_out) {
  constexpr int K = NC + 1;
  extern __shared__ __align__(16) float sm[];
  const int VP = odd_pitch(B_TX + 2 * r);   // V2 row pitch
  float* V2 = sm;                            // [K][B_TY][VP]
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * B_TX, y0 = blockIdx.y * B_TY;
  const long long HW = (long long)H * W;
  // owner: row oy, 8-pixel segment
  const int oy = tid / B_NSEG, seg = tid % B_NSEG;
  const int gy = y0 + oy;
  float g[NC][B_KX];
  float invN[B_KX], best[B_KX], z[B_KX];
  int32_t bl[B_KX];
#pragma unroll
  for (int j = 0; j < B_KX; ++j) {
    const int gx = x0 + seg * B_KX + j;
    const bool in = gy < H && gx < W;
    const long long p = in ? (long long)gy * W + gx : 0;
#pragma unroll
    for (int k = 0; k < NC; ++k) g[k][j] = in ? __ldg(G + k * HW + p) : 0.0f;
    invN[j] = in ? 1.0f / (float)window_count(gy, gx, H, W, r) : 0.0f;
    best[j] = INFINITY;
    bl[j] = 0;
    if (do_wta && !first && in) {
      best[j] = best_cost[p];
      bl[j] = best_label[p];
    }
  }

#pragma unroll 1
  for (int l = 0; l < L; ++l) {
    const float* wl = wbuf + (long long)l * K * HW;
    // ---- vertical sliding sums of every w plane over the tile's rows (+ r halo), from global
    switch (r) {
      case 1: agg_vpass<1>(wl, V2, VP, W, H, x0, y0, K, HW); break;
      case 2: agg_vpass<2>(wl, V2, VP, W, H, x0, y0, K, HW); break;
      case 3: agg_vpass<3>(wl, V2, VP, W, H, x0, y0, K, HW); break;
      case 4: agg_vpass<4>(wl, V2, VP, W, H, x0, y0, K, HW); break;
      case 5: agg_vpass<5>(wl, V2, VP, W, H, x0, y0, K, HW); break;
      case 6: agg_vpass<6>(wl, V2, VP, W, H, x0, y0, K, HW); break;
      case 7: agg_vpass<7>(wl, V2, VP, W, H, x0, y0, K, HW); break;
      case 8: agg_vpass<8>(wl, V2, VP, W, H, x0, y0, K, HW); break;
      default: agg_vpass<9>(wl, V2, VP, W, H, x0, y0, K, HW); break;
    }
    __syncthreads();
    // ---- horizontal sliding sums by the owners, Z and WTA
#pragma unroll
    for (int j = 0; j < B_KX; ++j) z[j] = 0.0f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float* row = V2 + (k * B_TY + oy) * VP + seg * B_KX;
      float acc = 0.0f;
      for (int dx = 0; dx <= 2 * r; ++dx) acc += row[dx];
      float bw[B_KX];
      bw[0] = acc;
#pragma unroll
      for (int s = 1; s < B_KX; ++s) {
        acc += row[s + 2 * r] - row[s - 1];
        bw[s] = acc;
      }
#pragma unroll
      for (int j = 0; j < B_KX; ++j) z[j] = (k == 0) ? bw[j] : fmaf(g[k - 1][j], bw[j], z[j]);
    }
#pragma unroll
    for (int j = 0; j < B_KX; ++j) {
      const int gx = x0 + seg * B_KX + j;
      if (gy >= H || gx >= W) continue;
      const float zz = z[j] * invN[j];
      if (filtered_out) filtered_out[(long long)l * HW + (long long)gy * W + gx] = zz;
      if (zz < best[j]) {
        best[j] = zz;
        bl[j] = label_base + l;
      }
    }
    __syncthreads();
  }
  if (!do_wta) return;
#pragma unroll
  for (int j = 0; j < B_KX; ++j) {
    const int gx = x0 + seg * B_KX + j;
    if (gy >= H || gx >= W) continue;
    const long long p = (long long)gy * W + gx;
    if (last) {
      if (labels_out) labels_out[p] = bl[j];
      if (min_cost_out) min_cost_out[p] = best[j];
      if (keys_out) keys_out[p] = pack_key_signed(best[j], bl[j]);
    } else {
      best_cost[p] = best[j];
      best_label[p] = bl[j];
    }
  }
}

template <int M, int D, int R>
cudaError_t coef2_r(const float* guide, const float* stats, const float* vol, float* wbuf, WLayout wo, int W, int H, int r,
                       int L, float lam0, cudaStream_t st) {
  using C = CoefCfg<M, D>;
  const size_t smem = sizeof(float) * coef2_smem_floats(M, D, r);
  cudaError_t e = cudaFuncSetAttribute(k_coef2<M, D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((W + A_TX - 1) / A_TX, (H + A_TY - 1) / A_TY);
  k_coef2<M, D, R><<<grid, C::THREADS, smem, st>>>(guide, stats, vol, wbuf, wo, W, H, r, L, lam0);
  return cudaGetLastError();
}

template <int M, int D>
cudaError_t coef2_impl(const float* guide, const float* stats, const float* vol, float* wbuf, WLayout wo, int W, int H,
                       int r, int L, float lam0, cudaStream_t st) {
  switch (r) {   // the BASELINE radii get compile-time kernels; others use the runtime-r instance
    case 2: return coef2_r<M, D, 2>(guide, stats, vol, wbuf, wo, W, H, r, L, lam0, st);
    case 4: return coef2_r<M, D, 4>(guide, stats, vol, wbuf, wo, W, H, r, L, lam0, st);
    case 7: return coef2_r<M, D, 7>(guide, stats, vol, wbuf, wo, W, H, r, L, lam0, st);
    case 9: return coef2_r<M, D, 9>(guide, stats, vol, wbuf, wo, W, H, r, L, lam0, st);
    default: return coef2_r<M, D, 0>(guide, stats, vol, wbuf, wo, W, H, r, L, lam0, st);
  }
}

template <int NC>
cudaError_t agg2_impl(const AggArgs& a, cudaStream_t st) {
  const size_t smem = sizeof(float) * agg2_smem_floats(NC, a.r);
  cudaError_t e = cudaFuncSetAttribute(k_agg2<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.W + B_TX - 1) / B_TX, (a.H + B_TY - 1) / B_TY);
  k_agg2<NC><<<grid, B_THREADS, smem, st>>>(a.G, a.wbuf, a.W, a.H, a.r, a.L, a.label_base, a.filtered_out, a.do_wta,
                                            a.first, a.last, a.best_cost, a.best_label, a.labels_out,
                                            a.min_cost_out, a.keys_out);
  return cudaGetLastError();
}

}  // namespace v2
}  // namespace hgf
