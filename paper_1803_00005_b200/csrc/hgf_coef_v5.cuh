// HGF per-slice coefficients, version 5 (k_coef5<n, R>): horizontal-first row marching.
//
// For each slice l and pixel p (Eq12 with G_{n+1} = p; Eq13 P:304 reassociated):
//     S_0 = B(p),  S_k = B(G_k p)  (k = 1..n),   w = P'(S - nu S_0),   w_0 = kappa S_0 - nu^T w
//
// The box sum B is separable; k_coef3 sums vertically first, so the n + 1 vertical sums of every column
// have to cross threads (shared memory) before the horizontal pass.  Here the order is swapped:
//   H_k(j, x) = sum_{|dx| <= R} G_k(j, x + dx) p(j, x + dx)      (horizontal, in registers)
//   S_k(y, x) = S_k(y - 1, x) + H_k(y + R, x) - H_k(y - R - 1, x)  (vertical running sum, in registers)
// so a thread that owns (label, 16-pixel segment) keeps S for its 16 pixels in registers and only READS the
// raw cost rows and guidance rows (one plane plus label-independent broadcasts) from shared memory.  The
// leaving row's horizontal sums are recomputed from the leaving cost row instead of being stored: FP32
// work (~2x the box-sum flops of k_coef3) is traded for the shared-memory traffic that bound k_coef3
// (its L1/SMEM data pipe was ~78 % busy, FMA ~25 %).
//
// A CTA owns a strip of TX = 128 columns x a band of BH rows x 32 labels (lane = label, warp = segment) and
// marches down the band one row per step.  One elected thread keeps a 3-stage TMA ring full: per step the
// entering row (y + R) and the leaving row (y - R - 1) of the 32 labels' cost slices and of the n guidance
// planes (boxes of 164 columns; out-of-image rows/columns/labels read as zero = clipped windows), plus the
// output row's per-pixel statistics records (one bulk copy).  The coefficients are stored into the
// label-interleaved layout (WLayout::il) that k_agg3 reads.
#pragma once
#include <cuda.h>

#include <cstdlib>

#include <cuda/ptx>

#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace v5 {

constexpr int TX = 128;          // owned columns per strip
constexpr int SEG = 16;          // pixels per thread (one group of the interleaved layout)
constexpr int NW = TX / SEG;     // warps (segments)
constexpr int LB = 32;           // labels per CTA (lane = label)
constexpr int XB = 164;          // TMA box width (>= TX + 2*9 + 3); 164 = 4 mod 8: conflict-free LDS.128
constexpr int RMAX = 9;
constexpr int NST = 3;           // TMA ring depth
static_assert(SEG == kWGroupPx, "a segment is one group of the interleaved layout");
static_assert(XB >= TX + 2 * RMAX + 3 && XB % 8 == 4, "box width");

template <int NC>
struct Geom {
  static constexpr int K = NC + 1, NP = NC * (NC + 1) / 2, NS = NP + NC;
  static constexpr int SPX = stats_aos_floats(NC);
  static constexpr int PROW = LB * XB;                         // one cost row of the 32 labels
  static constexpr int GROW = (3 * 2 * XB + 31) / 32 * 32;      // up to M = 3 channels (x2: d = 2 pairs)
  static constexpr int SROW = TX * SPX;
  static constexpr int STAGE = 2 * PROW + 2 * GROW + SROW;     // floats; every part 128-byte aligned
  static constexpr size_t SMEM = sizeof(float) * (size_t)NST * STAGE + 128;
};

__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
  const int32_t c[3] = {x, y, z};
  cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, dst, tm, c, bar);
}

// sum over the horizontal windows of one row into S (SIGN = +1 entering row, -1 leaving row):
// pr = this lane's cost row (window column 0 = image x xs - R), ir = the M raw guide rows (same columns).
// The products G_k p = I_i^j p (k = (i-1)D + j) are formed in registers from the raw guide, so only
// M (not n = M D) guidance values per column are read from shared memory.
template <int M, int D, int R, int SIGN>
__device__ __forceinline__ void hsum_row(const float* __restrict__ pr, const float* __restrict__ ir,
                                         float (&S)[M * D + 1][SEG]) {
  constexpr int K = M * D + 1;
  constexpr int SH = (4 - R % 4) % 4;            // SMEM column of window column 0 within its 16-byte chunk
  auto P = [&](int j) -> float {                  // cost at window column j (128-bit loads, CSE'd)
    const float4 v = reinterpret_cast<const float4*>(pr)[(SH + j) >> 2];
    const int e = (SH + j) & 3;
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
  };
  auto Ii = [&](int i, int j) -> float {          // raw guide channel i at window column j (broadcast loads)
    const float4 v = reinterpret_cast<const float4*>(ir + i * XB)[(SH + j) >> 2];
    const int e = (SH + j) & 3;
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
  };
  // acc += Q(j) (+1) or acc -= Q(j) (-1), Q_0 = p, Q_{iD+d} = I_i^d p
  auto add = [&](float (&acc)[K], int j, float sgn) {
    const float q = P(j);
    acc[0] = fmaf(sgn, q, acc[0]);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const float g = Ii(i, j);
      float t = sgn * q;                           // exact (sgn = +-1)
#pragma unroll
      for (int d = 0; d < D; ++d) {
        if (d + 1 < D) {
          acc[1 + i * D + d] = fmaf(g, t, acc[1 + i * D + d]);
          t = t * g;
        } else {
          acc[1 + i * D + d] = fmaf(g, t, acc[1 + i * D + d]);
        }
      }
    }
  };
  float acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0f;
#pragma unroll
  for (int j = 0; j <= 2 * R; ++j) add(acc, j, 1.0f);
#pragma unroll
  for (int k = 0; k < K; ++k) S[k][0] = SIGN > 0 ? S[k][0] + acc[k] : S[k][0] - acc[k];
#pragma unroll
  for (int i = 1; i < SEG; ++i) {
    add(acc, i + 2 * R, 1.0f);
    add(acc, i - 1, -1.0f);
#pragma unroll
    for (int k = 0; k < K; ++k) S[k][i] = SIGN > 0 ? S[k][i] + acc[k] : S[k][i] - acc[k];
  }
}

// Degree-2 guidance (the paper's RGB d = 2 setting): the guide rows are staged as pairs
// (I_i, I_i^2) per column, so each product pair (I_i p, I_i^2 p) is one packed FFMA2 with the cost as the
// broadcast scalar operand, and the running sums S of the two planes of a channel are updated with one FADD2.
// S0 = plane 0 (B(p)), S2[i] = planes (1 + 2i, 2 + 2i).
template <int M, int R, int SIGN>
__device__ __forceinline__ void hsum_row2(const float* __restrict__ pr, const float* __restrict__ gr,
                                          float (&S0)[SEG], float2 (&S2)[M][SEG]) {
  constexpr int SH = (4 - R % 4) % 4;
  auto P = [&](int j) -> float {
    const float4 v = reinterpret_cast<const float4*>(pr)[(SH + j) >> 2];
    const int e = (SH + j) & 3;
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
  };
  auto G2 = [&](int i, int j) -> float2 {          // (I_i, I_i^2) at window column j (broadcast loads)
    const float4 v = reinterpret_cast<const float4*>(gr + i * 2 * XB)[(SH + j) >> 1];
    return ((SH + j) & 1) ? make_float2(v.z, v.w) : make_float2(v.x, v.y);
  };
  float a0 = 0.0f;
  float2 a2[M];
#pragma unroll
  for (int i = 0; i < M; ++i) a2[i] = make_float2(0.0f, 0.0f);
  auto add = [&](int j, float sgn) {
    const float q = sgn * P(j);                    // exact (sgn = +-1)
    a0 += q;
#pragma unroll
    for (int i = 0; i < M; ++i) a2[i] = __ffma2_rn(make_float2(q, q), G2(i, j), a2[i]);
  };
  auto upd = [&](int i) {
    if (SIGN > 0) {
      S0[i] += a0;
#pragma unroll
      for (int c = 0; c < M; ++c) S2[c][i] = __fadd2_rn(S2[c][i], a2[c]);
    } else {
      S0[i] -= a0;
#pragma unroll
      for (int c = 0; c < M; ++c) S2[c][i] = __fadd2_rn(S2[c][i], make_float2(-a2[c].x, -a2[c].y));
    }
  };
#pragma unroll
  for (int j = 0; j <= 2 * R; ++j) add(j, 1.0f);
  upd(0);
#pragma unroll
  for (int i = 1; i < SEG; ++i) {
    add(i + 2 * R, 1.0f);
    add(i - 1, -1.0f);
    upd(i);
  }
}

// 256-bit global store (sm_100: STG.E.ENL2.256), p 32-byte aligned.
__device__ __forceinline__ void st_global_v8(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

template <int M, int D, int R>
__global__ void __launch_bounds__(NW * 32, 1)
    k_coef5(const __grid_constant__ CUtensorMap tm_vol, const __grid_constant__ CUtensorMap tm_i,
            const float* __restrict__ stats, float* __restrict__ wbuf, WLayout wo, int W, int H, int L, int BH) {
  constexpr int NC = M * D;
  using Gm = Geom<NC>;
  constexpr int K = Gm::K, NP = Gm::NP, NS = Gm::NS, SPX = Gm::SPX;
  constexpr int SH = (4 - R % 4) % 4;
  extern __shared__ __align__(128) float sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NST * Gm::STAGE);   // full barriers (TMA tx count)
  const int tid = threadIdx.x, lane = tid & 31, seg = tid >> 5;
  // grid (label batches, strips, bands): the batches of one (strip, band) are adjacent in launch order, so they
  // run at the same time and share each guidance row and statistics row through L2
  const int x0 = blockIdx.y * TX;
  const int Y0 = blockIdx.z * BH, Y1 = min(H, Y0 + BH);
  const int lb0 = blockIdx.x * LB;
  const int xt = x0 - R - SH;                       // TMA x start (16-byte aligned: x0 % 4 == 0)
  const int nsteps = 2 * R + (Y1 - Y0);             // entering rows Y0 - R .. Y1 - 1 + R
  const int nx = min(TX, W - x0);                   // pixels of the strip inside the image
  const unsigned sbytes = (unsigned)(nx * SPX * 4);

  uint64_t* empty = bar + NST;                      // consumer warps release a stage (count NW)
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      cuda::ptx::mbarrier_init(&bar[s], 1);
      cuda::ptx::mbarrier_init(&empty[s], NW);
    }
    cuda::ptx::fence_mbarrier_init(cuda::ptx::sem_release, cuda::ptx::scope_cluster);
  }
  // statistics records of pixels beyond the image stay zero (zero coefficients there)
  if (nx < TX) {
    for (int s = 0; s < NST; ++s)
      for (int e = nx * SPX + tid; e < TX * SPX; e += NW * 32) sm[s * Gm::STAGE + 2 * Gm::PROW + 2 * Gm::GROW + e] = 0.0f;
  }
  __syncthreads();

  // step t: entering row Y0 - R + t, leaving row Y0 - 2R - 1 + t (t >= 2R + 1), output row Y0 - 2R + t (t >= 2R)
  auto issue = [&](int t) {
    const int sl = t % NST;
    float* s = sm + sl * Gm::STAGE;
    uint64_t* b = &bar[sl];
    const int ye = Y0 - R + t;
    const bool leave = t >= 2 * R + 1, out = t >= 2 * R;
    const unsigned bytes = (unsigned)((leave ? 2 : 1) * (Gm::PROW + M * XB * (D == 2 ? 2 : 1)) * 4) + (out ? sbytes : 0u);
    cuda::ptx::mbarrier_arrive_expect_tx(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared, b,
                                         bytes);
    tma_3d(s, &tm_vol, xt, ye, lb0, b);
    if (D == 2) tma_3d(s + 2 * Gm::PROW, &tm_i, xt, 0, ye, b);      // pairs: dims (x, channel, y)
    else tma_3d(s + 2 * Gm::PROW, &tm_i, xt, ye, 0, b);             // raw planes: dims (x, y, channel)
    if (leave) {
      tma_3d(s + Gm::PROW, &tm_vol, xt, ye - 2 * R - 1, lb0, b);
      if (D == 2) tma_3d(s + 2 * Gm::PROW + Gm::GROW, &tm_i, xt, 0, ye - 2 * R - 1, b);
      else tma_3d(s + 2 * Gm::PROW + Gm::GROW, &tm_i, xt, ye - 2 * R - 1, 0, b);
    }
    if (out) {
      const int y = ye - R;
      cuda::ptx::cp_async_bulk(cuda::ptx::space_cluster, cuda::ptx::space_global, s + 2 * Gm::PROW + 2 * Gm::GROW,
                               stats + ((long long)y * W + x0) * SPX, sbytes, b);
    }
  };
  if (tid == 0)
    for (int t = 0; t < NST && t < nsteps; ++t) issue(t);

  // ===== consumer warps: lane = label, warp = 16-pixel segment =====
  // running window sums: S[k][i] (generic degree) or S0 / S2 pairs (degree 2)
  constexpr int KS = (D == 2) ? 1 : K;
  float S[KS][SEG];
  float2 S2[D == 2 ? M : 1][SEG];
#pragma unroll
  for (int k = 0; k < KS; ++k)
#pragma unroll
    for (int i = 0; i < SEG; ++i) S[k][i] = 0.0f;
#pragma unroll
  for (int c = 0; c < (D == 2 ? M : 1); ++c)
#pragma unroll
    for (int i = 0; i < SEG; ++i) S2[c][i] = make_float2(0.0f, 0.0f);
  auto Sk = [&](int k, int i) -> float {           // plane k of the window sums at segment pixel i
    if constexpr (D == 2) {
      if (k == 0) return S[0][i];
      return ((k - 1) & 1) ? S2[(k - 1) >> 1][i].y : S2[(k - 1) >> 1][i].x;
    } else {
      return S[k][i];
    }
  };

  const int l = lb0 + lane;
  const int grp = (x0 >> 4) + seg;                  // this segment's pixel group of the interleaved layout
  const bool store_ok = l < L && grp < wo.xg;
  const long long kstride = (long long)H * wo.xg * (kWGroupPx * kWGroupLabels);
  float* wl = wbuf + ((long long)(l / kWGroupLabels) * K * H * wo.xg + grp) * (kWGroupPx * kWGroupLabels) +
              (l % kWGroupLabels) * kWGroupPx;

  for (int t = 0; t < nsteps; ++t) {
    const float* s = sm + (t % NST) * Gm::STAGE;
    while (!cuda::ptx::mbarrier_try_wait_parity(&bar[t % NST], (t / NST) & 1)) {
    }
    if constexpr (D == 2) {
      hsum_row2<M, R, 1>(s + lane * XB + seg * SEG, s + 2 * Gm::PROW + 2 * seg * SEG, S[0], S2);
      if (t >= 2 * R + 1)
        hsum_row2<M, R, -1>(s + Gm::PROW + lane * XB + seg * SEG, s + 2 * Gm::PROW + Gm::GROW + 2 * seg * SEG, S[0],
                            S2);
    } else {
      hsum_row<M, D, R, 1>(s + lane * XB + seg * SEG, s + 2 * Gm::PROW + seg * SEG, S);
      if (t >= 2 * R + 1)
        hsum_row<M, D, R, -1>(s + Gm::PROW + lane * XB + seg * SEG, s + 2 * Gm::PROW + Gm::GROW + seg * SEG, S);
    }
    if (t >= 2 * R) {
      const int y = Y0 - 2 * R + t;                  // output row complete
      const float* st = s + 2 * Gm::PROW + 2 * Gm::GROW + seg * SEG * SPX;
      float* wrow = wl + (long long)y * wo.xg * (kWGroupPx * kWGroupLabels);
#pragma unroll
      for (int q8 = 0; q8 < SEG; q8 += 8) {
        float wv[K][8];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) {
          const int i = q8 + ii;
          float sp[SPX];
          const float4* s4 = reinterpret_cast<const float4*>(st + i * SPX);
#pragma unroll
          for (int q = 0; q < SPX / 4; ++q) {
            const float4 v = s4[q];
            sp[4 * q] = v.x; sp[4 * q + 1] = v.y; sp[4 * q + 2] = v.z; sp[4 * q + 3] = v.w;
          }
          float cc[NC > 0 ? NC : 1];
#pragma unroll
          for (int k = 0; k < NC; ++k) cc[k] = fmaf(-sp[NP + k], Sk(0, i), Sk(k + 1, i));
          float w0 = sp[NS] * Sk(0, i);
#pragma unroll
          for (int a = 0; a < NC; ++a) {
            float tt = 0.0f;
#pragma unroll
            for (int bq = 0; bq < NC; ++bq) {
              const int lo = a < bq ? a : bq, hi = a < bq ? bq : a;
              tt = fmaf(sp[lo * NC - lo * (lo - 1) / 2 + (hi - lo)], cc[bq], tt);
            }
            wv[a + 1][ii] = tt;
            w0 = fmaf(-sp[NP + a], tt, w0);
          }
          wv[0][ii] = w0;
        }
        if (store_ok) {
#pragma unroll
          for (int k = 0; k < K; ++k) st_global_v8(wrow + k * kstride + q8, wv[k]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) cuda::ptx::mbarrier_arrive(&empty[t % NST]);
    // thread 0 refills the stage once every warp has released it (no CTA-wide barrier: the other warps
    // run on into the stages already loaded)
    if (tid == 0 && t + NST < nsteps) {
      while (!cuda::ptx::mbarrier_try_wait_parity(&empty[t % NST], (t / NST) & 1)) {
      }
      issue(t + NST);
    }
  }
}

template <int M, int D, int R>
cudaError_t coef5_r(const void* tm_vol, const void* tm_i, const float* stats, float* wbuf, WLayout wo, int W, int H,
                    int L, int Lmodel, cudaStream_t st) {
  using Gm = Geom<M * D>;
  cudaError_t e = cudaFuncSetAttribute(k_coef5<M, D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::SMEM);
  if (e != cudaSuccess) return e;
  // band height: one CTA per SM; a band of BH rows costs BH + 2R steps (the vertical warm-up), so pick the
  // band count minimising waves x (BH + 2R), waves = ceil(CTAs / 148), among band counts giving >= 8 waves
  // (or, for small images, the most CTAs) -- the same wave model as k_coef3.
  // the band height depends on (W, H, R, Lmodel) only (see launch_coef_v5); the grid uses this chunk's batches
  const int strips = (W + TX - 1) / TX, batches = ((Lmodel > L ? Lmodel : L) + LB - 1) / LB;
  const int chunk_batches = (L + LB - 1) / LB;
  constexpr int kMaxBand = 320;
  int BH = H < kMaxBand ? H : kMaxBand;
  {
    long long best = -1;
    const int nbmax = H / 32 > 1 ? H / 32 : 1;
    // bands of at most kMaxBand rows: the fp32 running window sums are never restarted inside a band, so
    // their rounding drift grows with the band length (parity at 270 rows: tests/test_gpu_parity.py)
    const int nbmin = (H + kMaxBand - 1) / kMaxBand;
    const long long most = (long long)strips * ((H + (H + nbmax - 1) / nbmax - 1) / ((H + nbmax - 1) / nbmax)) * batches;
    const long long target = most < 8 * 148 ? most : 8 * 148;
    for (int nb = nbmin; nb <= (nbmax > nbmin ? nbmax : nbmin); ++nb) {
      const int bh = (H + nb - 1) / nb;
      const long long ctas = (long long)strips * ((H + bh - 1) / bh) * batches;
      if (ctas < target) continue;
      const long long cost = (ctas + 147) / 148 * (bh + 2 * R);
      if (best < 0 || cost < best) { best = cost; BH = bh; }
    }
    if (most < 148) {
      // small frames (less than one wave even at 32-row bands, e.g. the paper's 450 x 375 Middlebury size): bands
      // down to 8 rows, the count minimising waves x (band + warm-up) -- one full wave of short bands beats a
      // partial wave of long ones
      for (int nb = nbmin; nb <= H / 8; ++nb) {
        const int bh = (H + nb - 1) / nb;
        const long long ctas = (long long)strips * ((H + bh - 1) / bh) * batches;
        const long long cost = (ctas + 147) / 148 * (bh + 2 * R);
        if (cost < best) { best = cost; BH = bh; }
      }
    }
  }
  const int bh_env = std::getenv("HGF_COEF5_BH") ? std::atoi(std::getenv("HGF_COEF5_BH")) : 0;
  if (bh_env >= 8) BH = bh_env;                    // tuning / test runs only
  dim3 grid(chunk_batches, strips, (H + BH - 1) / BH);
  k_coef5<M, D, R><<<grid, NW * 32, Gm::SMEM, st>>>(*reinterpret_cast<const CUtensorMap*>(tm_vol),
                                                    *reinterpret_cast<const CUtensorMap*>(tm_i), stats, wbuf, wo, W, H,
                                                    L, BH);
  return cudaGetLastError();
}

template <int M, int D>
cudaError_t coef5_impl(const void* tm_vol, const void* tm_i, const float* stats, float* wbuf, WLayout wo, int W,
                       int H, int r, int L, int Lmodel, cudaStream_t st) {
  switch (r) {
    case 1: return coef5_r<M, D, 1>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    case 2: return coef5_r<M, D, 2>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    case 3: return coef5_r<M, D, 3>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    case 4: return coef5_r<M, D, 4>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    case 5: return coef5_r<M, D, 5>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    case 6: return coef5_r<M, D, 6>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    case 7: return coef5_r<M, D, 7>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    case 8: return coef5_r<M, D, 8>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    case 9: return coef5_r<M, D, 9>(tm_vol, tm_i, stats, wbuf, wo, W, H, L, Lmodel, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace v5
}  // namespace hgf
