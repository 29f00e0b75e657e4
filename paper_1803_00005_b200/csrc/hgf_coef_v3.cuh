// HGF per-slice coefficients, version 3 (k_coef3<n, R>): label-batched row marching, warp-specialised,
// TMA-fed.
//
// For each slice l and pixel p (Eq12 with G_{n+1} = p; Eq13 P:304 reassociated):
//     S_0 = B(p),  S_k = B(G_k p)  (k = 1..n),   w = P'(S - nu S_0),   w_0 = S_0/(lambda_0 + N) - nu^T w
//
// A CTA owns a strip of TX = 64 columns x a band of BH rows x a batch of LB = 32 labels and marches down
// the band one image row per step:
//   * TMA (one elected V thread): per step, the entering row (y+R) and the leaving row (y-R-1) of the
//     32 labels' cost slices and of the n guidance planes land in SMEM (2-stage ring, mbarrier-tracked,
//     issued two steps ahead).  Rows/labels/columns outside the image read as zero (clipped windows).
//   * V warps (producers): thread = (column c of the strip plus an R halo, group of 8 labels; groups are
//     warp-aligned); it keeps the vertical running sums V_k(c) = sum_{|dy|<=R} G_k p of its 8 labels in
//     registers, and per output row writes the V row of the 32 labels, copies the row's per-pixel
//     statistics records (k_stats2 aos: 27 floats + kappa = 1/(lambda_0+N)) into SMEM with coalesced
//     128-bit loads, and sums each segment's first 2R+1-column window (the H warps' starting sums).
//   * H warps (consumers): lane = label, warp = 16-pixel segment; slides the horizontal 2R+1 window over
//     the V row, reads each pixel's statistics with 128-bit broadcast loads (one wavefront per warp), does
//     the n x n matvec and stores w with 32-byte stores into the label-interleaved layout (WLayout::il:
//     the 32 lanes of one store instruction cover 2 KB contiguous) or 16-byte runs (planar layout).
//   * V and H warps run one row apart through a double-buffered SMEM V row (named barriers FULL/FREE).
// Label-invariant data (G, statistics) never costs per-label shared-memory traffic.
#pragma once
#include <cuda.h>

#include <cstdlib>

#include <cuda/ptx>

#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace v3 {

#ifndef HGF_EXP
#define HGF_EXP 0   // timing experiments only: 1 = V warps alone, 2 = H warps alone, 3 = neither (wrong results)
#endif
constexpr int C_TX = 64;                    // owned columns per strip
constexpr int C_LG = 8;                     // labels per V thread
constexpr int C_HSEG = 16;                  // pixels per H thread (two store groups of 8)
static_assert(C_HSEG % kWGroupPx == 0 && kWGroupPx % 8 == 0, "an H segment is whole groups of the interleaved layout");
constexpr int C_NSEG = C_TX / C_HSEG;       // segments per strip
constexpr int C_RMAX = 9;
constexpr int C_BXP = 88;                   // TMA box width: >= TX + 2*RMAX + 3 (x start rounded down to 16 B)
constexpr int C_BAR_V = 5;                  // named barrier among the V warps

template <int NC>
struct CoefGeom {
  static constexpr int K = NC + 1, NP = NC * (NC + 1) / 2, NS = NP + NC;
  // labels per CTA: 32 (H warp = one segment, lane = label) up to n = 6; 16 for n = 7..9 (H warp = two
  // segments x 16 labels) so that the V rows of n + 1 planes still double-buffer in SMEM
  static constexpr int LB = coef3_labels(NC);
  static_assert(kWGroupLabels % LB == 0, "a CTA's labels lie in one 32-label group of the layout");
  static constexpr int NG = LB / C_LG;                      // V label groups
  static constexpr int NHW = LB * C_NSEG / 32;              // H warps
  static constexpr int SPX = stats_aos_floats(NC);          // floats per pixel in the SMEM statistics row
  static_assert(NS + 1 <= SPX, "statistics + kappa must fit the per-pixel slot");
  // segment stride: consecutive segments 16 banks apart
  static constexpr int SSEG = C_HSEG * SPX + (16 - (C_HSEG * SPX) % 32 + 32) % 32;
  static constexpr int CXMAX = C_TX + 2 * C_RMAX;         // V columns (strip + halo), max 82
  static constexpr int CP = CXMAX;                          // SMEM column pitch
  static constexpr int LSTRIDE = K * CP + ((K * CP) % 2 == 0 ? 1 : 0);  // floats per label (odd)
  static constexpr int VROW = LB * LSTRIDE;                 // floats per V row buffer
  static constexpr int SROW = C_NSEG * SSEG;                // statistics row
  // one TMA stage: entering + leaving rows of the LB labels' cost slices and of the NC guidance planes
  // (every TMA destination 128-byte aligned: sizes rounded to 32 floats)
  static constexpr int PROW = LB * C_BXP, GROW = ((NC > 0 ? NC : 1) * C_BXP + 31) / 32 * 32;
  static constexpr int STAGE = 2 * PROW + 2 * GROW;
  // per (segment, label): the 2R+1 window sums of the segment's first pixel, computed by the V warps
  static constexpr int ISEG = LB * K + 16 + ((LB * K) % 32 == 16 ? 16 : 0);  // = 16 banks mod 32
  static constexpr int INI = C_NSEG * ISEG;
  static constexpr int CXP = (CXMAX + 31) / 32 * 32;        // V threads per label group (warp-aligned groups)
  static constexpr int NVW = (CXP * NG + 31) / 32;          // V warps
  static constexpr int THREADS = (NVW + NHW) * 32;
  static constexpr size_t SMEM =
      sizeof(float) * (2 * (size_t)STAGE + 2 * (size_t)VROW + 2 * (size_t)SROW + 2 * (size_t)INI) + 64;
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void c3_tma_3d(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
  const int32_t c[3] = {x, y, z};
  cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, dst, tm, c, bar);
}

// 256-bit global store (sm_100: STG.E.ENL2.256), p 32-byte aligned.
__device__ __forceinline__ void st_global_v8(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

// R > 0: compile-time radius; R == 0: runtime radius r_arg (<= C_RMAX).
template <int NC, int R>
__global__ void __launch_bounds__(CoefGeom<NC>::THREADS, 1)
    k_coef3(const __grid_constant__ CUtensorMap tm_vol, const __grid_constant__ CUtensorMap tm_g,
            const float* __restrict__ stats, float* __restrict__ wbuf, WLayout wo, int W, int H, int r_arg, int L,
            int BH, float lam0) {
  using Gm = CoefGeom<NC>;
  constexpr int K = Gm::K, NP = Gm::NP, NS = Gm::NS, CP = Gm::CP, LSTRIDE = Gm::LSTRIDE;
  constexpr int NV = Gm::NVW * 32, NH = Gm::NHW * 32, NALL = NV + NH;
  constexpr int C_LB = Gm::LB, C_NG = Gm::NG, C_SPX = Gm::SPX, C_SSEG = Gm::SSEG;
  const int r = (R > 0) ? R : r_arg;
  extern __shared__ __align__(128) float sm[];
  float* stage = sm;                              // [2][STAGE]: pe[32][BXP], pl[32][BXP], ge[NC][BXP], gl[NC][BXP]
  float* vrow = sm + 2 * Gm::STAGE;               // [2][LB][K][CP]
  float* srow = vrow + 2 * Gm::VROW;              // [2][NSEG][HSEG][SPX] (+16 pad per segment)
  float* ini = srow + 2 * Gm::SROW;               // [2][NSEG][ISEG]: [label][K] window sums per segment
  uint64_t* bar = reinterpret_cast<uint64_t*>(ini + 2 * Gm::INI);
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * C_TX;
  const int Y0 = blockIdx.y * BH, Y1 = min(H, Y0 + BH);
  const int lb0 = blockIdx.z * C_LB;
  const int CX = C_TX + 2 * r;                    // V columns used: image x = x0 - r + c
  const int xt = ((x0 - r) >> 2) << 2;            // TMA x start (16-byte aligned; arithmetic shift floors)
  const int sh = (x0 - r) - xt;                   // SMEM column of V column 0
  const int nsteps = 2 * r + (Y1 - Y0);           // entering rows Y0-r .. Y1-1+r

  if (tid < NV) {
    // ============================ V warps (producers) ============================
    const int g = tid / Gm::CXP, c = tid % Gm::CXP;  // groups warp-aligned: no bank straddles
    const bool active = g < C_NG && c < CX;
    const int cs = c + sh;
    if (tid == 0) {
      cuda::ptx::mbarrier_init(&bar[0], 1);
      cuda::ptx::mbarrier_init(&bar[1], 1);
      cuda::ptx::fence_mbarrier_init(cuda::ptx::sem_release, cuda::ptx::scope_cluster);
    }
    named_sync(C_BAR_V, NV);
    // step t: entering row Y0 - r + t, leaving row Y0 - 2r - 1 + t (from t = 2r + 1), output row Y0 - r + t - r
    auto issue = [&](int t) {
      float* s = stage + (t & 1) * Gm::STAGE;
      const int ye = Y0 - r + t;
      const bool leave = t >= 2 * r + 1;
      const unsigned bytes = (unsigned)(((leave ? 2 : 1) * (Gm::PROW + NC * C_BXP)) * 4);
      cuda::ptx::mbarrier_arrive_expect_tx(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared,
                                           &bar[t & 1], bytes);
      c3_tma_3d(s, &tm_vol, xt, ye, lb0, &bar[t & 1]);
      if (NC > 0) c3_tma_3d(s + 2 * Gm::PROW, &tm_g, xt, ye, 0, &bar[t & 1]);
      if (leave) {
        c3_tma_3d(s + Gm::PROW, &tm_vol, xt, ye - 2 * r - 1, lb0, &bar[t & 1]);
        if (NC > 0) c3_tma_3d(s + 2 * Gm::PROW + Gm::GROW, &tm_g, xt, ye - 2 * r - 1, 0, &bar[t & 1]);
      }
    };
    if (tid == 0) {
      issue(0);
      if (nsteps > 1) issue(1);
    }
    float acc[C_LG][K];
#pragma unroll
    for (int j = 0; j < C_LG; ++j)
#pragma unroll
      for (int k = 0; k < K; ++k) acc[j][k] = 0.0f;
    // statistics of output row y for the strip, prefetched one row ahead: k_stats2 stores them per pixel
    // (C_SPX floats: NS statistics, then kappa), so the strip's row is one contiguous run of 16-byte
    // chunks -> coalesced 128-bit loads and conflict-free 128-bit stores into the segment-padded srow.
    // Pixels beyond W read as zero, which makes their coefficients zero (the interleaved layout's padding).
    constexpr int SCH = C_SPX / 4;                       // 16-byte chunks per pixel
    constexpr int SPT = (C_TX * SCH + NV - 1) / NV;
    float4 spre[SPT];
    auto load_stats = [&](int y) {
#pragma unroll
      for (int q = 0; q < SPT; ++q) {
        const int e = tid + q * NV;
        const int x = e / SCH;
        float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (e < C_TX * SCH && y < Y1 && x0 + x < W)
          v = __ldg(reinterpret_cast<const float4*>(stats + ((long long)y * W + x0) * C_SPX) + e);
        spre[q] = v;
      }
    };
    load_stats(Y0);
    for (int t = 0; t < nsteps; ++t) {
      const float* s = stage + (t & 1) * Gm::STAGE;
      while (!cuda::ptx::mbarrier_try_wait_parity(&bar[t & 1], (t >> 1) & 1, uint32_t(kMbarSuspendNs))) {
      }
      const bool leave = t >= 2 * r + 1;
      if (active && (HGF_EXP & 2) == 0) {
        float ge[NC > 0 ? NC : 1], gl[NC > 0 ? NC : 1];
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          ge[k] = s[2 * Gm::PROW + k * C_BXP + cs];
          gl[k] = leave ? s[2 * Gm::PROW + Gm::GROW + k * C_BXP + cs] : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < C_LG; ++j) {
          const float pe = s[(g * C_LG + j) * C_BXP + cs];
          const float pl = leave ? s[Gm::PROW + (g * C_LG + j) * C_BXP + cs] : 0.0f;
          acc[j][0] += pe - pl;
#pragma unroll
          for (int k = 0; k < NC; ++k) acc[j][k + 1] = fmaf(ge[k], pe, fmaf(-gl[k], pl, acc[j][k + 1]));
        }
      }
      named_sync(C_BAR_V, NV);                         // every V thread is done with stage t & 1
      if (tid == 0 && t + 2 < nsteps) {
        cuda::ptx::fence_proxy_async(cuda::ptx::space_shared);
        issue(t + 2);
      }
      const int y = Y0 - r + t - r;                    // output row completed by this step
      if (y < Y0) continue;
      const int b = (y - Y0) & 1;
      if (y - Y0 >= 2) named_sync(3 + b, NALL);        // H warps released buffer b
      if (active && (HGF_EXP & 2) == 0) {
        float* dst = vrow + b * Gm::VROW + (g * C_LG) * LSTRIDE + c;
#pragma unroll
        for (int j = 0; j < C_LG; ++j)
#pragma unroll
          for (int k = 0; k < K; ++k) dst[j * LSTRIDE + k * CP] = acc[j][k];
      }
      float* sdst = srow + b * Gm::SROW;
#pragma unroll
      for (int q = 0; q < SPT; ++q) {
        const int e = tid + q * NV;
        if (e < C_TX * SCH) {
          const int x = e / SCH, c4 = e % SCH;
          *reinterpret_cast<float4*>(sdst + (x / C_HSEG) * C_SSEG + (x % C_HSEG) * C_SPX + 4 * c4) = spre[q];
        }
      }
      // window sums of every (segment, label, plane) at the segment's first pixel: the H warps start their
      // sliding windows from these instead of summing 2R+1 columns each (moves ~1/4 of the H work here)
      named_sync(C_BAR_V, NV);
      for (int item = tid; item < ((HGF_EXP & 2) ? 0 : C_NSEG * C_LB * K); item += NV) {
        // lanes walk labels (odd LSTRIDE: conflict-free loads; stride-K stores into ini: conflict-free)
        const int lab = item % C_LB, sk = item / C_LB, k = sk % K, sg = sk / K;
        const int rem = lab * K + k;
        const float* colp = vrow + b * Gm::VROW + lab * LSTRIDE + k * CP + sg * C_HSEG;
        float a = 0.0f;
        if (R > 0) {
#pragma unroll
          for (int j = 0; j <= 2 * R; ++j) a += colp[j];
        } else {
          for (int j = 0; j <= 2 * r; ++j) a += colp[j];
        }
        ini[b * Gm::INI + sg * Gm::ISEG + rem] = a;
      }
      named_arrive(1 + b, NALL);                       // row y ready in buffer b
      load_stats(y + 1);
    }
  } else {
    // ============================ H warps (consumers) ============================
    const int h = tid - NV, hw = h >> 5, ln = h & 31;
    // lane = label, warp = segment: each pixel's statistics are one broadcast per warp, and the odd
    // LSTRIDE keeps the 32 labels' V-row loads conflict-free
    const int lab = C_LB == 32 ? ln : (ln & 15);                   // label within the batch
    const int seg = C_LB == 32 ? hw : 2 * hw + (ln >> 4);          // 16-pixel segment 0..3
    const int l = lb0 + lab;
    const bool lok = l < L;
    const int xs = seg * C_HSEG;                      // first owned pixel (strip-relative)
    for (int y = Y0; y < Y1; ++y) {
      const int b = (y - Y0) & 1;
      named_sync(1 + b, NALL);
      if (HGF_EXP & 1) {
        named_arrive(3 + b, NALL);
        continue;
      }
      const float* vr = vrow + b * Gm::VROW + lab * LSTRIDE + xs;    // V column xs of plane 0
      const float* st = srow + b * Gm::SROW + seg * C_SSEG;
      const float* ip = ini + b * Gm::INI + seg * Gm::ISEG + lab * K;
      float S[K];
#pragma unroll
      for (int k = 0; k < K; ++k) S[k] = ip[k];
#pragma unroll 1
      for (int q8 = 0; q8 < C_HSEG; q8 += 8) {
      float wv[K][8];
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) {
        const int i = q8 + ii;
        if (i > 0) {
#pragma unroll
          for (int k = 0; k < K; ++k) S[k] += vr[k * CP + i + 2 * r] - vr[k * CP + i - 1];
        }
        float sp[C_SPX];
        const float4* s4 = reinterpret_cast<const float4*>(st + i * C_SPX);
#pragma unroll
        for (int q = 0; q < C_SPX / 4; ++q) {
          const float4 v = s4[q];
          sp[4 * q] = v.x; sp[4 * q + 1] = v.y; sp[4 * q + 2] = v.z; sp[4 * q + 3] = v.w;
        }
        float cc[NC > 0 ? NC : 1];
#pragma unroll
        for (int k = 0; k < NC; ++k) cc[k] = fmaf(-sp[NP + k], S[0], S[k + 1]);
        float w0 = sp[NS] * S[0];
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
      if (wo.il) {
        // label-interleaved layout (see WLayout): 32-byte stores of 8 pixels; G = 16: the 16 labels of a
        // half-warp cover one contiguous 1 KB run; G = 8: the 32 labels of a warp do (whole lines)
        const int grp = (x0 + xs + q8) / kWGroupPx;
        if (lok && grp < wo.xg) {
          float* wg = wbuf + (((long long)(l / kWGroupLabels) * K * H + y) * wo.xg + grp) *
                                 (kWGroupPx * kWGroupLabels) +
                      (l % kWGroupLabels) * kWGroupPx + q8 % kWGroupPx;
          const long long kstride = (long long)H * wo.xg * (kWGroupPx * kWGroupLabels);
#pragma unroll
          for (int k = 0; k < K; ++k) st_global_v8(wg + k * kstride, wv[k]);
        }
      } else if (lok) {
        float* wrow = wbuf + wo.origin + (long long)l * K * wo.plane + (long long)y * wo.pitch + x0 + xs + q8;
        if (x0 + xs + q8 + 8 <= W) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            float4* d4 = reinterpret_cast<float4*>(wrow + k * wo.plane);
            d4[0] = make_float4(wv[k][0], wv[k][1], wv[k][2], wv[k][3]);
            d4[1] = make_float4(wv[k][4], wv[k][5], wv[k][6], wv[k][7]);
          }
        } else {
#pragma unroll
          for (int k = 0; k < K; ++k)
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (x0 + xs + q8 + i < W) wrow[k * wo.plane + i] = wv[k][i];
        }
      }
      }
      named_arrive(3 + b, NALL);                   // buffer b free again
    }
  }
}

template <int NC, int R>
cudaError_t coef3_r(const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo, int W, int H,
                    int r, int L, float lam0, cudaStream_t st) {
  using Gm = CoefGeom<NC>;
  cudaError_t e = cudaFuncSetAttribute(k_coef3<NC, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::SMEM);
  if (e != cudaSuccess) return e;
  // band height: one CTA per SM (223 KB of SMEM), each band of BH rows costs BH + 2r row steps (the 2r-row
  // warm-up of the vertical sums), so pick the band count nb (balanced bands of ceil(H / nb) >= 32 rows)
  // minimising waves x (BH + 2r), waves = ceil(CTAs / 148), among the band counts that give at least 8
  // waves (fewer, longer CTAs measured slower: BH = 360 at C4) or, for small images, the most CTAs.
  // C4: nb = 8 (BH = 270, 12.97 waves) instead of BH = 128 (27.6 waves, 14 % warm-up): k_coef3
  // 22.97 -> 22.24 ms (HGF_COEF3_BH sweep, profiles/r01_coef3_bh_sweep.txt).
  const int strips = (W + C_TX - 1) / C_TX, batches = (L + Gm::LB - 1) / Gm::LB;
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
      const long long cost = (ctas + 147) / 148 * (bh + 2 * r);
      if (best < 0 || cost < best) { best = cost; BH = bh; }
    }
  }
  const int bh_env = std::getenv("HGF_COEF3_BH") ? std::atoi(std::getenv("HGF_COEF3_BH")) : 0;
  if (bh_env >= 8) BH = bh_env;                    // tuning runs only
  dim3 grid(strips, (H + BH - 1) / BH, batches);
  k_coef3<NC, R><<<grid, Gm::THREADS, Gm::SMEM, st>>>(*reinterpret_cast<const CUtensorMap*>(tm_vol),
                                                      *reinterpret_cast<const CUtensorMap*>(tm_g), stats, wbuf, wo, W,
                                                      H, r, L, BH, lam0);
  return cudaGetLastError();
}

template <int NC>
cudaError_t coef3_impl(const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo, int W,
                       int H, int r, int L, float lam0, cudaStream_t st) {
  switch (r) {
    case 2: return coef3_r<NC, 2>(tm_vol, tm_g, stats, wbuf, wo, W, H, r, L, lam0, st);
    case 4: return coef3_r<NC, 4>(tm_vol, tm_g, stats, wbuf, wo, W, H, r, L, lam0, st);
    case 7: return coef3_r<NC, 7>(tm_vol, tm_g, stats, wbuf, wo, W, H, r, L, lam0, st);
    case 9: return coef3_r<NC, 9>(tm_vol, tm_g, stats, wbuf, wo, W, H, r, L, lam0, st);
    default: return coef3_r<NC, 0>(tm_vol, tm_g, stats, wbuf, wo, W, H, r, L, lam0, st);
  }
}

}  // namespace v3
}  // namespace hgf
