// HGF per-slice coefficients, version 4 (k_coef4<n>): row marching with the horizontal box sums on the
// 5th-generation tensor cores (tcgen05.mma, TMEM accumulators).
//
// For each slice l and pixel p (Eq12 with G_{n+1} = p; Eq13 P:304 reassociated):
//     S_0 = B(p),  S_k = B(G_k p)  (k = 1..n),   w = P'(S - nu S_0),   w_0 = kappa S_0 - nu^T w
//
// A CTA owns a strip of TX = 128 output columns x a band of BH rows x a batch of LB = 16 labels and marches
// down the band one image row per step:
//   * TMA (one elected V thread): the entering (y+R) and leaving (y-R-1) rows of the 16 labels' cost slices
//     and of the n guidance planes land in SMEM (2-stage ring, mbarrier-tracked, issued two steps ahead).
//   * V warps: thread = (column c of the strip plus an R halo, group of 8 labels); vertical running sums
//     V_k(c) = sum_{|dy|<=R} G_k p in registers.  Per output row they write the V row as the B operand of
//     an MMA: B[n][c], n = label * (n+1) + plane, K-major core matrices, split x = hi + lo with hi
//     tf32-exact (hi, lo in two SMEM planes).
//   * one elected thread issues D[px][n] = sum_c Band[px][c] * (B_hi + B_lo)[n][c] as 2 x KC/8
//     tcgen05.mma.kind::tf32 (M = 128 pixels, N = 16 (n+1), K = 8 columns each): Band[px][c] = 1 for
//     px <= c <= px + 2R lives in TMEM (A operand), D in TMEM (double-buffered across rows).  The split
//     keeps the sums fp32-accurate (products by 1 are exact; lo carries the bits tf32 drops;
//     tools/umma_test.cu: max relative error 4.9e-7 on 19-term sums).
//   * epilogue warps: thread = pixel (TMEM lane); tcgen05.ld its n+1 window sums per label, reads its
//     per-pixel statistics record (k_stats2 aos) once per row into registers, does the n x n matvec and
//     stores w in the planar layout (the 32 lanes of a warp write one 128-byte line per plane).
// No shared-memory traffic for the horizontal pass, the statistics or the segment start sums: the V-row
// write (2 words per plane per column) is the only per-label exchange between threads.
//
// Status (opt-in, HGF_COEF4=1): parity-green and more accurate than k_coef3 (max normalised error 1.4e-5
// vs 2.3e-5 on the GPU parity cases), but slower at C4 (29 vs 23 ms per frame).  Measured with HGF_EXP4
// builds: V warps alone 11.7 ms, + MMAs 21.5 ms, + epilogue 24.4 ms -- the tf32 MMAs (2 x 19 per row, the
// banded A wastes 7/8 of the K extent) keep the tensor pipe busy ~9 ms per frame and the single B buffer
// (137 KB for hi + lo) serialises V-row writes with them.  A bf16 hi/lo split halves both (one B buffer of
// bf16x2 pairs, double-buffered) but its 2^-18 representation error fails the 1e-4 parity bound (1.1e-4
// on C1); see DESIGN.md §6.
#pragma once
#include <cuda.h>

#include <cuda/ptx>

#include "hgf_common.cuh"
#include "hgf_launch.h"
#include "hgf_tc.cuh"

#ifndef HGF_EXP4
#define HGF_EXP4 0   // timing experiments only: 5 = epilogue skips its work, 6 = no MMAs (wrong results)
#endif

namespace hgf {
namespace v4 {

constexpr int TX = 128;                      // output columns per strip = MMA M (TMEM lanes)
constexpr int LB = kCoef4LB;                 // labels per CTA
constexpr int LG = 8;                        // labels per V thread
constexpr int NG = LB / LG;                  // V label groups
constexpr int RMAX = 9;
constexpr int CXP = 160;                     // V threads per group (>= TX + 2 RMAX, warp-aligned)
constexpr int KCMAX = (TX + 2 * RMAX + 7) / 8 * 8;   // MMA K extent (columns), 152
constexpr int BXP = kCoef4BoxX;              // TMA box width (>= TX + 2 RMAX + 3, multiple of 4)
constexpr int NVW = NG * CXP / 32;           // 10 V warps
constexpr int MMAW = NVW;                    // warp that allocates TMEM and issues the MMAs
constexpr int NEW = 4;                       // epilogue warps (one per TMEM lane quadrant)
constexpr int EW0 = NVW + 1;                 // first epilogue warp
constexpr int THREADS = (NVW + 1 + NEW) * 32;   // 480

constexpr int BAR_V = 1;                     // named barrier among the V warps
constexpr int SPX = kStatsAos;               // floats per statistics record
static_assert(KCMAX <= BXP && TX + 2 * RMAX + 3 <= BXP && TX + 2 * RMAX <= CXP, "strip geometry");

template <int NC>
struct Geom4 {
  static constexpr int K = NC + 1, NP = NC * (NC + 1) / 2, NS = NP + NC;
  static constexpr int N = LB * K;                               // MMA N (multiple of 16)
  static constexpr int LBO = (N / 8) * 128 + 16;                 // bytes between 16-byte K chunks (+16: banks)
  static constexpr int BPLANE = ((KCMAX / 4) * LBO + 1023) / 1024 * 1024;   // bytes of one of B_hi / B_lo
  static constexpr int PROW = LB * BXP;                          // floats: one cost row of the 16 labels
  static constexpr int GROW = ((NC > 0 ? NC : 1) * BXP + 31) / 32 * 32;
  static constexpr int STAGE = 2 * PROW + 2 * GROW;              // floats per TMA stage
  static constexpr size_t SMEM = 2 * (size_t)BPLANE + 2 * (size_t)STAGE * 4 + 8 * sizeof(uint64_t);
  static_assert(N % 16 == 0 && N <= 128, "MMA N / TMEM double buffer");
  static_assert(LB == 16 && K <= 7, "epilogue: 4-label batches of <= 32 columns");
  static_assert(NS + 1 <= SPX, "statistics record");
};

__device__ __forceinline__ void nsync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
  const int32_t c[3] = {x, y, z};
  cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, dst, tm, c, bar);
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
  while (!cuda::ptx::mbarrier_try_wait_parity(bar, parity, uint32_t(kMbarSuspendNs))) {   // parked, not spinning
  }
}

template <int NC>
__global__ void __launch_bounds__(THREADS, 1)
    k_coef4(const __grid_constant__ CUtensorMap tm_vol, const __grid_constant__ CUtensorMap tm_g,
            const float* __restrict__ stats, float* __restrict__ wbuf, WLayout wo, int W, int H, int r, int L,
            int BH) {
  using Gm = Geom4<NC>;
  constexpr int K = Gm::K, NP = Gm::NP, NS = Gm::NS, N = Gm::N, LBO = Gm::LBO;
  constexpr int NV = NVW * 32;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* bhi = smraw;                                     // B_hi, then B_lo (BPLANE bytes each)
  unsigned char* blo = smraw + Gm::BPLANE;
  float* stage = reinterpret_cast<float*>(smraw + 2 * Gm::BPLANE);   // [2][STAGE]
  uint64_t* bar = reinterpret_cast<uint64_t*>(stage + 2 * Gm::STAGE);
  uint64_t* tma_full = bar;          // [2] stage landed
  uint64_t* mma_done = bar + 2;      // [2] MMAs of the row in D[b] completed (B free again)
  uint64_t* d_free = bar + 4;        // [2] epilogue warps finished reading D[b]
  uint64_t* b_full = bar + 6;        // [2] every V warp wrote row i's B (row parity i & 1)
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int x0 = blockIdx.x * TX;
  const int Y0 = blockIdx.y * BH, Y1 = min(H, Y0 + BH);
  const int lb0 = blockIdx.z * LB;
  const int CX = TX + 2 * r;                      // V columns used: image x = x0 - r + c
  const int KC = (CX + 7) / 8 * 8;                // MMA K extent
  const int xt = ((x0 - r) >> 2) << 2;            // TMA x start (16-byte aligned; arithmetic shift floors)
  const int sh = (x0 - r) - xt;                   // SMEM column of V column 0
  const int nsteps = 2 * r + (Y1 - Y0);           // entering rows Y0-r .. Y1-1+r

  // ---- setup: barriers, zeroed B (columns >= CX stay zero), TMEM (D double buffer + band A)
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      cuda::ptx::mbarrier_init(&tma_full[i], 1);
      cuda::ptx::mbarrier_init(&mma_done[i], 1);
      cuda::ptx::mbarrier_init(&d_free[i], NEW);
      cuda::ptx::mbarrier_init(&b_full[i], NVW);
    }
    cuda::ptx::fence_mbarrier_init(cuda::ptx::sem_release, cuda::ptx::scope_cluster);
  }
  {
    uint4* z = reinterpret_cast<uint4*>(smraw);
    for (int i = tid; i < 2 * Gm::BPLANE / 16; i += THREADS) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (warp == MMAW) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  constexpr uint32_t IDESC = tc::idesc_tf32(TX, N);
  const uint32_t a_col = tbase + 256;             // A: columns [256, 256 + KC); D[b]: columns [128 b, 128 b + N)
  if (warp >= EW0) {
    // band: lane m (= output pixel m of the strip) has ones at columns m .. m + 2r
    const int m = 32 * (warp & 3) + lane;
    const uint32_t lrow = (uint32_t)(32 * (warp & 3)) << 16;
    for (int c0 = 0; c0 < KCMAX; c0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + j;
        v[j] = __float_as_uint((c >= m && c <= m + 2 * r) ? 1.0f : 0.0f);
      }
      tc::st_x8(lrow + a_col + c0, v);
    }
    tc::wait_st();
  }
  tc::fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();

  if (tid < NV) {
    // ============================ V warps ============================
    const int g = tid / CXP, c = tid % CXP;
    const bool active = c < CX;
    const int cs = c + sh;
    auto issue = [&](int t) {
      float* s = stage + (t & 1) * Gm::STAGE;
      const int ye = Y0 - r + t;
      const bool leave = t >= 2 * r + 1;
      const unsigned bytes = (unsigned)(((leave ? 2 : 1) * (Gm::PROW + NC * BXP)) * 4);
      cuda::ptx::mbarrier_arrive_expect_tx(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared,
                                           &tma_full[t & 1], bytes);
      tma3(s, &tm_vol, xt, ye, lb0, &tma_full[t & 1]);
      if (NC > 0) tma3(s + 2 * Gm::PROW, &tm_g, xt, ye, 0, &tma_full[t & 1]);
      if (leave) {
        tma3(s + Gm::PROW, &tm_vol, xt, ye - 2 * r - 1, lb0, &tma_full[t & 1]);
        if (NC > 0) tma3(s + 2 * Gm::PROW + Gm::GROW, &tm_g, xt, ye - 2 * r - 1, 0, &tma_full[t & 1]);
      }
    };
    if (tid == 0) {
      issue(0);
      if (nsteps > 1) issue(1);
    }
    float acc[LG][K];
#pragma unroll
    for (int j = 0; j < LG; ++j)
#pragma unroll
      for (int k = 0; k < K; ++k) acc[j][k] = 0.0f;
    // this thread's B offsets: element (n, c) at (c/4)*LBO + (n/8)*128 + (n%8)*16 + (c%4)*4 bytes
    const int cbase = (c >> 2) * LBO + (c & 3) * 4;
    for (int t = 0; t < nsteps; ++t) {
      const float* s = stage + (t & 1) * Gm::STAGE;
      mbar_wait_parity(&tma_full[t & 1], (t >> 1) & 1);
      const bool leave = t >= 2 * r + 1;
      if (active) {
        float ge[NC > 0 ? NC : 1], gl[NC > 0 ? NC : 1];
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          ge[k] = s[2 * Gm::PROW + k * BXP + cs];
          gl[k] = leave ? s[2 * Gm::PROW + Gm::GROW + k * BXP + cs] : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < LG; ++j) {
          const float pe = s[(g * LG + j) * BXP + cs];
          const float pl = leave ? s[Gm::PROW + (g * LG + j) * BXP + cs] : 0.0f;
          acc[j][0] += pe - pl;
#pragma unroll
          for (int k = 0; k < NC; ++k) acc[j][k + 1] = fmaf(ge[k], pe, fmaf(-gl[k], pl, acc[j][k + 1]));
        }
      }
      nsync(BAR_V, NV);                                // every V thread is done with stage t & 1
      if (tid == 0 && t + 2 < nsteps) {
        cuda::ptx::fence_proxy_async(cuda::ptx::space_shared);
        issue(t + 2);
      }
      const int y = Y0 - r + t - r;                    // output row completed by this step
      if (y < Y0) continue;
      const int i = y - Y0;
      // B is free once the previous row's MMAs have completed
      if (i >= 1) mbar_wait_parity(&mma_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
      if (active) {
#pragma unroll
        for (int j = 0; j < LG; ++j)
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const int n = (g * LG + j) * K + k;
            const int off = cbase + (n >> 3) * 128 + (n & 7) * 16;
            float hi, lo;
            tc::split_tf32(acc[j][k], hi, lo);
            *reinterpret_cast<float*>(bhi + off) = hi;
            *reinterpret_cast<float*>(blo + off) = lo;
          }
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) cuda::ptx::mbarrier_arrive(&b_full[i & 1]);   // this warp's part of row i's B is written
    }
  } else if (warp == MMAW) {
    // ============================ MMA warp ============================
    // per output row: B written (named barrier) and D[b] drained (d_free) -> 2 x KC/8 MMAs -> commit
    const uint64_t dh0 = tc::sdesc(tc::smem_u32(bhi), LBO, 128), dl0 = tc::sdesc(tc::smem_u32(blo), LBO, 128);
    const uint64_t dstep = (uint64_t)((2 * LBO) >> 4);           // next 8-column K step (start address field)
    const int ksteps = KC / 8;
    for (int y = Y0; y < Y1; ++y) {
      const int i = y - Y0, b = i & 1;
      mbar_wait_parity(&b_full[b], (i >> 1) & 1);
      if (lane == 0) {
        if (i >= 2) mbar_wait_parity(&d_free[b], ((i - 2) >> 1) & 1);
        tc::fence_after();
        const uint32_t d_col = tbase + 128 * b;
#if HGF_EXP4 != 6
        for (int s8 = 0; s8 < ksteps; ++s8)
          tc::mma_tf32_ts(d_col, a_col + 8 * s8, dh0 + (uint64_t)s8 * dstep, IDESC, s8 > 0 ? 1u : 0u);
        for (int s8 = 0; s8 < ksteps; ++s8)
          tc::mma_tf32_ts(d_col, a_col + 8 * s8, dl0 + (uint64_t)s8 * dstep, IDESC, 1u);
#endif
        tc::mma_commit(&mma_done[b]);
      }
      __syncwarp();
    }
  } else {
    // ============================ epilogue warps ============================
    const int q = warp & 3;                           // TMEM lane quadrant of this warp
    const int px = 32 * q + lane;                     // output pixel of the strip = TMEM lane
    const int gx = x0 + px;
    const uint32_t lrow = (uint32_t)(32 * q) << 16;
    for (int y = Y0; y < Y1; ++y) {
      const int i = y - Y0, b = i & 1;
      float sp[SPX];
      {
        const bool in = gx < W;
        const float4* src = reinterpret_cast<const float4*>(stats + ((long long)y * W + (in ? gx : 0)) * SPX);
#pragma unroll
        for (int u = 0; u < SPX / 4; ++u) {
          const float4 v = in ? __ldg(src + u) : make_float4(0.f, 0.f, 0.f, 0.f);
          sp[4 * u] = v.x; sp[4 * u + 1] = v.y; sp[4 * u + 2] = v.z; sp[4 * u + 3] = v.w;
        }
      }
      mbar_wait_parity(&mma_done[b], (i >> 1) & 1);
      tc::fence_after();
      const uint32_t d_col = tbase + 128 * b;
#pragma unroll 1
      for (int half = 0; half < (HGF_EXP4 == 5 ? 0 : 2); ++half)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        // labels 8 half + 4 bb + [0, 4): D columns [c0, c0 + 4K), fetched as 8-column loads from c0 & ~7
        const int o = (4 * K * bb) & 7;               // compile-time per bb
        const int a0 = 8 * K * half + ((4 * K * bb) & ~7);
        float dv[32];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (8 * u < o + 4 * K) tc::ld_x8(lrow + d_col + a0 + 8 * u, *reinterpret_cast<float(*)[8]>(dv + 8 * u));
        tc::wait_ld();
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
        const int j = 8 * half + 4 * bb + jj;
        float S[K];
#pragma unroll
        for (int k = 0; k < K; ++k) S[k] = dv[o + jj * K + k];
        float cc[NC > 0 ? NC : 1];
#pragma unroll
        for (int k = 0; k < NC; ++k) cc[k] = fmaf(-sp[NP + k], S[0], S[k + 1]);
        float wv[K];
        float w0 = sp[NS] * S[0];
#pragma unroll
        for (int a = 0; a < NC; ++a) {
          float tt = 0.0f;
#pragma unroll
          for (int bq = 0; bq < NC; ++bq) {
            const int lo = a < bq ? a : bq, hi = a < bq ? bq : a;
            tt = fmaf(sp[lo * NC - lo * (lo - 1) / 2 + (hi - lo)], cc[bq], tt);
          }
          wv[a + 1] = tt;
          w0 = fmaf(-sp[NP + a], tt, w0);
        }
        wv[0] = w0;
        const int l = lb0 + j;
        if (l < L && gx < W) {
          float* dst = wbuf + wo.origin + (long long)l * K * wo.plane + (long long)y * wo.pitch + gx;
#pragma unroll
          for (int k = 0; k < K; ++k) dst[k * wo.plane] = wv[k];
        }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) cuda::ptx::mbarrier_arrive(&d_free[b]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == MMAW) {
    tc::fence_after();
    tc::tmem_dealloc(tbase, 512);
  }
}

template <int NC>
cudaError_t coef4_impl(const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo, int W,
                       int H, int r, int L, cudaStream_t st) {
  using Gm = Geom4<NC>;
  if (r < 1 || r > RMAX) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_coef4<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::SMEM);
  if (e != cudaSuccess) return e;
  const int strips = (W + TX - 1) / TX, batches = (L + LB - 1) / LB;
  int BH = 128;
  while (BH > 32 && (long long)strips * ((H + BH - 1) / BH) * batches < 4 * 148) BH /= 2;
  dim3 grid(strips, (H + BH - 1) / BH, batches);
  k_coef4<NC><<<grid, THREADS, Gm::SMEM, st>>>(*reinterpret_cast<const CUtensorMap*>(tm_vol),
                                               *reinterpret_cast<const CUtensorMap*>(tm_g), stats, wbuf, wo, W, H,
                                               r, L, BH);
  return cudaGetLastError();
}

}  // namespace v4
}  // namespace hgf
