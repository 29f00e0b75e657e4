// Label-independent statistics, version 5 (k_stats5<n, LP, R>): k_stats4's row march with its three phases run by
// separate warps and pipelined across iterations through mbarriers, instead of one CTA that does V, H and R in turn
// between CTA barriers (k_stats4 spent ~25 % of its H phase at the barrier and its V phase waiting on global loads).
//
//   G_ab = B(G_a G_b) (Prop 2; Eq12), then per pixel the Prop-1 recursion (Eq4, readings
//   F1/F2; stats_finish / filter_finish_m) -- the same arithmetic in the same order as k_stats4, so the two kernels
//   give the same bits (tests/test_gpu_parity.py::test_stats5_bit_identical_to_stats4).
//
// Per CTA: a strip of TX = 64 output columns x a band of BH rows, RB = 2 rows per iteration, and
//   * 3 V warps (thread = strip column incl. the 2r halo): float64 vertical running sums of the products, held in
//     REGISTERS across iterations (k_stats4 re-read them from shared memory), the next iteration's channel rows
//     loaded one iteration ahead; each iteration's RB rows of sums go to vertical-sum slot j % NBV;
//   * NHW H warps (item = (row, 32-pixel segment, pair), one per thread): sliding 2r + 1-column window sums of a
//     vertical-sum slot into horizontal-sum slot j % NBH;
//   * 4 R warps (thread = pixel): the pixel's sums from an H slot (released at once), the recursion and the record
//     (or, LP = 1, the fused single-slice coefficients).
// Slots are handed over with full/free mbarriers (phase parity (j / NB) & 1); the roles run up to NB - 1
// iterations apart.  One 352..384-thread CTA per SM (n <= 6, 2r <= 32).  Default for hgf_filter's fused single-slice
// pass (LP = 1; one whole frame, so tall bands with the warm-up amortised); the statistics pass keeps k_stats4, whose
// three CTAs per SM hide each other's warm-ups (HGF_STATS5=1 selects k_stats5 there too, bit-identical).
#pragma once
#include <cuda/ptx>

#include "hgf_stats_v4.cuh"

namespace hgf {
namespace st5 {

using st4::npair;
using st4::nsums;
constexpr int TX = 64, RB = 2, TXP = TX + 1, HS = 32, NVW = 3, NRW = RB * TX / 32, NBV = 2, NBH = 2;

template <int NC, int LP>
struct Cfg {
  static constexpr int NPAIR = nsums(NC, LP);
  static constexpr int ITEMS = RB * (TX / HS) * NPAIR;
  static constexpr int NHW = (ITEMS + 31) / 32;
  static constexpr int THREADS = 32 * (NVW + NHW + NRW);
};

__host__ __device__ inline int vxp(int r) { return (TX + 2 * r) | 1; }
__host__ __device__ inline size_t smem_bytes(int NC, int r, int lp) {
  return (size_t)nsums(NC, lp) * RB * (NBV * vxp(r) + NBH * TXP) * sizeof(double) + 64 * sizeof(uint64_t);
}

__device__ __forceinline__ void bwait(uint64_t* bar, unsigned parity) {
  while (!cuda::ptx::mbarrier_try_wait_parity(bar, parity, uint32_t(kMbarSuspendNs))) {
  }
}
__device__ __forceinline__ void barrive(uint64_t* bar) {
  (void)cuda::ptx::mbarrier_arrive(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared, bar);
}

template <int NC, int LP, int RT>
__global__ void __launch_bounds__(Cfg<NC, LP>::THREADS, 1)
    k_stats5(const float* __restrict__ G, float* __restrict__ stats, int W, int H, int r_arg, double lam, int mode,
             int aos, float lam0f, int yb0, int yb1, int BH, const float* __restrict__ P, float* __restrict__ wout,
             WLayout wo) {
  using C = Cfg<NC, LP>;
  const int r = RT > 0 ? RT : r_arg;
  constexpr int K = NC + 1, NG = npair(NC), NPAIR = C::NPAIR, NHW = C::NHW;
  extern __shared__ __align__(16) double sd[];
  const int VXP = vxp(r);
  double* vs = sd;                                       // [NBV][RB][NPAIR][VXP]
  double* hs = vs + NBV * RB * NPAIR * VXP;              // [NBH][RB][NPAIR][TXP]
  uint64_t* bars = reinterpret_cast<uint64_t*>(hs + NBH * RB * NPAIR * TXP);
  uint64_t* vfull = bars;                                // V wrote slot (NVW warps)
  uint64_t* vfree = vfull + NBV;                         // H done reading slot (NHW warps)
  uint64_t* hfull = vfree + NBV;                         // H wrote slot (NHW warps)
  uint64_t* hfree = hfull + NBH;                         // R read slot (NRW warps)
  const int tid = threadIdx.x, wq = tid >> 5, ln = tid & 31;
  const long long HW = (long long)H * W;
  // persistent CTAs: work item = (strip, band), strips fastest, items blockIdx.x, + gridDim.x, ...; every role walks
  // the same items, and the slot counter jg runs on across items, so a CTA's vertical warps start the next band's
  // warm-up while its horizontal / recursion warps finish the last one
  const int strips = (W + TX - 1) / TX;
  const int band0 = yb0 / BH, nbands = (yb1 + BH - 1) / BH - band0;
  const int nitems = strips * nbands;
  struct Item { int x0, Y0, Z0, Z1, nit, it0; };
  auto item_of = [&](int it_) {
    Item I;
    I.x0 = (it_ % strips) * TX;
    I.Y0 = (band0 + it_ / strips) * BH;
    const int Y1 = min(H, I.Y0 + BH);
    I.Z0 = max(I.Y0, yb0);
    I.Z1 = min(Y1, yb1);                                 // rows written
    // iterations yb = Y0 + it * RB while yb < Z1; those with yb + RB <= Z0 (rows before the requested range) are
    // vertical-only; the others go through the slots
    I.nit = I.Z1 > I.Y0 ? (I.Z1 - I.Y0 + RB - 1) / RB : 0;
    I.it0 = I.Z0 > I.Y0 ? (I.Z0 - I.Y0) / RB : 0;
    return I;
  };

  if (tid == 0) {
    for (int s = 0; s < NBV; ++s) {
      cuda::ptx::mbarrier_init(&vfull[s], NVW);
      cuda::ptx::mbarrier_init(&vfree[s], NHW);
    }
    for (int s = 0; s < NBH; ++s) {
      cuda::ptx::mbarrier_init(&hfull[s], NHW);
      cuda::ptx::mbarrier_init(&hfree[s], NRW);
    }
    cuda::ptx::fence_mbarrier_init(cuda::ptx::sem_release, cuda::ptx::scope_cluster);
  }
  __syncthreads();

  if (wq < NVW) {
    // ---- V warps: column c of the strip (image x = x0 - r + c)
    const int c = tid;
    const int CX = TX + 2 * r;
    const bool vcol = c < CX;
    int jg = 0;
    for (int itm = blockIdx.x; itm < nitems; itm += gridDim.x) {
      const Item I = item_of(itm);
      const int Y0 = I.Y0, nit = I.nit, it0 = I.it0;
      const int vx = I.x0 - r + c;
      const bool xin = vcol && vx >= 0 && vx < W;
      auto load_row = [&](int yy, float (&v)[K + LP]) {
        const bool in = xin && yy >= 0 && yy < H;
        v[0] = in ? 1.0f : 0.0f;
        const float* src = G + (long long)yy * W + vx;
#pragma unroll
        for (int k = 1; k < K; ++k) v[k] = in ? __ldg(src + (k - 1) * HW) : 0.0f;
        if (LP) v[K] = in ? __ldg(P + (long long)yy * W + vx) : 0.0f;
      };
      double acc[NPAIR];
#pragma unroll
      for (int q = 0; q < NPAIR; ++q) acc[q] = 0.0;
      // warm-up: the window of output row Y0 - 1 (rows Y0 - 1 - r .. Y0 - 1 + r)
      if (vcol) {
        for (int yy = Y0 - 1 - r; yy <= Y0 - 1 + r; ++yy) {
          float e[K + LP];
          load_row(yy, e);
          int q = 0;
#pragma unroll
          for (int a = 0; a < K; ++a)
#pragma unroll
            for (int b = a; b < K; ++b) {
              if (a == 0 && b == 0) continue;
              acc[q] = fma((double)e[a], (double)e[b], acc[q]);
              ++q;
            }
          if constexpr (LP == 1) {
#pragma unroll
            for (int a = 0; a < K; ++a) acc[NG + a] = fma((double)e[a], (double)e[K], acc[NG + a]);
          }
        }
      }
      float en[RB][K + LP], lnx[RB][K + LP];
      if (vcol && nit > 0) {
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          load_row(Y0 + rb + r, en[rb]);
          load_row(Y0 + rb - r - 1, lnx[rb]);
        }
      }
      for (int it = 0; it < nit; ++it) {
        const int yb = Y0 + it * RB;
        const bool slot = it >= it0;
        float e[RB][K + LP], l[RB][K + LP];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb)
#pragma unroll
          for (int a = 0; a < K + LP; ++a) {
            e[rb][a] = en[rb][a];
            l[rb][a] = lnx[rb][a];
          }
        if (vcol && it + 1 < nit) {
#pragma unroll
          for (int rb = 0; rb < RB; ++rb) {
            load_row(yb + RB + rb + r, en[rb]);
            load_row(yb + RB + rb - r - 1, lnx[rb]);
          }
        }
        const int sv = jg % NBV;
        double* dstb = vs + (size_t)sv * RB * NPAIR * VXP;
        if (slot && jg >= NBV) bwait(&vfree[sv], (jg / NBV - 1) & 1);
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          if (vcol) {
            int q = 0;
#pragma unroll
            for (int a = 0; a < K; ++a)
#pragma unroll
              for (int b = a; b < K; ++b) {
                if (a == 0 && b == 0) continue;
                acc[q] = fma((double)e[rb][a], (double)e[rb][b], fma(-(double)l[rb][a], (double)l[rb][b], acc[q]));
                ++q;
              }
            if constexpr (LP == 1) {
#pragma unroll
              for (int a = 0; a < K; ++a)
                acc[NG + a] =
                    fma((double)e[rb][a], (double)e[rb][K], fma(-(double)l[rb][a], (double)l[rb][K], acc[NG + a]));
            }
            if (slot) {
              double* dst = dstb + rb * NPAIR * VXP + c;
#pragma unroll
              for (int q2 = 0; q2 < NPAIR; ++q2) dst[q2 * VXP] = acc[q2];
            }
          }
        }
        if (slot) {
          __syncwarp();
          if (ln == 0) barrive(&vfull[sv]);
          ++jg;
        }
      }
    }
    return;
  }

  if (wq < NVW + NHW) {
    // ---- H warps: item t = (row rb, 32-pixel segment, pair q), pairs fastest
    const int t = tid - 32 * NVW;
    const bool act = t < C::ITEMS;
    const int q = t % NPAIR, sg = (t / NPAIR) % (TX / HS), rb = t / (NPAIR * (TX / HS));
    int j = 0;
    for (int itm = blockIdx.x; itm < nitems; itm += gridDim.x) {
     const Item I = item_of(itm);
     for (int jj0 = I.it0; jj0 < I.nit; ++jj0, ++j) {
      const int sv = j % NBV, sh = j % NBH;
      bwait(&vfull[sv], (j / NBV) & 1);
      if (j >= NBH) bwait(&hfree[sh], (j / NBH - 1) & 1);
      if (act) {
        const double* v = vs + (size_t)sv * RB * NPAIR * VXP + (rb * NPAIR + q) * VXP + sg * HS;
        double* o = hs + (size_t)sh * RB * NPAIR * TXP + (rb * NPAIR + q) * TXP + sg * HS;
        double a = 0.0;
        for (int jj = 0; jj <= 2 * r; ++jj) a += v[jj];
        o[0] = a;
#pragma unroll
        for (int i = 1; i < HS; ++i) {
          a += v[i + 2 * r] - v[i - 1];
          o[i] = a;
        }
      }
      __syncwarp();
      if (ln == 0) {
        barrive(&vfree[sv]);
        barrive(&hfull[sh]);
      }
     }
    }
    return;
  }

  // ---- R warps: pixel (rb, x) of each iteration
  const int p = tid - 32 * (NVW + NHW);
  const int rb = p / TX, x = p % TX;
  int j = 0;
  for (int itm = blockIdx.x; itm < nitems; itm += gridDim.x) {
   const Item I = item_of(itm);
   for (int it = I.it0; it < I.nit; ++it, ++j) {
    const int sh = j % NBH;
    bwait(&hfull[sh], (j / NBH) & 1);
    double g[NPAIR];
    const double* src = hs + (size_t)sh * RB * NPAIR * TXP + rb * NPAIR * TXP + x;
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) g[q] = src[q * TXP];
    __syncwarp();
    if (ln == 0) barrive(&hfree[sh]);
    const int gy = I.Y0 + it * RB + rb, gx = I.x0 + x;
    if (gy >= I.Z0 && gy < I.Z1 && gx < W) {
      const double N = (double)window_count(gy, gx, H, W, r);
      if constexpr (LP == 1) {
        float* wl = wout + wo.origin + (long long)gy * wo.pitch + gx;
        if (mode == 0) filter_finish_m<NC, 0>(g, N, lam, lam0f, wl, wo.plane);
        else filter_finish_m<NC, 1>(g, N, lam, lam0f, wl, wo.plane);
      } else {
        stats_finish<NC>(g, N, lam, mode, aos, lam0f, stats, (long long)gy * W + gx, HW);
      }
    }
   }
  }
}

// Same contract and band rule as st4::stats4_launch_r (bit-identical output); r <= 16.
template <int NC, int LP, int RT>
cudaError_t stats5_launch_r(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos,
                            float lam0f, int y0, int y1, const float* P, float* wout, WLayout wo, cudaStream_t st) {
  using C = Cfg<NC, LP>;
  if (aos && NC > kCoef3MaxN) return cudaErrorInvalidValue;
  if (TX + 2 * r > 32 * NVW) return cudaErrorInvalidValue;
  const size_t smem = smem_bytes(NC, r, LP);
  cudaError_t e = cudaFuncSetAttribute(k_stats5<NC, LP, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (y0 >= y1) return cudaSuccess;
  // LP = 0 (statistics, possibly row-sharded): k_stats4's band rule (the same bands whichever rows are requested);
  // LP = 1 (one whole frame): one CTA per SM, so the band count minimising waves x (band + warm-up rows)
  int BH = st4::band_height(W, H);
  if (LP == 1 && !std::getenv("HGF_STATS4_BH")) {
    const int strips = (W + TX - 1) / TX;
    long long best = -1;
    for (int nb = 1; nb <= (H + 31) / 32; ++nb) {
      const int bh = (H + nb - 1) / nb;
      const long long ctas = (long long)strips * ((H + bh - 1) / bh);
      const long long cost = (ctas + 147) / 148 * (bh + 2 * r + 1);
      if (best < 0 || cost < best) { best = cost; BH = bh; }
    }
  }
  const long long items = (long long)((W + TX - 1) / TX) * ((y1 + BH - 1) / BH - y0 / BH);
  int nsm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  dim3 grid((unsigned)(items < nsm ? items : nsm));     // persistent: one CTA per SM walking the work items
  k_stats5<NC, LP, RT><<<grid, C::THREADS, smem, st>>>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, BH, P, wout,
                                                      wo);
  return cudaGetLastError();
}

// Statistics of rows [y0, y1) (the st4::stats4_impl contract): k_stats5 for n <= 6 and r <= 16 (HGF_STATS5=0: k_stats4).
// k_stats5 only on request here (HGF_STATS5=1): at C4 its one CTA per SM loses to k_stats4's three (0.88 vs 0.84 ms
// at its best band height), while for the fused single-slice pass below it wins (C5: 0.33 -> 0.24 ms).
template <int NC>
cudaError_t stats_sel(const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos, float lam0f,
                      int y0, int y1, cudaStream_t st) {
  const char* e = std::getenv("HGF_STATS5");
  if (NC <= 6 && r <= 16 && (e && e[0] == '1')) {
    if (r == 9)
      return stats5_launch_r<NC, 0, 9>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, nullptr, nullptr, WLayout{},
                                       st);
    return stats5_launch_r<NC, 0, 0>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, nullptr, nullptr, WLayout{}, st);
  }
  return st4::stats4_impl<NC>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
}

// hgf_filter's fused single-slice pass (the st4::filter1_impl contract), k_stats5 where it applies.
template <int NC>
cudaError_t filter1_sel(const float* G, const float* P, float* wout, WLayout wo, int W, int H, int r, double lam,
                        int mode, float lam0f, cudaStream_t st) {
  // n = 6 (C5: 0.33 -> 0.24 ms; n = 5 even, 0.21 both); for fewer channels k_stats4's many small CTAs per SM win (n = 3: 0.12 vs
  // 0.19 ms, n = 1: 0.054 vs 0.080 ms)
  const char* e = std::getenv("HGF_STATS5");
  if (NC == 6 && r <= 16 && !(e && e[0] == '0')) {
    if (r == 9) return stats5_launch_r<NC, 1, 9>(G, nullptr, W, H, r, lam, mode, 0, lam0f, 0, H, P, wout, wo, st);
    return stats5_launch_r<NC, 1, 0>(G, nullptr, W, H, r, lam, mode, 0, lam0f, 0, H, P, wout, wo, st);
  }
  return st4::filter1_impl<NC>(G, P, wout, wo, W, H, r, lam, mode, lam0f, st);
}

}  // namespace st5
}  // namespace hgf
