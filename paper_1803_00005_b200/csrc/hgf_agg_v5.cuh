// HGF per-slice aggregation + WTA, version 5 (k_agg5<n, R>): row marching with the vertical window in registers.
//
// Per slice l (Eq14 P:328-333 == Eq8):  Z = (B(w_0) + sum_k G_k B(w_k)) / N, then the running WTA
// (ties -> lowest label).  B is separable; here the horizontal sums come first and the vertical window is
// a register ring:
//   Hw_k(j, x) = sum_{|dx| <= R} w_k(j, x + dx)                     (H warps, from the TMA'd coefficient row)
//   T_k(y, x)  = T_k(y - 1, x) + Hw_k(y + R, x) - Hw_k(y - R - 1, x) (V warps; Hw(y - R - 1) is the ring slot
//                                                                      the entering Hw(y + R) overwrites)
// so every coefficient value crosses shared memory once (TMA write, one read), every horizontal sum once (one
// write, one read), and nothing is re-read for the vertical pass.  k_agg3 instead filters 64 x 24 tiles whose
// 2R-row vertical halos are fetched and summed again for every tile (2.2x the coefficient traffic at R = 9).
//
// A CTA owns a strip of TX = 64 output columns x a band of rows x a group of labels, and marches the band once
// per batch of LB = 4 labels:
//   * one elected thread keeps a 3-stage TMA ring full: per step the entering coefficient row (4 labels x
//     K planes x 96 columns, one box of the label-interleaved layout, 64-byte swizzle) and the guidance row of
//     the output row;
//   * H warps (thread = label x plane x 16-pixel segment): slide the 2R+1 window along the row, write Hw into a
//     double-buffered row [K][4][72] (named barriers FULL/EMPTY);
//   * V warps (thread = label x pixel, lanes = 4 labels x 8 pixels): the ring of 2R+1 Hw rows per plane and
//     the window sums T in registers (the step loop is unrolled 2R+1 times so the ring index is static), Z,
//     then the batch minimum over the 4 labels by shuffles and the band's running minimum key per pixel in
//     shared memory; at the end one 64-bit atomic MIN per pixel into the frame's key buffer.
#pragma once
#include <cuda.h>

#include <cstdlib>

#include <cuda/ptx>

#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace v5a {

constexpr int TX = 64;                 // output columns per strip
constexpr int LB = 4;                  // labels per batch
constexpr int XG = 6;                  // 16-pixel groups per coefficient row (covers [x0 - 16, x0 + 80))
constexpr int HP = 72;                 // Hw row pitch per (plane, label): 72 = 8 mod 32 (conflict-free V reads)
constexpr int NST = 4;                 // TMA ring depth (refills two steps behind the H warps)
constexpr int NHB = 3;                 // Hw row buffers (H warps run up to two steps ahead of the V warps)
constexpr int NHW = 4, NVW = 8;        // H warps, V warps
constexpr int THREADS = (NHW + NVW) * 32;
constexpr int MAXBAND = 288;
constexpr int BAR_FULL = 1, BAR_EMPTY = 4, BAR_V = 7;   // named barriers 1-3 (FULL), 4-6 (EMPTY), 7 (V only)

template <int NC>
struct Geom {
  static constexpr int K = NC + 1;
  static constexpr int WROW = K * XG * LB * 16;                 // floats of one coefficient row box
  static constexpr int GROW = (NC > 0 ? NC : 1) * TX;          // guidance row of the output row
  static constexpr int STAGE = (WROW + GROW + 255) / 256 * 256;  // 1 KB aligned (64-byte swizzle)
  static constexpr int HROW = K * LB * HP;
  static constexpr size_t SMEM = sizeof(float) * ((size_t)NST * STAGE + NHB * (size_t)HROW) +
                                 sizeof(long long) * (size_t)MAXBAND * TX + 256 + 1024;
  static_assert(K <= 8, "H threads cover up to 8 planes");
};

__device__ __forceinline__ void nsync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void narrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// SMEM float index of element (plane k, group g, label j, pixel c) of a coefficient row box: the box is
// (16 px, LB labels, XG groups, 1 row, K planes) with the 64-byte swizzle (16-byte chunk q of 64-byte row r
// stored at q ^ ((r >> 1) & 3); rows r = j + LB (g + XG k)).
__device__ __forceinline__ int wbox_idx(int k, int g, int j, int c) {
  const int r = j + LB * (g + XG * k);
  return r * 16 + ((((c >> 2) ^ ((r >> 1) & 3))) << 2) + (c & 3);
}

template <int NC, int R>
__global__ void __launch_bounds__(THREADS, 1)
    k_agg5(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_g, int W, int H, int L,
           int label_base, int labels_per_cta, int BH, unsigned long long* __restrict__ keys,
           float* __restrict__ filtered_out) {
  using Gm = Geom<NC>;
  constexpr int K = Gm::K, RL = 2 * R + 1;
  extern __shared__ __align__(1024) float sm[];
  float* hrow = sm + NST * Gm::STAGE;                                   // [NHB][K][LB][HP]
  long long* best = reinterpret_cast<long long*>(hrow + NHB * Gm::HROW);  // [BH][TX] running minimum keys
  uint64_t* bar = reinterpret_cast<uint64_t*>(best + MAXBAND * TX);     // full[NST], empty[NST]
  uint64_t* empty = bar + NST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int x0 = blockIdx.x * TX;
  const int Y0 = blockIdx.y * BH, Y1 = min(H, Y0 + BH), bh = Y1 - Y0;
  const int la = blockIdx.z * labels_per_cta, lz = min(L, la + labels_per_cta);
  const int nbatch = (lz - la + LB - 1) / LB;
  const int nsteps = bh + 2 * R;                 // entering rows Y0 - R .. Y1 - 1 + R
  const int total = nbatch * nsteps;             // the TMA ring runs across batches
  const long long HW = (long long)W * H;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      cuda::ptx::mbarrier_init(&bar[s], 1);
      cuda::ptx::mbarrier_init(&empty[s], NHW + NVW);   // H warps read the w row, V warps the G row
    }
    cuda::ptx::fence_mbarrier_init(cuda::ptx::sem_release, cuda::ptx::scope_cluster);
  }
  for (int e = tid; e < bh * TX; e += THREADS) best[e] = LLONG_MAX;
  __syncthreads();

  // global step q = b * nsteps + t: batch b, entering row ye = Y0 - R + t, output row ye - R (t >= 2R)
  auto issue = [&](int q) {
    const int b = q / nsteps, t = q - b * nsteps;
    float* s = sm + (q % NST) * Gm::STAGE;
    const int l = la + b * LB;                   // first label of the batch (4 | 32: one group of the layout)
    const int ye = Y0 - R + t, y = ye - R;
    const bool out = t >= 2 * R;
    cuda::ptx::mbarrier_arrive_expect_tx(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared,
                                         &bar[q % NST], (unsigned)(Gm::WROW + (out ? NC * TX : 0)) * 4u);
    const int32_t cw[5] = {0, l % kWGroupLabels, (x0 >> 4) - 1, ye, (l / kWGroupLabels) * K};
    cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, s, &tm_w, cw, &bar[q % NST]);
    if (out && NC > 0) {
      const int32_t cg[3] = {x0, y, 0};
      cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, s + Gm::WROW, &tm_g, cg,
                                      &bar[q % NST]);
    }
  };

  if (warp < NHW) {
    // ===================== H warps: thread = (label j, plane k, segment s) =====================
    // 4 labels x 8 planes x 4 segments; a quarter-warp = 4 labels x 2 segments (adjacent groups: distinct
    // swizzled 16-byte slots, conflict-free box reads)
    const int j = lane & 3, s = 2 * (warp & 1) + ((lane >> 2) & 1), k = 4 * (warp >> 1) + (lane >> 3);
    if (tid == 0)
      for (int q = 0; q < NST && q < total; ++q) issue(q);
    for (int q = 0; q < total; ++q) {
      // refill: the stage of step q - 2 (released by every warp once it finished that step) for step q + 2
      if (tid == 0 && q >= 2 && q + 2 < total) {
        while (!cuda::ptx::mbarrier_try_wait_parity(&empty[(q - 2) % NST], ((q - 2) / NST) & 1)) {
        }
        issue(q + 2);
      }
      const float* st = sm + (q % NST) * Gm::STAGE;
      while (!cuda::ptx::mbarrier_try_wait_parity(&bar[q % NST], (q / NST) & 1)) {
      }
      const int hb = q % NHB;
      if (q >= NHB) nsync(BAR_EMPTY + hb, THREADS);                  // V warps done with Hw buffer hb
      if (k < K) {
        // window columns of output pixel i = 16 s + c: box columns [i + 16 - R, i + 16 + R]
        float v[48];
#pragma unroll
        for (int g = 0; g < 3; ++g)
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 f = *reinterpret_cast<const float4*>(st + wbox_idx(k, s + g, j, 4 * c4));
            v[16 * g + 4 * c4] = f.x; v[16 * g + 4 * c4 + 1] = f.y; v[16 * g + 4 * c4 + 2] = f.z;
            v[16 * g + 4 * c4 + 3] = f.w;
          }
        // two independent 8-pixel slides (starting sums as pairwise trees): short dependency chains
        float o[16];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          float part[2 * R + 1];
#pragma unroll
          for (int d = 0; d <= 2 * R; ++d) part[d] = v[8 * h2 + 16 - R + d];
#pragma unroll
          for (int w = 1; w <= 2 * R; w *= 2)
#pragma unroll
            for (int d = 0; d + w <= 2 * R; d += 2 * w) part[d] += part[d + w];
          float acc = part[0];
          o[8 * h2] = acc;
#pragma unroll
          for (int c = 1; c < 8; ++c) {
            acc += v[8 * h2 + c + 16 + R] - v[8 * h2 + c + 15 - R];
            o[8 * h2 + c] = acc;
          }
        }
        float* dst = hrow + hb * Gm::HROW + (k * LB + j) * HP + 16 * s;
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4)
          *reinterpret_cast<float4*>(dst + 4 * c4) = make_float4(o[4 * c4], o[4 * c4 + 1], o[4 * c4 + 2], o[4 * c4 + 3]);
      }
      narrive(BAR_FULL + hb, THREADS);
      __syncwarp();
      if (lane == 0) cuda::ptx::mbarrier_arrive(&empty[q % NST]);
    }
    return;
  }

  // ===================== V warps: thread = (label j, pixel px); lanes = 4 labels x 8 pixels =====================
  const int v = tid - NHW * 32;
  const int j = (v & 31) >> 3;                  // label within the batch
  const int px = ((v >> 5) << 3) | (v & 7);     // 0..63
  const int gx = x0 + px;
  const bool xin = gx < W;
  float ring[K][RL];
  float T[K];
  for (int q0 = 0; q0 < total; q0 += RL) {
#pragma unroll
    for (int u = 0; u < RL; ++u) {
      const int q = q0 + u;
      if (q >= total) break;
      const int b = q / nsteps, t = q - b * nsteps;
      if (t == 0) {
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          T[kk] = 0.0f;
#pragma unroll
          for (int uu = 0; uu < RL; ++uu) ring[kk][uu] = 0.0f;
        }
      }
      // ring slot u = q mod RL: the value leaving at step q (row ye - RL) was written at step q - RL into the
      // same slot; the slots are zeroed at each batch start, so the first RL steps subtract zeros
      const int hb = q % NHB;
      nsync(BAR_FULL + hb, THREADS);
      const float* hr = hrow + hb * Gm::HROW + j * HP + px;
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const float hw = hr[kk * LB * HP];
        T[kk] += hw - ring[kk][u];
        ring[kk][u] = hw;
      }
      narrive(BAR_EMPTY + hb, THREADS);
      const int y = Y0 - 2 * R + t;
      if (t >= 2 * R && y < Y1) {
        const float* gr = sm + (q % NST) * Gm::STAGE + Gm::WROW;
        float z = T[0];
#pragma unroll
        for (int kk = 0; kk < NC; ++kk) z = fmaf(gr[kk * TX + px], T[kk + 1], z);
        const int l = la + b * LB + j;                 // label within the chunk (slice index of w)
        const bool ok = xin && l < lz;
        z = z / (float)window_count(y, gx, H, W, R);
        if (filtered_out && ok) filtered_out[(long long)l * HW + (long long)y * W + gx] = z;
        unsigned long long key =
            ok ? ((unsigned long long)orderable_bits(z) << 32) | (unsigned)(label_base + l) : ~0ull;
        unsigned long long o = __shfl_xor_sync(0xffffffffu, key, 8);
        key = o < key ? o : key;
        o = __shfl_xor_sync(0xffffffffu, key, 16);
        key = o < key ? o : key;
        if (j == 0) {
          long long* bp = best + (y - Y0) * TX + px;
          const long long ks = (long long)(key ^ 0x8000000000000000ull);
          if (ks < *bp) *bp = ks;
        }
      }
      __syncwarp();
      if (lane == 0) cuda::ptx::mbarrier_arrive(&empty[q % NST]);   // done with this stage's guidance row
    }
  }
  // the band's minima -> the frame's key buffer (signed order: key ^ 2^63, hgf.h)
  asm volatile("bar.sync %0, %1;" ::"r"(BAR_V), "r"(NVW * 32) : "memory");
  for (int e = v; e < bh * TX; e += NVW * 32) {
    const int yy = e / TX, xx = e % TX;
    if (x0 + xx < W && best[e] != LLONG_MAX)
      atomicMin(reinterpret_cast<long long*>(keys) + (long long)(Y0 + yy) * W + x0 + xx, best[e]);
  }
}

}  // namespace v5a
}  // namespace hgf

namespace hgf {
namespace v5a {

template <int NC, int R>
cudaError_t agg5_r(const void* tm_w, const void* tm_g, int W, int H, int L, int label_base, int labels_per_cta,
                   unsigned long long* keys, float* filtered_out, cudaStream_t st) {
  using Gm = Geom<NC>;
  cudaError_t e = cudaFuncSetAttribute(k_agg5<NC, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::SMEM);
  if (e != cudaSuccess) return e;
  // bands (<= MAXBAND rows: the best-key rows live in shared memory) and label groups: one CTA per SM; a
  // band of BH rows costs (BH + 2R) steps per batch of 4 labels.  Pick the band count minimising
  // waves x (BH + 2R) among those giving >= 4 waves (or the most CTAs for small frames).
  const int strips = (W + TX - 1) / TX;
  const int groups = (L + labels_per_cta - 1) / labels_per_cta;
  int BH = H < MAXBAND ? H : MAXBAND;
  {
    long long best = -1;
    const int nbmin = (H + MAXBAND - 1) / MAXBAND, nbmax = H / 16 > nbmin ? H / 16 : nbmin;
    const long long most = (long long)strips * nbmax * groups;
    const long long target = most < 4 * 148 ? most : 4 * 148;
    for (int nb = nbmin; nb <= nbmax; ++nb) {
      const int bh = (H + nb - 1) / nb;
      const long long ctas = (long long)strips * ((H + bh - 1) / bh) * groups;
      if (ctas < target) continue;
      const long long cost = (ctas + 147) / 148 * (bh + 2 * R);
      if (best < 0 || cost < best) { best = cost; BH = bh; }
    }
  }
  const int bh_env = std::getenv("HGF_AGG5_BH") ? std::atoi(std::getenv("HGF_AGG5_BH")) : 0;
  if (bh_env >= 8 && bh_env <= MAXBAND) BH = bh_env;
  dim3 grid(strips, (H + BH - 1) / BH, groups);
  k_agg5<NC, R><<<grid, THREADS, Gm::SMEM, st>>>(*reinterpret_cast<const CUtensorMap*>(tm_w),
                                                 *reinterpret_cast<const CUtensorMap*>(tm_g), W, H, L, label_base,
                                                 labels_per_cta, BH, keys, filtered_out);
  return cudaGetLastError();
}

template <int NC>
cudaError_t agg5_impl(const void* tm_w, const void* tm_g, int W, int H, int r, int L, int label_base,
                      int labels_per_cta, unsigned long long* keys, float* filtered_out, cudaStream_t st) {
  switch (r) {
    case 1: return agg5_r<NC, 1>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 2: return agg5_r<NC, 2>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 3: return agg5_r<NC, 3>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 4: return agg5_r<NC, 4>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 5: return agg5_r<NC, 5>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 6: return agg5_r<NC, 6>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 7: return agg5_r<NC, 7>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 8: return agg5_r<NC, 8>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 9: return agg5_r<NC, 9>(tm_w, tm_g, W, H, L, label_base, labels_per_cta, keys, filtered_out, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace v5a
}  // namespace hgf
