// HGF per-slice aggregation + WTA, version 3 (k_agg3<n, R>): TMA-fed, compile-time radius.
//
// Per slice l and 64x24 output tile:  Z = (B(w_0) + sum_k G_k B(w_k)) / N   (Eq14 P:328-333 == Eq8),
// running WTA min/argmin in registers (ties -> lowest label).
//
// Data movement (the binding resource is the SM's ~128 B/clk shared-memory data path, measured in
// profiles/r01_microbench2.txt):
//   * one cp.async.bulk.tensor (TMA) per slice brings the K = n+1 planes of w for the tile plus an
//     R halo into SMEM (coefficient buffer rows pitched to 16 bytes).  TMA's out-of-bounds zero fill on
//     all four sides implements the clipped windows (F6).  The tile grid is shifted so that every
//     TMA x coordinate is 16-byte aligned: unaligned x offsets trap on this B200 stack
//     (tools/tma_test2.cu);
//     the next slice's TMA is issued before this slice's passes (double buffer, mbarrier-tracked);
//   * vertical pass in place: each (plane, column) item loads its column into registers once and
//     writes the 2R+1-row window sums back over the first TY rows;
//   * horizontal pass + Z + WTA by owner threads (one row x 8 pixels each) that keep G, 1/N and the
//     running (min, argmin) in registers; 128-bit shared loads, conflict-free by construction
//     (8 lanes of a quarter-warp read 8 different rows; the row pitch BX has BX/4 odd).
//
// IL = true reads the label-interleaved coefficient layout written by k_coef3 (WLayout::il): a rank-5
// tensor map (16 px, 32 labels, x groups, y, planes) with box (16, 1, BX/16, BY, K) lands the same
// [k][y][x] tile (BX a multiple of 32) with the 64-byte TMA swizzle: the 16-byte chunk c of 64-byte row
// R sits at chunk c ^ ((R >> 1) & 3), i.e. float index f -> f ^ ((f >> 3) & 12).  The swizzle keeps both
// passes conflict-free without a padded pitch; owners then map a quarter-warp to 4 rows x 2 segments that
// are 16 pixels apart (tools/swizzle_banks.py checks every access pattern).
#pragma once
#include <cuda.h>

#include <cuda/ptx>

#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace v3 {

constexpr int TX = 64, TY = 24, KX = 8, NSEG = TX / KX, THREADS = 256, NOWN = TY * NSEG;

__host__ __device__ constexpr int box_pitch(int wx) {
  int b = (wx + 3) / 4 * 4;
  while (((b / 4) & 1) == 0) b += 4;  // BX/4 odd -> quarter-warp 16-B loads from 8 rows hit distinct banks
  return b;
}

template <int NC, int R, bool IL = false>
struct AggGeom {
  static constexpr int K = NC + 1;
  static constexpr int WX = TX + 2 * R;
  static constexpr int BX = IL ? (WX + 31) / 32 * 32 : box_pitch(WX);   // IL: whole 128-B rows
  static constexpr int BY = TY + 2 * R;
  static constexpr int PLANE = BY * BX;                    // floats per plane in SMEM
  static constexpr int LABEL_FLOATS = K * PLANE;                 // bytes landed by one slice's TMA / 4
  static constexpr int BUF_STRIDE = (LABEL_FLOATS + 31) / 32 * 32; // keeps every TMA destination 128-B aligned
  // one slice buffer per CTA and two CTAs per SM: the co-resident CTA hides this one's TMA wait
  static constexpr int NBUF = 1;
  static constexpr int NV4 = (KX + 2 * R + 3) / 4;        // 128-bit loads per owner row segment
  static_assert(KX * (NSEG - 1) + 4 * NV4 <= BX, "owner loads stay inside the row");
  static_assert(BX <= 256 && BY <= 256, "TMA box limits");
  static_assert(!IL || (NBUF == 1 && (BX % 16) == 0), "swizzled tile: one 1024-B aligned buffer");
};

// SMEM float index of logical tile element f under the 64-byte TMA swizzle (identity without it).
template <bool IL>
__device__ __forceinline__ int swz(int f) {
  return IL ? (f ^ ((f >> 3) & 12)) : f;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// mbarrier / TMA wrappers over libcu++'s cuda::ptx (PTX ISA 8.0+, sm_90+).
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) { cuda::ptx::mbarrier_init(bar, count); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  cuda::ptx::mbarrier_arrive_expect_tx(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared, bar,
                                       bytes);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!cuda::ptx::mbarrier_try_wait_parity(bar, parity)) {
  }
}
__device__ __forceinline__ void fence_barrier_init() {
  cuda::ptx::fence_mbarrier_init(cuda::ptx::sem_release, cuda::ptx::scope_cluster);
}
__device__ __forceinline__ void fence_proxy_async() { cuda::ptx::fence_proxy_async(cuda::ptx::space_shared); }
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
  const int32_t c[3] = {x, y, z};
  cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, dst, tm, c, bar);
}

template <int NC, int R, bool IL>
__global__ void __launch_bounds__(THREADS, 2)
    k_agg3(const __grid_constant__ CUtensorMap tmw, const float* __restrict__ G, int W, int H, int pad, int L, int label_base,
           float* __restrict__ filtered_out, int do_wta, int first, int last, float* __restrict__ best_cost,
           int32_t* __restrict__ best_label, int32_t* __restrict__ labels_out, float* __restrict__ min_cost_out,
           int64_t* __restrict__ keys_out) {
  using Gm = AggGeom<NC, R, IL>;
  constexpr int K = Gm::K, BX = Gm::BX, BY = Gm::BY, PLANE = Gm::PLANE, NBUF = Gm::NBUF, NV4 = Gm::NV4;
  constexpr unsigned BYTES = Gm::LABEL_FLOATS * 4u;
  // Dynamic SMEM: NBUF slice buffers (each BUF_STRIDE floats, 128-B aligned) followed by the mbarriers.
  // Indexing the __shared__ array directly keeps every access in the shared state space (LDS/STS).
  extern __shared__ __align__(1024) float buf[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + NBUF * Gm::BUF_STRIDE);
  const int tid = threadIdx.x;
  // Tiles start at x0 = 64*bx - XSHIFT so that the TMA x coordinate x0 - R is a multiple of 4 (16 bytes):
  // TMA traps on x offsets that are not 16-byte aligned (tools/tma_test2.cu); negative coordinates and
  // the out-of-bounds zero fill are fine, and implement the clipped windows.
  constexpr int XALIGN = IL ? 16 : 4;   // IL: x groups of 16 pixels
  constexpr int XSHIFT = (XALIGN - R % XALIGN) % XALIGN;
  // Grouped tile order: consecutive CTAs walk down a column of GY tiles before moving right, so the ~148
  // CTAs resident at once cover a compact ~12 x 12-tile block and the R-halos they share (the coefficient
  // tiles overlap by 2R) are L2 hits instead of repeated HBM reads (ncu r01: 1.64x re-read with row order).
  constexpr int GY = 12;
  int tile_x, tile_y;
  {
    const int id = blockIdx.y * gridDim.x + blockIdx.x;
    const int per_group = GY * gridDim.x;
    const int first = (id / per_group) * GY;
    const int rows = min(GY, (int)gridDim.y - first);
    const int in = id % per_group;
    tile_y = first + in % rows;
    tile_x = in / rows;
  }
  const int x0 = tile_x * TX - XSHIFT, y0 = tile_y * TY;
  const int tx0 = x0 - R + pad, ty0 = y0 - R + pad;   // pad = 0 in the pitched layout
  const long long HW = (long long)H * W;

  if (tid == 0) {
    for (int b = 0; b < NBUF; ++b) mbar_init(&bar[b], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // label l of the chunk: plane coordinate l * K (planar) or group coordinates (l % 32, (l / 32) * K) (IL)
  auto load = [&](float* dst, int l, uint64_t* bb) {
    mbar_expect_tx(bb, BYTES);
    if (IL) {
      const int32_t c[5] = {0, l % kWGroupLabels, tx0 / kWGroupPx, ty0, (l / kWGroupLabels) * K};
      cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, dst, &tmw, c, bb);
    } else {
      tma_load_3d(dst, &tmw, tx0, ty0, l * K, bb);
    }
  };
  if (tid == 0 && L > 0) load(buf, 0, &bar[0]);

  // owner role: row oy, pixels x0 + 8*seg + [0, 8)
  const bool is_owner = tid < NOWN;
  const int wq = tid >> 5, ln = tid & 31;
  // planar: a quarter-warp = 8 rows of one segment (odd BX/4 pitch); IL: 4 rows x segments s, s + 2
  const int oy = IL ? (ln & 3) + 4 * wq : (ln & 7) + 8 * (wq % 3);
  const int seg = IL ? ((ln >> 3) & 1) + 4 * (ln >> 4) + 2 * ((ln >> 2) & 1) : (ln >> 3) + 4 * (wq / 3);
  const int gy = y0 + oy;
  float g[NC > 0 ? NC : 1][KX];
  float invN[KX], best[KX];
  int32_t bl[KX];
#pragma unroll
  for (int j = 0; j < KX; ++j) {
    const int gx = x0 + seg * KX + j;
    const bool in = is_owner && gy < H && gx >= 0 && gx < W;
    const long long p = in ? (long long)gy * W + gx : 0;
#pragma unroll
    for (int k = 0; k < NC; ++k) g[k][j] = in ? __ldg(G + k * HW + p) : 0.0f;
    invN[j] = in ? 1.0f / (float)window_count(gy, gx, H, W, R) : 0.0f;
    best[j] = INFINITY;
    bl[j] = 0;
    if (do_wta && !first && in) {
      best[j] = best_cost[p];
      bl[j] = best_label[p];
    }
  }

#pragma unroll 1
  for (int l = 0; l < L; ++l) {
    const int b = (NBUF == 2) ? (l & 1) : 0;
    const unsigned parity = (NBUF == 2) ? ((l >> 1) & 1) : (l & 1);
    float* lb = buf + b * Gm::BUF_STRIDE;
    mbar_wait(&bar[b], parity);
    if (NBUF == 2 && tid == 0 && l + 1 < L) {           // prefetch the next slice into the other buffer
      fence_proxy_async();
      load(buf + (b ^ 1) * Gm::BUF_STRIDE, l + 1, &bar[b ^ 1]);
    }
    // ---- vertical window sums, in place: rows [0, TY) <- sum of rows [y, y + 2R]
    for (int item = tid; item < K * Gm::WX; item += THREADS) {
      const int k = item / Gm::WX, c = item % Gm::WX;
      const int f0 = k * PLANE + c;
      float col[BY];
#pragma unroll
      for (int y = 0; y < BY; ++y) col[y] = lb[swz<IL>(f0 + y * BX)];
      float acc = 0.0f;
#pragma unroll
      for (int y = 0; y <= 2 * R; ++y) acc += col[y];
      lb[swz<IL>(f0)] = acc;
#pragma unroll
      for (int y = 1; y < TY; ++y) {
        acc += col[y + 2 * R] - col[y - 1];
        lb[swz<IL>(f0 + y * BX)] = acc;
      }
    }
    __syncthreads();
    // ---- horizontal window sums + Z + WTA (owners)
    if (is_owner) {
      float z[KX];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int f0 = k * PLANE + oy * BX + seg * KX;
        float f[4 * NV4];
#pragma unroll
        for (int q = 0; q < NV4; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(lb + swz<IL>(f0 + 4 * q));
          f[4 * q] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
        }
        float acc = 0.0f;
#pragma unroll
        for (int dx = 0; dx <= 2 * R; ++dx) acc += f[dx];
#pragma unroll
        for (int s = 0; s < KX; ++s) {
          if (s > 0) acc += f[s + 2 * R] - f[s - 1];
          if (k == 0) z[s] = acc;
          else z[s] = fmaf(g[k - 1][s], acc, z[s]);
        }
      }
#pragma unroll
      for (int s = 0; s < KX; ++s) {
        const int gx = x0 + seg * KX + s;
        if (gy < H && gx >= 0 && gx < W) {
          const float zz = z[s] * invN[s];
          if (filtered_out) filtered_out[(long long)l * HW + (long long)gy * W + gx] = zz;
          if (zz < best[s]) {
            best[s] = zz;
            bl[s] = label_base + l;
          }
        }
      }
    }
    __syncthreads();
    if (NBUF == 1 && tid == 0 && l + 1 < L) {
      fence_proxy_async();
      load(buf, l + 1, &bar[0]);
    }
  }
  if (!do_wta || !is_owner) return;
#pragma unroll
  for (int s = 0; s < KX; ++s) {
    const int gx = x0 + seg * KX + s;
    if (gy >= H || gx < 0 || gx >= W) continue;
    const long long p = (long long)gy * W + gx;
    if (last) {
      if (labels_out) labels_out[p] = bl[s];
      if (min_cost_out) min_cost_out[p] = best[s];
      if (keys_out) keys_out[p] = pack_key_signed(best[s], bl[s]);
    } else {
      best_cost[p] = best[s];
      best_label[p] = bl[s];
    }
  }
}

template <int NC, int R, bool IL>
size_t agg3_smem_bytes() {
  using Gm = AggGeom<NC, R, IL>;
  return (size_t)Gm::NBUF * Gm::BUF_STRIDE * 4 + 128;
}

template <int NC, int R, bool IL>
cudaError_t agg3_launch(const void* tmap, const AggArgs& a, cudaStream_t st) {
  const size_t smem = agg3_smem_bytes<NC, R, IL>();
  cudaError_t e = cudaFuncSetAttribute(k_agg3<NC, R, IL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  constexpr int XALIGN = IL ? 16 : 4;
  dim3 grid((a.W + (XALIGN - R % XALIGN) % XALIGN + TX - 1) / TX, (a.H + TY - 1) / TY);
  k_agg3<NC, R, IL><<<grid, THREADS, smem, st>>>(*reinterpret_cast<const CUtensorMap*>(tmap), a.G, a.W, a.H, a.pad, a.L,
                                             a.label_base, a.filtered_out, a.do_wta, a.first, a.last, a.best_cost,
                                             a.best_label, a.labels_out, a.min_cost_out, a.keys_out);
  return cudaGetLastError();
}

template <int NC, int R>
cudaError_t agg3_impl(const void* tmap, const AggArgs& a, cudaStream_t st) {
  return a.il ? agg3_launch<NC, R, true>(tmap, a, st) : agg3_launch<NC, R, false>(tmap, a, st);
}

}  // namespace v3
}  // namespace hgf
