// HGF per-slice aggregation + WTA, version 3 (k_agg3<n, R, IL>): TMA-fed, compile-time radius.
//
// Per slice l and 64x24 output tile:  Z = (B(w_0) + sum_k G_k B(w_k)) / N   (Eq14 P:328-333 == Eq8),
// running WTA min/argmin in registers (ties -> lowest label).
//
// Data movement (the binding resource is the SM's L1/shared data pipe, ~1 wavefront per clock; see
// profiles/r01_microbench2.txt and the ncu summaries):
//   * the K = n+1 planes of w for the tile plus an R halo arrive by TMA in two plane groups
//     [0, KA) and [KA, K), each in its own buffer with its own mbarrier: while one group is filtered,
//     the next slice's copy of the other group is in flight (double buffering at the SMEM cost of one
//     slice, so two CTAs still fit per SM).  TMA's out-of-bounds zero fill on all four sides implements
//     the clipped windows (F6).  The tile grid is shifted so that every TMA x coordinate is
//     16-byte aligned (IL: 64-byte): unaligned x offsets trap on this B200 stack (tools/tma_test2.cu);
//   * vertical pass in place: each (plane, column) item loads its column into registers once and
//     writes the 2R+1-row window sums back over the first TY rows; a warp covers 32 consecutive
//     columns of one plane (conflict-free);
//   * horizontal pass + Z + WTA by owner threads (one row x 8 pixels each) that keep G, 1/N and the
//     running (min, argmin) in registers; 128-bit shared loads, conflict-free by construction
//     (planar: 8 lanes of a quarter-warp read 8 different rows; the row pitch BX has BX/4 odd).
//
// IL = true reads the label-interleaved coefficient layout written by k_coef3 (WLayout::il): a rank-5
// tensor map (G px, 32 labels, x groups, y, planes) with box (G, 1, BX/G, BY, planes), G = kWGroupPx, lands the same
// [k][y][x] tile (BX a multiple of 32) with the 64-byte TMA swizzle: the 16-byte chunk c of 64-byte row
// R sits at chunk c ^ ((R >> 1) & 3), i.e. float index f -> f ^ ((f >> 3) & 12) from a 1 KB aligned
// buffer.  The swizzle keeps both passes conflict-free without a padded pitch; owners then map a
// quarter-warp to 4 rows x 2 segments that are 16 pixels apart (tools/swizzle_banks.py checks it).
#pragma once
#include <cuda.h>

#include <cuda/ptx>

#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace v3 {

constexpr int TX = 64, KX = 8, NSEG = TX / KX;
// Tile height: 48 rows at one 512-thread CTA per SM for n <= HGF_AGG3_TALL_N (the 2R-row vertical halo then costs
// 1.375x instead of 1.75x of TMA and vertical-pass traffic), else 24 rows at two 256-thread CTAs per SM.
#ifndef HGF_AGG3_TALL_N
#define HGF_AGG3_TALL_N 6
#endif
__host__ __device__ constexpr int agg3_ty(int NC) { return NC <= HGF_AGG3_TALL_N ? 48 : 24; }
__host__ __device__ constexpr int agg3_threads(int NC) { return NC <= HGF_AGG3_TALL_N ? 512 : 256; }

__host__ __device__ constexpr int box_pitch(int wx) {
  int b = (wx + 3) / 4 * 4;
  while (((b / 4) & 1) == 0) b += 4;  // BX/4 odd -> quarter-warp 16-B loads from 8 rows hit distinct banks
  return b;
}

template <int NC, int R, bool IL = false>
struct AggGeom {
  static constexpr int K = NC + 1;
  static constexpr int KA = agg3_ka(K), KB = K - KA;
  static constexpr int WX = TX + 2 * R;
  static constexpr int VX = (WX + 31) / 32 * 32;                     // vertical-pass columns per plane
  static constexpr int BX = IL ? VX : box_pitch(WX);                   // IL: whole 128-B rows
  static constexpr int TY = agg3_ty(NC), THREADS = agg3_threads(NC), NOWN = TY * NSEG;
  static constexpr int BY = TY + 2 * R;
  static constexpr int PLANE = BY * BX;                                // floats per plane in SMEM
  static constexpr int OFF_B = (KA * PLANE + 255) / 256 * 256;         // group B buffer: 1 KB aligned
  static constexpr int FLOATS = OFF_B + (KB * PLANE + 31) / 32 * 32;
  static constexpr int NV4 = (KX + 2 * R + 3) / 4;                     // 128-bit loads per owner row segment
  static_assert(KX * (NSEG - 1) + 4 * NV4 <= BX, "owner loads stay inside the row");
  static_assert(BX <= 256 && BY <= 256, "TMA box limits");
  static_assert(K >= 2, "two plane groups");
};

// 8-pixel groups (HGF_WG8) give 32-byte TMA inner runs, which take the 32-byte swizzle instead (the 64-byte
// one needs 64-byte rows and faults on 32-byte ones: tools/tma_swz8.cu, profiles/r01_tma_swz8.txt): the
// 16-byte chunk c of 32-byte row R sits at c ^ ((R >> 2) & 1), i.e. f -> f ^ ((f >> 3) & 4).
constexpr bool kSw32 = kWGroupPx == 8;
// SMEM float index of logical tile element f under the TMA swizzle (identity without it).
template <bool IL>
__device__ __forceinline__ int swz(int f) {
  return IL ? (kSw32 ? (f ^ ((f >> 3) & 4)) : (f ^ ((f >> 3) & 12))) : f;
}

// mbarrier / TMA wrappers over libcu++'s cuda::ptx (PTX ISA 8.0+, sm_90+).
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) { cuda::ptx::mbarrier_init(bar, count); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  cuda::ptx::mbarrier_arrive_expect_tx(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared, bar,
                                       bytes);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  // the suspend-time hint parks the waiting warp in hardware instead of spinning through issue slots
  while (!cuda::ptx::mbarrier_try_wait_parity(bar, parity, uint32_t(kMbarSuspendNs))) {
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

// tmA / tmB: tensor maps whose box covers planes [0, KA) / [KA, K) of one slice.
template <int NC, int R, bool IL>
__global__ void __launch_bounds__(agg3_threads(NC), agg3_threads(NC) == 512 ? 1 : ((NC + 1) * 42 * 96 * 4 <= 113 * 1024 ? 2 : 1))
    k_agg3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const float* __restrict__ G, int W, int H, int pad, int L, int label_base, float* __restrict__ filtered_out,
           int do_wta, int first, int last, float* __restrict__ best_cost, int32_t* __restrict__ best_label,
           int32_t* __restrict__ labels_out, float* __restrict__ min_cost_out, int64_t* __restrict__ keys_out,
           long long* const* __restrict__ peer_keys, int rows_per_owner) {
  using Gm = AggGeom<NC, R, IL>;
  constexpr int K = Gm::K, KA = Gm::KA, BX = Gm::BX, BY = Gm::BY, PLANE = Gm::PLANE, NV4 = Gm::NV4;
  constexpr int TY = Gm::TY, THREADS = Gm::THREADS, NOWN = Gm::NOWN;
  constexpr unsigned BYTES_A = Gm::KA * PLANE * 4u, BYTES_B = Gm::KB * PLANE * 4u;
  // Dynamic SMEM: group A buffer, group B buffer (1 KB aligned), then the two mbarriers.
  // Indexing the __shared__ array directly keeps every access in the shared state space (LDS/STS).
  extern __shared__ __align__(1024) float buf[];
  float* const bufs[2] = {buf, buf + Gm::OFF_B};
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + Gm::FLOATS);
  const int tid = threadIdx.x;
  // Tiles start at x0 = 64*bx - XSHIFT so that the TMA x coordinate x0 - R is a multiple of 4 (16 bytes;
  // IL: of one kWGroupPx-pixel group): TMA traps on x offsets that are not 16-byte aligned (tools/tma_test2.cu);
  // negative coordinates and the out-of-bounds zero fill are fine, and implement the clipped windows.
  constexpr int XALIGN = IL ? kWGroupPx : 4;
  constexpr int XSHIFT = (XALIGN - R % XALIGN) % XALIGN;
  // Grouped tile order: consecutive CTAs walk down a column of GY tiles before moving right, so the ~148
  // CTAs resident at once cover a compact ~12 x 12-tile block and the R-halos they share (the coefficient
  // tiles overlap by 2R) are L2 hits instead of repeated HBM reads (ncu r01: 1.64x re-read with row order).
  constexpr int GY = 12;
  int tile_x, tile_y;
  {
    const int id = blockIdx.y * gridDim.x + blockIdx.x;
    const int per_group = GY * gridDim.x;
    const int first_row = (id / per_group) * GY;
    const int rows = min(GY, (int)gridDim.y - first_row);
    const int in = id % per_group;
    tile_y = first_row + in % rows;
    tile_x = in / rows;
  }
  const int x0 = tile_x * TX - XSHIFT, y0 = tile_y * TY;
  const int tx0 = x0 - R + pad, ty0 = y0 - R + pad;   // pad = 0 in the pitched layout
  const long long HW = (long long)H * W;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // group h of label l: plane coordinate l*K + h*KA (planar) or group coordinates (l % 32, (l/32)*K + h*KA)
  auto load = [&](int h, int l) {
    mbar_expect_tx(&bar[h], h == 0 ? BYTES_A : BYTES_B);
    const CUtensorMap* tm = h == 0 ? &tmA : &tmB;
    if (IL) {
      const int32_t c[5] = {0, l % kWGroupLabels, tx0 / kWGroupPx, ty0, (l / kWGroupLabels) * K + h * KA};
      cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, bufs[h], tm, c, &bar[h]);
    } else {
      tma_load_3d(bufs[h], tm, tx0, ty0, l * K + h * KA, &bar[h]);
    }
  };
  if (tid == 0 && L > 0) {
    load(0, 0);
    load(1, 0);
  }

  // owner role: row oy, pixels x0 + 8*seg + [0, 8)
  const bool is_owner = tid < NOWN;
  const int wq = tid >> 5, ln = tid & 31;
  // planar: a quarter-warp = 8 rows of one segment (odd BX/4 pitch); IL: 4 rows x segments s, s + 2;
  // IL with the 32-byte swizzle: one row x all 8 segments (segments s and s + 4 share a chunk index and are
  // told apart by the swizzle bit; tools/swizzle_banks.py checks R = 1..32)
  constexpr int NRG = TY / 8;     // planar: row groups of 8 per segment half
  const int oy = IL ? (kSw32 ? (ln >> 3) + 4 * wq : (ln & 3) + 4 * wq) : (ln & 7) + 8 * (wq % NRG);
  const int seg = IL ? (kSw32 ? (ln & 7) : ((ln >> 3) & 1) + 4 * (ln >> 4) + 2 * ((ln >> 2) & 1))
                     : (ln >> 3) + 4 * (wq / NRG);
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

  // owner row-segment offsets of plane 0 (swizzled); PLANE/32 is even, so other planes differ by bit 3 at most
  static_assert(!IL || kSw32 || ((PLANE / 32) & 1) == 0, "plane swizzle phase");
  int ofs[NV4];
#pragma unroll
  for (int q = 0; q < NV4; ++q) ofs[q] = swz<IL>(oy * BX + seg * KX + 4 * q);
  float z[KX];
  // per (label l, plane group h): the in-place vertical pass (all threads), then the owners' horizontal pass
  auto vpass = [&](int h, int l) {
    const int k0 = h == 0 ? 0 : KA, k1 = h == 0 ? KA : K;
    float* lb = bufs[h];
    mbar_wait(&bar[h], l & 1);
    // ---- vertical window sums, in place: rows [0, TY) <- sum of rows [y, y + 2R]
    for (int item = tid; item < (k1 - k0) * Gm::VX; item += THREADS) {
      const int kk = item / Gm::VX, c = item % Gm::VX;
      if (c >= Gm::WX) continue;
      const int f0 = kk * PLANE + c;
      // swizzled address of row y: (f0 ^ m(y)) + y*BX, the XOR mask m depending only on y mod 4
      // (BX is a multiple of 32 floats, so adding y*BX never carries into the swizzled bits)
      int fb[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        fb[j] = IL ? (kSw32 ? (f0 ^ ((((f0 >> 5) + j * (BX / 32)) & 1) << 2))
                            : (f0 ^ ((((f0 >> 5) + j * (BX / 32)) & 3) << 2)))
                   : f0;
      // the column is read once; the outputs in two halves for 48-row tiles, the second half's input rows
      // loaded after the first half's stores (rows below them), so at most ~TY/2 + 2R + 1 values are live
      constexpr int VCH = TY > 24 ? TY / 2 : TY;
      float col[BY];
#pragma unroll
      for (int y = 0; y < VCH + 2 * R; ++y) col[y] = lb[fb[y & 3] + y * BX];
      float acc = 0.0f;
#pragma unroll
      for (int y = 0; y <= 2 * R; ++y) acc += col[y];
      lb[fb[0]] = acc;
#pragma unroll
      for (int y = 1; y < VCH; ++y) {
        acc += col[y + 2 * R] - col[y - 1];
        lb[fb[y & 3] + y * BX] = acc;
      }
      if constexpr (VCH < TY) {
#pragma unroll
        for (int y = VCH + 2 * R; y < BY; ++y) col[y] = lb[fb[y & 3] + y * BX];
#pragma unroll
        for (int y = VCH; y < TY; ++y) {
          acc += col[y + 2 * R] - col[y - 1];
          lb[fb[y & 3] + y * BX] = acc;
        }
      }
    }
  };
  auto hpass = [&](int h, int l) {
    const int k0 = h == 0 ? 0 : KA;
    float* lb = bufs[h];
    // ---- horizontal window sums, accumulated into Z (owners)
    if (is_owner) {
#pragma unroll
      for (int k = (h == 0 ? 0 : KA); k < (h == 0 ? KA : K); ++k) {
        // plane kk of the group: swizzle mask of plane 0 flipped in bit 3 when kk * PLANE/32 = 2 mod 4
        const int kk = k - k0;
        // (32-byte swizzle: flipped in bit 2 when kk * PLANE/32 is odd)
        const int flip = !IL ? 0
                         : kSw32 ? (((kk * (PLANE / 32)) & 1) ? 4 : 0)
                                 : ((((kk * ((PLANE / 32) & 3)) & 3) == 2) ? 8 : 0);
        float f[4 * NV4];
#pragma unroll
        for (int q = 0; q < NV4; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(lb + kk * PLANE + (ofs[q] ^ flip));
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
      if (h == 1) {
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
    }
  };
#pragma unroll 1
  for (int l = 0; l < L; ++l) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      vpass(h, l);
      __syncthreads();
      hpass(h, l);
      __syncthreads();
      // group h of this slice consumed: fetch group h of the next slice while the other group is filtered (a
      // single-barrier variant that overlapped the next group's vertical pass with this group's owner work left
      // the tile loads less time to land: 18.7 -> 20.5 ms at C4)
      if (tid == 0 && l + 1 < L) {
        fence_proxy_async();
        load(h, l + 1);
      }
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
      if (peer_keys) {
        // fused merge: a 64-bit atomic MIN on the owner GPU's key buffer (over NVLink for remote owners).
        // System scope: the owners' buffers are written by several GPUs (ATOM.E.MIN.S64.STRONG.SYS).
        const int owner = gy / rows_per_owner;
        atomicMin_system(peer_keys[owner] + (long long)(gy - owner * rows_per_owner) * W + gx,
                         (long long)pack_key_signed(best[s], bl[s]));
      }
    } else {
      best_cost[p] = best[s];
      best_label[p] = bl[s];
    }
  }
  if (last && peer_keys) __threadfence_system();
}

template <int NC, int R, bool IL>
size_t agg3_smem_bytes() {
  using Gm = AggGeom<NC, R, IL>;
  return (size_t)Gm::FLOATS * 4 + 128;
}

template <int NC, int R, bool IL>
cudaError_t agg3_launch(const void* tmaps, const AggArgs& a, cudaStream_t st) {
  const size_t smem = agg3_smem_bytes<NC, R, IL>();
  cudaError_t e = cudaFuncSetAttribute(k_agg3<NC, R, IL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  constexpr int XALIGN = IL ? kWGroupPx : 4;
  using Gm = AggGeom<NC, R, IL>;
  dim3 grid((a.W + (XALIGN - R % XALIGN) % XALIGN + TX - 1) / TX, (a.H + Gm::TY - 1) / Gm::TY);
  const CUtensorMap* tm = reinterpret_cast<const CUtensorMap*>(tmaps);
  k_agg3<NC, R, IL><<<grid, Gm::THREADS, smem, st>>>(tm[0], tm[1], a.G, a.W, a.H, a.pad, a.L, a.label_base,
                                                 a.filtered_out, a.do_wta, a.first, a.last, a.best_cost,
                                                 a.best_label, a.labels_out, a.min_cost_out, a.keys_out,
                                                 a.peer_keys, a.rows_per_owner);
  return cudaGetLastError();
}

// tmaps: two consecutive CUtensorMaps (plane groups [0, KA) and [KA, K)).
template <int NC, int R>
cudaError_t agg3_impl(const void* tmaps, const AggArgs& a, cudaStream_t st) {
  return a.il ? agg3_launch<NC, R, true>(tmaps, a, st) : agg3_launch<NC, R, false>(tmaps, a, st);
}

}  // namespace v3
}  // namespace hgf
