// HGF per-slice aggregation + WTA, version 6 (k_agg6<n, R>): k_agg3's arithmetic and tile (64 x 48 outputs,
// label-interleaved coefficient layout, 64-byte TMA swizzle) with the CTA split into warp roles that run as a
// per-plane pipeline instead of in CTA-wide lock step.
//
//   Z = (B(w_0) + sum_k G_k B(w_k)) / N   (Eq14 P:328-333 == Eq8), running WTA min/argmin (ties -> lowest label,
//   P:26), box sums clipped at the borders (F6) through TMA's out-of-bounds zero fill.
//
// Why: k_agg3 is bound by the SM's shared-memory pipe (LSU, ~1 wavefront per clock), but at one 512-thread CTA
// per SM it spends a third of its time in the four CTA barriers per slice (vertical pass on 16 warps with 21
// warp-items of work, horizontal pass on 12 owner warps) and waiting for the next plane group's TMA, which it
// can only issue half a slice ahead.  Here:
//   * the coefficient planes arrive one TMA box each (plane-step s = lK + k: plane k of slice l) into a ring of NB
//     1 KB-aligned slots (as many as shared memory holds: 9 at r = 9, NB >= K), slot s % NB with three mbarriers:
//     full (TMA landed), vdone (vertical sums written), hdone (owners finished reading); each completes once per
//     NB plane-steps (phase parity (s / NB) & 1);
//   * the last warp's lane 0 (producer) refills a slot as soon as the owners release it, NB - 1 plane-steps before
//     it is needed (k_agg3: one plane group, half a slice);
//   * 3 vertical warps (96 threads = the tile's 96 swizzled columns) do the in-place vertical window sums of a
//     plane, then arrive on vdone;
//   * owner warps (rows x 8 or 16 pixels, conflict-free swizzled mappings) wait on vdone, do the horizontal sums,
//     Z and (after the last plane of a slice) the WTA, then arrive on hdone.
// The vertical warps run up to NB - 1 plane-steps ahead of the owners, so both passes keep the LSU busy without CTA
// barriers; that slack is what pays (cutting it to two plane-steps cost 18 %, growing it from K - 1 = 6 to 8: -2 %).
#pragma once
#include <cuda.h>

#include <cuda/ptx>

#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {
namespace v6a {

// Tile height 48 (= kAgg6TY; 36-row tiles with two vertical teams measured the same C4 time).
constexpr int TX = 64, TY = 48;
constexpr int NVW = 3;                     // vertical warps (one column each of the 96-column tile)
static_assert(TY == kAgg6TY, "host box height");
static_assert(kWGroupPx == 16, "64-byte swizzle (16-pixel groups)");

// Owner configuration.  D = 0: owners of 8 pixels holding the n guidance planes G_k (any n <= 6), 512 threads.
// D >= 1: owners of 16 pixels holding only the m = NC / D raw channels I_i (G_{(i-1)D+j} = I_i^j formed by the same
// repeated multiplication as k_poly_guidance, so bit-identical), m <= 3: half the owners, each loading 16 + 2R
// columns per plane for 16 outputs instead of 8 + 2R for 8 (-35 % of the horizontal pass's shared wavefronts), at
// 320 threads so the wider owners get ~200 registers.  Either way the owner's horizontal sums restart every 8
// pixels, as k_agg3's owners do.
template <int NC, int D>
struct Roles {
  static constexpr int KX = D == 0 ? 8 : 16, NSEG = TX / KX;
  static constexpr int NOWN = TY * NSEG;             // owner threads = warps [0, NOWN / 32)
  static constexpr int THREADS = D == 0 ? 512 : NOWN + 32 * NVW + 32;   // the last warp is the TMA producer

  static constexpr int MG = D == 0 ? NC : NC / (D > 0 ? D : 1);    // guide values held per owner pixel
  static_assert(NOWN % 32 == 0 && NOWN + 32 * NVW + 32 == THREADS, "warp roles");
  static_assert(D == 0 || (NC % (D > 0 ? D : 1) == 0 && NC / (D > 0 ? D : 1) <= 3), "raw-channel owners: m <= 3");
  // registers per thread: each SM sub-partition holds 16384, and takes up to ceil(warps / 4) of the CTA's warps
  static constexpr int MAXREG = (16384 / (32 * ((THREADS / 32 + 3) / 4))) / 8 * 8 > 255
                                    ? 255
                                    : (16384 / (32 * ((THREADS / 32 + 3) / 4))) / 8 * 8;
};

template <int NC, int R, int D>
struct Geom {
  static constexpr int K = NC + 1;
  static constexpr int KX = Roles<NC, D>::KX, NSEG = Roles<NC, D>::NSEG;
  static constexpr int WX = TX + 2 * R;
  static constexpr int BX = (WX + 31) / 32 * 32;
  static constexpr int BY = TY + 2 * R;
  static constexpr int PLANE = BX * BY;                        // floats per plane tile
  static constexpr int PSTRIDE = (PLANE + 255) / 256 * 256;    // 1 KB-aligned plane buffers
  // ring slots: as many plane buffers as fit next to the barriers and the 1 KB static reservation (<= 16)
  static constexpr int NBFIT = (227 * 1024 - 1024 - 16 * 3 * 8) / (PSTRIDE * 4);
  static constexpr int NB = NBFIT > 16 ? 16 : NBFIT;
  static_assert(NB >= K, "one slice of planes in flight");
  static constexpr int FLOATS = NB * PSTRIDE;
  static constexpr int NV4 = (KX + 2 * R + 3) / 4;
  static_assert(BX == 32 * NVW, "one vertical thread per tile column");
  static_assert(KX * (NSEG - 1) + 4 * NV4 <= BX, "owner loads stay inside the row");
  static_assert(BX <= 256 && BY <= 256, "TMA box limits");
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) { cuda::ptx::mbarrier_init(bar, count); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!cuda::ptx::mbarrier_try_wait_parity(bar, parity, uint32_t(kMbarSuspendNs))) {
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  (void)cuda::ptx::mbarrier_arrive(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared, bar);
}

// tm: rank-5 map over the interleaved coefficient buffer, box (16 px, 1 label, BX/16 groups, BY rows, 1 plane).
template <int NC, int R, int D>
__global__ void __maxnreg__((Roles<NC, D>::MAXREG))
    k_agg6(const __grid_constant__ CUtensorMap tm, const float* __restrict__ G, int W, int H, int L, int label_base,
           float* __restrict__ filtered_out, int do_wta, int first, int last, float* __restrict__ best_cost,
           int32_t* __restrict__ best_label, int32_t* __restrict__ labels_out, float* __restrict__ min_cost_out,
           int64_t* __restrict__ keys_out, long long* const* __restrict__ peer_keys, int rows_per_owner,
           long long* __restrict__ fkeys) {
  using Gm = Geom<NC, R, D>;
  using Ro = Roles<NC, D>;
  constexpr int K = Gm::K, BX = Gm::BX, BY = Gm::BY, PSTRIDE = Gm::PSTRIDE, NV4 = Gm::NV4, KX = Gm::KX;
  constexpr int NOWN = Ro::NOWN, THREADS = Ro::THREADS, MG = Ro::MG, NB = Gm::NB;
  extern __shared__ __align__(1024) float buf[];
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + Gm::FLOATS);
  uint64_t* vdone = full + NB;        // per ring slot: TMA landed / vertical sums written / owners released
  uint64_t* hdone = vdone + NB;
  const int tid = threadIdx.x, wq = tid >> 5, ln = tid & 31;
  // tile origin shifted so the TMA x coordinate x0 - R is a whole 16-pixel group (unaligned x traps); grouped
  // tile order (GY tiles down a column) so the CTAs resident at once share their R-halos through L2 (k_agg3)
  constexpr int XSHIFT = (kWGroupPx - R % kWGroupPx) % kWGroupPx;
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
  const int tx0 = x0 - R, ty0 = y0 - R;
  const long long HW = (long long)H * W;

  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&vdone[b], NVW);
      mbar_init(&hdone[b], NOWN / 32);
    }
    cuda::ptx::fence_mbarrier_init(cuda::ptx::sem_release, cuda::ptx::scope_cluster);
  }
  __syncthreads();
  // label split (small frames, fewer tiles than ~1.5 waves): CTA z takes labels [la, la + LL) of the chunk and
  // atomic-MINs its per-pixel minimum keys into fkeys (k_keys_finalize writes the outputs); ties keep the lowest
  // label either way (the key's low word), so the result equals the unsplit scan
  const int la = (int)(((long long)L * blockIdx.z) / gridDim.z);
  const int LL = (int)(((long long)L * (blockIdx.z + 1)) / gridDim.z) - la;
  const int S = K * LL;

  if (wq == THREADS / 32 - 1) {
    // ---- producer: plane k of slice l into buffer k once the owners have released slice l - 1's plane k
    if (ln != 0) return;
    for (int s = 0; s < S; ++s) {
      const int ll = s / K, k = s - ll * K, b = s % NB, l = la + ll;
      if (s >= NB) {
        mbar_wait(&hdone[b], (s / NB - 1) & 1);
        cuda::ptx::fence_proxy_async(cuda::ptx::space_shared);
      }
      cuda::ptx::mbarrier_arrive_expect_tx(cuda::ptx::sem_release, cuda::ptx::scope_cta, cuda::ptx::space_shared,
                                           &full[b], (uint32_t)(Gm::PLANE * 4));
      const int32_t c[5] = {0, l % kWGroupLabels, tx0 / kWGroupPx, ty0, (l / kWGroupLabels) * K + k};
      cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, buf + b * PSTRIDE, &tm, c,
                                      &full[b]);
    }
    return;
  }

  if (wq >= NOWN / 32) {
    // ---- vertical warps: column c of every plane, in place: rows [0, TY) <- sum of rows [y, y + 2R].  The whole
    // column is loaded before the first sum (one shared-memory round trip per plane); same summation order as
    // k_agg3, so the two kernels are bit-identical.  (Two independent half-column chains were measured: no gain.)
    const int c = tid - NOWN;
    // swizzled address of row y: (c ^ m(y)) + y*BX, the XOR mask depending only on y mod 4 (BX = 96 floats)
    int fb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) fb[j] = c ^ ((((c >> 5) + j * (BX / 32)) & 3) << 2);
    for (int s = 0; s < S; ++s) {
      const int b = s % NB;
      float* lb = buf + b * PSTRIDE;
      mbar_wait(&full[b], (s / NB) & 1);
      if (c < Gm::WX) {
        float col[BY];
#pragma unroll
        for (int y = 0; y < BY; ++y) col[y] = lb[fb[y & 3] + y * BX];
        float acc = 0.0f;
#pragma unroll
        for (int y = 0; y <= 2 * R; ++y) acc += col[y];
        lb[fb[0]] = acc;
#pragma unroll
        for (int y = 1; y < TY; ++y) {
          acc += col[y + 2 * R] - col[y - 1];
          lb[fb[y & 3] + y * BX] = acc;
        }
      }
      __syncwarp();
      if (ln == 0) mbar_arrive(&vdone[b]);
    }
    return;
  }

  // ---- owners: row oy, pixels x0 + KX*seg + [0, KX).  D = 0: a quarter-warp = 4 rows x segments s, s + 2; D >= 1:
  // 4 rows x 2 segments of one 8-row block.  Both conflict-free for the 128-bit loads under the 64-byte swizzle
  // (tools/swizzle_banks.py).
  const int oy = D == 0 ? (ln & 3) + 4 * wq : (ln & 3) + 4 * (ln >> 4) + 8 * wq;
  const int seg = D == 0 ? ((ln >> 3) & 1) + 4 * (ln >> 4) + 2 * ((ln >> 2) & 1) : (ln >> 2) & 3;
  const int gy = y0 + oy;
  float g[MG][KX];
  float invN[KX], best[KX];
  int32_t bl[KX];
#pragma unroll
  for (int j = 0; j < KX; ++j) {
    const int gx = x0 + seg * KX + j;
    const bool in = gy < H && gx >= 0 && gx < W;
    const long long p = in ? (long long)gy * W + gx : 0;
#pragma unroll
    for (int k = 0; k < MG; ++k) g[k][j] = in ? __ldg(G + (long long)(D == 0 ? k : k * D) * HW + p) : 0.0f;
    invN[j] = in ? 1.0f / (float)window_count(gy, gx, H, W, R) : 0.0f;
    best[j] = INFINITY;
    bl[j] = 0;
    if (do_wta && !first && !fkeys && in) {
      best[j] = best_cost[p];
      bl[j] = best_label[p];
    }
  }
  // G_k at pixel s (k >= 1): the held plane, or I_i^j by repeated multiplication (k_poly_guidance's order)
  auto guide = [&](int k, int s) -> float {
    if constexpr (D == 0) {
      return g[k - 1][s];
    } else {
      const int i = (k - 1) / D, j = (k - 1) % D;
      float t = g[i][s];
#pragma unroll
      for (int e = 0; e < j; ++e) t = t * g[i][s];
      return t;
    }
  };
  int ofs[NV4];
#pragma unroll
  for (int q = 0; q < NV4; ++q) {
    const int f = oy * BX + seg * KX + 4 * q;
    ofs[q] = f ^ ((f >> 3) & 12);
  }
  float z[KX];
#pragma unroll 1
  for (int l = la; l < la + LL; ++l) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int sg = (l - la) * K + k, b = sg % NB;
      const float* lb = buf + b * PSTRIDE;
      mbar_wait(&vdone[b], (sg / NB) & 1);
      float f[4 * NV4];
#pragma unroll
      for (int q = 0; q < NV4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(lb + ofs[q]);
        f[4 * q] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
      }
      // horizontal window sums, restarted every 8 pixels (k_agg3's owner order)
#pragma unroll
      for (int h8 = 0; h8 < KX; h8 += 8) {
        float acc = 0.0f;
#pragma unroll
        for (int dx = 0; dx <= 2 * R; ++dx) acc += f[h8 + dx];
#pragma unroll
        for (int s = h8; s < h8 + 8; ++s) {
          if (s > h8) acc += f[s + 2 * R] - f[s - 1];
          if (k == 0) z[s] = acc;
          else z[s] = fmaf(guide(k, s), acc, z[s]);
        }
      }
      // release the plane once its loaded values have been consumed
      __syncwarp();
      if (ln == 0) mbar_arrive(&hdone[b]);
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
  if (!do_wta) return;
#pragma unroll
  for (int s = 0; s < KX; ++s) {
    const int gx = x0 + seg * KX + s;
    if (gy >= H || gx < 0 || gx >= W) continue;
    const long long p = (long long)gy * W + gx;
    if (fkeys) {
      if (LL > 0) atomicMin(fkeys + p, (long long)pack_key_signed(best[s], bl[s]));
    } else if (last) {
      if (labels_out) labels_out[p] = bl[s];
      if (min_cost_out) min_cost_out[p] = best[s];
      if (keys_out) keys_out[p] = pack_key_signed(best[s], bl[s]);
      if (peer_keys) {
        // fused merge (k_agg3): system-scope 64-bit atomic MIN into the row owner's key buffer
        const int owner = gy / rows_per_owner;
        atomicMin_system(peer_keys[owner] + (long long)(gy - owner * rows_per_owner) * W + gx,
                         (long long)pack_key_signed(best[s], bl[s]));
      }
    } else {
      best_cost[p] = best[s];
      best_label[p] = bl[s];
    }
  }
  if (last && peer_keys && !fkeys) __threadfence_system();
}

template <int NC, int R, int D>
cudaError_t agg6_launch(const void* tmap, const AggArgs& a, cudaStream_t st) {
  using Gm = Geom<NC, R, D>;
  using Ro = Roles<NC, D>;
  const size_t smem = (size_t)Gm::FLOATS * 4 + 3 * Gm::NB * sizeof(uint64_t);
  cudaError_t e = cudaFuncSetAttribute(k_agg6<NC, R, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  constexpr int XSHIFT = (kWGroupPx - R % kWGroupPx) % kWGroupPx;
  dim3 grid((a.W + XSHIFT + TX - 1) / TX, (a.H + TY - 1) / TY, a.fkeys && a.nsplit > 1 ? a.nsplit : 1);
  k_agg6<NC, R, D><<<grid, Ro::THREADS, smem, st>>>(*reinterpret_cast<const CUtensorMap*>(tmap), a.G, a.W, a.H, a.L,
                                                    a.label_base, a.filtered_out, a.do_wta, a.first, a.last,
                                                    a.best_cost, a.best_label, a.labels_out, a.min_cost_out,
                                                    a.keys_out, a.peer_keys, a.rows_per_owner, a.fkeys);
  return cudaGetLastError();
}

}  // namespace v6a

template <int NC, int D>
inline cudaError_t agg6_r(int r, const void* tm, const AggArgs& a, cudaStream_t st) {
  switch (r) {
    case 1: return v6a::agg6_launch<NC, 1, D>(tm, a, st); case 2: return v6a::agg6_launch<NC, 2, D>(tm, a, st);
    case 3: return v6a::agg6_launch<NC, 3, D>(tm, a, st); case 4: return v6a::agg6_launch<NC, 4, D>(tm, a, st);
    case 5: return v6a::agg6_launch<NC, 5, D>(tm, a, st); case 6: return v6a::agg6_launch<NC, 6, D>(tm, a, st);
    case 7: return v6a::agg6_launch<NC, 7, D>(tm, a, st); case 8: return v6a::agg6_launch<NC, 8, D>(tm, a, st);
    case 9: return v6a::agg6_launch<NC, 9, D>(tm, a, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace hgf
