// Internal device helpers for the HGF kernels (sm_100a).  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hgf {

// Clipped-window pixel count N_p = |Omega_p| = B(G_0)(p) (border reading F6).
__device__ __forceinline__ int window_count(int y, int x, int H, int W, int r) {
  const int ny = min(y + r, H - 1) - max(y - r, 0) + 1;
  const int nx = min(x + r, W - 1) - max(x - r, 0) + 1;
  return ny * nx;
}

// Monotone float -> uint32 map used by the packed WTA keys (hgf.h, hgf_aggregate_wta_ex).
__device__ __forceinline__ uint32_t orderable_bits(float f) {
  f = f + 0.0f;  // canonicalise -0.0 to +0.0
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float from_orderable_bits(uint32_t o) {
  const uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(b);
}
__device__ __forceinline__ uint64_t pack_key(float cost, int32_t label) {
  return (static_cast<uint64_t>(orderable_bits(cost)) << 32) | static_cast<uint32_t>(label);
}

// Signed-order key (hgf.h keys_out): unsigned key XOR 2^63, so int64 MIN == unsigned MIN.
__device__ __forceinline__ int64_t pack_key_signed(float cost, int32_t label) {
  return static_cast<int64_t>(pack_key(cost, label) ^ 0x8000000000000000ull);
}

// Layout of the per-slice coefficient buffer.
// Planar (il == 0): element (label l, plane k, y, x) of a chunk lives at
//   origin + (l*(n+1) + k)*plane + y*pitch + x.
// Label-interleaved (il == 1, k_coef3 -> k_agg3): 32 labels share each G-pixel group (G = kWGroupPx),
//   ((((l/32)*(n+1) + k)*H + y)*xg + x/G)*(32*G) + (l%32)*G + x%G.
// G = 16 (default): the 16 labels of a k_coef3 half-warp store one contiguous 1 KB run per instruction
// (each 128-byte line half-written by the two 8-pixel stores of a lane), k_agg3's TMA reads 64-byte runs.
// G = 8 (-DHGF_WG8=1): the 32 labels of a warp store 1 KB of whole lines per instruction, k_agg3's TMA
// reads 32-byte runs (profiles/r01_tma_run_rate.txt: ~1 run per clock per SM for either length).
#ifndef HGF_WG8
#define HGF_WG8 0
#endif
constexpr int kWGroupPx = HGF_WG8 ? 8 : 16, kWGroupLabels = 32;
// Suspend-time hint (ns) for mbarrier.try_wait: a waiting warp is parked until the phase completes (or
// the hint elapses) instead of spinning through issue slots the working warps need.
constexpr unsigned kMbarSuspendNs = 20000;
// Floats per pixel record of the per-pixel ("AoS") statistics layout read by k_coef3 / k_coef4 (n <= 6).
constexpr int kStatsAos = 28;
struct WLayout {
  long long origin;   // = pad * pitch + pad
  long long plane;
  int pitch;          // multiple of 4 in the padded layout (16-byte rows)
  int pad;            // zero margin above / left of the image (0 = flat layout; else roundup(r, 4))
  int il;             // 1 = label-interleaved layout
  int xg;             // 16-pixel groups per row (il == 1)
};

// Number of statistics planes stored per pixel for n channels: P' (upper triangle) + nu.
__host__ __device__ constexpr int stats_planes(int n) { return n * (n + 1) / 2 + n; }
// Floats per per-pixel statistics record (the statistics, then kappa, padded to 16 bytes): 28 for n <= 6.
__host__ __device__ constexpr int stats_aos_floats(int n) {
  return n <= 6 ? kStatsAos : (stats_planes(n) + 1 + 3) / 4 * 4;
}
// k_coef3: labels per CTA (32 up to n = 6; 16 for n = 7..9 so the V rows of n + 1 planes fit SMEM).
constexpr int kCoef3MaxN = 9;
__host__ __device__ constexpr int coef3_labels(int n) { return n <= 6 ? 32 : 16; }

}  // namespace hgf
