// Non-template kernels (K1 guidance, key unpacking) and the n -> template dispatch.
// The per-n template instantiations live in hgf_inst.cu (compiled once per n with -DHGF_N=n).
#include <cstdlib>

#include "hgf_common.cuh"
#include "hgf_launch.h"

namespace hgf {

// ------------------------------------------------------------------ K1: polynomial guidance
// Gp (optional, d = 2): the same powers as (I_i, I_i^2) pairs, layout [H][m][gp][2] (k_coef5's guide rows).
__global__ void k_poly_guidance(const float* __restrict__ I, float* __restrict__ G, float2* __restrict__ Gp, int gp, int m,
                                int d, int W, long long HW) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < HW; p += (long long)gridDim.x * blockDim.x) {
    for (int i = 0; i < m; ++i) {
      const float v = I[i * HW + p];
      float t = v;                       // repeated multiplication: I^1, I^2, ... (exact powers order)
      G[(long long)(i * d) * HW + p] = t;
      for (int j = 1; j < d; ++j) {
        t = t * v;
        G[(long long)(i * d + j) * HW + p] = t;
      }
      if (Gp) {
        const long long y = p / W, x = p - y * W;
        Gp[(y * m + i) * gp + x] = make_float2(v, v * v);
      }
    }
  }
}

__global__ void k_unpack_keys(const int64_t* __restrict__ keys, int32_t* __restrict__ labels, float* __restrict__ cost,
                              long long HW) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < HW; p += (long long)gridDim.x * blockDim.x) {
    const uint64_t k = (uint64_t)keys[p] ^ 0x8000000000000000ull;
    if (labels) labels[p] = (int32_t)(uint32_t)(k & 0xffffffffull);
    if (cost) cost[p] = from_orderable_bits((uint32_t)(k >> 32));
  }
}

// Final WTA outputs from the merged per-pixel keys (k_agg5 path): labels / min cost / keys, and the fused
// label-sharded merge into the row owners' key buffers (system scope: several GPUs' atomics meet there).
__global__ void k_keys_finalize(const int64_t* __restrict__ keys, int W, long long HW, int32_t* __restrict__ labels,
                                float* __restrict__ cost, int64_t* __restrict__ keys_out,
                                long long* const* __restrict__ peer_keys, int rows_per_owner) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < HW; p += (long long)gridDim.x * blockDim.x) {
    const int64_t ks = keys[p];
    const uint64_t k = (uint64_t)ks ^ 0x8000000000000000ull;
    if (labels) labels[p] = (int32_t)(uint32_t)(k & 0xffffffffull);
    if (cost) cost[p] = from_orderable_bits((uint32_t)(k >> 32));
    if (keys_out) keys_out[p] = ks;
    if (peer_keys) {
      const int y = (int)(p / W), x = (int)(p - (long long)y * W);
      const int owner = y / rows_per_owner;
      atomicMin_system(peer_keys[owner] + (long long)(y - owner * rows_per_owner) * W + x, (long long)ks);
    }
  }
  if (peer_keys) __threadfence_system();
}

__global__ void k_fill_i64(int64_t* __restrict__ p, long long n, long long v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

// ------------------------------------------------------------------ launchers
static int grid_1d(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  return (int)(b < 148LL * 32 ? (b < 1 ? 1 : b) : 148LL * 32);
}

cudaError_t launch_keys_finalize(const int64_t* keys, int W, int H, int32_t* labels_out, float* min_cost_out,
                                 int64_t* keys_out, long long* const* peer_keys, int rows_per_owner, cudaStream_t st) {
  const long long HW = (long long)W * H;
  k_keys_finalize<<<grid_1d(HW, 256), 256, 0, st>>>(keys, W, HW, labels_out, min_cost_out, keys_out, peer_keys,
                                                    rows_per_owner);
  return cudaGetLastError();
}

cudaError_t launch_poly_guidance(const float* I, float* G, float* Gp, int gp_pitch, int m, int d, int W, int H,
                                 cudaStream_t st) {
  const long long HW = (long long)W * H;
  k_poly_guidance<<<grid_1d(HW, 256), 256, 0, st>>>(I, G, reinterpret_cast<float2*>(d == 2 ? Gp : nullptr), gp_pitch,
                                                      m, d, W, HW);
  return cudaGetLastError();
}

#define HGF_DISPATCH(n, CALL)                                                          \
  switch (n) {                                                                         \
    case 1: return CALL(1); case 2: return CALL(2); case 3: return CALL(3);            \
    case 4: return CALL(4); case 5: return CALL(5); case 6: return CALL(6);            \
    case 7: return CALL(7); case 8: return CALL(8); case 9: return CALL(9);            \
    case 10: return CALL(10); case 11: return CALL(11); case 12: return CALL(12);      \
    case 13: return CALL(13); case 14: return CALL(14); case 15: return CALL(15);      \
    case 16: return CALL(16); case 17: return CALL(17); case 18: return CALL(18);      \
    case 19: return CALL(19); case 20: return CALL(20);                                \
    default: return cudaErrorInvalidValue;                                             \
  }

cudaError_t launch_filter1(int n, const float* G, const float* P, float* wout, WLayout wo, int W, int H, int r,
                           double lam, int mode, float lam0f, cudaStream_t st) {
  if (n > kStats4MaxN || 64 + 2 * r > 128 || stats4_smem(n, r, 1) > 200 * 1024) return cudaErrorInvalidValue;
  switch (n) {
#define F1(N) \
  case N: return st5::filter1_sel<N>(G, P, wout, wo, W, H, r, lam, mode, lam0f, st);
    F1(1) F1(2) F1(3) F1(4) F1(5) F1(6) F1(7) F1(8) F1(9)
#undef F1
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_stats(int n, const float* G, float* stats, int W, int H, int r, double lam, int mode, int aos,
                         float lam0f, int y0, int y1, double* scratch3, cudaStream_t st) {
  const int TS = 16 + 2 * r;
  // = st2::smem_bytes(n, r): odd-pitch channel tiles, 17-double rows of horizontal sums, vertical sums
  const size_t smem2 = ((size_t)(n + 1) * TS * (TS | 1) * 4 + 15) / 16 * 16 + (size_t)7 * TS * 17 * 8 +
                       (size_t)7 * 16 * 16 * 8 + 16;
  // k_stats4 (row-marching Gram sums, hgf_stats_v4.cuh) for n <= kStats4MaxN; HGF_STATS2=1 keeps the
  // tiled k_stats2 (comparison runs)
  const bool force2 = std::getenv("HGF_STATS2") != nullptr && std::getenv("HGF_STATS2")[0] == '1';
  if (!force2 && n <= kStats4MaxN && 64 + 2 * r <= 128 && stats4_smem(n, r) <= 200 * 1024) {
    switch (n) {
      case 1: return st5::stats_sel<1>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      case 2: return st5::stats_sel<2>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      case 3: return st5::stats_sel<3>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      case 4: return st5::stats_sel<4>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      case 5: return st5::stats_sel<5>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      case 6: return st5::stats_sel<6>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      case 7: return st5::stats_sel<7>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      case 8: return st5::stats_sel<8>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      case 9: return st5::stats_sel<9>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st);
      default: break;
    }
  }
  // k_stats3 (Gram planes + warp-per-pixel recursion) where k_stats2 would spill heavily (n >= kStats3MinN)
  // or not fit its channel tiles in shared memory (the O(r) v1 kernel) -- measured on the C5 sweep
  const int s3min = std::getenv("HGF_STATS3_MIN_N") ? std::atoi(std::getenv("HGF_STATS3_MIN_N")) : kStats3MinN;
  if (scratch3 && !aos && y0 == 0 && y1 == H && (n >= s3min || (n >= 7 && smem2 > 200 * 1024))) {
#define CALL(N) st3::stats3_impl<N>(G, stats, scratch3, W, H, r, lam, mode, st)
    HGF_DISPATCH(n, CALL)
#undef CALL
  }
  // sliding-sum version when all n+1 channel tiles fit in shared memory, else the pairwise v1 kernel
  if (smem2 <= 200 * 1024) {
#define CALL(N) st2::stats2_impl<N>(G, stats, W, H, r, lam, mode, aos, lam0f, y0, y1, st)
    HGF_DISPATCH(n, CALL)
#undef CALL
  }
  if (aos || y0 != 0 || y1 != H) return cudaErrorInvalidValue;
#define CALL(N) stats_impl<N>(G, stats, W, H, r, lam, mode, st)
  HGF_DISPATCH(n, CALL)
#undef CALL
}

cudaError_t launch_coef(int n, const float* G, const float* stats, const float* vol, float* wbuf, int W, int H, int r,
                        int L, float lam0, cudaStream_t st) {
#define CALL(N) coef_impl<N>(G, stats, vol, wbuf, W, H, r, L, lam0, st)
  HGF_DISPATCH(n, CALL)
#undef CALL
}

cudaError_t launch_agg(int n, const AggArgs& a, cudaStream_t st) {
#define CALL(N) agg_impl<N>(a, st)
  HGF_DISPATCH(n, CALL)
#undef CALL
}

cudaError_t launch_fill_i64(int64_t* p, long long n, long long v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_fill_i64<<<grid_1d(n, 256), 256, 0, st>>>(p, n, v);
  return cudaGetLastError();
}

cudaError_t launch_unpack_keys(const int64_t* keys, int32_t* labels, float* cost, int W, int H, cudaStream_t st) {
  const long long HW = (long long)W * H;
  k_unpack_keys<<<grid_1d(HW, 256), 256, 0, st>>>(keys, labels, cost, HW);
  return cudaGetLastError();
}

}  // namespace hgf

namespace hgf {

// Must match v2::RMAX in hgf_slice_v2.cuh (register arrays of k_agg2 are sized by it).
constexpr int kV2RMax = 9;

// raw-guide channels x degree with a k_coef2 instantiation (hgf_inst2.cu): m, d <= 3, plus m = 4..6 at d = 1 and
// m = 4 at d = 2 (BASELINE config 5 sweeps m up to 20 at d = 1; beyond these the generic kernels run)
bool fast_path_ok(int m, int d, int r) {
  const bool md = (m >= 1 && m <= 3 && d >= 1 && d <= 3) || (d == 1 && m >= 4 && m <= 6) || (m == 4 && d == 2);
  return md && r >= 1 && r <= kV2RMax;
}

cudaError_t launch_coef_fast(int m, int d, const float* guide, const float* stats, const float* vol, float* wbuf, WLayout wo,
                             int W, int H, int r, int L, float lam0, cudaStream_t st) {
#define C2(M, D) return v2::coef2_impl<M, D>(guide, stats, vol, wbuf, wo, W, H, r, L, lam0, st)
  switch (m * 10 + d) {
    case 11: C2(1, 1); case 12: C2(1, 2); case 13: C2(1, 3);
    case 21: C2(2, 1); case 22: C2(2, 2); case 23: C2(2, 3);
    case 31: C2(3, 1); case 32: C2(3, 2); case 33: C2(3, 3);
    case 41: C2(4, 1); case 51: C2(5, 1); case 61: C2(6, 1); case 42: C2(4, 2);
    default: return cudaErrorInvalidValue;
  }
#undef C2
}

cudaError_t launch_agg_fast(int n, const AggArgs& a, cudaStream_t st) {
  switch (n) {
    case 1: return v2::agg2_impl<1>(a, st); case 2: return v2::agg2_impl<2>(a, st);
    case 3: return v2::agg2_impl<3>(a, st); case 4: return v2::agg2_impl<4>(a, st);
    case 5: return v2::agg2_impl<5>(a, st); case 6: return v2::agg2_impl<6>(a, st);
    case 7: return v2::agg2_impl<7>(a, st); case 8: return v2::agg2_impl<8>(a, st);
    case 9: return v2::agg2_impl<9>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hgf

namespace hgf {

template <int NC>
static cudaError_t agg3_r(int r, const void* tmap, const AggArgs& a, cudaStream_t st) {
  switch (r) {
    case 1: return v3::agg3_impl<NC, 1>(tmap, a, st);
    case 2: return v3::agg3_impl<NC, 2>(tmap, a, st);
    case 3: return v3::agg3_impl<NC, 3>(tmap, a, st);
    case 4: return v3::agg3_impl<NC, 4>(tmap, a, st);
    case 5: return v3::agg3_impl<NC, 5>(tmap, a, st);
    case 6: return v3::agg3_impl<NC, 6>(tmap, a, st);
    case 7: return v3::agg3_impl<NC, 7>(tmap, a, st);
    case 8: return v3::agg3_impl<NC, 8>(tmap, a, st);
    case 9: return v3::agg3_impl<NC, 9>(tmap, a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_agg_v3(int n, int r, const void* tmap, const AggArgs& a, cudaStream_t st) {
  switch (n) {
    case 1: return agg3_r<1>(r, tmap, a, st); case 2: return agg3_r<2>(r, tmap, a, st);
    case 3: return agg3_r<3>(r, tmap, a, st); case 4: return agg3_r<4>(r, tmap, a, st);
    case 5: return agg3_r<5>(r, tmap, a, st); case 6: return agg3_r<6>(r, tmap, a, st);
    case 7: return agg3_r<7>(r, tmap, a, st); case 8: return agg3_r<8>(r, tmap, a, st);
    case 9: return agg3_r<9>(r, tmap, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hgf

namespace hgf {

cudaError_t launch_coef_v3(int n, const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo,
                           int W, int H, int r, int L, float lam0, cudaStream_t st) {
#define C3(N) return v3::coef3_impl<N>(tm_vol, tm_g, stats, wbuf, wo, W, H, r, L, lam0, st)
  switch (n) {
    case 1: C3(1); case 2: C3(2); case 3: C3(3); case 4: C3(4); case 5: C3(5); case 6: C3(6);
    case 7: C3(7); case 8: C3(8); case 9: C3(9);
    default: return cudaErrorInvalidValue;
  }
#undef C3
}

cudaError_t launch_coef_v4(int n, const void* tm_vol, const void* tm_g, const float* stats, float* wbuf, WLayout wo,
                           int W, int H, int r, int L, cudaStream_t st) {
#define C4(N) return v4::coef4_impl<N>(tm_vol, tm_g, stats, wbuf, wo, W, H, r, L, st)
  switch (n) {
    case 1: C4(1); case 2: C4(2); case 3: C4(3); case 4: C4(4); case 5: C4(5); case 6: C4(6);
    default: return cudaErrorInvalidValue;
  }
#undef C4
}

}  // namespace hgf
