// k_agg6 instantiations and its launcher (hgf_agg_v6.cuh): 8-pixel owners (D = 0) for n = 1..6 here, 16-pixel
// raw-channel owners (D = d, m <= 3) in hgf_agg6w.cu.
#include <cstdlib>
#include <cstring>

#include "hgf_agg_v6.cuh"

namespace hgf {
cudaError_t launch_agg_v6w(int m, int d, int r, const void* tm, const AggArgs& a, cudaStream_t st);

cudaError_t launch_agg_v6(int m, int d, int r, const void* tm, const AggArgs& a, cudaStream_t st) {
  // 16-pixel raw-channel owners where they apply (m <= 3); HGF_AGG6_KX=8 keeps the 8-pixel owners (A/B, tests)
  const char* kx = std::getenv("HGF_AGG6_KX");
  if (m <= 3 && !(kx && !strcmp(kx, "8"))) return launch_agg_v6w(m, d, r, tm, a, st);
  switch (m * d) {
    case 1: return agg6_r<1, 0>(r, tm, a, st); case 2: return agg6_r<2, 0>(r, tm, a, st);
    case 3: return agg6_r<3, 0>(r, tm, a, st); case 4: return agg6_r<4, 0>(r, tm, a, st);
    case 5: return agg6_r<5, 0>(r, tm, a, st); case 6: return agg6_r<6, 0>(r, tm, a, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace hgf
