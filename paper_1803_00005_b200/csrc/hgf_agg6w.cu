// k_agg6 with 16-pixel raw-channel owners (D = d >= 1, m <= 3, n = m d <= 6; hgf_agg_v6.cuh).
#include "hgf_agg_v6.cuh"

namespace hgf {
cudaError_t launch_agg_v6w(int m, int d, int r, const void* tm, const AggArgs& a, cudaStream_t st) {
#define A6(M, D) \
  if (m == M && d == D) return agg6_r<M * D, D>(r, tm, a, st)
  A6(1, 1); A6(2, 1); A6(3, 1);
  A6(1, 2); A6(2, 2); A6(3, 2);
  A6(1, 3); A6(2, 3);
#undef A6
  return cudaErrorInvalidValue;
}
}  // namespace hgf
