// k_coef5 instantiations (raw guide channels m <= 3, degree d <= 3, n = m d <= 6, r = 1..9) and its launcher
// (hgf_coef_v5.cuh).
#include "hgf_coef_v5.cuh"

namespace hgf {
bool coef5_ok(int m, int d, int r) { return m >= 1 && m <= 3 && d >= 1 && d <= 3 && m * d <= kCoef5MaxN && r >= 1 && r <= 9; }

cudaError_t launch_coef_v5(int m, int d, const void* tm_vol, const void* tm_i, const float* stats, float* wbuf,
                           WLayout wo, int W, int H, int r, int L, int Lmodel, cudaStream_t st) {
#define C5(M, D) \
  if (m == M && d == D) return v5::coef5_impl<M, D>(tm_vol, tm_i, stats, wbuf, wo, W, H, r, L, Lmodel, st)
  C5(1, 1); C5(1, 2); C5(1, 3); C5(2, 1); C5(2, 2); C5(2, 3); C5(3, 1); C5(3, 2);
#undef C5
  return cudaErrorInvalidValue;
}
}  // namespace hgf
