// k_agg6 instantiations (n = 1..6, r = 1..9) and its launcher (hgf_agg_v6.cuh).
#include "hgf_agg_v6.cuh"

namespace hgf {
namespace {
template <int N>
cudaError_t agg6_r(int r, const void* tm, const AggArgs& a, cudaStream_t st) {
  switch (r) {
    case 1: return v6a::agg6_launch<N, 1>(tm, a, st); case 2: return v6a::agg6_launch<N, 2>(tm, a, st);
    case 3: return v6a::agg6_launch<N, 3>(tm, a, st); case 4: return v6a::agg6_launch<N, 4>(tm, a, st);
    case 5: return v6a::agg6_launch<N, 5>(tm, a, st); case 6: return v6a::agg6_launch<N, 6>(tm, a, st);
    case 7: return v6a::agg6_launch<N, 7>(tm, a, st); case 8: return v6a::agg6_launch<N, 8>(tm, a, st);
    case 9: return v6a::agg6_launch<N, 9>(tm, a, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t launch_agg_v6(int n, int r, const void* tm, const AggArgs& a, cudaStream_t st) {
  switch (n) {
    case 1: return agg6_r<1>(r, tm, a, st); case 2: return agg6_r<2>(r, tm, a, st);
    case 3: return agg6_r<3>(r, tm, a, st); case 4: return agg6_r<4>(r, tm, a, st);
    case 5: return agg6_r<5>(r, tm, a, st); case 6: return agg6_r<6>(r, tm, a, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace hgf
