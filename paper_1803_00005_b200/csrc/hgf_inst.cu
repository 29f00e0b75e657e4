// Explicit instantiation of the per-channel-count kernels for n = HGF_N (set by the Makefile).
#include "hgf_kernels.cuh"
#include "hgf_slice_v2.cuh"
#include "hgf_stats_v3.cuh"

#ifndef HGF_N
#error "compile with -DHGF_N=<n>"
#endif

namespace hgf {
template cudaError_t stats_impl<HGF_N>(const float*, float*, int, int, int, double, int, cudaStream_t);
template cudaError_t coef_impl<HGF_N>(const float*, const float*, const float*, float*, int, int, int, int, float,
                                      cudaStream_t);
template cudaError_t agg_impl<HGF_N>(const AggArgs&, cudaStream_t);
namespace st3 {
template cudaError_t stats3_impl<HGF_N>(const float*, float*, double*, int, int, int, double, int, cudaStream_t);
}  // namespace st3
#if HGF_N <= 9
namespace v2 {
template cudaError_t agg2_impl<HGF_N>(const AggArgs&, cudaStream_t);
}  // namespace v2
#endif
}  // namespace hgf

#include "hgf_agg_v3.cuh"
#include "hgf_coef_v3.cuh"
#include "hgf_coef_v4.cuh"
#if HGF_N <= 9
namespace hgf {
namespace v3 {
template cudaError_t coef3_impl<HGF_N>(const void*, const void*, const float*, float*, WLayout, int, int, int, int,
                                       float, cudaStream_t);
}  // namespace v3
}  // namespace hgf
#endif
#if HGF_N <= 6
namespace hgf {
namespace v4 {
template cudaError_t coef4_impl<HGF_N>(const void*, const void*, const float*, float*, WLayout, int, int, int, int,
                                       cudaStream_t);
}  // namespace v4
}  // namespace hgf
#endif
#if HGF_N <= 9
namespace hgf {
namespace v3 {
template cudaError_t agg3_impl<HGF_N, 1>(const void*, const AggArgs&, cudaStream_t);
template cudaError_t agg3_impl<HGF_N, 2>(const void*, const AggArgs&, cudaStream_t);
template cudaError_t agg3_impl<HGF_N, 3>(const void*, const AggArgs&, cudaStream_t);
template cudaError_t agg3_impl<HGF_N, 4>(const void*, const AggArgs&, cudaStream_t);
template cudaError_t agg3_impl<HGF_N, 5>(const void*, const AggArgs&, cudaStream_t);
template cudaError_t agg3_impl<HGF_N, 6>(const void*, const AggArgs&, cudaStream_t);
template cudaError_t agg3_impl<HGF_N, 7>(const void*, const AggArgs&, cudaStream_t);
template cudaError_t agg3_impl<HGF_N, 8>(const void*, const AggArgs&, cudaStream_t);
template cudaError_t agg3_impl<HGF_N, 9>(const void*, const AggArgs&, cudaStream_t);
}  // namespace v3
#if HGF_N == 1
void agg3_box(int n, int R, int il, int* bx, int* by) {
  *bx = il ? (v3::TX + 2 * R + 31) / 32 * 32 : v3::box_pitch(v3::TX + 2 * R);
  *by = v3::agg3_ty(n) + 2 * R;
}
#endif
}  // namespace hgf
#endif

#include "hgf_stats_v2.cuh"
namespace hgf {
namespace st2 {
template cudaError_t stats2_impl<HGF_N>(const float*, float*, int, int, int, double, int, int, float, int, int,
                                        cudaStream_t);
}  // namespace st2
}  // namespace hgf

#if HGF_N <= 9
#include "hgf_stats_v4.cuh"
namespace hgf {
namespace st4 {
template cudaError_t stats4_impl<HGF_N>(const float*, float*, int, int, int, double, int, int, float, int, int,
                                        cudaStream_t);
template cudaError_t filter1_impl<HGF_N>(const float*, const float*, float*, WLayout, int, int, int, double, int,
                                         float, cudaStream_t);
}  // namespace st4
}  // namespace hgf
#include "hgf_stats_v5.cuh"
namespace hgf {
namespace st5 {
template cudaError_t stats_sel<HGF_N>(const float*, float*, int, int, int, double, int, int, float, int, int,
                                      cudaStream_t);
template cudaError_t filter1_sel<HGF_N>(const float*, const float*, float*, WLayout, int, int, int, double, int,
                                        float, cudaStream_t);
}  // namespace st5
}  // namespace hgf
#endif
