// Explicit instantiation of the per-channel-count kernels for n = HGF_N (set by the Makefile).
#include "hgf_kernels.cuh"
#include "hgf_slice_v2.cuh"

#ifndef HGF_N
#error "compile with -DHGF_N=<n>"
#endif

namespace hgf {
template cudaError_t stats_impl<HGF_N>(const float*, float*, int, int, int, double, int, cudaStream_t);
template cudaError_t coef_impl<HGF_N>(const float*, const float*, const float*, float*, int, int, int, int, float,
                                      cudaStream_t);
template cudaError_t agg_impl<HGF_N>(const AggArgs&, cudaStream_t);
#if HGF_N <= 9
namespace v2 {
template cudaError_t agg2_impl<HGF_N>(const AggArgs&, cudaStream_t);
}  // namespace v2
#endif
}  // namespace hgf
