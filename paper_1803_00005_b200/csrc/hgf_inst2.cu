// Explicit instantiation of the v2 coefficient kernel for raw-guide channels HGF_M and degree HGF_D.
#include "hgf_slice_v2.cuh"

#if !defined(HGF_M) || !defined(HGF_D)
#error "compile with -DHGF_M=<m> -DHGF_D=<d>"
#endif

namespace hgf {
namespace v2 {
template cudaError_t coef2_impl<HGF_M, HGF_D>(const float*, const float*, const float*, float*, WLayout, int, int, int, int,
                                              float, cudaStream_t);
}  // namespace v2
}  // namespace hgf
