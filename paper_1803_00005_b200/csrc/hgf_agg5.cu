// k_agg5 instantiations (n = 1..6, r = 1..9) and its launcher (hgf_agg_v5.cuh).
#include "hgf_agg_v5.cuh"

namespace hgf {
cudaError_t launch_agg_v5(int n, const void* tm_w, const void* tm_g, int W, int H, int r, int L, int label_base,
                          int labels_per_cta, unsigned long long* keys, float* filtered_out, cudaStream_t st) {
  switch (n) {
    case 1: return v5a::agg5_impl<1>(tm_w, tm_g, W, H, r, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 2: return v5a::agg5_impl<2>(tm_w, tm_g, W, H, r, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 3: return v5a::agg5_impl<3>(tm_w, tm_g, W, H, r, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 4: return v5a::agg5_impl<4>(tm_w, tm_g, W, H, r, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 5: return v5a::agg5_impl<5>(tm_w, tm_g, W, H, r, L, label_base, labels_per_cta, keys, filtered_out, st);
    case 6: return v5a::agg5_impl<6>(tm_w, tm_g, W, H, r, L, label_base, labels_per_cta, keys, filtered_out, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace hgf
