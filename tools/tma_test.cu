// Standalone check of the TMA + mbarrier helpers used by k_agg3 (hgf_agg_v3.cuh).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1803_00005_b200/csrc -o tools/tma_test tools/tma_test.cu
#include <cstdio>
#include <vector>

#include <cudaTypedefs.h>

#include "hgf_agg_v3.cuh"

using namespace hgf::v3;

__global__ void k_tma(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, float* out, int bx, int by, int bz, int x, int y, int z,
                      int variant) {
  extern __shared__ unsigned char smem_raw[];
  float* buf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    if (variant != 1) fence_barrier_init();
  }
  __syncthreads();
  const unsigned bytes = bx * by * bz * 4;
  if (variant == 2) {                      // barrier only: plain arrive, no TMA
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[0])) : "memory");
    mbar_wait(&bar[0], 0);
    return;
  }
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar[0], bytes);
    if (variant == 3) {
      uint64_t desc = reinterpret_cast<uint64_t>(&tm);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(buf)),
          "l"(desc), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar[0]))
          : "memory");
    } else {
      tma_load_3d(buf, variant == 4 ? gtm : &tm, x, y, z, &bar[0]);
    }
  }
  mbar_wait(&bar[0], 0);
  for (int i = threadIdx.x; i < bx * by * bz; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int W = 64, H = 48, P = 7;
  std::vector<float> h((size_t)W * H * P);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int bx = TBX, by = 28, bz = 4;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)P};
  const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  const cuuint32_t box[3] = {bx, by, bz};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaMalloc(&o, bx * by * bz * 4);
  CUtensorMap* gtm;
  cudaMalloc(&gtm, sizeof(CUtensorMap));
  cudaMemcpy(gtm, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  for (int variant : {VARIANT}) {
    cudaMemset(o, 0xff, bx * by * bz * 4);
    const int x = -2, y = -2, z = 1;
    k_tma<<<1, 128, bx * by * bz * 4 + 128>>>(tm, gtm, o, bx, by, bz, x, y, z, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> got((size_t)bx * by * bz);
    cudaMemcpy(got.data(), o, got.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int zz = 0; zz < bz; ++zz)
      for (int yy = 0; yy < by; ++yy)
        for (int xx = 0; xx < bx; ++xx) {
          const int gx = x + xx, gy = y + yy, gz = z + zz;
          const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H && gz < P;
          const float want = in ? h[((size_t)gz * H + gy) * W + gx] : 0.0f;
          if (got[((size_t)zz * by + yy) * bx + xx] != want) ++bad;
        }
    printf("variant %d mismatches %d\n", variant, bad);
  }
  return 0;
}
