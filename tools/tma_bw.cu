// TMA load throughput vs the length of the contiguous inner run (tensor-map dim 0).
// Every case moves the same box volume (~84 x 42 x 7 floats) per request into a 2-deep SMEM ring,
// one CTA per SM, L2-resident source; prints GB/s for the whole GPU.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tma_bw.cu -o tools/tma_bw -lcuda
#include <cstdio>
#include <vector>

#include <cuda/ptx>
#include <cudaTypedefs.h>

namespace ptx = cuda::ptx;

template <int RANK>
__global__ void k_bw(const __grid_constant__ CUtensorMap tm, unsigned bytes, int iters, int e, int nxg, int bx1,
                     int stride_floats, int* sink) {
  extern __shared__ __align__(128) float buf[];
  __shared__ alignas(8) uint64_t bar[2];
  if (threadIdx.x != 0) return;
  ptx::mbarrier_init(&bar[0], 1);
  ptx::mbarrier_init(&bar[1], 1);
  ptx::fence_mbarrier_init(ptx::sem_release, ptx::scope_cluster);
  auto issue = [&](int it) {
    const int b = it & 1;
    const int l = (blockIdx.x + it) & 31;
    const int xg = (blockIdx.x * 7 + it * 3) % (nxg - bx1);
    const int y = it % 22;
    ptx::mbarrier_arrive_expect_tx(ptx::sem_release, ptx::scope_cta, ptx::space_shared, &bar[b], bytes);
    if (RANK == 4) {
      const int32_t c[4] = {l * e, xg, y, (it >> 1) & 1};
      ptx::cp_async_bulk_tensor(ptx::space_cluster, ptx::space_global, buf + b * stride_floats, &tm, c, &bar[b]);
    } else {
      const int32_t c[3] = {xg * 4, y, l * 8 + ((it >> 1) & 1)};
      ptx::cp_async_bulk_tensor(ptx::space_cluster, ptx::space_global, buf + b * stride_floats, &tm, c, &bar[b]);
    }
  };
  issue(0);
  issue(1);
  for (int it = 0; it < iters; ++it) {
    while (!ptx::mbarrier_try_wait_parity(&bar[it & 1], (it >> 1) & 1)) {
    }
    if (it + 2 < iters) issue(it + 2);
  }
  if (buf[5] == 12345.f) sink[0] = 1;
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  float* d;
  const size_t N = (size_t)64 << 20;  // 256 MB allocation; each case touches <= ~40 MB of it
  cudaMalloc(&d, N * 4);
  cudaMemset(d, 0, N * 4);
  int* sink;
  cudaMalloc(&sink, 4);
  const int iters = 400;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int es[] = {4, 8, 16, 32, 0};
  for (int e : es) {
    CUtensorMap tm;
    CUresult r;
    unsigned bytes;
    int nxg, bx1;
    if (e > 0) {
      nxg = 512 / e;
      bx1 = (84 + e - 1) / e;
      const cuuint64_t dims[4] = {(cuuint64_t)32 * e, (cuuint64_t)nxg, 64, 8};
      const cuuint64_t strides[3] = {(cuuint64_t)32 * e * 4, (cuuint64_t)32 * e * 4 * nxg,
                                     (cuuint64_t)32 * e * 4 * nxg * 64};
      const cuuint32_t box[4] = {(cuuint32_t)e, (cuuint32_t)bx1, 42, 7};
      const cuuint32_t es1[4] = {1, 1, 1, 1};
      r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es1, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      bytes = (unsigned)(e * bx1 * 42 * 7 * 4);
    } else {
      nxg = 128;
      bx1 = 21;
      const cuuint64_t dims[3] = {512, 64, 256};
      const cuuint64_t strides[2] = {512 * 4, 512 * 64 * 4};
      const cuuint32_t box[3] = {84, 42, 7};
      const cuuint32_t es1[3] = {1, 1, 1};
      r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es1, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      bytes = 84 * 42 * 7 * 4;
    }
    if (r != CUDA_SUCCESS) {
      printf("e=%d encode failed %d\n", e, (int)r);
      continue;
    }
    const int stride_floats = ((int)(bytes / 4) + 31) / 32 * 32;
    const size_t smem = (size_t)2 * stride_floats * 4;
    auto kern = (e > 0) ? k_bw<4> : k_bw<3>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      kern<<<148, 32, smem>>>(tm, bytes, iters, e, nxg, bx1, stride_floats, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t err = cudaGetLastError();
      const double gbs = 148.0 * iters * bytes / (ms * 1e-3) / 1e9;
      const double runs = 148.0 * iters * bytes / (e > 0 ? e * 4 : 336) / (ms * 1e-3) / 148 / 1.965e9;
      if (rep == 1)
        printf("inner run %4d B: box %u B  %.3f ms  %.0f GB/s  %.2f runs/clk/SM  %s\n", e > 0 ? e * 4 : 336, bytes, ms,
               gbs, runs, cudaGetErrorString(err));
    }
  }
  return 0;
}
