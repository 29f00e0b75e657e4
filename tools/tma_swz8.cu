// Does a rank-5 TMA load of the 8-pixel label-interleaved layout (8 px, 32 labels, x groups, y, planes)
// with 32-byte inner runs land the same [plane][y][x] tile, and under which shared-memory address
// function, for SWIZZLE_NONE / 32B / 64B?  Checks the candidates f, f ^ ((f >> 3) & 4) and
// f ^ ((f >> 3) & 12) (float index f from a 1 KB aligned buffer) and reports mismatches for each.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma_swz8 tools/tma_swz8.cu -lcuda
#include <cstdio>
#include <vector>

#include <cuda/ptx>
#include <cudaTypedefs.h>

namespace ptx = cuda::ptx;

__global__ void k_load(float* out, int n, const __grid_constant__ CUtensorMap tm, int lab, int gx, int y, int p,
                       unsigned bytes) {
  extern __shared__ unsigned char raw[];
  float* buf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbarrier_init(&bar, 1);
    ptx::fence_mbarrier_init(ptx::sem_release, ptx::scope_cluster);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbarrier_arrive_expect_tx(ptx::sem_release, ptx::scope_cta, ptx::space_shared, &bar, bytes);
    const int32_t c[5] = {0, lab, gx, y, p};
    ptx::cp_async_bulk_tensor(ptx::space_cluster, ptx::space_global, buf, &tm, c, &bar);
  }
  while (!ptx::mbarrier_try_wait_parity(&bar, 0)) {
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int G = 8, NL = 32, W = 256, H = 40, P = 4, XG = W / G;
  const int BX = 96, BY = 12, BP = 2;  // box: (8, 1, BX/8, BY, BP)
  std::vector<float> h((size_t)G * NL * XG * H * P);
  // value = logical id of (label, plane, y, x): encodes everything so misplacement is visible
  for (int p = 0; p < P; ++p)
    for (int y = 0; y < H; ++y)
      for (int g = 0; g < XG; ++g)
        for (int l = 0; l < NL; ++l)
          for (int i = 0; i < G; ++i)
            h[((((size_t)p * H + y) * XG + g) * NL + l) * G + i] = (float)(((p * 64 + l) * 64 + y) * 1024 + g * G + i);
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const CUtensorMapSwizzle modes[3] = {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_SWIZZLE_64B};
  const char* names[3] = {"none", "32B", "64B"};
  const int n = BX * BY * BP;
  cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, n * 4 + 2048);
  for (int m = 0; m < 3; ++m) {
    CUtensorMap tm;
    const cuuint64_t dims[5] = {(cuuint64_t)G, (cuuint64_t)NL, (cuuint64_t)XG, (cuuint64_t)H, (cuuint64_t)P};
    const cuuint64_t strides[4] = {(cuuint64_t)G * 4, (cuuint64_t)G * NL * 4, (cuuint64_t)G * NL * 4 * XG,
                                   (cuuint64_t)G * NL * 4 * XG * H};
    const cuuint32_t box[5] = {(cuuint32_t)G, 1, (cuuint32_t)(BX / G), (cuuint32_t)BY, (cuuint32_t)BP};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        modes[m], CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("swizzle %s: encode failed (%d)\n", names[m], (int)r);
      continue;
    }
    const int lab = 5, gx = -1, y0 = -3, p0 = 1;
    cudaMemset(o, 0xff, n * 4);
    k_load<<<1, 256, n * 4 + 2048>>>(o, n, tm, lab, gx, y0, p0, (unsigned)(n * 4));
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("swizzle %s: %s\n", names[m], cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> s(n);
    cudaMemcpy(s.data(), o, n * 4, cudaMemcpyDeviceToHost);
    int bad[3] = {0, 0, 0};
    for (int f = 0; f < n; ++f) {
      const int xx = f % BX, yy = (f / BX) % BY, pp = f / (BX * BY);
      const int x = gx * G + xx, y = y0 + yy, p = p0 + pp;
      const bool oob = x < 0 || x >= W || y < 0 || y >= H;
      const float want = oob ? 0.0f : (float)(((p * 64 + lab) * 64 + y) * 1024 + x);
      const int cand[3] = {f, f ^ ((f >> 3) & 4), f ^ ((f >> 3) & 12)};
      for (int c = 0; c < 3; ++c) bad[c] += s[cand[c]] != want;
    }
    printf("swizzle %s: mismatches identity %d, f^((f>>3)&4) %d, f^((f>>3)&12) %d (of %d)\n", names[m], bad[0], bad[1],
           bad[2], n);
  }
  return 0;
}
