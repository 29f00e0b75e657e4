// Standalone check of the tcgen05 pieces a banded-ones horizontal box sum needs (sm_100a):
//   D[m][n] = sum_c A[m][c] * B[n][c],  A = band of ones (A[m][c] = 1 for m <= c <= m + 2R) in TMEM,
//   B = data in SMEM (K-major, no swizzle, core matrices 8 rows x 16 B, custom LBO), split hi/lo tf32,
//   D in TMEM (fp32), read back with tcgen05.ld.32x32b.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/umma_test.cu -o tools/umma_test
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 112, R = 9, KC = 152;  // KC: K columns (multiple of 8), >= M + 2R
constexpr int LBO = (N / 8) * 128 + 16;            // bytes between 16-B K chunks (+16: conflict-free lanes)
constexpr int SBO = 128;                           // bytes between 8-row groups
constexpr int BBYTES = (KC / 4) * LBO;             // one of hi / lo

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void k_test(const float* __restrict__ bin, float* __restrict__ dout, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* bhi = reinterpret_cast<float*>(sm);
  float* blo = reinterpret_cast<float*>(sm + BBYTES);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // B: element (n, c) at (c/4)*LBO + (n/8)*SBO + (n%8)*16 + (c%4)*4 bytes; hi = tf32(x), lo = x - hi
  for (int e = tid; e < N * KC; e += blockDim.x) {
    const int n = e / KC, c = e % KC;
    const float x = bin[e];
    uint32_t hb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
    const float hi = __uint_as_float(hb);
    const float lo = x - hi;
    const int off = ((c / 4) * LBO + (n / 8) * SBO + (n % 8) * 16 + (c % 4) * 4) / 4;
    bhi[off] = hi;
    blo[off] = lo;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  const uint32_t d_col = tb, a_col = tb + 256;    // D: columns [0, 112), A: columns [256, 256 + KC)
  // A (band) into TMEM: thread = lane m (4 warps cover the 4 lane quadrants)
  {
    const int m = tid;  // 128 threads
    const uint32_t lane_addr = ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < KC; c0 += 8) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + j;
        v[j] = __float_as_uint((c >= m && c <= m + 2 * R) ? 1.0f : 0.0f);
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                       lane_addr + a_col + c0),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  // generic-proxy SMEM writes -> visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const int nparts = mode == 0 ? 1 : 2;
    for (int part = 0; part < nparts; ++part) {
      const uint32_t base = smem_u32(part == 0 ? bhi : blo);
      for (int s = 0; s < KC / 8; ++s) {
        const uint64_t bd = sdesc(base + 2 * s * LBO, LBO, SBO);
        const uint32_t acc = (part > 0 || s > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_col),
            "r"(a_col + 8 * s), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const uint32_t lane_addr = ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(lane_addr + d_col + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 8; ++j) dout[tid * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

int main() {
  std::vector<float> b((size_t)N * KC);
  srand(1);
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < KC; ++c) {
      const float u = (float)rand() / RAND_MAX;
      b[(size_t)n * KC + c] = (c < M + 2 * R) ? (0.1f + 3.0f * u) * (n % 3 == 0 ? 1000.0f : 1.0f) : 0.0f;
    }
  float *db, *dd;
  cudaMalloc(&db, b.size() * 4);
  cudaMalloc(&dd, (size_t)M * N * 4);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 2 * BBYTES;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dd, 0, (size_t)M * N * 4);
    k_test<<<1, 128, smem>>>(db, dd, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> d((size_t)M * N);
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    int bad = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int c = m; c <= m + 2 * R; ++c) ref += b[(size_t)n * KC + c];
        const double err = std::fabs(d[(size_t)m * N + n] - ref) / std::fabs(ref);
        if (err > worst) worst = err;
        if (err > 1e-3 && bad < 5) {
          printf("  m=%d n=%d got %.6f want %.6f\n", m, n, d[(size_t)m * N + n], ref);
          ++bad;
        }
      }
    printf("mode %d (%s): max rel err %.3e\n", mode, mode == 0 ? "hi only" : "hi + lo", worst);
  }
  return 0;
}
