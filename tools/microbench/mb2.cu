// Microbenchmark 2: on-chip data-path throughput per SM on B200 (decides how the HGF box passes move data).
//   LDS.32 / LDS.64 / LDS.128 bandwidth, SHFL throughput, LDS + SHFL concurrently, L1-hit LDG bandwidth.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb2 mb2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 2048;

template <int V>
struct Vec;
template <> struct Vec<1> { using T = float; };
template <> struct Vec<2> { using T = float2; };
template <> struct Vec<4> { using T = float4; };

__device__ __forceinline__ float hsum(float a) { return a; }
__device__ __forceinline__ float hsum(float2 a) { return a.x + a.y; }
__device__ __forceinline__ float hsum(float4 a) { return (a.x + a.y) + (a.z + a.w); }

template <int V>
__global__ void k_lds(float* out, int stride) {
  using T = typename Vec<V>::T;
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
  __syncthreads();
  const T* sv = reinterpret_cast<const T*>(s);
  const int n = 8192 / V;
  float acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  int idx = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < ITER; ++i) {
    T a = sv[(idx) & (n - 1)];
    T b = sv[(idx + stride) & (n - 1)];
    T c = sv[(idx + 2 * stride) & (n - 1)];
    T d = sv[(idx + 3 * stride) & (n - 1)];
    acc0 += hsum(a); acc1 += hsum(b); acc2 += hsum(c); acc3 += hsum(d);
    idx += 4 * stride;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

__global__ void k_shfl(float* out) {
  float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
#pragma unroll 1
  for (int i = 0; i < ITER; ++i) {
    a += __shfl_down_sync(0xffffffffu, b, 1);
    b += __shfl_down_sync(0xffffffffu, c, 2);
    c += __shfl_down_sync(0xffffffffu, d, 3);
    d += __shfl_down_sync(0xffffffffu, a, 4);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

// LDS.32 and SHFL interleaved (are they separate data paths?)
__global__ void k_lds_shfl(float* out) {
  __shared__ float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
  __syncthreads();
  float a = threadIdx.x, b = a + 1, acc0 = 0, acc1 = 0;
  int idx = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < ITER; ++i) {
    acc0 += s[idx & 8191];
    a += __shfl_down_sync(0xffffffffu, b, 1);
    acc1 += s[(idx + 256) & 8191];
    b += __shfl_down_sync(0xffffffffu, a, 2);
    idx += 512;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + acc0 + acc1;
}

// L1-resident global loads (each CTA re-reads its own 32 KB slice)
__global__ void k_ldg_l1(const float* __restrict__ g, float* out) {
  const float* base = g + blockIdx.x * 8192;
  float acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  int idx = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < ITER; ++i) {
    acc0 += __ldg(base + (idx & 8191));
    acc1 += __ldg(base + ((idx + 256) & 8191));
    acc2 += __ldg(base + ((idx + 512) & 8191));
    acc3 += __ldg(base + ((idx + 768) & 8191));
    idx += 1024;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount, blocks = sms * 4, thr = 256;
  const double per_sm_clk = (double)sms * clk * 1e3;  // SM-cycles per second (all SMs)
  float *out, *g;
  cudaMalloc(&out, 64 << 20);
  cudaMalloc(&g, (size_t)blocks * 8192 * 4);
  cudaMemset(g, 0, (size_t)blocks * 8192 * 4);
  const double thr_total = (double)blocks * thr;
  for (int stride : {256, 512}) {
    float ms = timeit([&] { k_lds<1><<<blocks, thr>>>(out, stride); });
    printf("LDS.32  %.1f B/clk/SM\n", thr_total * ITER * 4 * 4 / (ms * 1e-3) / per_sm_clk);
    ms = timeit([&] { k_lds<2><<<blocks, thr>>>(out, stride); });
    printf("LDS.64  %.1f B/clk/SM\n", thr_total * ITER * 4 * 8 / (ms * 1e-3) / per_sm_clk);
    ms = timeit([&] { k_lds<4><<<blocks, thr>>>(out, stride); });
    printf("LDS.128 %.1f B/clk/SM\n", thr_total * ITER * 4 * 16 / (ms * 1e-3) / per_sm_clk);
  }
  float ms = timeit([&] { k_shfl<<<blocks, thr>>>(out); });
  printf("SHFL    %.2f warp-instr/clk/SM\n", thr_total / 32 * ITER * 4 / (ms * 1e-3) / per_sm_clk);
  ms = timeit([&] { k_lds_shfl<<<blocks, thr>>>(out); });
  printf("LDS+SHFL mixed: %.2f (LDS+SHFL) warp-instr/clk/SM  (1.0 = shared path, 2.0 = separate)\n",
         thr_total / 32 * ITER * 4 / (ms * 1e-3) / per_sm_clk);
  ms = timeit([&] { k_ldg_l1<<<blocks, thr>>>(g, out); });
  printf("LDG L1-hit %.1f B/clk/SM\n", thr_total * ITER * 4 * 4 / (ms * 1e-3) / per_sm_clk);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
