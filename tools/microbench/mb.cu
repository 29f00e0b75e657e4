// Microbenchmarks used to pick the HGF kernel design on B200 (sm_100a).
// Measures: FP32 FFMA / FFMA2 / FADD throughput, FP64 DFMA, SMEM LDS bandwidth,
// L2-resident and HBM read bandwidth, DSMEM (cluster) read bandwidth.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb mb.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITER = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// three-distinct-register form (a, b vary per thread)
__global__ void k_ffma3(float* out, const float* ab) {
  float a = ab[threadIdx.x & 31], b = ab[32 + (threadIdx.x & 31)];
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma2(float* out, const float* ab) {
  float2 a = make_float2(ab[threadIdx.x & 31], ab[(threadIdx.x + 1) & 31]);
  float2 b = make_float2(ab[32 + (threadIdx.x & 31)], ab[32 + ((threadIdx.x + 3) & 31)]);
  float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, threadIdx.x), x2 = make_float2(3, 4), x3 = make_float2(5, 6);
  float2 x4 = make_float2(7, 8), x5 = make_float2(9, 10), x6 = make_float2(11, 12), x7 = make_float2(13, 14);
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = __ffma2_rn(x0, a, b); x1 = __ffma2_rn(x1, a, b); x2 = __ffma2_rn(x2, a, b); x3 = __ffma2_rn(x3, a, b);
      x4 = __ffma2_rn(x4, a, b); x5 = __ffma2_rn(x5, a, b); x6 = __ffma2_rn(x6, a, b); x7 = __ffma2_rn(x7, a, b);
    }
  }
  float2 s = make_float2(x0.x + x1.x + x2.x + x3.x + x4.x + x5.x + x6.x + x7.x, x0.y + x1.y + x2.y + x3.y + x4.y + x5.y + x6.y + x7.y);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s.x + s.y;
}
__global__ void k_fadd(float* out, const float* ab) {
  float a = ab[threadIdx.x & 31];
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 += a; x1 -= a; x2 += a; x3 -= a; x4 += a; x5 -= a; x6 += a; x7 -= a;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_fadd2(float* out, const float* ab) {
  float2 a = make_float2(ab[threadIdx.x & 31], ab[(threadIdx.x + 5) & 31]);
  float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, threadIdx.x), x2 = make_float2(3, 4), x3 = make_float2(5, 6);
  float2 x4 = make_float2(7, 8), x5 = make_float2(9, 10), x6 = make_float2(11, 12), x7 = make_float2(13, 14);
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = __fadd2_rn(x0, a); x1 = __fadd2_rn(x1, a); x2 = __fadd2_rn(x2, a); x3 = __fadd2_rn(x3, a);
      x4 = __fadd2_rn(x4, a); x5 = __fadd2_rn(x5, a); x6 = __fadd2_rn(x6, a); x7 = __fadd2_rn(x7, a);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0.x + x1.x + x2.x + x3.x + x4.x + x5.x + x6.x + x7.x + x0.y + x7.y;
}
__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITER / 8; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// SMEM read bandwidth: LDS.32 conflict-free
__global__ void k_lds32(float* out) {
  __shared__ float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
  __syncthreads();
  float acc = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += s[(idx + j * 256) & 8191];
    idx += 32;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_lds128(float* out) {
  __shared__ float4 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i, i, i);
  __syncthreads();
  float acc = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < ITER / 4; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { float4 v = s[(idx + j * 256) & 2047]; acc += v.x + v.w; }
    idx += 32;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
// streaming read of n float4 (grid-stride)
__global__ void k_read(const float4* __restrict__ p, size_t n, float* out, int reps) {
  float acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(p + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.f) out[0] = acc;
}
// DSMEM read bandwidth (cluster of 2): each CTA reads peer's smem
__global__ void __cluster_dims__(2, 1, 1) k_dsmem(float* out) {
  __shared__ float4 s[2048];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i, i, i);
  cl.sync();
  float4* peer = cl.map_shared_rank(s, cl.block_rank() ^ 1);
  float acc = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < ITER / 16; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { float4 v = peer[(idx + j * 256) & 2047]; acc += v.x + v.w; }
    idx += 32;
  }
  cl.sync();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d L2 %d MB smem/SM %zu clock %d MHz\n", prop.name, sms, prop.l2CacheSize >> 20,
         prop.sharedMemPerMultiprocessor, clk_khz / 1000);
  float *out, *ab; double* dout;
  CK(cudaMalloc(&out, 64 << 20)); CK(cudaMalloc(&dout, 64 << 20)); CK(cudaMalloc(&ab, 256));
  CK(cudaMemset(ab, 0, 256));
  int blocks = sms * 8, thr = 256;
  double nthr = (double)blocks * thr;
  float ms;
  ms = timeit([&] { k_ffma<<<blocks, thr>>>(out, 0.999f, 0.001f); });
  printf("FFMA(imm-ish)  %.1f TFLOP/s\n", nthr * ITER * 32 * 2 / ms / 1e9);
  ms = timeit([&] { k_ffma3<<<blocks, thr>>>(out, ab); });
  printf("FFMA(3reg)     %.1f TFLOP/s\n", nthr * ITER * 32 * 2 / ms / 1e9);
  ms = timeit([&] { k_ffma2<<<blocks, thr>>>(out, ab); });
  printf("FFMA2          %.1f TFLOP/s\n", nthr * ITER * 32 * 4 / ms / 1e9);
  ms = timeit([&] { k_fadd<<<blocks, thr>>>(out, ab); });
  printf("FADD           %.1f TFLOP/s (adds)\n", nthr * ITER * 32 / ms / 1e9);
  ms = timeit([&] { k_fadd2<<<blocks, thr>>>(out, ab); });
  printf("FADD2          %.1f TFLOP/s (adds)\n", nthr * ITER * 32 * 2 / ms / 1e9);
  ms = timeit([&] { k_dfma<<<blocks, thr>>>(dout, 0.999, 0.001); });
  printf("DFMA           %.2f TFLOP/s\n", nthr * (ITER / 8) * 32 * 2 / ms / 1e9);
  ms = timeit([&] { k_lds32<<<blocks, thr>>>(out); });
  printf("LDS.32         %.1f TB/s  (%.1f B/clk/SM @%d MHz)\n", nthr * ITER * 8 * 4 / ms / 1e9,
         nthr * ITER * 8 * 4 / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
  ms = timeit([&] { k_lds128<<<blocks, thr>>>(out); });
  printf("LDS.128        %.1f TB/s  (%.1f B/clk/SM)\n", nthr * (ITER / 4) * 8 * 16 / ms / 1e9,
         nthr * (ITER / 4) * 8 * 16 / (ms * 1e-3) / sms / (clk_khz * 1e3));
  ms = timeit([&] { k_dsmem<<<blocks, thr>>>(out); });
  printf("DSMEM LD.128   %.1f TB/s  (%.1f B/clk/SM)\n", nthr * (ITER / 16) * 8 * 16 / ms / 1e9,
         nthr * (ITER / 16) * 8 * 16 / (ms * 1e-3) / sms / (clk_khz * 1e3));
  for (size_t mb : {8, 32, 64, 96, 4096}) {
    size_t bytes = mb << 20;
    float4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
    int reps = mb >= 1024 ? 1 : 20;
    ms = timeit([&] { k_read<<<sms * 8, 512>>>(buf, bytes / 16, out, reps); });
    printf("read %5zu MB x%d: %.2f TB/s\n", mb, reps, (double)bytes * reps / ms / 1e9);
    cudaFree(buf);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
