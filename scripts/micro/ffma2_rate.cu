// Microbenchmark: issue/throughput of packed FFMA2 (fma.rn.f32x2) vs scalar FFMA on sm_100a.
// Each thread runs 8 independent chains; reports lane-FMAs per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__global__ void k_scalar(float* out, float b, float c, int iters) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __fmaf_rn(x[i], b, c);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_packed(float* out, float b, float c, int iters) {
  uint64_t x[4];
  float2 bb = make_float2(b, b), cc = make_float2(c, c);
  uint64_t B = *reinterpret_cast<uint64_t*>(&bb), C = *reinterpret_cast<uint64_t*>(&cc);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v = make_float2(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
    x[i] = *reinterpret_cast<uint64_t*>(&v);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = ffma2(x[i], B, C);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v = *reinterpret_cast<float2*>(&x[i]);
    s += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int nt = 256, nb = sms * 8, iters = 1 << 14;
  float* out;
  cudaMalloc(&out, sizeof(float) * nt * nb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) k_scalar<<<nb, nt>>>(out, 0.999f, 1e-3f, iters);
      else k_packed<<<nb, nt>>>(out, 0.999f, 1e-3f, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fmas = double(nt) * nb * iters * 8;
      double per_sm_clk = fmas / (ms * 1e-3) / sms / (clk * 1e3);
      if (rep == 2) printf("%s: %.3f ms, %.1f lane-FMA per SM per clock (at %d MHz max)\n",
                           v ? "FFMA2 packed" : "FFMA scalar", ms, per_sm_clk, clk / 1000);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
