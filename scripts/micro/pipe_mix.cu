// Microbenchmark: throughput of FFMA2 / FFMA / IMAD.WIDE.U32 alone and mixed on sm_100a,
// to see which FP32 pipes (fmaheavy / fmalite) each uses. 8 independent chains per thread.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, float b, float c, uint32_t m, int iters) {
  float2 x[4];
  float y[8];
  uint32_t u[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[i] = make_float2(threadIdx.x * 1e-3f + i, threadIdx.x * 2e-3f + i);
    u[i] = threadIdx.x * 7 + i;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = threadIdx.x * 1e-3f + i;
  const float2 B = make_float2(b, b), C = make_float2(c, c);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (MODE == 0 || MODE == 3) x[i] = __ffma2_rn(x[i], B, C);                 // FFMA2
      if (MODE == 1 || MODE == 4) {                                              // 2 FFMA
        y[2 * i] = __fmaf_rn(y[2 * i], b, c);
        y[2 * i + 1] = __fmaf_rn(y[2 * i + 1], b, c);
      }
      if (MODE == 2 || MODE == 3 || MODE == 4) {                                 // IMAD.WIDE
        const uint64_t p = static_cast<uint64_t>(m) * u[i];
        u[i] = static_cast<uint32_t>(p >> 32) ^ static_cast<uint32_t>(p);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += x[i].x + x[i].y + (float)u[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, float* out, int sms, int clk) {
  const int nt = 256, nb = sms * 8, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<MODE><<<nb, nt>>>(out, 0.999f, 1e-3f, 0xD2511F53u, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double warp_iters = double(nt / 32) * nb * iters * 4;  // per-chain-step warp instructions (x4 chains)
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s %.3f ms  %.2f chain-steps per SM-clock (one step = 1 FFMA2 | 2 FFMA | 1 IMAD.WIDE + LOP)\n", name, ms,
         warp_iters / sms / cyc);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * 256 * sms * 8);
  run<0>("FFMA2 only", out, sms, clk);
  run<1>("2x FFMA only", out, sms, clk);
  run<2>("IMAD.WIDE only", out, sms, clk);
  run<3>("FFMA2 + IMAD.WIDE", out, sms, clk);
  run<4>("2x FFMA + IMAD.WIDE", out, sms, clk);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
