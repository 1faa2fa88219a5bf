// Microbenchmark: issue cost of the 32x32->64 products Philox needs on sm_100a:
// IMAD.WIDE.U32 vs IMAD.HI.U32 + IMAD (lo) vs lo-only / hi-only. 4 chains per thread.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(uint32_t* out, uint32_t m, int iters) {
  uint32_t u[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) u[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (MODE == 0) {
        const uint64_t p = static_cast<uint64_t>(m) * u[i];
        u[i] = static_cast<uint32_t>(p >> 32) ^ static_cast<uint32_t>(p);
      } else if (MODE == 1) {
        uint32_t hi, lo;
        asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(u[i]), "r"(m));
        asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(u[i]), "r"(m));
        u[i] = hi ^ lo;
      } else if (MODE == 2) {
        u[i] = (u[i] * m) ^ 0x9E3779B9u;
      } else if (MODE == 3) {
        u[i] = __umulhi(u[i], m) ^ 0x9E3779B9u;
      } else {
        u[i] = (u[i] + m) ^ 0x9E3779B9u;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = u[0] ^ u[1] ^ u[2] ^ u[3];
}

template <int MODE>
void run(const char* name, uint32_t* out, int sms, int clk) {
  const int nt = 256, nb = sms * 8, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<MODE><<<nb, nt>>>(out, 0xD2511F53u, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double steps = double(nt / 32) * nb * iters * 4;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-34s %.3f ms  %.3f warp-steps per SMSP-clock\n", name, ms, steps / (sms * 4) / cyc);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, sizeof(uint32_t) * 256 * sms * 8);
  run<0>("IMAD.WIDE.U32 + LOP3", out, sms, clk);
  run<1>("IMAD.HI.U32 + IMAD + LOP3", out, sms, clk);
  run<2>("IMAD (lo) + LOP3", out, sms, clk);
  run<3>("IMAD.HI.U32 + LOP3", out, sms, clk);
  run<4>("IADD + LOP3", out, sms, clk);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
