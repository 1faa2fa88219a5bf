// calib.cu — row f2: the e(T) calibration curve built on the GPU (reading R2: the T <-> e
// relation that the energy matching of PAPER.md:90 inverts; construction deferred by the
// paper to [mz-dth18]).
//
// K temperatures x `reps` replicas of an open L x L MPR lattice with every site free,
// started ordered (phi = pi), are swept together: checkerboard Metropolis with a
// symmetric local move phi' = phi + step*(2u-1), step = min(2pi, 3 sqrt T), rejected
// outside [0, 2pi] (same Gibbs law as the conditional simulation's independence proposal,
// far faster to equilibrate at low T). After every sweep each lattice's whole-grid energy
// is summed in exact fixed point (ARITH §J). The host averages the measurement sweeps,
// averages replicas, and makes the curve strictly increasing (pool-adjacent-violators,
// then one fp32 ulp between ties) — the recipe of scripts/make_calibration.py, written
// independently here.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_math.cuh"
#include "internal.cuh"

namespace mpr {

namespace {

struct CalibLattice {
  float beta;   // 1 / T (fp32 division)
  float step;   // local-move half-width
  uint32_t rep; // replica index: the Philox realization counter
};

__device__ __forceinline__ float cos_q(float q, float d) { return cos_spec(__fmul_rn(q, d)); }

// One colour half of sweep `sweep` on every lattice; one thread per (lattice, site of colour).
__global__ void __launch_bounds__(256) k_calib_half(float* __restrict__ phi, const CalibLattice* __restrict__ lat,
                                                    int nlat, int L, int colour, uint32_t sweep, uint32_t k0,
                                                    uint32_t k1, float q) {
  const int half = (L + 1) / 2;
  const int64_t per_lat = static_cast<int64_t>(L) * half;
  const int64_t total = per_lat * nlat;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int l = static_cast<int>(t / per_lat);
    const int64_t rem = t - static_cast<int64_t>(l) * per_lat;
    const int r = static_cast<int>(rem / half);
    const int c = 2 * static_cast<int>(rem - static_cast<int64_t>(r) * half) + ((r + colour) & 1);
    if (c >= L) continue;
    float* P = phi + static_cast<int64_t>(l) * L * L;
    const int64_t i = static_cast<int64_t>(r) * L + c;
    const CalibLattice cl = lat[l];
    const Words4 w = philox4x32_10(static_cast<uint32_t>(i), sweep, cl.rep, 3u, k0, k1);
    const float cur = P[i];
    const float prop = __fadd_rn(cur, __fmul_rn(cl.step, __fsub_rn(__fmul_rn(2.0f, u24(w.w0)), 1.0f)));
    if (prop < 0.0f || prop > kTwoPiF) continue;
    const int nr[4] = {r - 1, r + 1, r, r};
    const int nc[4] = {c, c, c - 1, c + 1};
    float s_cur = 0.0f, s_new = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (nr[k] < 0 || nr[k] >= L || nc[k] < 0 || nc[k] >= L) continue;
      const float pj = P[static_cast<int64_t>(nr[k]) * L + nc[k]];
      s_cur = __fadd_rn(s_cur, cos_q(q, __fsub_rn(cur, pj)));
      s_new = __fadd_rn(s_new, cos_q(q, __fsub_rn(prop, pj)));
    }
    const float dE = __fmul_rn(1.0f, __fsub_rn(s_cur, s_new));
    const bool accept = (dE <= 0.0f) || (u24(w.w1) < exp_spec(-__fmul_rn(dE, cl.beta)));
    if (accept) P[i] = prop;
  }
}

// Fixed-point whole-grid bond sum of every lattice (ARITH §J); one CTA row per lattice.
__global__ void __launch_bounds__(256) k_calib_energy(const float* __restrict__ phi, int L, float q,
                                                      long long* __restrict__ out) {
  const int l = blockIdx.y;
  const float* P = phi + static_cast<int64_t>(l) * L * L;
  long long acc = 0;
  const int64_t n = static_cast<int64_t>(L) * L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / L), c = static_cast<int>(i - static_cast<int64_t>(r) * L);
    if (c + 1 < L) acc += __float2ll_rn(__fmul_rn(cos_q(q, __fsub_rn(P[i], P[i + 1])), 0x1p32f));
    if (r + 1 < L) acc += __float2ll_rn(__fmul_rn(cos_q(q, __fsub_rn(P[i], P[i + L])), 0x1p32f));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc)
    atomicAdd(reinterpret_cast<unsigned long long*>(out + l), static_cast<unsigned long long>(acc));
}

__global__ void k_fill(float* __restrict__ p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace

cudaError_t run_calibration(const float* T_host, int K, int L, float q, int n_eq, int n_meas, int reps,
                            uint64_t seed, long long* fx_host, cudaStream_t st) {
  const int nlat = K * reps;
  const int S = n_eq + n_meas;
  const int64_t n = static_cast<int64_t>(L) * L;
  float* phi = nullptr;
  CalibLattice* lat = nullptr;
  long long* fx = nullptr;
  cudaError_t e = cudaMalloc(&phi, sizeof(float) * n * nlat);
  if (e == cudaSuccess) e = cudaMalloc(&lat, sizeof(CalibLattice) * nlat);
  if (e == cudaSuccess) e = cudaMalloc(&fx, sizeof(long long) * nlat * S);
  if (e == cudaSuccess) {
    CalibLattice* h = new CalibLattice[nlat];
    for (int k = 0; k < K; ++k)
      for (int r = 0; r < reps; ++r) {
        const double Td = static_cast<double>(T_host[k]);
        const double st_d = 3.0 * __builtin_sqrt(Td);
        h[k * reps + r].beta = 1.0f / T_host[k];
        h[k * reps + r].step = static_cast<float>(st_d < 6.283185307179586 ? st_d : 6.283185307179586);
        h[k * reps + r].rep = static_cast<uint32_t>(r);
      }
    e = cudaMemcpyAsync(lat, h, sizeof(CalibLattice) * nlat, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    delete[] h;
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(fx, 0, sizeof(long long) * nlat * S, st);
  if (e == cudaSuccess) {
    k_fill<<<1184, 256, 0, st>>>(phi, n * nlat, 0x1.921fb6p+1f);  // ordered start: phi = pi
    const uint32_t k0 = static_cast<uint32_t>(seed & 0xffffffffu), k1 = static_cast<uint32_t>(seed >> 32);
    const int64_t half_items = static_cast<int64_t>(L) * ((L + 1) / 2) * nlat;
    const int grid_h = static_cast<int>((half_items + 255) / 256 < 148 * 16 ? (half_items + 255) / 256 : 148 * 16);
    const dim3 grid_e(static_cast<unsigned>((n + 255) / 256 < 16 ? (n + 255) / 256 : 16), static_cast<unsigned>(nlat));
    for (int s = 1; s <= S && e == cudaSuccess; ++s) {
      k_calib_half<<<grid_h, 256, 0, st>>>(phi, lat, nlat, L, 0, static_cast<uint32_t>(s), k0, k1, q);
      k_calib_half<<<grid_h, 256, 0, st>>>(phi, lat, nlat, L, 1, static_cast<uint32_t>(s), k0, k1, q);
      // energies of sweep s land in fx[(s-1)*nlat + l]
      k_calib_energy<<<grid_e, 256, 0, st>>>(phi, L, q, fx + static_cast<int64_t>(s - 1) * nlat);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(fx_host, fx, sizeof(long long) * nlat * S, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (phi) cudaFree(phi);
  if (lat) cudaFree(lat);
  if (fx) cudaFree(fx);
  return e;
}

}  // namespace mpr
