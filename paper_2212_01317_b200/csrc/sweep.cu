// sweep.cu — the hot loop of the LE-MPR conditional simulation.
//
// One launch = one colour half-sweep ("the updating algorithm can be
// applied to all the spins on the same sub-grid in parallel") over ALL realizations
// of a batch. Layout: the state G is gap-site major and
// realization minor, G[g][r], so
//   * only gap sites are stored and updated (samples are frozen, and
//     shared by all realizations: their angles live in the 32-byte GapRec of each
//     gap neighbour);
//   * one work item = (gap site g, realization pair j): a float2 of the state, one
//     Philox4x32-10 call whose four words serve both realizations (ARITH §A), eight
//     cos_spec evaluations per realization (ARITH §B, H) and one exp_spec;
//   * consecutive lanes take consecutive items, so the self and neighbour float2
//     accesses of a warp are contiguous runs of G (coalesced), and every lane of a
//     warp does useful work whatever the gap pattern (no idle lanes on frozen sites).
// The whole-grid energy (a8) and the last-n_avg accumulation (a9) are fused into the
// epilogue; the energy of each bond is the value of the branch the Metropolis step
// already chose, so the diagnostic costs no extra cos evaluation.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_math.cuh"
#include "internal.cuh"

namespace mpr {

namespace {

constexpr int kMaxPairs = 512;  // batch <= 1024 realizations

template <bool QHALF>
__device__ __forceinline__ float cosq(float d, float q) {
  if (QHALF) return cos_half_spec(d);
  return cos_spec(__fmul_rn(q, d));
}

// ARITH §H for one realization. FULL: all four neighbours exist (interior site), so
// the sums need no masking and start from the first term (+0 + c == c exactly, since
// cos_spec never returns -0). Returns the new angle; `sel` selects the bonds whose
// chosen-branch cos is added to *e_sel (energy epilogue).
template <bool QHALF, bool ENERGY, bool FULL, bool BFEXP>
__device__ __forceinline__ float metropolis(float cur, const float (&nbv)[4], uint32_t flags,
                                            uint32_t sel, float beta, float q, float J,
                                            uint32_t wa, uint32_t wb, bool& accepted,
                                            long long& e_sel) {
  const float prop = proposal_angle(wa);
  float s_cur = 0.0f, s_new = 0.0f;
  long long ec = 0, en = 0;  // ARITH §J fixed-point bond sums of the selected bonds
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float cc = cosq<QHALF>(__fsub_rn(cur, nbv[k]), q);
    float cn = cosq<QHALF>(__fsub_rn(prop, nbv[k]), q);
    if (!FULL) {
      const bool has = ((flags >> (2 * k)) & 3u) != 0u;
      cc = has ? cc : 0.0f;
      cn = has ? cn : 0.0f;
    }
    if (FULL && k == 0) {
      s_cur = cc;
      s_new = cn;
    } else {
      s_cur = __fadd_rn(s_cur, cc);
      s_new = __fadd_rn(s_new, cn);
    }
    if (ENERGY && ((sel >> k) & 1u)) {
      ec += __float2ll_rn(__fmul_rn(cc, 0x1p32f));
      en += __float2ll_rn(__fmul_rn(cn, 0x1p32f));
    }
  }
  const float dE = __fmul_rn(J, __fsub_rn(s_cur, s_new));
  const float x = -__fmul_rn(dE, beta);
  if (BFEXP) {  // branch-free: exp evaluated by every lane (no divergence around it)
    const float e = exp_spec_fast(x);
    accepted = (dE <= 0.0f) | (u24(wb) < e);
  } else {
    accepted = (dE <= 0.0f) || (u24(wb) < exp_spec_fast(x));
  }
  if (ENERGY) e_sel += accepted ? en : ec;
  return accepted ? prop : cur;
}

// Every neighbour present: each 2-bit field of flags is non-zero.
__device__ __forceinline__ bool all_present(uint32_t f) {
  return ((f | (f >> 1)) & 0x55u) == 0x55u;
}

// One work item (gap site, realization pair) once its record and the states it reads
// are in registers: Philox, two Metropolis updates, store, fused epilogues.
template <bool QHALF, bool ENERGY, bool BFEXP>
__device__ __forceinline__ void process_item(const SweepArgs& a, const GapRec& rec, float2 cur,
                                             const float (&nv0)[4], const float (&nv1)[4],
                                             uint32_t self_off, uint32_t pair, long long& e0, long long& e1,
                                             bool accum0, bool accum1) {
  uint32_t sel = 0;
  if (ENERGY) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
      sel |= (a.is_b ? (ty != NB_NONE) : (ty == NB_KNOWN)) ? (1u << k) : 0u;
    }
  }
  const Words4 w = philox4x32_10(rec.site, a.sweep, pair, 2u, a.k0, a.k1);
  bool acc0, acc1;
  float n0, n1;
  if (all_present(rec.flags)) {
    n0 = metropolis<QHALF, ENERGY, true, BFEXP>(cur.x, nv0, rec.flags, sel, rec.beta, a.q, a.J, w.w0, w.w1, acc0, e0);
    n1 = metropolis<QHALF, ENERGY, true, BFEXP>(cur.y, nv1, rec.flags, sel, rec.beta, a.q, a.J, w.w2, w.w3, acc1, e1);
  } else {
    n0 = metropolis<QHALF, ENERGY, false, BFEXP>(cur.x, nv0, rec.flags, sel, rec.beta, a.q, a.J, w.w0, w.w1, acc0, e0);
    n1 = metropolis<QHALF, ENERGY, false, BFEXP>(cur.y, nv1, rec.flags, sel, rec.beta, a.q, a.J, w.w2, w.w3, acc1, e1);
  }
  if (acc0 || acc1) *reinterpret_cast<float2*>(a.G + self_off) = make_float2(n0, n1);
  if (accum0 || accum1) {
    float2* ap = reinterpret_cast<float2*>(a.A + self_off);
    float2 av = *ap;
    if (accum0) av.x = __fadd_rn(av.x, n0);
    if (accum1) av.y = __fadd_rn(av.y, n1);
    *ap = av;
  }
}

// Accumulation flags of the realization pair j for this sweep: the fixed window of the
// last n_avg sweeps, or (adaptive protocol, ARITH §K) each realization's own window
// (win_lo, win_hi].
__device__ __forceinline__ void accum_flags(const SweepArgs& a, int j, bool& f0, bool& f1) {
  if (a.win_lo) {
    const int s = static_cast<int>(a.sweep);
    f0 = a.win_lo[2 * j] < s && s <= a.win_hi[2 * j];
    f1 = a.win_lo[2 * j + 1] < s && s <= a.win_hi[2 * j + 1];
  } else {
    f0 = f1 = a.accumulate != 0;
  }
}

// a8: per-realization fixed-point bond sums of this CTA -> global int64 atomics, one per
// realization (exact, so the result does not depend on the order: ARITH §J).
__device__ __forceinline__ void energy_epilogue(const SweepArgs& a, int npairs, bool active, int j, long long e0,
                                                long long e1) {
  __shared__ unsigned long long es[2 * kMaxPairs];
  for (int t = threadIdx.x; t < 2 * npairs; t += blockDim.x) es[t] = 0ull;
  __syncthreads();
  if (active && (e0 != 0 || e1 != 0)) {
    atomicAdd(&es[2 * j], static_cast<unsigned long long>(e0));
    atomicAdd(&es[2 * j + 1], static_cast<unsigned long long>(e1));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 2 * npairs; t += blockDim.x)
    if (t >= a.r_valid_lo && t < a.r_valid_hi && es[t] != 0ull)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.energy + static_cast<int64_t>(t) * a.energy_stride), es[t]);
}

// Work split: thread tid owns realization pair j = tid % npairs and gap sites
// g = tid / npairs + k * gstride; consecutive lanes -> consecutive (g, j) items.
struct Split {
  int j;
  bool active;
  uint32_t g0, gstride;
};
__device__ __forceinline__ Split split_work(int npairs) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = gridDim.x * blockDim.x;
  const int active = (total / npairs) * npairs;
  Split s;
  s.j = tid % npairs;
  s.active = tid < active;
  s.g0 = static_cast<uint32_t>(tid / npairs);
  s.gstride = static_cast<uint32_t>(active / npairs);
  return s;
}

// Direct-load variant: record, own state and neighbour states loaded from global memory
// at the start of each item (PF: register-free prefetch of the next item).
template <bool QHALF, bool ENERGY, int MINB, int PF, int NT, bool BFEXP, bool LIST>
__global__ void __launch_bounds__(NT, MINB) k_sweep_half(const SweepArgs a) {
  const Split sp = split_work(a.npairs);
  // 32-bit element offsets: the host caps the batch so that P * R < 2^31
  const uint32_t R = static_cast<uint32_t>(a.R);
  const uint32_t j2 = 2u * static_cast<uint32_t>(sp.j);
  const uint32_t gcount = static_cast<uint32_t>(a.g_count);
  const uint32_t gbegin = static_cast<uint32_t>(a.g_begin);
  long long e0 = 0, e1 = 0;
  bool accum0 = false, accum1 = false;
  bool live = sp.active;
  if (live) {
    accum_flags(a, sp.j, accum0, accum1);
    // adaptive protocol: a pair whose two realizations have finished is frozen
    if (a.win_hi) live = static_cast<int>(a.sweep) <= max(a.win_hi[2 * sp.j], a.win_hi[2 * sp.j + 1]);
  }
  if (live) {
    const uint32_t pair = a.pair_base + static_cast<uint32_t>(sp.j);
    for (uint32_t g = sp.g0; g < gcount; g += sp.gstride) {
      // DC order (row f3): the phase's gap ids come from a list; SC: a contiguous range
      const uint32_t gg = LIST ? a.glist[g] : gbegin + g;
      const GapRec rec = a.rec[gg];
      const uint32_t self_off = gg * R + j2;
      const float2 cur = *reinterpret_cast<const float2*>(a.G + self_off);
      if (PF && !LIST) {
        const uint32_t gn = gg + sp.gstride;
        if (gn < gbegin + gcount) {
          if (PF == 1) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.rec + gn));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.G + (gn * R + j2)));
          } else {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.rec + gn));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.G + (gn * R + j2)));
          }
        }
      }
      float nv0[4], nv1[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
        if (ty == NB_GAP) {
          const float2 v = *reinterpret_cast<const float2*>(a.G + (static_cast<uint32_t>(rec.nb[k]) * R + j2));
          nv0[k] = v.x;
          nv1[k] = v.y;
        } else {
          const float f = __int_as_float(rec.nb[k]);
          nv0[k] = f;
          nv1[k] = f;
        }
      }
      process_item<QHALF, ENERGY, BFEXP>(a, rec, cur, nv0, nv1, self_off, pair, e0, e1, accum0, accum1);
    }
  }
  if (ENERGY) energy_epilogue(a, a.npairs, sp.active && live, sp.j, e0, e1);
}

// a6: initial states of a batch (ARITH §G).
__global__ void __launch_bounds__(256) k_init_states(const GapRec* __restrict__ rec,
                                                     float* __restrict__ G, float* __restrict__ A,
                                                     int64_t P, int R, int npairs,
                                                     uint32_t pair_base, int random_init,
                                                     uint32_t k0, uint32_t k1) {
  const int64_t items = P * npairs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < items;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t / npairs;
    const int j = static_cast<int>(t - g * npairs);
    float2 v;
    if (random_init) {
      const Words4 w = philox4x32_10(rec[g].site, 0u, pair_base + static_cast<uint32_t>(j), 1u, k0, k1);
      v = make_float2(proposal_angle(w.w0), proposal_angle(w.w2));
    } else {
      const float f = rec[g].init;
      v = make_float2(f, f);
    }
    *reinterpret_cast<float2*>(G + g * R + 2 * j) = v;
    if (A) *reinterpret_cast<float2*>(A + g * R + 2 * j) = make_float2(0.0f, 0.0f);
  }
}

// a9 (realization sum): acc[g] += sum_{r in [r_lo, r_hi)} X[g][r], fp64, r ascending —
// the same summation order as the oracle (ARITH §I).
__global__ void __launch_bounds__(256) k_acc_reduce(const float* __restrict__ X, int64_t g_begin,
                                                    int64_t g_end, int R, int r_lo, int r_hi,
                                                    double* __restrict__ acc) {
  for (int64_t g = g_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < g_end;
       g += (int64_t)gridDim.x * blockDim.x) {
    double s = acc[g];
    const float* x = X + g * R;
    for (int r = r_lo; r < r_hi; ++r) s = __dadd_rn(s, static_cast<double>(x[r]));
    acc[g] = s;
  }
}

}  // namespace

// Kernel variants (tuning knob, MPR_SWEEP_VARIANT; profiles/r01_summary.md records every
// alternative measured): 0 = plain, 2 = + register-free L2 prefetch of the next item,
// 5 (default) = 2 + branch-free exp, 8 = 5 capped at 64 registers (32 warps/SM).
// C2 half-sweep: v0 106.5, v2 103.3, v5 99.3, v8 101.8 us; C4: v5 4.15, v8 4.02 ms.
// LIST: the gap ids of the phase come from a list (double-checkerboard order, row f3).
template <bool Q, bool E, bool LIST>
static void* sweep_kernel_ptr(int variant) {
  switch (variant) {
    case 0: return reinterpret_cast<void*>(k_sweep_half<Q, E, 1, 0, 256, false, LIST>);
    case 2: return reinterpret_cast<void*>(k_sweep_half<Q, E, 1, 2, 256, false, LIST>);
    case 8: return reinterpret_cast<void*>(k_sweep_half<Q, E, 4, 2, 256, true, LIST>);
    default: return reinterpret_cast<void*>(k_sweep_half<Q, E, 1, 2, 256, true, LIST>);  // 5
  }
}

static int sweep_threads(int) { return 256; }

static size_t sweep_smem(int) { return 0; }

static void* sweep_kernel(bool qhalf, bool energy, bool list, int variant) {
  if (list) {
    if (qhalf) return energy ? sweep_kernel_ptr<true, true, true>(variant) : sweep_kernel_ptr<true, false, true>(variant);
    return energy ? sweep_kernel_ptr<false, true, true>(variant) : sweep_kernel_ptr<false, false, true>(variant);
  }
  if (qhalf) return energy ? sweep_kernel_ptr<true, true, false>(variant) : sweep_kernel_ptr<true, false, false>(variant);
  return energy ? sweep_kernel_ptr<false, true, false>(variant) : sweep_kernel_ptr<false, false, false>(variant);
}

int sweep_grid_size(int device, int variant) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sweep_kernel(true, false, false, variant), sweep_threads(variant),
                                                sweep_smem(variant));
  if (per < 1) per = 1;
  return sms * per;
}

void launch_sweep_half(const SweepArgs& a, int grid, int variant, cudaStream_t st) {
  const int nt = sweep_threads(variant);
  const int64_t items = a.g_count * a.npairs;
  int64_t g = (items + nt - 1) / nt;
  if (g > grid) g = grid;
  const int64_t need = (a.npairs + nt - 1) / nt;  // active threads >= npairs
  if (g < need) g = need;
  if (g < 1) g = 1;
  const bool qhalf = (a.q == 0.5f);
  const bool energy = (a.energy != nullptr);
  void* fn = sweep_kernel(qhalf, energy, a.glist != nullptr, variant);
  void* args[] = {const_cast<SweepArgs*>(&a)};
  cudaLaunchKernel(fn, dim3(static_cast<unsigned>(g)), dim3(nt), args, sweep_smem(variant), st);
}

void launch_init_states(const GapRec* rec, float* G, float* A, int64_t P, int R, int npairs,
                        uint32_t pair_base, int random_init, uint32_t k0, uint32_t k1,
                        cudaStream_t st) {
  const int64_t items = P * npairs;
  int64_t g = (items + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  k_init_states<<<static_cast<unsigned>(g), 256, 0, st>>>(rec, G, A, P, R, npairs, pair_base,
                                                          random_init, k0, k1);
}

void launch_acc_reduce(const float* X, int64_t g_begin, int64_t g_count, int R, int r_lo, int r_hi,
                       double* acc, cudaStream_t st) {
  if (g_count <= 0) return;
  int64_t g = (g_count + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  k_acc_reduce<<<static_cast<unsigned>(g), 256, 0, st>>>(X, g_begin, g_begin + g_count, R, r_lo, r_hi, acc);
}

}  // namespace mpr
