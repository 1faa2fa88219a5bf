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
//     Philox4x32-10 call whose four words serve both realizations (ARITH §A), five
//     sin_spec evaluations per realization (ΔE in the product form, ARITH §B2, H) and
//     one exp_spec;
//   * consecutive lanes take consecutive items, so the self and neighbour float2
//     accesses of a warp are contiguous runs of G (coalesced), and every lane of a
//     warp does useful work whatever the gap pattern (no idle lanes on frozen sites).
// The whole-grid energy (a8) and the last-n_avg accumulation (a9) are fused into the
// epilogue; the energy of each selected bond is its cos_spec at the angle the Metropolis
// step chose (evaluated only in the ENERGY kernels).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "device_math.cuh"
#include "internal.cuh"

namespace mpr {

namespace {


// Programmatic dependent launch (the batch's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, see launch_pdl): a kernel may be
// scheduled while its predecessor drains; pdl_wait() blocks until the predecessor's
// memory operations are complete and visible, pdl_trigger() (after a CTA's last global
// write) lets the successor start launching. Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <bool QHALF>
__device__ __forceinline__ float cosq(float d, float q) {
  if (QHALF) return cos_half_spec(d);
  return cos_spec(__fmul_rn(q, d));
}

// ARITH §H for one realization: the product form
//   dE = 2J * sin[q(phi' - phi)/2] * sum_j sin[q((phi' + phi)/2 - phi_j)]
// with sin_spec(a) = a * S(a*a) (ARITH §B2) and the neighbour sum accumulated by fmaf in the
// order N, S, W, E; QHALF folds the products by h = q/2 = 1/4 into S4. FULL: all four
// neighbours exist (interior site), so no term is masked. Returns the new angle; `sel` selects
// the bonds whose cos (ARITH §B) at the chosen angle is added to *e_sel (energy epilogue).
template <bool QHALF, bool ENERGY, bool FULL, bool BFEXP>
__device__ __forceinline__ float metropolis(float cur, const float (&nbv)[4], uint32_t flags,
                                            uint32_t sel, float beta, float q, float J,
                                            uint32_t wa, uint32_t wb, bool& accepted,
                                            long long& e_sel) {
  const float prop = proposal_angle(wa);
  const float h = __fmul_rn(q, 0.5f);
  const float d = __fsub_rn(prop, cur);
  float S1;
  if (QHALF) {
    S1 = __fmul_rn(d, sin_poly_quarter(__fmul_rn(d, d)));
  } else {
    const float a0 = __fmul_rn(h, d);
    S1 = __fmul_rn(a0, sin_poly(__fmul_rn(a0, a0)));
  }
  const float sm = __fadd_rn(prop, cur);
  float sig = 0.0f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float x = __fmaf_rn(-2.0f, nbv[k], sm);
    float t;
    if (QHALF) {
      t = __fmaf_rn(x, sin_poly_quarter(__fmul_rn(x, x)), sig);
    } else {
      const float a = __fmul_rn(h, x);
      t = __fmaf_rn(a, sin_poly(__fmul_rn(a, a)), sig);
    }
    if (!FULL) {
      const bool has = ((flags >> (2 * k)) & 3u) != 0u;
      sig = has ? t : sig;
    } else {
      sig = t;
    }
  }
  const float dE = __fmul_rn(__fmul_rn(2.0f, J), __fmul_rn(S1, sig));
  const float x = -__fmul_rn(dE, beta);
  if (BFEXP) {  // branch-free: exp evaluated by every lane (no divergence around it)
    const float e = exp_spec_fast(x);
    accepted = (dE <= 0.0f) | (u24(wb) < e);
  } else {
    accepted = (dE <= 0.0f) || (u24(wb) < exp_spec_fast(x));
  }
  const float nv = accepted ? prop : cur;
  if (ENERGY) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if ((sel >> k) & 1u) e_sel += __float2ll_rn(__fmul_rn(cosq<QHALF>(__fsub_rn(nv, nbv[k]), q), 0x1p32f));
  }
  return nv;
}

// ARITH §H for both realizations of a pair at once, on packed f32x2 instructions: the
// x / y components follow exactly the scalar operation sequence of metropolis() above
// (each FFMA2/FADD2/FMUL2 component rounds like its scalar twin), so the results are
// bit-identical while the FP instruction count of an item halves. No packed product feeds
// a packed add (device_math.cuh: the ptxas FMUL2 -> FADD2 contraction).
template <bool QHALF, bool ENERGY, bool FULL>
__device__ __forceinline__ float2 metropolis_pair(float2 cur, const float2 (&nb)[4], uint32_t flags,
                                                  uint32_t sel, float beta, float q, float J,
                                                  const Words4& w, bool& acc0, bool& acc1,
                                                  long long& e0, long long& e1) {
  // the proposal product is scalar: it feeds the adds below
  const float2 prop = make_float2(__fmul_rn(__uint2float_rn(w.w0 >> 8), 0x1.921fb6p-22f),
                                  __fmul_rn(__uint2float_rn(w.w2 >> 8), 0x1.921fb6p-22f));
  const float2 d = __fadd2_rn(prop, make_float2(-cur.x, -cur.y));
  float2 S1;
  if (QHALF) {
    S1 = __fmul2_rn(d, sin_poly_quarter2(__fmul2_rn(d, d)));
  } else {
    const float2 a0 = __fmul2_rn(f2(__fmul_rn(q, 0.5f)), d);
    S1 = __fmul2_rn(a0, sin_poly2(__fmul2_rn(a0, a0)));
  }
  const float2 sm = __fadd2_rn(prop, cur);
  float2 sig = f2(0.0f);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 x = __ffma2_rn(f2(-2.0f), nb[k], sm);
    float2 t;
    if (QHALF) {
      t = __ffma2_rn(x, sin_poly_quarter2(__fmul2_rn(x, x)), sig);
    } else {
      const float2 a = __fmul2_rn(f2(__fmul_rn(q, 0.5f)), x);
      t = __ffma2_rn(a, sin_poly2(__fmul2_rn(a, a)), sig);
    }
    if (!FULL) {
      const bool has = ((flags >> (2 * k)) & 3u) != 0u;
      sig = has ? t : sig;
    } else {
      sig = t;
    }
  }
  const float2 dE = __fmul2_rn(f2(__fmul_rn(2.0f, J)), __fmul2_rn(S1, sig));
  const float2 xe = __fmul2_rn(dE, f2(-beta));  // == -(dE * beta): RN is sign-symmetric
  // u(w) < exp_spec(x)  <=>  (w >> 8) < exp_spec(x) * 2^24 (exact power-of-two scalings)
  const float2 e24 = exp_spec_fast2_x24(xe);
  acc0 = (dE.x <= 0.0f) | (__uint2float_rn(w.w1 >> 8) < e24.x);
  acc1 = (dE.y <= 0.0f) | (__uint2float_rn(w.w3 >> 8) < e24.y);
  const float2 nv = make_float2(acc0 ? prop.x : cur.x, acc1 ? prop.y : cur.y);
  if (ENERGY) {  // a8: the selected bonds' cos at the chosen angles
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if ((sel >> k) & 1u) {
        const float2 dk = __fadd2_rn(nv, make_float2(-nb[k].x, -nb[k].y));
        const float2 c = QHALF ? cos_half_spec2(dk) : cos_spec2(__fmul2_rn(f2(q), dk));
        const float2 ch = __fmul2_rn(c, f2(0x1p32f));
        e0 += __float2ll_rn(ch.x);
        e1 += __float2ll_rn(ch.y);
      }
  }
  return nv;
}

// Every neighbour present: each 2-bit field of flags is non-zero.
__device__ __forceinline__ bool all_present(uint32_t f) {
  return ((f | (f >> 1)) & 0x55u) == 0x55u;
}

// One work item (gap site, realization pair) once its record and the states it reads
// are in registers: Philox, two Metropolis updates, store, fused epilogues.
template <bool QHALF, bool ENERGY, bool BFEXP, bool PK>
__device__ __forceinline__ void process_item_w(const SweepArgs& a, const GapRec& rec, float2 cur,
                                               const float2 (&nb)[4], uint32_t self_off, const Words4& w,
                                               long long& e0, long long& e1, bool accum0, bool accum1);

template <bool QHALF, bool ENERGY, bool BFEXP, bool PK>
__device__ __forceinline__ void process_item(const SweepArgs& a, const GapRec& rec, float2 cur,
                                             const float2 (&nb)[4], uint32_t self_off, uint32_t pair,
                                             long long& e0, long long& e1, bool accum0, bool accum1) {
  const Words4 w = philox4x32_10_rk(rec.site, a.sweep, pair, 2u, a.rk0, a.rk1);
  process_item_w<QHALF, ENERGY, BFEXP, PK>(a, rec, cur, nb, self_off, w, e0, e1, accum0, accum1);
}

// The item once its Philox words are known (the quad kernel may draw them early).
template <bool QHALF, bool ENERGY, bool BFEXP, bool PK>
__device__ __forceinline__ void process_item_w(const SweepArgs& a, const GapRec& rec, float2 cur,
                                               const float2 (&nb)[4], uint32_t self_off, const Words4& w,
                                               long long& e0, long long& e1, bool accum0, bool accum1) {
  uint32_t sel = 0;
  if (ENERGY) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
      sel |= (a.is_b ? (ty != NB_NONE) : (ty == NB_KNOWN)) ? (1u << k) : 0u;
    }
  }
  bool acc0, acc1;
  float n0, n1;
  if (PK) {
    const float2 nn = all_present(rec.flags)
        ? metropolis_pair<QHALF, ENERGY, true>(cur, nb, rec.flags, sel, rec.beta, a.q, a.J, w, acc0, acc1, e0, e1)
        : metropolis_pair<QHALF, ENERGY, false>(cur, nb, rec.flags, sel, rec.beta, a.q, a.J, w, acc0, acc1, e0, e1);
    n0 = nn.x;
    n1 = nn.y;
  } else if (all_present(rec.flags)) {
    const float nv0[4] = {nb[0].x, nb[1].x, nb[2].x, nb[3].x};
    const float nv1[4] = {nb[0].y, nb[1].y, nb[2].y, nb[3].y};
    n0 = metropolis<QHALF, ENERGY, true, BFEXP>(cur.x, nv0, rec.flags, sel, rec.beta, a.q, a.J, w.w0, w.w1, acc0, e0);
    n1 = metropolis<QHALF, ENERGY, true, BFEXP>(cur.y, nv1, rec.flags, sel, rec.beta, a.q, a.J, w.w2, w.w3, acc1, e1);
  } else {
    const float nv0[4] = {nb[0].x, nb[1].x, nb[2].x, nb[3].x};
    const float nv1[4] = {nb[0].y, nb[1].y, nb[2].y, nb[3].y};
    n0 = metropolis<QHALF, ENERGY, false, BFEXP>(cur.x, nv0, rec.flags, sel, rec.beta, a.q, a.J, w.w0, w.w1, acc0, e0);
    n1 = metropolis<QHALF, ENERGY, false, BFEXP>(cur.y, nv1, rec.flags, sel, rec.beta, a.q, a.J, w.w2, w.w3, acc1, e1);
  }
  float2* const gp = reinterpret_cast<float2*>(a.G + self_off);
  if (acc0 || acc1) {
    const float2 nv = make_float2(n0, n1);
    *gp = nv;
  }
  if (accum0 || accum1) {
    float2* ap = reinterpret_cast<float2*>(a.A + self_off);
    float2 av = *ap;
    if (accum0) av.x = __fadd_rn(av.x, n0);
    if (accum1) av.y = __fadd_rn(av.y, n1);
    *ap = av;
  }
}

// Both pairs of a two-pair item (variant 33) as one block of straight-line arithmetic, so
// the serial steps of one pair (the neighbour sum, exp) overlap the other pair's instead of
// running back to back behind the per-pair branches; then each pair's store and a9
// accumulation as before. Each pair's arithmetic is metropolis_pair's: bit-identical.
// (Merging the two stores into one float4 store was measured slower: 72.0 vs 69.5 us.)
template <bool QHALF, bool ENERGY>
__device__ __forceinline__ void process_quad_w2(const SweepArgs& a, const GapRec& rec, float4 cur, const float2 (&nbA)[4],
                                                const float2 (&nbB)[4], uint32_t self_off, const Words4& wA,
                                                const Words4& wB, bool liveA, bool liveB, long long (&e)[2][2],
                                                const bool (&acc)[2][2]) {
  uint32_t sel = 0;
  if (ENERGY) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
      sel |= (a.is_b ? (ty != NB_NONE) : (ty == NB_KNOWN)) ? (1u << k) : 0u;
    }
  }
  const float2 cA = make_float2(cur.x, cur.y), cB = make_float2(cur.z, cur.w);
  bool a0, a1, b0, b1;
  long long eA0 = 0, eA1 = 0, eB0 = 0, eB1 = 0;
  float2 nA, nB;
  if (all_present(rec.flags)) {
    nA = metropolis_pair<QHALF, ENERGY, true>(cA, nbA, rec.flags, sel, rec.beta, a.q, a.J, wA, a0, a1, eA0, eA1);
    nB = metropolis_pair<QHALF, ENERGY, true>(cB, nbB, rec.flags, sel, rec.beta, a.q, a.J, wB, b0, b1, eB0, eB1);
  } else {
    nA = metropolis_pair<QHALF, ENERGY, false>(cA, nbA, rec.flags, sel, rec.beta, a.q, a.J, wA, a0, a1, eA0, eA1);
    nB = metropolis_pair<QHALF, ENERGY, false>(cB, nbB, rec.flags, sel, rec.beta, a.q, a.J, wB, b0, b1, eB0, eB1);
  }
  if (liveA) {
    if (ENERGY) {
      e[0][0] += eA0;
      e[0][1] += eA1;
    }
    if (a0 || a1) *reinterpret_cast<float2*>(a.G + self_off) = nA;
    if (acc[0][0] || acc[0][1]) {
      float2* ap = reinterpret_cast<float2*>(a.A + self_off);
      float2 av = *ap;
      if (acc[0][0]) av.x = __fadd_rn(av.x, nA.x);
      if (acc[0][1]) av.y = __fadd_rn(av.y, nA.y);
      *ap = av;
    }
  }
  if (liveB) {
    if (ENERGY) {
      e[1][0] += eB0;
      e[1][1] += eB1;
    }
    if (b0 || b1) *reinterpret_cast<float2*>(a.G + self_off + 2u) = nB;
    if (acc[1][0] || acc[1][1]) {
      float2* ap = reinterpret_cast<float2*>(a.A + self_off + 2u);
      float2 av = *ap;
      if (acc[1][0]) av.x = __fadd_rn(av.x, nB.x);
      if (acc[1][1]) av.y = __fadd_rn(av.y, nB.y);
      *ap = av;
    }
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
// realization and CTA (exact, so the result does not depend on the order: ARITH §J).
// Thread tid holds the K values of realizations K*u .. K*u+K-1, u = tid % nunits (`unit`),
// added into one shared slot per realization. When nunits divides 32 (a batch of 2, 4,
// ..., 32 / K realizations), up to 256 threads would hit each slot, so the lanes of a
// warp that share a unit (lanes equal mod nunits) are first reduced with shuffles and only
// lanes < nunits issue the shared atomics. Needs blockDim.x == 256 and every thread.
constexpr int kMaxRealizations = 1024;
template <int K>
__device__ __forceinline__ void energy_epilogue_k(const SweepArgs& a, int nunits, int unit, bool active,
                                                  long long (&v)[K]) {
  __shared__ unsigned long long es[kMaxRealizations];
  for (int t = threadIdx.x; t < K * nunits; t += blockDim.x) es[t] = 0ull;
  __syncthreads();
  if (!active)
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = 0;
  bool issue = active;
  if (nunits <= 16 && (32 % nunits) == 0) {  // lane l has unit (l + const) % nunits: warp-periodic
#pragma unroll
    for (int k = 0; k < K; ++k)
      for (int off = 16; off >= nunits; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    issue = (threadIdx.x & 31) < nunits;
  }
  if (issue)
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (v[k] != 0) atomicAdd(&es[unit * K + k], static_cast<unsigned long long>(v[k]));
  __syncthreads();
  for (int t = threadIdx.x; t < K * nunits; t += blockDim.x)
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

// One realization pair per thread. PF = 2: record, own and neighbour states loaded at the
// start of each item, with a register-free L2 prefetch of the next item; PF = 3: the next
// item's record is loaded one item ahead (below).
template <bool QHALF, bool ENERGY, int MINB, int PF, int NT, bool BFEXP, bool LIST, bool PK>
__global__ void __launch_bounds__(NT, MINB) k_sweep_half(const SweepArgs a) {
  pdl_wait();
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
  if (live && PF == 3) {
    // Record one item ahead: the 32-byte record of item g + gstride is loaded into registers
    // while item g computes, so an item waits for one dependent round trip (its neighbour
    // states), not two (record, then states). Plus the L2 prefetch of the next own state.
    const uint32_t pair = a.pair_base + static_cast<uint32_t>(sp.j);
    uint32_t g = sp.g0;
    uint32_t gg = 0;
    GapRec rec{};
    if (g < gcount) {
      gg = LIST ? a.glist[g] : gbegin + g;
      rec = a.rec[gg];
    }
    for (; g < gcount; g += sp.gstride) {
      const uint32_t gn = g + sp.gstride;
      uint32_t ggn = 0;
      GapRec recn{};
      if (gn < gcount) {
        ggn = LIST ? a.glist[gn] : gbegin + gn;
        recn = a.rec[ggn];
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.G + (ggn * R + j2)));
      }
      const uint32_t self_off = gg * R + j2;
      const float2 cur = *reinterpret_cast<const float2*>(a.G + self_off);
      float2 nb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
        if (ty == NB_GAP) {
          nb[k] = *reinterpret_cast<const float2*>(a.G + (static_cast<uint32_t>(rec.nb[k]) * R + j2));
        } else {
          nb[k] = f2(__int_as_float(rec.nb[k]));
        }
      }
      process_item<QHALF, ENERGY, BFEXP, PK>(a, rec, cur, nb, self_off, pair, e0, e1, accum0, accum1);
      rec = recn;
      gg = ggn;
    }
  } else if (live) {
    const uint32_t pair = a.pair_base + static_cast<uint32_t>(sp.j);
    for (uint32_t g = sp.g0; g < gcount; g += sp.gstride) {
      // DC order (row f3): the phase's gap ids come from a list; SC: a contiguous range
      const uint32_t gg = LIST ? a.glist[g] : gbegin + g;
      const GapRec rec = a.rec[gg];
      const uint32_t self_off = gg * R + j2;
      const float2 cur = *reinterpret_cast<const float2*>(a.G + self_off);
      if (PF == 2 && !LIST) {  // register-free L2 prefetch of the next item's record and state
        const uint32_t gn = gg + sp.gstride;
        if (gn < gbegin + gcount) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.rec + gn));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.G + (gn * R + j2)));
        }
      }
      float2 nb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
        if (ty == NB_GAP) {
          nb[k] = *reinterpret_cast<const float2*>(a.G + (static_cast<uint32_t>(rec.nb[k]) * R + j2));
        } else {
          nb[k] = f2(__int_as_float(rec.nb[k]));
        }
      }
      process_item<QHALF, ENERGY, BFEXP, PK>(a, rec, cur, nb, self_off, pair, e0, e1, accum0, accum1);
    }
  }
  if (ENERGY) {
    long long v[2] = {e0, e1};
    energy_epilogue_k<2>(a, a.npairs, sp.j, sp.active && live, v);
  }
  pdl_trigger();
}

// Variant 14: the one-pair item of variant 13 two at a time. A thread takes its items g and
// g + gstride per loop trip (the same items, in the same split, as variant 13), draws both
// Philox calls, loads both, and runs both metropolis_pair in one block so that the two
// chains interleave. The fallback of the two-pair kernels for an odd pair count (the C4
// tail batch); no energy epilogue (energy sweeps keep variant 13).
template <bool QHALF, bool LIST>
__global__ void __launch_bounds__(256, 3) k_sweep_half2(const SweepArgs a) {
  pdl_wait();
  const Split sp = split_work(a.npairs);
  const uint32_t R = static_cast<uint32_t>(a.R);
  const uint32_t j2 = 2u * static_cast<uint32_t>(sp.j);
  const uint32_t gcount = static_cast<uint32_t>(a.g_count);
  const uint32_t gbegin = static_cast<uint32_t>(a.g_begin);
  bool acc0 = false, acc1 = false;
  bool live = sp.active;
  if (live) {
    accum_flags(a, sp.j, acc0, acc1);
    if (a.win_hi) live = static_cast<int>(a.sweep) <= max(a.win_hi[2 * sp.j], a.win_hi[2 * sp.j + 1]);
  }
  if (live) {
    const uint32_t pair = a.pair_base + static_cast<uint32_t>(sp.j);
    const uint32_t gs = sp.gstride;
    uint32_t g = sp.g0;
    uint32_t ga = 0, gb = 0;
    GapRec ra{}, rb{};
    if (g < gcount) {
      ga = LIST ? a.glist[g] : gbegin + g;
      ra = a.rec[ga];
    }
    if (g + gs < gcount) {
      gb = LIST ? a.glist[g + gs] : gbegin + g + gs;
      rb = a.rec[gb];
    }
    for (; g < gcount; g += 2u * gs) {
      const bool vb = g + gs < gcount;
      const uint32_t g2 = g + 2u * gs, g3 = g + 3u * gs;
      uint32_t ga2 = 0, gb2 = 0;
      GapRec ra2{}, rb2{};
      if (g2 < gcount) {
        ga2 = LIST ? a.glist[g2] : gbegin + g2;
        ra2 = a.rec[ga2];
      }
      if (g3 < gcount) {
        gb2 = LIST ? a.glist[g3] : gbegin + g3;
        rb2 = a.rec[gb2];
      }
      const Words4 wa = philox4x32_10_rk(ra.site, a.sweep, pair, 2u, a.rk0, a.rk1);
      const Words4 wb = philox4x32_10_rk(rb.site, a.sweep, pair, 2u, a.rk0, a.rk1);
      const uint32_t offa = ga * R + j2, offb = gb * R + j2;
      const float2 ca = *reinterpret_cast<const float2*>(a.G + offa);
      const float2 cb = vb ? *reinterpret_cast<const float2*>(a.G + offb) : f2(0.0f);
      float2 na[4], nbv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t ta = (ra.flags >> (2 * k)) & 3u, tb = (rb.flags >> (2 * k)) & 3u;
        na[k] = ta == NB_GAP ? *reinterpret_cast<const float2*>(a.G + (static_cast<uint32_t>(ra.nb[k]) * R + j2))
                             : f2(__int_as_float(ra.nb[k]));
        nbv[k] = (vb && tb == NB_GAP) ? *reinterpret_cast<const float2*>(a.G + (static_cast<uint32_t>(rb.nb[k]) * R + j2))
                                      : f2(__int_as_float(rb.nb[k]));
      }
      bool a0, a1, b0, b1;
      long long e = 0;
      float2 xa, xb;
      if (all_present(ra.flags) && all_present(rb.flags)) {
        xa = metropolis_pair<QHALF, false, true>(ca, na, ra.flags, 0u, ra.beta, a.q, a.J, wa, a0, a1, e, e);
        xb = metropolis_pair<QHALF, false, true>(cb, nbv, rb.flags, 0u, rb.beta, a.q, a.J, wb, b0, b1, e, e);
      } else {
        xa = metropolis_pair<QHALF, false, false>(ca, na, ra.flags, 0u, ra.beta, a.q, a.J, wa, a0, a1, e, e);
        xb = metropolis_pair<QHALF, false, false>(cb, nbv, rb.flags, 0u, rb.beta, a.q, a.J, wb, b0, b1, e, e);
      }
      if (a0 || a1) *reinterpret_cast<float2*>(a.G + offa) = xa;
      if (vb && (b0 || b1)) *reinterpret_cast<float2*>(a.G + offb) = xb;
      if (acc0 || acc1) {
        float2* pa = reinterpret_cast<float2*>(a.A + offa);
        float2 av = *pa;
        if (acc0) av.x = __fadd_rn(av.x, xa.x);
        if (acc1) av.y = __fadd_rn(av.y, xa.y);
        *pa = av;
        if (vb) {
          float2* pb = reinterpret_cast<float2*>(a.A + offb);
          float2 bv = *pb;
          if (acc0) bv.x = __fadd_rn(bv.x, xb.x);
          if (acc1) bv.y = __fadd_rn(bv.y, xb.y);
          *pb = bv;
        }
      }
      ra = ra2;
      rb = rb2;
      ga = ga2;
      gb = gb2;
    }
  }
  pdl_trigger();
}

// NP realization pairs (2 NP realizations) of one gap site per thread (NP = 2 is built;
// NP = 4 measured no faster, profiles/r01_summary.md). The record, the flag decoding, the
// neighbour addresses and the loop overhead are shared by the NP pairs, and the own /
// neighbour states move as float4 (two pairs each). Each pair still draws its own Philox
// call and runs metropolis_pair, so the results are those of k_sweep_half bit for bit.
// Requires npairs % NP == 0 (launch_sweep_half falls back). EARLY: every pair's Philox
// words are drawn right after the record arrives.
template <bool QHALF, bool ENERGY, int MINB, bool LIST, int NP = 2, bool EARLY = false, bool IL = false>
__global__ void __launch_bounds__(256, MINB) k_sweep_quad(const SweepArgs a) {
  pdl_wait();
  constexpr int NQ = NP / 2;  // float4 quads per thread
  const int nq = a.npairs / NP;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = gridDim.x * blockDim.x;
  const int nactive = (total / nq) * nq;
  const bool active = tid < nactive;
  const int jq = tid % nq;
  const uint32_t gstride = static_cast<uint32_t>(nactive / nq);
  const uint32_t R = static_cast<uint32_t>(a.R), j4 = 2u * NP * static_cast<uint32_t>(jq);
  const uint32_t gcount = static_cast<uint32_t>(a.g_count), gbegin = static_cast<uint32_t>(a.g_begin);
  bool acc[NP][2];
  bool live[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    acc[p][0] = acc[p][1] = false;
    live[p] = active;
  }
  if (active) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      accum_flags(a, NP * jq + p, acc[p][0], acc[p][1]);
      if (a.win_hi) {  // adaptive protocol: a pair whose two realizations have finished is frozen
        const int sw = static_cast<int>(a.sweep), r = 2 * (NP * jq + p);
        live[p] = sw <= max(a.win_hi[r], a.win_hi[r + 1]);
      }
    }
  }
  bool any_live = false;
#pragma unroll
  for (int p = 0; p < NP; ++p) any_live |= live[p];
  const uint32_t pair0 = a.pair_base + static_cast<uint32_t>(NP * jq);
  long long e[NP][2];
#pragma unroll
  for (int p = 0; p < NP; ++p) e[p][0] = e[p][1] = 0;
  if (any_live) {
    uint32_t g = static_cast<uint32_t>(tid / nq);
    uint32_t gg = 0;
    GapRec rec{};
    if (g < gcount) {
      gg = LIST ? a.glist[g] : gbegin + g;
      rec = a.rec[gg];
    }
    for (; g < gcount; g += gstride) {
      const uint32_t gn = g + gstride;
      uint32_t ggn = 0;
      GapRec recn{};
      if (gn < gcount) {
        ggn = LIST ? a.glist[gn] : gbegin + gn;
        recn = a.rec[ggn];
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.G + (ggn * R + j4)));
      }
      // EARLY: draw every pair's Philox words as soon as the record is here, before the
      // state loads are consumed, so the load latency is covered by the integer work
      Words4 wpre[NP];
      if (EARLY) {
#pragma unroll
        for (int p = 0; p < NP; ++p) wpre[p] = philox4x32_10_rk(rec.site, a.sweep, pair0 + p, 2u, a.rk0, a.rk1);
      }
      const uint32_t self_off = gg * R + j4;
      uint32_t nb_off[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) nb_off[k] = static_cast<uint32_t>(rec.nb[k]) * R + j4;
#pragma unroll
      for (int qd = 0; qd < NQ; ++qd) {
        const float4 cur = *reinterpret_cast<const float4*>(a.G + self_off + 4u * qd);
        float2 nbA[4], nbB[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
          if (ty == NB_GAP) {
            const float4 v = *reinterpret_cast<const float4*>(a.G + nb_off[k] + 4u * qd);
            nbA[k] = make_float2(v.x, v.y);
            nbB[k] = make_float2(v.z, v.w);
          } else {
            nbA[k] = nbB[k] = f2(__int_as_float(rec.nb[k]));
          }
        }
        const int pa = 2 * qd, pb = 2 * qd + 1;
        if (EARLY && IL && NP == 2) {
          process_quad_w2<QHALF, ENERGY>(a, rec, cur, nbA, nbB, self_off, wpre[0], wpre[NP - 1], live[0], live[NP - 1],
                                         reinterpret_cast<long long(&)[2][2]>(e[0][0]),
                                         reinterpret_cast<const bool(&)[2][2]>(acc[0][0]));
        } else if (EARLY) {
          if (live[pa])
            process_item_w<QHALF, ENERGY, true, true>(a, rec, make_float2(cur.x, cur.y), nbA, self_off + 4u * qd,
                                                      wpre[pa], e[pa][0], e[pa][1], acc[pa][0], acc[pa][1]);
          if (live[pb])
            process_item_w<QHALF, ENERGY, true, true>(a, rec, make_float2(cur.z, cur.w), nbB,
                                                      self_off + 4u * qd + 2u, wpre[pb], e[pb][0], e[pb][1],
                                                      acc[pb][0], acc[pb][1]);
        } else {
          if (live[pa])
            process_item<QHALF, ENERGY, true, true>(a, rec, make_float2(cur.x, cur.y), nbA, self_off + 4u * qd,
                                                    pair0 + pa, e[pa][0], e[pa][1], acc[pa][0], acc[pa][1]);
          if (live[pb])
            process_item<QHALF, ENERGY, true, true>(a, rec, make_float2(cur.z, cur.w), nbB, self_off + 4u * qd + 2u,
                                                    pair0 + pb, e[pb][0], e[pb][1], acc[pb][0], acc[pb][1]);
        }
      }
      rec = recn;
      gg = ggn;
    }
  }
  if (ENERGY) {  // a8 epilogue for realizations 2 NP jq .. 2 NP jq + 2 NP - 1
    long long v[2 * NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      v[2 * p] = e[p][0];
      v[2 * p + 1] = e[p][1];
    }
    energy_epilogue_k<2 * NP>(a, nq, jq, active, v);
  }
  pdl_trigger();
}

// ---- Variant 40: the SFU rejection filter (DESIGN.md §7 "Filtered sweep") -------------
// At the temperatures the method estimates (T ~ 1e-4 .. 1e-2 against bond energies of
// order J), almost every proposal of the independence sampler is rejected by a wide
// margin: -beta dE < -17 for 93 % of the updates at C2 and ~98 % at C3/C4. For those the
// Metropolis decision is known without the exact fp32 arithmetic of ARITH §H: when
// x = -beta dE_spec <= -17, exp_spec(x) * 2^24 < 1, so u(w) < exp_spec(x) holds only for
// w >> 8 == 0. The filter evaluates dE with the SFU sine (MUFU.SIN, a pipe of its own)
// and a rigorous error bound B against the exact form, and certifies "reject" when
//   (w >> 8) != 0  and  fl(fl(dE_m - B) * beta) > 17.5.
// Only the pairs it cannot certify (C2: ~6 % measured) run the exact metropolis_pair,
// compacted per warp through a shared-memory queue so that the exact path runs on full
// warps. The exact path is untouched, so the states are the oracle's bit for bit; the
// bound holds by construction once sfu_filter_check() has measured the SFU sine's error
// over every fp32 argument the filter can see (mpr_init only selects variant 40 when it
// passed).
// Measured (profiles/r02_summary.md): 79.4 us per C2 half-sweep against 72.1 us for variant
// 28, so it is opt-in (MPR_SWEEP_VARIANT=40). The FMA-heavy pipe drops from 71 % to 48 %
// busy, but the kernel is issue-bound: each SFU sine costs two issue slots (FMUL.RZ +
// MUFU.SIN, scalar) against four for a packed polynomial sine pair, the queue adds ~18
// slots per item, so the instruction count stays at v28's (52.8 M vs 53.7 M per launch)
// and the thinner arithmetic no longer hides the state loads (long-scoreboard stalls
// 0.95 -> 2.7 per issue). Deeper register pipelines (2 CTAs/SM) were slower still.
constexpr int kFiltQ = 64;          // queue entries per warp (< 32 left + <= 32 appended)
constexpr float kFiltX = 17.5f;     // threshold on beta * (dE_m - B)
constexpr float kFiltB = 6.0e-5f;   // B = kFiltB * 2J (>= 1.7x the bound)
constexpr double kFiltEps = 4.0e-6; // largest SFU sine error the bound B allows

// dE of both realizations of a pair from SFU sines: the same proposal, difference and sum
// as metropolis_pair; the sine arguments are y0 = fl(h d) and y_k = fl(-2h nb_k + fl(h sm))
// (for q = 1/2 exactly the arguments of ARITH §B2's S4 form, x / 4; for other q within two
// units in the last place of them, which the bound allows for). Packed f32x2 throughout
// except the SFU sines; a contraction ptxas may apply here only removes a rounding.
// Returns true when both updates are certain rejections.
struct FiltConst {
  float h;
  float2 m2h, hh, twoJ, nBj;
};
template <bool FULL>
__device__ __forceinline__ bool filter_rejects(float2 cur, const float2 (&nb)[4], uint32_t flags, float beta,
                                               const FiltConst& fc, const Words4& w) {
  const float2 prop = make_float2(__fmul_rn(__uint2float_rn(w.w0 >> 8), 0x1.921fb6p-22f),
                                  __fmul_rn(__uint2float_rn(w.w2 >> 8), 0x1.921fb6p-22f));
  const float2 y0 = __fmul2_rn(fc.hh, __fadd2_rn(prop, make_float2(-cur.x, -cur.y)));
  const float2 hs = __fmul2_rn(fc.hh, __fadd2_rn(prop, cur));
  float2 sg = f2(0.0f);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 y = __ffma2_rn(fc.m2h, nb[k], hs);
    float2 t = make_float2(__sinf(y.x), __sinf(y.y));
    if (!FULL && ((flags >> (2 * k)) & 3u) == 0u) t = f2(0.0f);
    sg = k == 0 ? t : __fadd2_rn(sg, t);
  }
  const float2 s1 = make_float2(__sinf(y0.x), __sinf(y0.y));
  const float2 e = __fmul2_rn(__fmul2_rn(fc.twoJ, s1), sg);
  const float2 xb = __fmul2_rn(__fadd2_rn(e, fc.nBj), f2(beta));
  return min(w.w1, w.w3) > 255u && xb.x > kFiltX && xb.y > kFiltX;
}

// One queued pair on the exact path: its record and states are re-read (L1/L2 hits: the
// item was visited moments ago, and nothing it reads changes during the half-sweep).
template <bool QHALF>
__device__ __forceinline__ void filt_exact(const SweepArgs& a, uint32_t R, const uint4 wq, const uint2 m) {
  const uint32_t gg = m.x, col = m.y & 0x3fffffffu;
  const bool acc0 = (m.y >> 30) & 1u, acc1 = (m.y >> 31) & 1u;
  const GapRec rec = a.rec[gg];
  const uint32_t self_off = gg * R + col;
  const float2 cur = *reinterpret_cast<const float2*>(a.G + self_off);
  float2 nb[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
    nb[k] = ty == NB_GAP ? *reinterpret_cast<const float2*>(a.G + (static_cast<uint32_t>(rec.nb[k]) * R + col))
                         : f2(__int_as_float(rec.nb[k]));
  }
  long long e0 = 0, e1 = 0;
  process_item_w<QHALF, false, true, true>(a, rec, cur, nb, self_off, Words4{wq.x, wq.y, wq.z, wq.w}, e0,
                                                  e1, acc0, acc1);
}

// NP realization pairs of one gap site per thread (NP = 2: float4 state moves as in
// k_sweep_quad; NP = 1: float2, for odd pair counts). Every lane runs the same number of
// loop trips (warp-uniform), so the queue's ballots see the whole warp.
template <bool QHALF, int MINB, bool LIST, int NP>
__global__ void __launch_bounds__(256, MINB) k_sweep_filt(const SweepArgs a) {
  __shared__ uint4 qw[8][kFiltQ];  // Philox words of the queued pairs
  __shared__ uint2 qm[8][kFiltQ];  // (gap id, column | accumulation bits)
  pdl_wait();
  const int lane = threadIdx.x & 31;
  uint4* const myqw = qw[threadIdx.x >> 5];
  uint2* const myqm = qm[threadIdx.x >> 5];
  const unsigned below = (1u << lane) - 1u;
  const int nq = a.npairs / NP;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = gridDim.x * blockDim.x;
  const int nactive = (total / nq) * nq;
  const bool active = tid < nactive;
  const int jq = tid % nq;
  const uint32_t gstride = static_cast<uint32_t>(nactive / nq);
  const uint32_t R = static_cast<uint32_t>(a.R), j0 = 2u * NP * static_cast<uint32_t>(jq);
  const uint32_t gcount = static_cast<uint32_t>(a.g_count), gbegin = static_cast<uint32_t>(a.g_begin);
  FiltConst fc;
  fc.h = __fmul_rn(a.q, 0.5f);
  fc.hh = f2(fc.h);
  fc.m2h = f2(-2.0f * fc.h);
  fc.twoJ = f2(__fmul_rn(2.0f, a.J));
  fc.nBj = f2(-__fmul_rn(kFiltB, fc.twoJ.x));
  // per pair: live (adaptive windows), the queue word (column | accumulation bits) and
  // whether a certified rejection accumulates its unchanged state (a9)
  bool live[NP];
  uint32_t qbits[NP];
  bool anyacc[NP];
  bool any_live = false;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    bool f0 = false, f1 = false;
    live[p] = active;
    if (active) {
      accum_flags(a, NP * jq + p, f0, f1);
      if (a.win_hi) {
        const int sw = static_cast<int>(a.sweep), r = 2 * (NP * jq + p);
        live[p] = sw <= max(a.win_hi[r], a.win_hi[r + 1]);
      }
    }
    qbits[p] = (j0 + 2u * p) | (f0 ? 1u << 30 : 0u) | (f1 ? 1u << 31 : 0u);
    anyacc[p] = f0 || f1;
    any_live |= live[p];
  }
  const uint32_t pair0 = a.pair_base + static_cast<uint32_t>(NP * jq);
  uint32_t g = any_live ? static_cast<uint32_t>(tid / nq) : gcount;
  uint32_t gg = 0;
  GapRec rec{};
  if (g < gcount) {
    gg = LIST ? a.glist[g] : gbegin + g;
    rec = a.rec[gg];
  }
  int cnt = 0;  // queued pairs of this warp (warp-uniform)
  uint32_t n_exact = 0, n_live = 0;  // MPR_FILTER_STATS
  while (__any_sync(0xffffffffu, g < gcount)) {
    const bool have = g < gcount;
    const uint32_t gn = g + gstride;
    uint32_t ggn = 0;
    GapRec recn{};
    if (have && gn < gcount) {
      ggn = LIST ? a.glist[gn] : gbegin + gn;
      recn = a.rec[ggn];
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.G + (ggn * R + j0)));
    }
    Words4 w[NP];
    bool cand[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) cand[p] = false;
    if (have) {
#pragma unroll
      for (int p = 0; p < NP; ++p) w[p] = philox4x32_10_rk(rec.site, a.sweep, pair0 + p, 2u, a.rk0, a.rk1);
      const uint32_t self_off = gg * R + j0;
      float2 cur[NP];
      float2 nb[NP][4];
      if (NP == 2) {
        const float4 c4 = *reinterpret_cast<const float4*>(a.G + self_off);
        cur[0] = make_float2(c4.x, c4.y);
        cur[NP - 1] = make_float2(c4.z, c4.w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
          if (ty == NB_GAP) {
            const float4 v = *reinterpret_cast<const float4*>(a.G + (static_cast<uint32_t>(rec.nb[k]) * R + j0));
            nb[0][k] = make_float2(v.x, v.y);
            nb[NP - 1][k] = make_float2(v.z, v.w);
          } else {
            nb[0][k] = nb[NP - 1][k] = f2(__int_as_float(rec.nb[k]));
          }
        }
      } else {
        cur[0] = *reinterpret_cast<const float2*>(a.G + self_off);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t ty = (rec.flags >> (2 * k)) & 3u;
          nb[0][k] = ty == NB_GAP
              ? *reinterpret_cast<const float2*>(a.G + (static_cast<uint32_t>(rec.nb[k]) * R + j0))
              : f2(__int_as_float(rec.nb[k]));
        }
      }
      const bool full = all_present(rec.flags);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const bool rej = full ? filter_rejects<true>(cur[p], nb[p], rec.flags, rec.beta, fc, w[p])
                              : filter_rejects<false>(cur[p], nb[p], rec.flags, rec.beta, fc, w[p]);
        cand[p] = live[p] && !rej;
        if (a.fstats) n_live += live[p] ? 1u : 0u;
        // a certain rejection keeps the state: no store; the fused a9 epilogue adds it
        if (live[p] && rej && anyacc[p]) {
          float2* ap = reinterpret_cast<float2*>(a.A + self_off + 2u * p);
          float2 av = *ap;
          if (qbits[p] >> 30 & 1u) av.x = __fadd_rn(av.x, cur[p].x);
          if (qbits[p] >> 31) av.y = __fadd_rn(av.y, cur[p].y);
          *ap = av;
        }
      }
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const unsigned m = __ballot_sync(0xffffffffu, cand[p]);
      if (cand[p]) {
        const int pos = cnt + __popc(m & below);
        myqw[pos] = make_uint4(w[p].w0, w[p].w1, w[p].w2, w[p].w3);
        myqm[pos] = make_uint2(gg, qbits[p]);
      }
      cnt += __popc(m);
      if (a.fstats) n_exact += cand[p] ? 1u : 0u;
      if (cnt >= 32) {  // a full warp of exact updates
        __syncwarp();
        const int e = cnt - 32 + lane;
        filt_exact<QHALF>(a, R, myqw[e], myqm[e]);
        cnt -= 32;
        __syncwarp();
      }
    }
    rec = recn;
    gg = ggn;
    g = gn;
  }
  __syncwarp();
  if (lane < cnt) filt_exact<QHALF>(a, R, myqw[lane], myqm[lane]);
  if (a.fstats) {
    n_exact = __reduce_add_sync(0xffffffffu, n_exact);
    n_live = __reduce_add_sync(0xffffffffu, n_live);
    if (lane == 0) {
      atomicAdd(&a.fstats[0], static_cast<unsigned long long>(n_exact));
      atomicAdd(&a.fstats[1], static_cast<unsigned long long>(n_live));
    }
  }
  pdl_trigger();
}

// Self-check of the filter's premises on this device, over every argument it can see:
//   err[0] = max |y * S(fl(y*y)) - sinf_sfu(y)| over every fp32 y, |y| <= 3.2 (the sine
//            arguments fl(h x) lie in [-TWO_PI_F/2, TWO_PI_F/2] for q <= 1/2);
//   err[1] = max over every fp32 x in [-80, -17] of exp_spec(x) * 2^24 (must be < 1).
__global__ void k_filter_check(unsigned long long* err) {
  const uint32_t lim = __float_as_uint(3.2f);
  double e = 0.0;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= lim; b += gridDim.x * blockDim.x) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const float y = __uint_as_float(b | (s ? 0x80000000u : 0u));
      const float P = sin_poly(__fmul_rn(y, y));
      const double t = __dmul_rn(static_cast<double>(y), static_cast<double>(P));
      e = fmax(e, fabs(__dsub_rn(t, static_cast<double>(__sinf(y)))));
    }
  }
  float ex = 0.0f;
  const uint32_t x0 = __float_as_uint(17.0f), x1 = __float_as_uint(80.0f);
  for (uint32_t b = x0 + blockIdx.x * blockDim.x + threadIdx.x; b <= x1; b += gridDim.x * blockDim.x) {
    const float x = -__uint_as_float(b);
    ex = fmaxf(ex, exp_spec_fast2_x24(make_float2(x, x)).x);
  }
  for (int off = 16; off > 0; off >>= 1) {
    e = fmax(e, __shfl_xor_sync(0xffffffffu, e, off));
    ex = fmaxf(ex, __shfl_xor_sync(0xffffffffu, ex, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&err[0], static_cast<unsigned long long>(__double_as_longlong(e)));
    atomicMax(&err[1], static_cast<unsigned long long>(__double_as_longlong(static_cast<double>(ex))));
  }
}

// Row f3, the paper's DC scheme with shared-memory tiles ("Each tile can be
// loaded into the block's shared memory ... looking up the neighboring spins uses shared
// instead of global memory"). One CTA per (l_b x l_b tile of parity tau, chunk of Rc
// realizations): the tile and its one-site halo are staged densely in shared memory (gap
// states of the chunk, the frozen angles of the samples), the tile's colour-A gaps are
// updated, then its colour-B gaps against the new A states, and the tile's gap states are
// written back. During the tau phase the other parity's tiles do not change, so this is
// exactly the phases (tau, A), (tau, B) of ARITH §H's DC order — and each update is the
// same metropolis_pair with the same Philox words as the list kernels: bit-identical.
// The halo ring holds only the neighbours of tile sites, so out-of-grid cells are never read.
struct DcTileArgs {
  const int32_t* gid;   // gap id per site (-1: sample)
  const float* phiK;    // frozen angles of the samples
  const float* T;       // temperature field (beta = 1 / T, as the records hold it)
  float* G;             // state [P][R]
  float* A;             // last-n_avg accumulator [P][R] (nullable)
  int64_t Lx, Ly;
  int lb, tau, R, Rc;   // tile side, parity; batch stride; realizations per CTA chunk (even)
  int nchunks;          // chunks of Rc realizations covering the npairs * 2 of the batch
  int npairs;
  uint32_t pair_base, sweep;
  uint32_t rk0[10], rk1[10];
  float q, J;
  int accumulate;
};

template <bool QHALF>
__global__ void __launch_bounds__(256) k_sweep_dc_tile(const DcTileArgs a) {
  extern __shared__ float ds[];
  pdl_wait();
  const int W = a.lb + 2;            // tile + halo width (cells)
  const int chunk = blockIdx.z;
  const int tr = blockIdx.y;
  const int s0 = (a.tau + tr) & 1;   // first tile column of parity tau in this tile row
  const int tc = s0 + 2 * blockIdx.x;
  const int64_t r0 = static_cast<int64_t>(tr) * a.lb, c0 = static_cast<int64_t>(tc) * a.lb;
  if (c0 >= a.Lx) return;
  const int hr = static_cast<int>(min(static_cast<int64_t>(a.lb), a.Ly - r0)), hc = static_cast<int>(min(static_cast<int64_t>(a.lb), a.Lx - c0));
  const int rc0 = chunk * a.Rc;                 // first realization of the chunk in the batch
  const int nr = min(a.Rc, 2 * a.npairs - rc0);  // realizations of this chunk (even)
  const int Rc = a.Rc;
  // shared layout: [W * W cells][Rc] floats, then two lists of tile gap cells (A, B)
  float* S = ds;
  int* list = reinterpret_cast<int*>(ds + W * W * Rc);
  __shared__ int ncol[2];
  if (threadIdx.x < 2) ncol[threadIdx.x] = 0;
  __syncthreads();
  // stage: cells of the tile and its halo ring inside the grid (corners are never read)
  for (int t = threadIdx.x; t < W * W; t += blockDim.x) {
    const int y = t / W, x = t - y * W;
    const int64_t r = r0 - 1 + y, c = c0 - 1 + x;
    const bool intile = y >= 1 && y <= hr && x >= 1 && x <= hc;
    const bool ring = !intile && (y >= 1 && y <= hr ? (x == 0 || x == hc + 1) : (x >= 1 && x <= hc && (y == 0 || y == hr + 1)));
    if (!(intile || ring) || r < 0 || r >= a.Ly || c < 0 || c >= a.Lx) continue;
    const int64_t i = r * a.Lx + c;
    const int g = a.gid[i];
    float* cell = S + t * Rc;
    if (g < 0) {
      const float v = a.phiK[i];
      for (int k = 0; k < nr; ++k) cell[k] = v;
    } else {
      const float* src = a.G + static_cast<int64_t>(g) * a.R + rc0;
      for (int k = 0; k < nr; k += 2) *reinterpret_cast<float2*>(cell + k) = *reinterpret_cast<const float2*>(src + k);
      if (intile) {  // a tile gap: onto its colour's list
        const int col = static_cast<int>((r + c) & 1);
        const int pos = atomicAdd(&ncol[col], 1);
        list[col * a.lb * a.lb + pos] = t;
      }
    }
  }
  __syncthreads();
  const int npc = nr / 2;  // pairs of the chunk
  const uint32_t pair0 = a.pair_base + static_cast<uint32_t>(rc0 / 2);
  const float* gA = nullptr;
  for (int col = 0; col < 2; ++col) {
    const int n = ncol[col];
    for (int it = threadIdx.x; it < n * npc; it += blockDim.x) {
      const int li = it / npc, j = it - li * npc;
      const int t = list[col * a.lb * a.lb + li];
      const int y = t / W, x = t - y * W;
      const int64_t r = r0 - 1 + y, c = c0 - 1 + x;
      const uint32_t site = static_cast<uint32_t>(r * a.Lx + c);
      const Words4 w = philox4x32_10_rk(site, a.sweep, pair0 + j, 2u, a.rk0, a.rk1);
      const int nbc[4] = {t - W, t + W, t - 1, t + 1};
      const bool has[4] = {r > 0, r + 1 < a.Ly, c > 0, c + 1 < a.Lx};
      uint32_t flags = 0;
      float2 nb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        flags |= (has[k] ? 1u : 0u) << (2 * k);
        nb[k] = has[k] ? *reinterpret_cast<const float2*>(S + nbc[k] * Rc + 2 * j) : make_float2(0.f, 0.f);
      }
      float2* cp = reinterpret_cast<float2*>(S + t * Rc + 2 * j);
      const float2 cur = *cp;
      const float beta = __fdiv_rn(1.0f, a.T[r * a.Lx + c]);
      bool acc0, acc1;
      long long e0 = 0, e1 = 0;
      const float2 nv = (flags == 0x55u)
          ? metropolis_pair<QHALF, false, true>(cur, nb, flags, 0u, beta, a.q, a.J, w, acc0, acc1, e0, e1)
          : metropolis_pair<QHALF, false, false>(cur, nb, flags, 0u, beta, a.q, a.J, w, acc0, acc1, e0, e1);
      *cp = nv;
    }
    __syncthreads();  // colour B reads the new colour-A states
  }
  (void)gA;
  // write back the tile's gap states (and the last-n_avg accumulation)
  for (int col = 0; col < 2; ++col) {
    const int n = ncol[col];
    for (int it = threadIdx.x; it < n * npc; it += blockDim.x) {
      const int li = it / npc, j = it - li * npc;
      const int t = list[col * a.lb * a.lb + li];
      const int y = t / W, x = t - y * W;
      const int64_t i = (r0 - 1 + y) * a.Lx + (c0 - 1 + x);
      const int64_t off = static_cast<int64_t>(a.gid[i]) * a.R + rc0 + 2 * j;
      const float2 v = *reinterpret_cast<const float2*>(S + t * Rc + 2 * j);
      *reinterpret_cast<float2*>(a.G + off) = v;
      if (a.accumulate) {
        float2 av = *reinterpret_cast<float2*>(a.A + off);
        av.x = __fadd_rn(av.x, v.x);
        av.y = __fadd_rn(av.y, v.y);
        *reinterpret_cast<float2*>(a.A + off) = av;
      }
    }
  }
  pdl_trigger();
}

// a6: initial states of a batch (ARITH §G).
// U realization pairs per work item (U = 2: float4 stores, needs an even pair count).
// Items t = g * nunits + u are visited with a grid stride; (g, u) advance incrementally, so
// the loop has no integer division (items < 2^31: the host caps P * R).
template <int U>
// ginit: the BLOCK_MEAN angle of every gap as a compact array (4 bytes per gap instead of
// the 32-byte record sector that holds it).
__global__ void __launch_bounds__(256) k_init_states(const GapRec* __restrict__ rec,
                                                     const float* __restrict__ ginit,
                                                     float* __restrict__ G, float* __restrict__ A,
                                                     int64_t P, int R, int npairs,
                                                     uint32_t pair_base, int random_init,
                                                     uint32_t k0, uint32_t k1) {
  pdl_wait();
  const uint32_t nunits = static_cast<uint32_t>(npairs / U);
  const uint32_t items = static_cast<uint32_t>(P) * nunits;
  const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  uint32_t g = t0 / nunits, u = t0 - g * nunits;
  const uint32_t sg = stride / nunits, su = stride - sg * nunits;
  for (uint32_t t = t0; t < items; t += stride) {
    float v[2 * U];
    if (random_init) {
#pragma unroll
      for (int h = 0; h < U; ++h) {
        const Words4 w = philox4x32_10(rec[g].site, 0u, pair_base + U * u + h, 1u, k0, k1);
        v[2 * h] = proposal_angle(w.w0);
        v[2 * h + 1] = proposal_angle(w.w2);
      }
    } else {
      const float f = ginit[g];
#pragma unroll
      for (int h = 0; h < 2 * U; ++h) v[h] = f;
    }
    float* gp = G + static_cast<int64_t>(g) * R + 2 * U * u;
    if (U == 2) {
      *reinterpret_cast<float4*>(gp) = make_float4(v[0], v[1], v[2 % (2 * U)], v[3 % (2 * U)]);
      if (A) *reinterpret_cast<float4*>(A + static_cast<int64_t>(g) * R + 4 * u) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      *reinterpret_cast<float2*>(gp) = make_float2(v[0], v[1]);
      if (A) *reinterpret_cast<float2*>(A + static_cast<int64_t>(g) * R + 2 * u) = make_float2(0.f, 0.f);
    }
    g += sg;
    u += su;
    if (u >= nunits) {
      u -= nunits;
      ++g;
    }
  }
  pdl_trigger();
}

// a9 (realization sum) for short rows (a few realizations per batch): one thread per gap
// site adds its row directly, r ascending (the row is at most a 32-byte sector or two).
__global__ void __launch_bounds__(256) k_acc_reduce_short(const float* __restrict__ X, int64_t g_begin,
                                                          int64_t g_end, int R, int r_lo, int r_hi,
                                                          double* __restrict__ acc) {
  pdl_wait();
  for (int64_t g = g_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < g_end;
       g += (int64_t)gridDim.x * blockDim.x) {
    double s = acc[g];
    const float* x = X + g * R;
    for (int r = r_lo; r < r_hi; ++r) s = __dadd_rn(s, static_cast<double>(x[r]));
    acc[g] = s;
  }
  pdl_trigger();
}

// a9 (realization sum): acc[g] += sum_{r in [r_lo, r_hi)} X[g][r], fp64, r ascending —
// the same summation order as the oracle (ARITH §I). A CTA owns 256 gap sites; their
// rows are staged through shared memory 32 realizations at a time (each warp reads
// 128-byte row segments, coalesced), then every thread adds its own row in order. The
// padded row stride (33) makes the per-thread reads bank-conflict free.
constexpr int kAccTile = 256, kAccChunk = 32;
__global__ void __launch_bounds__(kAccTile) k_acc_reduce(const float* __restrict__ X, int64_t g_begin,
                                                         int64_t g_end, int R, int r_lo, int r_hi,
                                                         double* __restrict__ acc) {
  pdl_wait();
  __shared__ float sm[kAccTile * (kAccChunk + 1)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t g0 = g_begin + (int64_t)blockIdx.x * kAccTile; g0 < g_end; g0 += (int64_t)gridDim.x * kAccTile) {
    const int64_t g = g0 + threadIdx.x;
    double s = g < g_end ? acc[g] : 0.0;
    for (int rc = r_lo; rc < r_hi; rc += kAccChunk) {
      const int nr = min(kAccChunk, r_hi - rc);
      __syncthreads();
      for (int row = warp; row < kAccTile; row += kAccTile / 32) {
        const int64_t gg = g0 + row;
        if (gg < g_end && lane < nr) sm[row * (kAccChunk + 1) + lane] = X[gg * R + rc + lane];
      }
      __syncthreads();
      if (g < g_end) {
        const float* x = sm + threadIdx.x * (kAccChunk + 1);
        for (int r = 0; r < nr; ++r) s = __dadd_rn(s, static_cast<double>(x[r]));
      }
    }
    if (g < g_end) acc[g] = s;
  }
  pdl_trigger();
}

// Row f1 check on the device: the host's ARITH §K test (api.cu equilibrium_reached), every
// fp64 operation an explicit round-to-nearest intrinsic in the same order, so the
// decisions are the host's (and the oracle's) bit for bit.
__device__ double energy_from_fx_dev(long long E_fx, double n_bonds) {
  return __ddiv_rn(__dmul_rn(-__ll2double_rn(E_fx), 0x1p-32), n_bonds);
}

__global__ void k_adaptive_check(const AdaptiveCheckArgs a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.r_hi || a.eq[r] != 0) return;
  bool ok = false;
  if (a.check) {
    const long long* e = a.energy + static_cast<int64_t>(r) * a.energy_stride + (a.s - a.n_fit);
    const int n = a.n_fit;
    const double xbar = __ddiv_rn(static_cast<double>(n - 1), 2.0);
    double sy = 0.0;
    for (int t = 0; t < n; ++t) sy = __dadd_rn(sy, energy_from_fx_dev(a.sum_known_fx + e[t], a.n_bonds));
    const double ybar = __ddiv_rn(sy, static_cast<double>(n));
    double sxx = 0.0, sxy = 0.0;
    for (int t = 0; t < n; ++t) {
      const double y = energy_from_fx_dev(a.sum_known_fx + e[t], a.n_bonds);
      const double dx = __dsub_rn(static_cast<double>(t), xbar);
      sxx = __dadd_rn(sxx, __dmul_rn(dx, dx));
      sxy = __dadd_rn(sxy, __dmul_rn(dx, __dsub_rn(y, ybar)));
    }
    const double b = __ddiv_rn(sxy, sxx);
    const double ai = __dsub_rn(ybar, __dmul_rn(b, xbar));
    double sse = 0.0;
    for (int t = 0; t < n; ++t) {
      const double y = energy_from_fx_dev(a.sum_known_fx + e[t], a.n_bonds);
      const double res = __dsub_rn(__dsub_rn(y, ai), __dmul_rn(b, static_cast<double>(t)));
      sse = __dadd_rn(sse, __dmul_rn(res, res));
    }
    double tau = __ddiv_rn(__dmul_rn(2.0, __dsqrt_rn(__ddiv_rn(sse, static_cast<double>(n - 2)))),
                           static_cast<double>(n));
    if (a.slope_tol > tau) tau = a.slope_tol;
    ok = b >= -tau;
  }
  if (ok || a.forced) {
    a.eq[r] = ok ? a.s : -a.s;
    a.win_lo[r] = a.s;
    a.win_hi[r] = a.s + a.n_avg;
    atomicSub(&a.status[0], 1);
    atomicMax(&a.status[1], a.s + a.n_avg);
  }
}

}  // namespace

void launch_adaptive_check(const AdaptiveCheckArgs& a, cudaStream_t st) {
  const int nt = 128;
  k_adaptive_check<<<(a.r_hi + nt - 1) / nt, nt, 0, st>>>(a);
}

// Kernel variants (tuning knob, MPR_SWEEP_VARIANT). profiles/r01_summary.md records every
// alternative measured, including the ones no longer built: 32-bit byte offsets, register
// caps at 3/5 CTAs, two records ahead with neighbour prefetch, four pairs per thread, and
// split IMAD.HI/IMAD Philox products. All variants are bit-identical.
//   5  = one pair per thread, scalar arithmetic, L2 prefetch of the next item
//        (the first optimised kernel, kept as the scalar reference);
//   13 = one pair per thread, packed f32x2, record one item ahead, 4 CTAs/SM
//        (the fallback of 22/28/33 for odd pair counts in energy sweeps);
//   14 = 13 two items per loop trip, both chains in one block (the odd-pair fallback
//        otherwise);
//   22 = k_sweep_quad: two pairs per thread, float4 state moves, 4 CTAs/SM;
//   28 = 22 with both pairs' Philox words drawn before the state loads are used,
//        3 CTAs/SM (the energy-trace sweeps of 33);
//   33 = 28 with both pairs' arithmetic in one block (the two chains interleave), per-pair
//        stores (default: C2 69.25 -> 67.98 us, C4 equal within noise);
//   40 / 41 = the SFU rejection filter (two / one pair per thread; opt-in, slower).
// Half-sweep, us (C2 / C3 / C4 at M = 10), product-form dE (ARITH §H), one resident wave:
//   v5  92.6 (C2);  v13 89.7 / 1965 / 3525;  v28 72.2 / 1509 / 3082
//   (v28 with the resident waves of launch_sweep_half: 69.3 / 1367 / ~2707).
// Direct form (8 cos per update), for comparison:
//   v5  99.5 / 2229 / 4127;  v13 93.9 / 2071 / 3717;
//   v22 87.1 / 1838 / 3402;  v28 84.5 / 1780 / 3351.
template <bool Q, bool E, bool LIST>
static void* sweep_kernel_ptr(int variant) {
  if (variant == 14 && !E) return reinterpret_cast<void*>(k_sweep_half2<Q, LIST>);
  if (variant == 5) return reinterpret_cast<void*>(k_sweep_half<Q, E, 1, 2, 256, true, LIST, false>);
  return reinterpret_cast<void*>(k_sweep_half<Q, E, 4, 3, 256, true, LIST, true>);  // 13 (and 22/28's fallback)
}

static int sweep_threads(int) { return 256; }

static size_t sweep_smem(int) { return 0; }

static bool is_quad(int variant) { return variant == 22 || variant == 28 || variant == 33; }
static bool is_filt(int variant) { return variant == 40 || variant == 41; }
static int pairs_per_thread(int variant) { return (is_quad(variant) || variant == 40) ? 2 : 1; }

// Variant 40 (SFU filter, two pairs per thread) / 41 (one pair per thread, also 40's
// fallback for odd pair counts); 3 CTAs/SM like 28.
static void* filt_kernel(bool qhalf, bool list, int variant) {
  if (variant == 40) {
    if (qhalf) return list ? reinterpret_cast<void*>(k_sweep_filt<true, 3, true, 2>) : reinterpret_cast<void*>(k_sweep_filt<true, 3, false, 2>);
    return list ? reinterpret_cast<void*>(k_sweep_filt<false, 3, true, 2>) : reinterpret_cast<void*>(k_sweep_filt<false, 3, false, 2>);
  }
  if (qhalf) return list ? reinterpret_cast<void*>(k_sweep_filt<true, 3, true, 1>) : reinterpret_cast<void*>(k_sweep_filt<true, 3, false, 1>);
  return list ? reinterpret_cast<void*>(k_sweep_filt<false, 3, true, 1>) : reinterpret_cast<void*>(k_sweep_filt<false, 3, false, 1>);
}

template <bool Q, bool E>
static void* quad_kernel_ptr(bool list, int variant) {
  if (variant == 28)
    return list ? reinterpret_cast<void*>(k_sweep_quad<Q, E, 3, true, 2, true>) : reinterpret_cast<void*>(k_sweep_quad<Q, E, 3, false, 2, true>);
  if (variant == 33)
    return list ? reinterpret_cast<void*>(k_sweep_quad<Q, E, 3, true, 2, true, true>) : reinterpret_cast<void*>(k_sweep_quad<Q, E, 3, false, 2, true, true>);
  return list ? reinterpret_cast<void*>(k_sweep_quad<Q, E, 4, true, 2, false>) : reinterpret_cast<void*>(k_sweep_quad<Q, E, 4, false, 2, false>);  // 22
}

static void* sweep_kernel(bool qhalf, bool energy, bool list, int variant) {
  if (is_filt(variant)) return filt_kernel(qhalf, list, variant);  // launch_sweep_half: no energy
  if (is_quad(variant)) {
    if (qhalf) return energy ? quad_kernel_ptr<true, true>(list, variant) : quad_kernel_ptr<true, false>(list, variant);
    return energy ? quad_kernel_ptr<false, true>(list, variant) : quad_kernel_ptr<false, false>(list, variant);
  }
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
  // the two-pair kernels fall back to 13 for an odd pair count, the filter kernels to 41
  // (odd pair counts) and to 28 / 13 (energy trace): size the grid for all of them
  if (is_filt(variant)) {
    for (int v : {41, 28}) {
      int perf = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perf, sweep_kernel(true, v == 28, false, v), 256, 0);
      if (perf < per) per = perf;
    }
  }
  const int fb = (is_quad(variant) || is_filt(variant)) ? 13 : -1;
  if (fb >= 0) {
    for (int e = 0; e < 2; ++e) {
      int perf = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perf, sweep_kernel(true, e != 0, false, fb), sweep_threads(fb),
                                                    sweep_smem(fb));
      if (perf < per) per = perf;
    }
  }
  if (per < 1) per = 1;
  return sms * per;
}

// Launch with the programmatic-stream-serialization attribute (PDL, see pdl_wait).
static void launch_pdl(const void* fn, unsigned grid, unsigned block, void** args, size_t smem, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelExC(&cfg, fn, args);
}

void launch_sweep_half(const SweepArgs& a, int grid, int variant, cudaStream_t st, int waves_forced) {
  const bool qhalf = (a.q == 0.5f);
  const bool energy = (a.energy != nullptr);
  // the filter kernels carry no energy epilogue: the exact kernels run energy sweeps
  if (is_filt(variant) && energy) variant = 28;
  // the interleaved form spills in its energy instantiations: energy sweeps run variant 28
  if (variant == 33 && energy) variant = 28;
  if (variant == 40 && (a.npairs & 1)) variant = 41;
  // the two-pair kernels need an even pair count (float4 alignment)
  // (variant 14, the two-items-per-trip form of 13: the C2 grid at M = 10, where the whole
  // batch runs it, 11.9 -> 10.5 us per half-sweep; MPR_TAIL_VARIANT=13 selects the old one)
  static const int tail_variant = [] {
    const char* v = std::getenv("MPR_TAIL_VARIANT");
    return v ? std::atoi(v) : 14;
  }();
  if (is_quad(variant) && (a.npairs & 1)) variant = (energy ? 13 : tail_variant);
  const int nt = sweep_threads(variant);
  const int64_t units = a.npairs / pairs_per_thread(variant);  // threads per gap site
  const int64_t items = a.g_count * units;
  int64_t g = (items + nt - 1) / nt;
  // Several resident waves of CTAs instead of one persistent wave: a CTA that finishes early
  // is replaced by a fresh one, so the slowest warps no longer set the launch's tail. About
  // 16 items per thread (C2: 3 waves, 72.1 -> 69.3 us; C3: 16 waves, 1505 -> 1365 us; C4:
  // 32 waves, 1529 -> 1354 us per half-sweep; profiles/r02_summary.md). Energy launches too
  // (their per-CTA global atomics cost less than the tail: the adaptive protocol at 2048^2,
  // M = 100, 57.9 -> 54.5 ms). waves_forced > 0 (MPR_SWEEP_WAVES, read at mpr_init) overrides.
  {
    const int64_t per_thread = items / (static_cast<int64_t>(grid) * nt);
    const int64_t waves =
        waves_forced > 0 ? waves_forced : std::min<int64_t>(32, std::max<int64_t>(1, (per_thread + 15) / 16));
    grid = static_cast<int>(grid * waves);
  }
  if (g > grid) g = grid;
  const int64_t need = (units + nt - 1) / nt;  // active threads >= units
  if (g < need) g = need;
  if (g < 1) g = 1;
  void* fn = sweep_kernel(qhalf, energy, a.glist != nullptr, variant);
  SweepArgs b = a;
  for (int i = 0; i < 10; ++i) {
    b.rk0[i] = a.k0 + static_cast<uint32_t>(i) * 0x9E3779B9u;
    b.rk1[i] = a.k1 + static_cast<uint32_t>(i) * 0xBB67AE85u;
  }
  void* args[] = {&b};
  launch_pdl(fn, static_cast<unsigned>(g), static_cast<unsigned>(nt), args, sweep_smem(variant), st);
}

int sfu_filter_check(int device, double* err) {
  // once per device and process: ~2.2e9 SFU sines, a few ms
  static std::mutex mu;
  static int state[64];      // 0 unknown, 1 passed, -1 failed
  static double errs[64][2];
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) return 0;
  if (state[device] == 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    unsigned long long* d = nullptr;
    unsigned long long h[2] = {0, 0};
    bool ok = cudaMalloc(&d, sizeof(h)) == cudaSuccess;
    if (ok) ok = cudaMemset(d, 0, sizeof(h)) == cudaSuccess;
    if (ok) {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      k_filter_check<<<sms * 8, 256>>>(d);
      ok = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    if (d) cudaFree(d);
    cudaSetDevice(prev);
    double e0 = 1.0, e1 = 1.0;
    if (ok) {
      std::memcpy(&e0, &h[0], 8);
      std::memcpy(&e1, &h[1], 8);
    }
    errs[device][0] = e0;
    errs[device][1] = e1;
    // the general-q arguments add up to 2 ulp of |y| <= pi (< 4e-7) to the sine error
    state[device] = (ok && e0 + 4.0e-7 <= kFiltEps && e1 < 1.0) ? 1 : -1;
  }
  if (err) {
    err[0] = errs[device][0];
    err[1] = errs[device][1];
  }
  return state[device] > 0;
}

// Shared memory of one DC tile CTA: (l_b + 2)^2 cells x Rc realizations + the two gap lists.
static size_t dc_tile_smem(int lb, int Rc) {
  return sizeof(float) * static_cast<size_t>(lb + 2) * (lb + 2) * Rc + sizeof(int) * 2 * static_cast<size_t>(lb) * lb;
}

int dc_tile_chunk(int lb, int R) {
  // the largest even chunk (<= R, <= MPR_DC_RC, default 4) whose tile fits 200 KB of shared
  // memory; 0: none fits
  static const int cap = [] {
    const char* v = std::getenv("MPR_DC_RC");
    const int c = v ? std::atoi(v) : 4;
    return c >= 2 ? c : 2;
  }();
  for (int rc = std::min(R, cap) & ~1; rc >= 2; rc -= 2)
    if (dc_tile_smem(lb, rc) <= 200 * 1024) return rc;
  return 0;
}

void launch_sweep_dc_tiles(const SweepArgs& s, const int32_t* gid, const float* phiK, const float* T, int64_t Lx,
                           int64_t Ly, int lb, int tau, int Rc, cudaStream_t st) {
  DcTileArgs a{};
  a.gid = gid;
  a.phiK = phiK;
  a.T = T;
  a.G = s.G;
  a.A = s.A;
  a.Lx = Lx;
  a.Ly = Ly;
  a.lb = lb;
  a.tau = tau;
  a.R = s.R;
  a.Rc = Rc;
  a.npairs = s.npairs;
  a.nchunks = (2 * s.npairs + Rc - 1) / Rc;
  a.pair_base = s.pair_base;
  a.sweep = s.sweep;
  for (int i = 0; i < 10; ++i) {
    a.rk0[i] = s.k0 + static_cast<uint32_t>(i) * 0x9E3779B9u;
    a.rk1[i] = s.k1 + static_cast<uint32_t>(i) * 0xBB67AE85u;
  }
  a.q = s.q;
  a.J = s.J;
  a.accumulate = s.accumulate;
  const int nbx = static_cast<int>((Lx + lb - 1) / lb), nby = static_cast<int>((Ly + lb - 1) / lb);
  const size_t smem = dc_tile_smem(lb, Rc);
  const bool qhalf = (s.q == 0.5f);
  const void* fn = qhalf ? reinterpret_cast<const void*>(k_sweep_dc_tile<true>)
                         : reinterpret_cast<const void*>(k_sweep_dc_tile<false>);
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((nbx + 1) / 2), static_cast<unsigned>(nby), static_cast<unsigned>(a.nchunks));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void* args[] = {&a};
  cudaLaunchKernelExC(&cfg, fn, args);
}

void launch_init_states(const GapRec* rec, const float* ginit, float* G, float* A, int64_t P, int R, int npairs,
                        uint32_t pair_base, int random_init, uint32_t k0, uint32_t k1,
                        cudaStream_t st) {
  const bool quad = (npairs % 2) == 0;  // float4 items (R % 4 == 0: 16-byte aligned rows)
  const int64_t items = P * (quad ? npairs / 2 : npairs);
  int64_t g = (items + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  void* args[] = {const_cast<GapRec**>(&rec), const_cast<float**>(&ginit), &G, &A, &P, &R, &npairs, &pair_base,
                  &random_init, &k0, &k1};
  launch_pdl(quad ? reinterpret_cast<const void*>(k_init_states<2>) : reinterpret_cast<const void*>(k_init_states<1>),
             static_cast<unsigned>(g), 256, args, 0, st);
}

void launch_acc_reduce(const float* X, int64_t g_begin, int64_t g_count, int R, int r_lo, int r_hi,
                       double* acc, cudaStream_t st) {
  if (g_count <= 0) return;
  int64_t g = (g_count + kAccTile - 1) / kAccTile;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  int64_t g_end = g_begin + g_count;
  void* args[] = {const_cast<float**>(&X), &g_begin, &g_end, &R, &r_lo, &r_hi, &acc};
  // rows of <= 16 realizations: the direct kernel (staging would leave most lanes idle;
  // C4 at R = 8: 1.1 vs 4.1 ms); longer rows: staged through shared memory
  const bool shortrows = R <= 16;
  launch_pdl(shortrows ? reinterpret_cast<const void*>(k_acc_reduce_short) : reinterpret_cast<const void*>(k_acc_reduce),
             static_cast<unsigned>(g), kAccTile, args, 0, st);
}

}  // namespace mpr
