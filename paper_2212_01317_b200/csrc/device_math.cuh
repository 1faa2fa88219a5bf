// device_math.cuh — sm_100a device implementations of the docs/ARITH.md primitives
// (Philox4x32-10, cos_spec, exp_spec, fixed-point conversions). Written from the
// text of docs/ARITH.md; shares no code with oracle/. Every floating-point operation
// that feeds a decision is an explicit round-to-nearest intrinsic, so nvcc can
// neither contract nor reorder it.
#pragma once
#include <cstdint>

namespace mpr {

constexpr float kTwoPiF = 0x1.921fb6p+2f;  // ARITH notation TWO_PI_F

// ARITH §A — Philox4x32-10. The 32x32->64 products are single IMAD.WIDE.U32 (the split
// IMAD.HI.U32 + IMAD form was measured slower inside the packed sweep kernel:
// profiles/r01_summary.md).
struct Words4 {
  uint32_t w0, w1, w2, w3;
};

__device__ __forceinline__ Words4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return Words4{c0, c1, c2, c3};
}

// The same function with the round keys precomputed (rk0[i] = k0 + i * 0x9E3779B9,
// rk1[i] = k1 + i * 0xBB67AE85). Passed as kernel parameters they are constant-bank operands
// of the LOP3s instead of 20 live registers.
__device__ __forceinline__ Words4 philox4x32_10_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                   const uint32_t (&rk0)[10], const uint32_t (&rk1)[10]) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    c0 = hi1 ^ c1 ^ rk0[round];
    c1 = lo1;
    c2 = hi0 ^ c3 ^ rk1[round];
    c3 = lo0;
  }
  return Words4{c0, c1, c2, c3};
}

// ARITH §B2 — the even part S of sin_spec(x) = x * S(x*x) (degree 5 in t), and S4 for q = 1/2 (the
// products by h = 1/4 folded into the coefficients c_k * 2^-(4k+2): x * S4(x*x) is
// (x/4) * S((x/4)^2) with the exact power-of-two scalings done in the constants).
__device__ __forceinline__ float sin_poly(float t) {
  float p = -0x1.610f4ap-26f;
  p = __fmaf_rn(p, t, 0x1.6b1478p-19f);
  p = __fmaf_rn(p, t, -0x1.9f8a18p-13f);
  p = __fmaf_rn(p, t, 0x1.110ba2p-7f);
  p = __fmaf_rn(p, t, -0x1.55550cp-3f);
  p = __fmaf_rn(p, t, 1.0f);
  return p;
}

__device__ __forceinline__ float sin_poly_quarter(float t) {
  float p = -0x1.610f4ap-48f;
  p = __fmaf_rn(p, t, 0x1.6b1478p-37f);
  p = __fmaf_rn(p, t, -0x1.9f8a18p-27f);
  p = __fmaf_rn(p, t, 0x1.110ba2p-17f);
  p = __fmaf_rn(p, t, -0x1.55550cp-9f);
  p = __fmaf_rn(p, t, 0x1p-2f);
  return p;
}

// u(w) = (w >> 8) * 2^-24, exact.
__device__ __forceinline__ float u24(uint32_t w) {
  return __fmul_rn(__uint2float_rn(w >> 8), 0x1p-24f);
}

// ARITH §B — cos_spec(x) = P(x*x).
__device__ __forceinline__ float cos_spec(float x) {
  const float t = __fmul_rn(x, x);
  float p = 0x1.e0c79cp-30f;
  p = __fmaf_rn(p, t, -0x1.2392p-22f);
  p = __fmaf_rn(p, t, 0x1.9fb7a2p-16f);
  p = __fmaf_rn(p, t, -0x1.6c12aep-10f);
  p = __fmaf_rn(p, t, 0x1.555536p-5f);
  p = __fmaf_rn(p, t, -0.5f);
  p = __fmaf_rn(p, t, 1.0f);
  return p;
}

// cos_spec(0.5 * d) evaluated as P'(d*d) with coefficients c_k * 4^-k: bit-identical
// to cos_spec(__fmul_rn(0.5f, d)) (ARITH §B "implementation latitude").
__device__ __forceinline__ float cos_half_spec(float d) {
  const float t = __fmul_rn(d, d);
  float p = 0x1.e0c79cp-42f;                // c6 * 4^-6
  p = __fmaf_rn(p, t, -0x1.2392p-32f);      // c5 * 4^-5
  p = __fmaf_rn(p, t, 0x1.9fb7a2p-24f);     // c4 * 4^-4
  p = __fmaf_rn(p, t, -0x1.6c12aep-16f);    // c3 * 4^-3
  p = __fmaf_rn(p, t, 0x1.555536p-9f);      // c2 * 4^-2
  p = __fmaf_rn(p, t, -0.125f);             // c1 * 4^-1
  p = __fmaf_rn(p, t, 1.0f);                // c0
  return p;
}

// phi' = u(w) * TWO_PI_F computed as one multiply: (w>>8) * (TWO_PI_F * 2^-24). The
// 2^-24 scaling is exact, so the single rounding is the one of ARITH §H.
__device__ __forceinline__ float proposal_angle(uint32_t w) {
  return __fmul_rn(__uint2float_rn(w >> 8), 0x1.921fb6p-22f);
}

// ARITH §C — exp_spec(x), x <= 0. rint() is done with the 1.5*2^23 magic constant:
// for |v| < 2^22, (v + 1.5*2^23) rounds v to the nearest integer (ties to even) in
// round-to-nearest mode, so n equals rintf(v) bit for bit; the integer n is read
// from the low mantissa bits. No XU (FRND/F2I) instructions.
__device__ __forceinline__ float exp_spec_fast(float x) {
  const float v = __fmul_rn(x, 0x1.715476p+0f);
  const float tm = __fadd_rn(v, 12582912.0f);
  const float n = __fsub_rn(tm, 12582912.0f);
  const int ni = __float_as_int(tm) - 0x4b400000;
  float f = __fmaf_rn(-n, 0x1.62e430p-1f, x);
  f = __fmaf_rn(-n, -0x1.05c610p-29f, f);
  float p = 0x1.6ac2a0p-10f;
  p = __fmaf_rn(p, f, 0x1.126e38p-7f);
  p = __fmaf_rn(p, f, 0x1.555890p-5f);
  p = __fmaf_rn(p, f, 0x1.555408p-3f);
  p = __fmaf_rn(p, f, 0x1.fffffap-2f);
  p = __fmaf_rn(p, f, 1.0f);
  p = __fmaf_rn(p, f, 1.0f);
  const float r = __fmul_rn(p, __int_as_float((ni + 127) << 23));
  return x < -80.0f ? 0.0f : r;
}

__device__ __forceinline__ float exp_spec(float x) {
  const float n = rintf(__fmul_rn(x, 0x1.715476p+0f));
  float f = __fmaf_rn(-n, 0x1.62e430p-1f, x);
  f = __fmaf_rn(-n, -0x1.05c610p-29f, f);
  float p = 0x1.6ac2a0p-10f;
  p = __fmaf_rn(p, f, 0x1.126e38p-7f);
  p = __fmaf_rn(p, f, 0x1.555890p-5f);
  p = __fmaf_rn(p, f, 0x1.555408p-3f);
  p = __fmaf_rn(p, f, 0x1.fffffap-2f);
  p = __fmaf_rn(p, f, 1.0f);
  p = __fmaf_rn(p, f, 1.0f);
  const int ni = static_cast<int>(n);
  const float scale = __int_as_float((ni + 127) << 23);
  const float r = __fmul_rn(p, scale);
  return x < -80.0f ? 0.0f : r;
}

// ---- Packed f32x2 forms (sm_100a FFMA2 / FADD2 / FMUL2) ------------------------------
// Each component is rounded exactly like the scalar __fmaf_rn / __fadd_rn / __fmul_rn, so
// the two realizations of a pair can share one instruction without changing a bit.
// ptxas 12.9 caveat (checked in SASS): a FMUL2 whose result feeds a FADD2 is contracted
// into one FFMA2 even with explicit .rn, which would drop a rounding. The packed code
// below therefore never feeds a packed product into a packed add; where ARITH has a
// product followed by an add (exp_spec's x*log2e + 1.5*2^23) the add is scalar.
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }

// cos_half_spec on both components (ARITH §B with the 4^-k coefficients).
__device__ __forceinline__ float2 cos_half_spec2(float2 d) {
  const float2 t = __fmul2_rn(d, d);
  float2 p = __ffma2_rn(f2(0x1.e0c79cp-42f), t, f2(-0x1.2392p-32f));
  p = __ffma2_rn(p, t, f2(0x1.9fb7a2p-24f));
  p = __ffma2_rn(p, t, f2(-0x1.6c12aep-16f));
  p = __ffma2_rn(p, t, f2(0x1.555536p-9f));
  p = __ffma2_rn(p, t, f2(-0.125f));
  p = __ffma2_rn(p, t, f2(1.0f));
  return p;
}

// S and S4 of ARITH §B2 on both components.
__device__ __forceinline__ float2 sin_poly2(float2 t) {
  float2 p = __ffma2_rn(f2(-0x1.610f4ap-26f), t, f2(0x1.6b1478p-19f));
  p = __ffma2_rn(p, t, f2(-0x1.9f8a18p-13f));
  p = __ffma2_rn(p, t, f2(0x1.110ba2p-7f));
  p = __ffma2_rn(p, t, f2(-0x1.55550cp-3f));
  p = __ffma2_rn(p, t, f2(1.0f));
  return p;
}

__device__ __forceinline__ float2 sin_poly_quarter2(float2 t) {
  float2 p = __ffma2_rn(f2(-0x1.610f4ap-48f), t, f2(0x1.6b1478p-37f));
  p = __ffma2_rn(p, t, f2(-0x1.9f8a18p-27f));
  p = __ffma2_rn(p, t, f2(0x1.110ba2p-17f));
  p = __ffma2_rn(p, t, f2(-0x1.55550cp-9f));
  p = __ffma2_rn(p, t, f2(0x1p-2f));
  return p;
}

// cos_spec on both components (ARITH §B).
__device__ __forceinline__ float2 cos_spec2(float2 x) {
  const float2 t = __fmul2_rn(x, x);
  float2 p = __ffma2_rn(f2(0x1.e0c79cp-30f), t, f2(-0x1.2392p-22f));
  p = __ffma2_rn(p, t, f2(0x1.9fb7a2p-16f));
  p = __ffma2_rn(p, t, f2(-0x1.6c12aep-10f));
  p = __ffma2_rn(p, t, f2(0x1.555536p-5f));
  p = __ffma2_rn(p, t, f2(-0.5f));
  p = __ffma2_rn(p, t, f2(1.0f));
  return p;
}

// exp_spec_fast on both components (ARITH §C): the rounding add is scalar (see above),
// everything after it packed.
__device__ __forceinline__ float2 exp_spec_fast2(float2 x) {
  const float vx = __fmul_rn(x.x, 0x1.715476p+0f);
  const float vy = __fmul_rn(x.y, 0x1.715476p+0f);
  const float2 tm = make_float2(__fadd_rn(vx, 12582912.0f), __fadd_rn(vy, 12582912.0f));
  const float2 n = __fadd2_rn(tm, f2(-12582912.0f));  // exact
  const float2 nn = make_float2(-n.x, -n.y);
  float2 f = __ffma2_rn(nn, f2(0x1.62e430p-1f), x);
  f = __ffma2_rn(nn, f2(-0x1.05c610p-29f), f);
  float2 p = __ffma2_rn(f2(0x1.6ac2a0p-10f), f, f2(0x1.126e38p-7f));
  p = __ffma2_rn(p, f, f2(0x1.555890p-5f));
  p = __ffma2_rn(p, f, f2(0x1.555408p-3f));
  p = __ffma2_rn(p, f, f2(0x1.fffffap-2f));
  p = __ffma2_rn(p, f, f2(1.0f));
  p = __ffma2_rn(p, f, f2(1.0f));
  const int nx = __float_as_int(tm.x) - 0x4b400000, ny = __float_as_int(tm.y) - 0x4b400000;
  const float2 r = __fmul2_rn(p, make_float2(__int_as_float((nx + 127) << 23), __int_as_float((ny + 127) << 23)));
  return make_float2(x.x < -80.0f ? 0.0f : r.x, x.y < -80.0f ? 0.0f : r.y);
}

// exp_spec_fast2(x) * 2^24, exactly: the power-of-two scale of the last step carries the
// extra 2^24 (n >= -116 keeps p * 2^(n+24) normal, so the product is the same exact scaling
// of p * 2^n). Compared with (float)(w >> 8) it decides u(w) < exp_spec(x) without forming
// u(w) = (w >> 8) * 2^-24 (ARITH §A/§C: both sides are exact power-of-two scalings).
__device__ __forceinline__ float2 exp_spec_fast2_x24(float2 x) {
  const float2 v = __fmul2_rn(x, f2(0x1.715476p+0f));  // packed product, scalar adds below
  const float2 tm = make_float2(__fadd_rn(v.x, 12582912.0f), __fadd_rn(v.y, 12582912.0f));
  const float2 n = __fadd2_rn(tm, f2(-12582912.0f));  // exact
  const float2 nn = make_float2(-n.x, -n.y);
  float2 f = __ffma2_rn(nn, f2(0x1.62e430p-1f), x);
  f = __ffma2_rn(nn, f2(-0x1.05c610p-29f), f);
  float2 p = __ffma2_rn(f2(0x1.6ac2a0p-10f), f, f2(0x1.126e38p-7f));
  p = __ffma2_rn(p, f, f2(0x1.555890p-5f));
  p = __ffma2_rn(p, f, f2(0x1.555408p-3f));
  p = __ffma2_rn(p, f, f2(0x1.fffffap-2f));
  p = __ffma2_rn(p, f, f2(1.0f));
  p = __ffma2_rn(p, f, f2(1.0f));
  const int nx = __float_as_int(tm.x) - 0x4b400000, ny = __float_as_int(tm.y) - 0x4b400000;
  const float2 r = __fmul2_rn(p, make_float2(__int_as_float((nx + 127 + 24) << 23), __int_as_float((ny + 127 + 24) << 23)));
  return make_float2(x.x < -80.0f ? 0.0f : r.x, x.y < -80.0f ? 0.0f : r.y);
}

// Order-preserving key of a float for integer atomicMin/atomicMax.
__device__ __forceinline__ int float_to_ordered(float f) {
  const int b = __float_as_int(f);
  return b >= 0 ? b : (b ^ 0x7fffffff);
}
__device__ __host__ __forceinline__ float ordered_to_float(int k) {
  const int b = k >= 0 ? k : (k ^ 0x7fffffff);
#ifdef __CUDA_ARCH__
  return __int_as_float(b);
#else
  float f;
  __builtin_memcpy(&f, &b, 4);
  return f;
#endif
}

}  // namespace mpr
