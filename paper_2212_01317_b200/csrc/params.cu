// params.cu — parameter-stage kernels of the LE-MPR hot path (a1-a5, a11 of SURVEY §8(a)).
//
//  k_minmax_count   a1  sample min/max + counts          (ARITH §D)
//  k_transform      a2  data -> spin angles at samples   (ARITH §D)
//  k_row_* / scan   gap-site index (colour, row-major) used by the sweep layout
//  k_block_stats    a3  block sample-bond sums, exact fixed point (ARITH §E-F)
//  k_block_T        a4  energy matching by table inversion (ARITH §F)
//  k_median_fill    a4  lower-median fallback, radix select
//  k_expand/k_smooth a5 BST step field and SST window smoothing
//  k_build_records      per-gap records: neighbours, beta = 1/T, BLOCK_MEAN init (ARITH §G)
//  k_predict        a11 back-transform of the conditional mean (ARITH §I)
//
// All of these are HBM-bound streaming/stencil kernels that run once per problem;
// the hot loop is in sweep.cu.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "device_math.cuh"
#include "internal.cuh"

namespace mpr {

namespace {

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_ull(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------------- a1: min/max
// 16 sites per thread per iteration: 4 x LDG.128 of z + 1 x LDG.128 of the mask.
template <bool VEC>
__global__ void __launch_bounds__(256) k_minmax_count(const float* __restrict__ z,
                                                      const uint8_t* __restrict__ mask,
                                                      int64_t Lx, int64_t n, int64_t row_base,
                                                      DevScalars* sc) {
  int kmin = 0x7fffffff, kmax = static_cast<int>(0x80000000u);
  unsigned long long nk = 0, ng0 = 0, ng1 = 0;
  int bad = 0;
  const int64_t nchunks = (n + 15) / 16;
  for (int64_t ch = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ch < nchunks;
       ch += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = ch * 16;
    float zv[16];
    uint8_t mv[16];
    if (VEC && i0 + 16 <= n) {
      const float4* z4 = reinterpret_cast<const float4*>(z + i0);
      const uint4 m4 = *reinterpret_cast<const uint4*>(mask + i0);
      const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
      for (int k = 0; k < 16; ++k) mv[k] = static_cast<uint8_t>(mw[k >> 2] >> (8 * (k & 3)));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // z at gaps is never used: load all 4 (the bytes are in range), select below.
        const float4 v = __ldg(z4 + k);
        zv[4 * k] = v.x; zv[4 * k + 1] = v.y; zv[4 * k + 2] = v.z; zv[4 * k + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int64_t i = i0 + k;
        mv[k] = i < n ? mask[i] : 1;  // out of range: treated below via i < n
        zv[k] = (i < n && mv[k]) ? z[i] : 0.0f;
      }
    }
    int64_t r = i0 / Lx + row_base, c = i0 - (i0 / Lx) * Lx;  // r: global row (colour parity)
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const bool in = (i0 + k) < n;
      if (in) {
        if (mv[k]) {
          const float v = zv[k];
          if (!isfinite(v)) bad = 1;
          const int key = float_to_ordered(v);
          kmin = min(kmin, key);
          kmax = max(kmax, key);
          ++nk;
        } else if (((r + c) & 1) == 0) {
          ++ng0;
        } else {
          ++ng1;
        }
      }
      if (++c == Lx) { c = 0; ++r; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  nk = warp_sum_ull(nk);
  ng0 = warp_sum_ull(ng0);
  ng1 = warp_sum_ull(ng1);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&sc->zmin_key, kmin);
    atomicMax(&sc->zmax_key, kmax);
    if (bad) atomicOr(&sc->bad_sample, 1);
    atomicAdd(&sc->n_known, nk);
    atomicAdd(&sc->n_gap[0], ng0);
    atomicAdd(&sc->n_gap[1], ng1);
  }
}

__device__ __forceinline__ void range_params(const DevScalars* sc, float* zmin, float* zmax,
                                             float* s) {
  // ARITH §D: canonicalise -0 to +0, then s = TWO_PI_F / (z_max - z_min).
  *zmin = __fadd_rn(ordered_to_float(sc->zmin_key), 0.0f);
  *zmax = __fadd_rn(ordered_to_float(sc->zmax_key), 0.0f);
  *s = (*zmax == *zmin) ? 0.0f : __fdiv_rn(kTwoPiF, __fsub_rn(*zmax, *zmin));
}

// ----------------------------------------------------------------- a2: transform
template <bool VEC>
__global__ void __launch_bounds__(256) k_transform(const float* __restrict__ z,
                                                   const uint8_t* __restrict__ mask, int64_t n,
                                                   const DevScalars* __restrict__ sc,
                                                   float* __restrict__ phi) {
  float zmin, zmax, s;
  range_params(sc, &zmin, &zmax, &s);
  const int64_t nch = (n + 3) / 4;
  for (int64_t ch = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ch < nch;
       ch += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = ch * 4;
    if (VEC && i0 + 4 <= n) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(z + i0));
      const uint32_t m = *reinterpret_cast<const uint32_t*>(mask + i0);
      const float zz[4] = {v.x, v.y, v.z, v.w};
      float o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool known = (m >> (8 * k)) & 0xffu;
        const float p = fminf(__fmul_rn(__fsub_rn(zz[k], zmin), s), kTwoPiF);
        o[k] = known ? p : 0.0f;
      }
      *reinterpret_cast<float4*>(phi + i0) = make_float4(o[0], o[1], o[2], o[3]);
    } else {
      for (int64_t i = i0; i < n && i < i0 + 4; ++i)
        phi[i] = mask[i] ? fminf(__fmul_rn(__fsub_rn(z[i], zmin), s), kTwoPiF) : 0.0f;
    }
  }
}

// ------------------------------------------------------------ gap-site index
// Gap ids: colour A ((r+c) even) first, then colour B; row-major within a colour.
// Local rows r = 0 .. Ly-1 of a buffer whose row 0 is global row row_base (row slabs);
// colours are global: (row_base + r + c) & 1.
__global__ void __launch_bounds__(256) k_row_counts(const uint8_t* __restrict__ mask, int64_t Lx,
                                                    int64_t Ly, int64_t row_base,
                                                    int* __restrict__ rowcnt) {
  const int64_t r = blockIdx.x;
  int cnt[2] = {0, 0};
  for (int64_t c = threadIdx.x; c < Lx; c += blockDim.x)
    if (!mask[r * Lx + c]) ++cnt[(row_base + r + c) & 1];
  __shared__ int s[2][8];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    int v = cnt[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s[k][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    int v = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += s[threadIdx.x][w];
    rowcnt[threadIdx.x * Ly + r] = v;
  }
}

// Exclusive scan of m ints (single CTA, 1024 threads, chunked with carry).
__global__ void __launch_bounds__(1024) k_scan_excl(const int* __restrict__ in, int64_t m,
                                                    int* __restrict__ out) {
  __shared__ int warp_tot[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < m; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int v = i < m ? in[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive
    }
    __syncthreads();
    const int wbase = wid ? warp_tot[wid - 1] : 0;
    if (i < m) out[i] = static_cast<int>(carry) + wbase + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_tot[31];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_row_compact(const uint8_t* __restrict__ mask, int64_t Lx,
                                                     int64_t Ly, int64_t row_base,
                                                     const int* __restrict__ rowoff,
                                                     int32_t* __restrict__ gid) {
  const int64_t r = blockIdx.x;
  __shared__ int wcnt[2][8];
  __shared__ int base[2];
  if (threadIdx.x < 2) base[threadIdx.x] = rowoff[threadIdx.x * Ly + r];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  for (int64_t c0 = 0; c0 < Lx; c0 += blockDim.x) {
    const int64_t c = c0 + threadIdx.x;
    const int64_t i = r * Lx + c;
    const bool in = c < Lx;
    const bool gap = in && !mask[i];
    const int col = static_cast<int>((row_base + r + c) & 1);
    const unsigned b0 = __ballot_sync(0xffffffffu, gap && col == 0);
    const unsigned b1 = __ballot_sync(0xffffffffu, gap && col == 1);
    if (lane == 0) { wcnt[0][wid] = __popc(b0); wcnt[1][wid] = __popc(b1); }
    __syncthreads();
    int pre = 0;
    for (int w = 0; w < wid; ++w) pre += wcnt[col][w];
    const unsigned below = (1u << lane) - 1u;
    const int rank = pre + __popc((col ? b1 : b0) & below);
    if (in) {
      if (gap) {
        const int g = base[col] + rank;
        gid[i] = g;
      } else {
        gid[i] = -1;
      }
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      int t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wcnt[threadIdx.x][w];
      base[threadIdx.x] += t;
    }
    __syncthreads();
  }
}

// The same compaction with one WARP per row and no block barriers (Lx % 4 == 0, 4-byte
// aligned mask rows): each lane takes 4 columns (one 32-bit mask load) per step, the lanes'
// per-colour gap counts are scanned with shuffles, and the ids go out as one int4 per lane
// (512 contiguous bytes per warp step). The next step's mask word is loaded ahead.
__global__ void __launch_bounds__(256) k_row_compact4(const uint8_t* __restrict__ mask, int64_t Lx,
                                                      int64_t Ly, int64_t row_base,
                                                      const int* __restrict__ rowoff,
                                                      int32_t* __restrict__ gid) {
  const int64_t r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= Ly) return;
  const int lane = threadIdx.x & 31;
  const uint8_t* mrow = mask + r * Lx;
  int32_t* grow = gid + r * Lx;
  int base0 = rowoff[r], base1 = rowoff[Ly + r];  // first id of colour 0 / 1 in this row
  // colour of column c: (row_base + r + c) & 1; lane columns 4l .. 4l+3 alternate from par
  const int par = static_cast<int>((row_base + r) & 1);
  uint32_t w = 0;
  if (4 * lane < Lx) w = *reinterpret_cast<const uint32_t*>(mrow + 4 * lane);
  for (int64_t c0 = 0; c0 < Lx; c0 += 128) {
    const int64_t c = c0 + 4 * lane;
    const bool in = c < Lx;
    const uint32_t cur = w;
    if (c + 128 < Lx) w = *reinterpret_cast<const uint32_t*>(mrow + c + 128);
    int gaps[4];
    int n0 = 0, n1 = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      gaps[k] = in && ((cur >> (8 * k)) & 0xffu) == 0;
      if (((par + k) & 1) == 0) n0 += gaps[k];  // c is a multiple of 4: (c + k) & 1 == k & 1
      else n1 += gaps[k];
    }
    int x0 = n0, x1 = n1;  // inclusive scans over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
      if (lane >= o) { x0 += y0; x1 += y1; }
    }
    int i0 = base0 + x0 - n0, i1 = base1 + x1 - n1;
    int out[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool col0 = ((par + k) & 1) == 0;
      out[k] = gaps[k] ? (col0 ? i0++ : i1++) : -1;
    }
    if (in) *reinterpret_cast<int4*>(grow + c) = make_int4(out[0], out[1], out[2], out[3]);
    base0 += __shfl_sync(0xffffffffu, x0, 31);
    base1 += __shfl_sync(0xffffffffu, x1, 31);
  }
}

// ----------------------------------------------------- a3: block bond statistics
constexpr int kTile = 32;            // 32 x 32 sites per CTA
constexpr int kMaxSlots = 17 * 17;   // blocks a tile can touch when l_b >= 2

// Rows [row0, row1) (global) of a local buffer whose row 0 is global row lrow0; the buffer
// also holds row row1 when row1 < Ly (the down bonds of the last own row read it). Tiles are
// aligned to global multiples of 32 rows, so a tile lies in one l_b block whenever l_b is a
// multiple of 32, wherever the slab starts.
__global__ void __launch_bounds__(256) k_block_stats(const float* __restrict__ phi,
                                                     const uint8_t* __restrict__ mask, int64_t Lx,
                                                     int64_t Ly, int64_t lrow0, int64_t row0,
                                                     int64_t row1, int lb, float q,
                                                     long long* __restrict__ SB,
                                                     long long* __restrict__ NB,
                                                     long long* __restrict__ SP,
                                                     long long* __restrict__ NK, DevScalars* sc) {
  __shared__ long long sSB[kMaxSlots], sNB[kMaxSlots], sSP[kMaxSlots], sNK[kMaxSlots];
  long long tsb2 = 0;  // this thread's squared sample-bond cosines (fixed point, R22)
  const int64_t c0 = (int64_t)blockIdx.x * kTile, r0 = (row0 / kTile) * kTile + (int64_t)blockIdx.y * kTile;
  const int64_t nbx = (Lx + lb - 1) / lb;
  const int64_t bc0 = c0 / lb, br0 = max(r0, row0) / lb;
  const int64_t cl = min(c0 + kTile, Lx) - 1, rl = min(r0 + kTile, row1) - 1;
  const int nbc = static_cast<int>(cl / lb - bc0 + 1), nbr = static_cast<int>(rl / lb - br0 + 1);
  const int nslots = nbc * nbr;
  for (int t = threadIdx.x; t < nslots; t += blockDim.x) { sSB[t] = 0; sNB[t] = 0; sSP[t] = 0; sNK[t] = 0; }
  __syncthreads();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (nslots == 1) {
    // the whole tile lies in one l_b block (l_b a multiple of 32, the default 32 included):
    // each thread sums its 4 sites in registers, then one warp reduction per warp (the sums
    // are exact integers, so the grouping does not matter)
    long long vsb = 0, vsp = 0;
    int vnb = 0, vnk = 0;
#pragma unroll
    for (int k = 0; k < kTile / 8; ++k) {
      const int64_t r = r0 + ty + 8 * k, c = c0 + tx;
      if (r >= row0 && r < row1 && c < Lx) {
        const int64_t i = (r - lrow0) * Lx + c;
        if (mask[i]) {
          const float pi = phi[i];
          vsp += __float2ll_rn(__fmul_rn(pi, 0x1p28f));
          vnk += 1;
          if (c + 1 < Lx && mask[i + 1]) {
            const float bnd = cos_spec(__fmul_rn(q, __fsub_rn(pi, phi[i + 1])));
            vsb += __float2ll_rn(__fmul_rn(bnd, 0x1p32f));
            tsb2 += __float2ll_rn(__fmul_rn(__fmul_rn(bnd, bnd), 0x1p32f));
            vnb += 1;
          }
          if (r + 1 < Ly && mask[i + Lx]) {
            const float bnd = cos_spec(__fmul_rn(q, __fsub_rn(pi, phi[i + Lx])));
            vsb += __float2ll_rn(__fmul_rn(bnd, 0x1p32f));
            tsb2 += __float2ll_rn(__fmul_rn(__fmul_rn(bnd, bnd), 0x1p32f));
            vnb += 1;
          }
        }
      }
    }
    vsb = warp_sum_ll(vsb);
    vsp = warp_sum_ll(vsp);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      vnb += __shfl_xor_sync(0xffffffffu, vnb, off);
      vnk += __shfl_xor_sync(0xffffffffu, vnk, off);
    }
    if (tx == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&sSB[0]), static_cast<unsigned long long>(vsb));
      atomicAdd(reinterpret_cast<unsigned long long*>(&sNB[0]), static_cast<unsigned long long>(vnb));
      atomicAdd(reinterpret_cast<unsigned long long*>(&sSP[0]), static_cast<unsigned long long>(vsp));
      atomicAdd(reinterpret_cast<unsigned long long*>(&sNK[0]), static_cast<unsigned long long>(vnk));
    }
  } else {
  // block column of this thread's site column: one 32-bit division per thread (Lx, Ly < 2^31)
  const int cbl = static_cast<int>(static_cast<uint32_t>(c0 + tx) / static_cast<uint32_t>(lb) - bc0);
  for (int k = 0; k < kTile / 8; ++k) {
    const int64_t r = r0 + ty + 8 * k, c = c0 + tx;
    long long vsb = 0, vnb = 0, vsp = 0, vnk = 0;
    int slot = 0;
    const bool in = r >= row0 && r < row1 && c < Lx;
    if (in) {
      const int rbl = static_cast<int>(static_cast<uint32_t>(r) / static_cast<uint32_t>(lb) - br0);
      slot = rbl * nbc + cbl;
      const int64_t i = (r - lrow0) * Lx + c;
      if (mask[i]) {
        const float pi = phi[i];
        vsp = __float2ll_rn(__fmul_rn(pi, 0x1p28f));
        vnk = 1;
        if (c + 1 < Lx && mask[i + 1]) {
          const float b = cos_spec(__fmul_rn(q, __fsub_rn(pi, phi[i + 1])));
          vsb += __float2ll_rn(__fmul_rn(b, 0x1p32f));
          tsb2 += __float2ll_rn(__fmul_rn(__fmul_rn(b, b), 0x1p32f));
          vnb += 1;
        }
        if (r + 1 < Ly && mask[i + Lx]) {
          const float b = cos_spec(__fmul_rn(q, __fsub_rn(pi, phi[i + Lx])));
          vsb += __float2ll_rn(__fmul_rn(b, 0x1p32f));
          tsb2 += __float2ll_rn(__fmul_rn(__fmul_rn(b, b), 0x1p32f));
          vnb += 1;
        }
      }
    }
    const int slot0 = __shfl_sync(0xffffffffu, slot, 0);
    if (!in) slot = slot0;
    if (__all_sync(0xffffffffu, slot == slot0)) {
      vsb = warp_sum_ll(vsb); vnb = warp_sum_ll(vnb); vsp = warp_sum_ll(vsp); vnk = warp_sum_ll(vnk);
      if (tx == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&sSB[slot0]), static_cast<unsigned long long>(vsb));
        atomicAdd(reinterpret_cast<unsigned long long*>(&sNB[slot0]), static_cast<unsigned long long>(vnb));
        atomicAdd(reinterpret_cast<unsigned long long*>(&sSP[slot0]), static_cast<unsigned long long>(vsp));
        atomicAdd(reinterpret_cast<unsigned long long*>(&sNK[slot0]), static_cast<unsigned long long>(vnk));
      }
    } else if (in) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&sSB[slot]), static_cast<unsigned long long>(vsb));
      atomicAdd(reinterpret_cast<unsigned long long*>(&sNB[slot]), static_cast<unsigned long long>(vnb));
      atomicAdd(reinterpret_cast<unsigned long long*>(&sSP[slot]), static_cast<unsigned long long>(vsp));
      atomicAdd(reinterpret_cast<unsigned long long*>(&sNK[slot]), static_cast<unsigned long long>(vnk));
    }
  }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nslots; t += blockDim.x) {
    const int64_t b = (br0 + t / nbc) * nbx + (bc0 + t % nbc);
    if (sSB[t]) atomicAdd(reinterpret_cast<unsigned long long*>(&SB[b]), static_cast<unsigned long long>(sSB[t]));
    if (sNB[t]) atomicAdd(reinterpret_cast<unsigned long long*>(&NB[b]), static_cast<unsigned long long>(sNB[t]));
    if (sSP[t]) atomicAdd(reinterpret_cast<unsigned long long*>(&SP[b]), static_cast<unsigned long long>(sSP[t]));
    if (sNK[t]) atomicAdd(reinterpret_cast<unsigned long long*>(&NK[b]), static_cast<unsigned long long>(sNK[t]));
  }
  tsb2 = warp_sum_ll(tsb2);
  if ((threadIdx.x & 31) == 0 && tsb2)
    atomicAdd(reinterpret_cast<unsigned long long*>(&sc->sum_SB2), static_cast<unsigned long long>(tsb2));
}

// Streaming form of a3 for l_b % 4 == 0 and Lx % 4 == 0 (16-byte aligned rows): a thread owns
// 4 adjacent columns and walks kRowsPerWarp rows, loading phi (float4) and mask (4 bytes) of
// each row ONCE — the row below of one step is the current row of the next — and the right
// neighbour of its 4th column from the next lane (lane 31 loads it). Sums stay in registers
// until the thread's block row changes, then go to per-CTA shared slots (one warp-reduction
// per group of lanes sharing a block when l_b / 4 is a power of two) and once per CTA to
// global memory. A CTA covers 128 columns x 8 warps x kRowsPerWarp rows, aligned to global
// row multiples so that l_b = 32 tiles never straddle a block row. Integer sums: the result
// is k_block_stats' bit for bit.
constexpr int kRowsPerWarp = 8;
constexpr int kBs4Cols = 128, kBs4Rows = 8 * kRowsPerWarp;
constexpr int kBs4Slots = (kBs4Cols / 4 + 1) * (kBs4Rows / 4 + 1);  // l_b >= 4
__global__ void __launch_bounds__(256) k_block_stats4(const float* __restrict__ phi,
                                                      const uint8_t* __restrict__ mask, int64_t Lx64,
                                                      int64_t Ly64, int64_t lrow064, int64_t row064,
                                                      int64_t row164, int lb, float q,
                                                      long long* __restrict__ SB,
                                                      long long* __restrict__ NB,
                                                      long long* __restrict__ SP,
                                                      long long* __restrict__ NK, DevScalars* sc) {
  __shared__ unsigned long long sl[4][kBs4Slots];
  long long tsb2 = 0;  // this thread's squared sample-bond cosines (fixed point, R22)
  // 32-bit index arithmetic (< 2^30 sites)
  const int Lx = static_cast<int>(Lx64), Ly = static_cast<int>(Ly64), lrow0 = static_cast<int>(lrow064);
  const int row0 = static_cast<int>(row064), row1 = static_cast<int>(row164);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int cbase = blockIdx.x * kBs4Cols;
  const int rbase = (row0 / kBs4Rows) * kBs4Rows + blockIdx.y * kBs4Rows;
  const int nbx = (Lx + lb - 1) / lb;
  const int bc0 = cbase / lb, br0 = max(rbase, row0) / lb;
  const int clast = min(cbase + kBs4Cols, Lx) - 1, rlast = min(rbase + kBs4Rows, row1) - 1;
  const int nbc = clast / lb - bc0 + 1;
  const int nslots = nbc * (rlast / lb - br0 + 1);
  for (int t = threadIdx.x; t < 4 * kBs4Slots; t += blockDim.x) sl[t / kBs4Slots][t % kBs4Slots] = 0ull;
  __syncthreads();
  const int c = cbase + 4 * lane;  // first of this thread's 4 columns
  const bool cin = c < Lx;         // Lx % 4 == 0: all 4 or none
  const int bcl = cin ? c / lb - bc0 : 0;
  const int grp = lb / 4;                                      // lanes per block column
  const bool pow2 = grp <= 32 && (grp & (grp - 1)) == 0 && (cbase % lb) == 0;
  const int ra = max(rbase + wp * kRowsPerWarp, row0), rz = min(rbase + (wp + 1) * kRowsPerWarp, row1);
  long long sb = 0, sp = 0;
  int nb = 0, nk = 0;
  int cur_br = ra < rz ? ra / lb : -1;
  auto flush = [&](int br) {
    // every lane of the warp calls this together (warp-uniform row loop)
    const int slot = (br - br0) * nbc + bcl;
    long long v[4] = {sb, static_cast<long long>(nb), sp, static_cast<long long>(nk)};
    if (pow2) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        for (int o = 1; o < grp; o <<= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (cin && (!pow2 || (lane % grp) == 0)) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (v[k]) atomicAdd(&sl[k][slot], static_cast<unsigned long long>(v[k]));
    }
    sb = sp = 0;
    nb = nk = 0;
  };
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t m = 0;
  if (ra < rz && cin) {
    const int i = (ra - lrow0) * Lx + c;
    p = *reinterpret_cast<const float4*>(phi + i);
    m = *reinterpret_cast<const uint32_t*>(mask + i);
  }
  for (int r = ra; r < rz; ++r) {
    const int br = r / lb;
    if (br != cur_br) {
      flush(cur_br);
      cur_br = br;
    }
    const bool down = r + 1 < Ly;
    const int i = (r - lrow0) * Lx + c;
    float4 pn = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t mn = 0;
    if (down && cin) {
      pn = *reinterpret_cast<const float4*>(phi + i + Lx);
      mn = *reinterpret_cast<const uint32_t*>(mask + i + Lx);
    }
    // right neighbour of the 4th column: the next lane's first, lane 31 loads it
    float pr = __shfl_down_sync(0xffffffffu, p.x, 1);
    uint32_t mr = __shfl_down_sync(0xffffffffu, m, 1) & 0xffu;
    if (lane == 31) {
      pr = 0.f;
      mr = 0;
      if (cin && c + 4 < Lx) {
        pr = phi[i + 4];
        mr = mask[i + 4];
      }
    }
    const float pv[5] = {p.x, p.y, p.z, p.w, pr};
    const float pd[4] = {pn.x, pn.y, pn.z, pn.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool kj = (m >> (8 * j)) & 0xffu;
      if (!kj) continue;
      sp += __float2ll_rn(__fmul_rn(pv[j], 0x1p28f));
      nk += 1;
      const bool kr = j < 3 ? ((m >> (8 * (j + 1))) & 0xffu) != 0 : mr != 0;
      if (kr) {  // right bond (c + j + 1 < Lx: a column past the edge has mask 0)
        const float b = cos_spec(__fmul_rn(q, __fsub_rn(pv[j], pv[j + 1])));
        sb += __float2ll_rn(__fmul_rn(b, 0x1p32f));
        tsb2 += __float2ll_rn(__fmul_rn(__fmul_rn(b, b), 0x1p32f));
        nb += 1;
      }
      if ((mn >> (8 * j)) & 0xffu) {  // down bond
        const float b = cos_spec(__fmul_rn(q, __fsub_rn(pv[j], pd[j])));
        sb += __float2ll_rn(__fmul_rn(b, 0x1p32f));
        tsb2 += __float2ll_rn(__fmul_rn(__fmul_rn(b, b), 0x1p32f));
        nb += 1;
      }
    }
    p = pn;
    m = mn;
  }
  if (cur_br >= 0) flush(cur_br);
  __syncthreads();
  for (int t = threadIdx.x; t < nslots; t += blockDim.x) {
    const int64_t b = static_cast<int64_t>(br0 + t / nbc) * nbx + (bc0 + t % nbc);
    if (sl[0][t]) atomicAdd(reinterpret_cast<unsigned long long*>(&SB[b]), sl[0][t]);
    if (sl[1][t]) atomicAdd(reinterpret_cast<unsigned long long*>(&NB[b]), sl[1][t]);
    if (sl[2][t]) atomicAdd(reinterpret_cast<unsigned long long*>(&SP[b]), sl[2][t]);
    if (sl[3][t]) atomicAdd(reinterpret_cast<unsigned long long*>(&NK[b]), sl[3][t]);
  }
  tsb2 = warp_sum_ll(tsb2);
  if ((threadIdx.x & 31) == 0 && tsb2)
    atomicAdd(reinterpret_cast<unsigned long long*>(&sc->sum_SB2), static_cast<unsigned long long>(tsb2));
}

// ------------------------------------------------- a4: e_b -> T_b (table inversion)
__global__ void __launch_bounds__(256) k_block_T(const long long* __restrict__ SB,
                                                 const long long* __restrict__ NB,
                                                 const long long* __restrict__ SP,
                                                 const long long* __restrict__ NK, int64_t nblocks,
                                                 const float* __restrict__ calT,
                                                 const float* __restrict__ cale, int K,
                                                 float* __restrict__ Tb, DevScalars* sc) {
  __shared__ float sT[256], se[256];
  for (int k = threadIdx.x; k < K; k += blockDim.x) { sT[k] = calT[k]; se[k] = cale[k]; }
  __syncthreads();
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long avail = 0;
  long long sb = 0, sp = 0, nk = 0, nbs = 0;
  if (b < nblocks) {
    const long long nbv = NB[b];
    sb = SB[b]; sp = SP[b]; nk = NK[b]; nbs = nbv;
    float T = -1.0f;  // marker: no sample bond in this block
    if (nbv > 0) {
      const double a = -__ll2double_rn(sb) * 0x1p-32;
      const float e = __double2float_rn(__ddiv_rn(a, __ll2double_rn(nbv)));
      if (e <= se[0]) {
        T = sT[0];
      } else if (e >= se[K - 1]) {
        T = sT[K - 1];
      } else {
        int k = 0;
        for (int j = 1; j < K; ++j)
          if (se[j] <= e) k = j;
        const float w = __fdiv_rn(__fsub_rn(e, se[k]), __fsub_rn(se[k + 1], se[k]));
        T = __fadd_rn(sT[k], __fmul_rn(w, __fsub_rn(sT[k + 1], sT[k])));
      }
      avail = 1;
    }
    Tb[b] = T;
  }
  avail = warp_sum_ull(avail);
  sb = warp_sum_ll(sb); sp = warp_sum_ll(sp); nk = warp_sum_ll(nk); nbs = warp_sum_ll(nbs);
  if ((threadIdx.x & 31) == 0) {
    if (avail) atomicAdd(&sc->n_avail, avail);
    if (nbs) atomicAdd(reinterpret_cast<unsigned long long*>(&sc->sum_NB), static_cast<unsigned long long>(nbs));
    if (sb) atomicAdd(reinterpret_cast<unsigned long long*>(&sc->sum_SB), static_cast<unsigned long long>(sb));
    if (sp) atomicAdd(reinterpret_cast<unsigned long long*>(&sc->sum_SP), static_cast<unsigned long long>(sp));
    if (nk) atomicAdd(reinterpret_cast<unsigned long long*>(&sc->sum_NK), static_cast<unsigned long long>(nk));
  }
}

// a6 BLOCK_MEAN initial angle of every block (ARITH §G): the block's mean known angle, or the
// global sample mean for a block without samples — one fp64 division per block instead of
// one per gap site in the record builder.
__global__ void __launch_bounds__(256) k_block_init(const long long* __restrict__ SP,
                                                    const long long* __restrict__ NK, int64_t nblocks,
                                                    const DevScalars* __restrict__ sc,
                                                    float* __restrict__ binit) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  const long long nk = NK[b];
  binit[b] = nk ? __double2float_rn(__ddiv_rn(__ll2double_rn(SP[b]) * 0x1p-28, __ll2double_rn(nk)))
                : __double2float_rn(__ddiv_rn(__ll2double_rn(sc->sum_SP) * 0x1p-28, __ll2double_rn(sc->sum_NK)));
}

// ------------------------------------------- a4: lower median + fallback (1 CTA)
// Radix select (4 passes of 8 bits) on the bit patterns of the positive available T_b.
__global__ void __launch_bounds__(1024) k_median_fill(float* __restrict__ Tb,
                                                      const long long* __restrict__ NB,
                                                      int64_t nblocks, DevScalars* sc) {
  __shared__ unsigned hist[256];
  __shared__ unsigned prefix, pmask;
  __shared__ unsigned long long rank;
  const unsigned long long n = sc->n_avail;
  if (n == 0) return;
  if (threadIdx.x == 0) { prefix = 0; pmask = 0; rank = (n - 1) / 2; }
  __syncthreads();
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    const unsigned pf = prefix, pm = pmask;
    for (int64_t b = threadIdx.x; b < nblocks; b += blockDim.x) {
      const float v = Tb[b];
      if (v > 0.0f) {
        const unsigned bits = __float_as_uint(v);
        if ((bits & pm) == pf) atomicAdd(&hist[(bits >> shift) & 255u], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long cum = 0;
      unsigned bin = 0;
      for (; bin < 256; ++bin) {
        if (cum + hist[bin] > rank) break;
        cum += hist[bin];
      }
      rank -= cum;
      prefix |= bin << shift;
      pmask |= 255u << shift;
    }
    __syncthreads();
  }
  const float med = __uint_as_float(prefix);
  unsigned long long nf = 0;
  for (int64_t b = threadIdx.x; b < nblocks; b += blockDim.x)
    if (NB[b] == 0) { Tb[b] = med; ++nf; }
  nf = warp_sum_ull(nf);
  if ((threadIdx.x & 31) == 0 && nf) atomicAdd(&sc->n_fallback, nf);
  if (threadIdx.x == 0) sc->median_T = med;
}

// ---------------------------------------------------- a5: expand + SST smoothing
// Local temperature rows [trow0, trow1) (global): T[(r - trow0) * Lx + c] = Tb(block(r, c)).
__global__ void __launch_bounds__(256) k_expand(const float* __restrict__ Tb, int64_t Lx,
                                                int64_t trow0, int64_t trow1, int lb,
                                                float* __restrict__ T) {
  const int64_t n = Lx * (trow1 - trow0), nbx = (Lx + lb - 1) / lb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lr = i / Lx, c = i - lr * Lx;
    T[i] = Tb[((lr + trow0) / lb) * nbx + c / lb];
  }
}

// One SST pass: clipped (2rs+1)^2 window mean with exact int64 window sums (ARITH §F).
// Output tile of 32 columns x TY rows per CTA of 32 x 8 threads: the
// (32 + 2rs) x (TY + 2rs) input tile is converted once to fixed point in shared
// memory, summed horizontally (one column per lane), then vertically with a sliding window
// over the TY / 8 output rows of each thread. Integer sums are exact, so the order of
// the additions does not change a bit. A tall tile (TY = 64) amortises the vertical halo and
// the two barriers on large grids; small grids keep TY = 32 for more CTAs. Interior tiles
// use 32-bit offsets from the tile origin.
// Row slabs: the buffer holds rows [row_base, row_base + Ly) of a grid of Ly_g rows. Windows
// clip at the GRID edges (the counts); rows outside the buffer contribute 0, which only
// corrupts the outermost r_s buffer rows per pass (the halo that the slab does not consume).
template <int TY>
__global__ void __launch_bounds__(256) k_smooth(const float* __restrict__ Tin,
                                                float* __restrict__ Tout, int64_t Lx, int64_t Ly,
                                                int64_t row_base, int64_t Ly_g, int rs) {
  extern __shared__ long long smem[];
  const int W = kTile + 2 * rs, HY = TY + 2 * rs, w = 2 * rs + 1;
  long long* Q = smem;             // HY rows x W cols
  long long* H = smem + HY * W;    // HY rows x kTile cols
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * kTile, r0 = (int64_t)blockIdx.y * TY;
  const bool interior = r0 - rs >= 0 && c0 - rs >= 0 && r0 + TY + rs <= Ly && c0 + kTile + rs <= Lx;
  if (interior) {  // whole halo tile inside the grid: no bounds checks, 32-bit offsets
    const float* base = Tin + (r0 - rs) * Lx + (c0 - rs);
    const uint32_t lx = static_cast<uint32_t>(Lx);
    for (int y = ty; y < HY; y += 8) {
      const float* row = base + static_cast<uint32_t>(y) * lx;
      long long* q = Q + y * W;
      q[tx] = __float2ll_rn(__fmul_rn(__ldg(row + tx), 0x1p40f));
      if (tx < 2 * rs) q[32 + tx] = __float2ll_rn(__fmul_rn(__ldg(row + 32 + tx), 0x1p40f));
    }
  } else {
    for (int y = ty; y < HY; y += 8) {
      const int64_t r = r0 - rs + y;
      const bool rin = r >= 0 && r < Ly;
      for (int x = tx; x < W; x += 32) {
        const int64_t c = c0 - rs + x;
        Q[y * W + x] = (rin && c >= 0 && c < Lx) ? __float2ll_rn(__fmul_rn(Tin[r * Lx + c], 0x1p40f)) : 0;
      }
    }
  }
  __syncthreads();
  for (int y = ty; y < HY; y += 8) {
    const long long* q = Q + y * W + tx;
    long long s = 0;
    for (int d = 0; d < w; ++d) s += q[d];
    H[y * kTile + tx] = s;
  }
  __syncthreads();
  const int64_t c = c0 + tx;
  if (c >= Lx) return;
  const int64_t ca = c - rs > 0 ? c - rs : 0, cb = c + rs < Lx - 1 ? c + rs : Lx - 1;
  const int ncol = static_cast<int>(cb - ca + 1);
  constexpr int kRowsPerThread = TY / 8;
  const int yb = ty * kRowsPerThread;
  float* out = Tout + (r0 + yb) * Lx + c;
  long long s = 0;
  for (int d = 0; d < w; ++d) s += H[(yb + d) * kTile + tx];
  const double full = static_cast<double>(w * ncol);  // rows unclipped (interior of the grid rows)
#pragma unroll 4
  for (int k = 0; k < kRowsPerThread; ++k) {
    const int64_t r = r0 + yb + k;
    if (k > 0) s += H[(yb + k + w - 1) * kTile + tx] - H[(yb + k - 1) * kTile + tx];
    if (r >= Ly) break;
    double cnt = full;
    const int64_t rg = r + row_base;
    if (rg - rs < 0 || rg + rs > Ly_g - 1) {
      const int64_t ra = rg - rs > 0 ? rg - rs : 0, rb = rg + rs < Ly_g - 1 ? rg + rs : Ly_g - 1;
      cnt = static_cast<double>(static_cast<int>(rb - ra + 1) * ncol);
    }
    out[static_cast<int64_t>(k) * Lx] = __double2float_rn(__ddiv_rn(__ll2double_rn(s) * 0x1p-40, cnt));
  }
}

// One SST pass with a compile-time radius RS (1..8; the generic k_smooth above serves the
// rest). Same exact integer window sums as k_smooth (ARITH §F), fewer instructions per site:
// each warp converts its halo row to fixed point into a per-warp staging row and sums it
// horizontally at once (no block barrier between the two), the w-term sums unroll, and the
// vertical pass slides over TY / 8 rows per thread. FROM_TB: the input is the step field
// T(r, c) = T_b(block(r, c)) itself, read from the block temperatures (the a5 expansion
// fused into the first pass: the expanded field is never written). Buffer rows
// [row_base, row_base + Ly) of a grid of Ly_g rows (row slabs; see k_smooth).
//
// F64 (host-checked: every T in [2^-17, T_max] with (2 RS + 1)^2 T_max < 2^13): the terms
// llrint(T 2^40) are the floats T 2^40 themselves (integer-valued from 2^23 up) and every
// partial window sum stays below 2^53, so the sums are formed EXACTLY in fp64 — one DADD
// per term instead of a 64-bit integer add (two heavy-pipe IMADs on sm_100a) and no F2I /
// I2F conversions — and equal ARITH §F's int64 sums bit for bit.
template <typename Acc>
__device__ __forceinline__ Acc smooth_term(float v);
template <>
__device__ __forceinline__ long long smooth_term<long long>(float v) { return __float2ll_rn(__fmul_rn(v, 0x1p40f)); }
template <>
__device__ __forceinline__ double smooth_term<double>(float v) { return static_cast<double>(__fmul_rn(v, 0x1p40f)); }
__device__ __forceinline__ double smooth_value(long long s) { return __ll2double_rn(s); }
__device__ __forceinline__ double smooth_value(double s) { return s; }

template <int RS, int TY, bool FROM_TB, bool F64>
__global__ void __launch_bounds__(256) k_smooth_rs(const float* __restrict__ Tin, const float* __restrict__ Tb,
                                                   float* __restrict__ Tout, int64_t Lx64, int64_t Ly64,
                                                   int64_t row_base64, int64_t Ly_g64, int lb) {
  using Acc = typename std::conditional<F64, double, long long>::type;
  constexpr int W = kTile + 2 * RS, HY = TY + 2 * RS, w = 2 * RS + 1;
  __shared__ Acc Qw[8][W];
  __shared__ Acc H[HY][kTile];
  // 32-bit index arithmetic throughout: buffers hold < 2^30 sites (the API's Lx*Ly bound)
  const int Lx = static_cast<int>(Lx64), Ly = static_cast<int>(Ly64);
  const int row_base = static_cast<int>(row_base64), Ly_g = static_cast<int>(Ly_g64);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c0 = blockIdx.x * kTile, r0 = blockIdx.y * TY;
  const int ca = c0 - RS + tx, cb = c0 + kTile - RS + tx;  // this lane's one or two columns
  const bool ina = ca >= 0 && ca < Lx, inb = tx < 2 * RS && cb < Lx;
  const int nbx = (Lx + lb - 1) / lb;
  int bca = 0, bcb = 0;
  if (FROM_TB) {
    bca = ina ? ca / lb : 0;
    bcb = inb ? cb / lb : 0;
  }
  // every load of this warp's halo rows is issued before the first is used (the rows'
  // values sit in registers: the loads overlap instead of one round trip per row)
  constexpr int NYW = (HY + 7) / 8;
  float va[NYW], vb[NYW];
  // interior tiles (the halo tile inside the buffer): unguarded loads
  const bool interior = r0 - RS >= 0 && r0 + TY + RS <= Ly && c0 - RS >= 0 && c0 + kTile + RS <= Lx;
  if (interior && !FROM_TB) {
    const float* row = Tin + (r0 - RS + ty) * Lx;
#pragma unroll
    for (int t = 0; t < NYW; ++t) {
      vb[t] = 0.0f;
      if (ty + 8 * t < HY) {
        va[t] = __ldg(row + ca);
        if (tx < 2 * RS) vb[t] = __ldg(row + cb);
      }
      row += 8 * Lx;
    }
  } else {
#pragma unroll
    for (int t = 0; t < NYW; ++t) {
      const int y = ty + 8 * t;
      const int r = r0 - RS + y;
      va[t] = vb[t] = 0.0f;
      if (y < HY && static_cast<unsigned>(r) < static_cast<unsigned>(Ly)) {
        if (FROM_TB) {
          const float* tb = Tb + ((r + row_base) / lb) * nbx;
          if (ina) va[t] = __ldg(tb + bca);
          if (inb) vb[t] = __ldg(tb + bcb);
        } else {
          const float* row = Tin + r * Lx;
          if (ina) va[t] = __ldg(row + ca);
          if (inb) vb[t] = __ldg(row + cb);
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < NYW; ++t) {
    const int y = ty + 8 * t;
    if (y >= HY) break;
    // outside the grid (or the buffer) the value is 0 and so is its fixed-point term
    Qw[ty][tx] = smooth_term<Acc>(va[t]);
    if (tx < 2 * RS) Qw[ty][kTile + tx] = smooth_term<Acc>(vb[t]);
    __syncwarp();
    Acc h = Qw[ty][tx];
#pragma unroll
    for (int d = 1; d < w; ++d) h += Qw[ty][tx + d];
    H[y][tx] = h;
    __syncwarp();
  }
  __syncthreads();
  const int c = c0 + tx;
  if (c >= Lx) return;
  const int cl = c - RS > 0 ? c - RS : 0, cr = c + RS < Lx - 1 ? c + RS : Lx - 1;
  const int ncol = cr - cl + 1;
  constexpr int kRows = TY / 8;
  const int yb = ty * kRows;
  float* out = Tout + (r0 + yb) * Lx + c;
  Acc sum = H[yb][tx];
#pragma unroll
  for (int d = 1; d < w; ++d) sum += H[yb + d][tx];
  const double full = static_cast<double>(w * ncol);
  // The window mean's IEEE division by the unclipped count, with the reciprocal hoisted:
  // y = RN(1 / cnt), q0 = RN(a y), rem = a - cnt q0 (exact by fma), q = RN(q0 + rem y) is
  // RN(a / cnt) (Markstein's theorem: y within half an ulp of 1 / cnt, q0 within one ulp of
  // a / cnt, no over- / underflow — a is a window sum of temperatures times 2^-40, cnt an
  // integer <= 1089). Clipped rows divide with __ddiv_rn. Bit-identical to ARITH §F.
  const double yfull = __drcp_rn(full);
#pragma unroll 4
  for (int k = 0; k < kRows; ++k) {
    if (k > 0) sum += H[yb + k + w - 1][tx] - H[yb + k - 1][tx];
    const int r = r0 + yb + k;
    if (r >= Ly) break;
    const int rg = r + row_base;
    const double a = smooth_value(sum) * 0x1p-40;
    double q;
    if (rg - RS < 0 || rg + RS > Ly_g - 1) {
      const int ra = rg - RS > 0 ? rg - RS : 0, rb = rg + RS < Ly_g - 1 ? rg + RS : Ly_g - 1;
      q = __ddiv_rn(a, static_cast<double>((rb - ra + 1) * ncol));
    } else {
      const double q0 = __dmul_rn(a, yfull);
      const double rem = __fma_rn(-full, q0, a);
      q = __fma_rn(rem, yfull, q0);
    }
    out[k * Lx] = __double2float_rn(q);
  }
}

// SST pass with 4 columns per thread (RS <= 4, Lx % 4 == 0, 16-byte aligned buffers): the
// thread's columns arrive as one float4, the RS halo values on each side come from the
// adjacent lanes by shuffle (the warp's outer lanes load theirs), and the 4 horizontal window
// sums slide in registers (2 adds per column after the first), so shared memory holds only
// the horizontal sums. The vertical pass slides down 16 rows per thread. Same exact sums
// (F64 or int64, see k_smooth_rs), same division, same clipping: bit-identical.
constexpr int kWideCols = 128, kWideRows = 32;
template <int RS, bool F64, bool FROM_TB>
__global__ void __launch_bounds__(256) k_smooth_wide(const float* __restrict__ Tin, const float* __restrict__ Tb,
                                                     float* __restrict__ Tout, int64_t Lx64, int64_t Ly64,
                                                     int64_t row_base64, int64_t Ly_g64, int lb) {
  using Acc = typename std::conditional<F64, double, long long>::type;
  constexpr int HY = kWideRows + 2 * RS, w = 2 * RS + 1;
  __shared__ __align__(16) Acc H[HY][kWideCols];
  const int Lx = static_cast<int>(Lx64), Ly = static_cast<int>(Ly64);
  const int row_base = static_cast<int>(row_base64), Ly_g = static_cast<int>(Ly_g64);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int c0 = blockIdx.x * kWideCols, r0 = blockIdx.y * kWideRows;
  const int c = c0 + 4 * lane;
  const bool cin = c < Lx;  // all 4 columns or none (Lx % 4 == 0)
  // every load of the warp's halo rows first (they overlap instead of one round trip per
  // row): the float4 of the thread's columns, and for the outer lanes their RS halo columns
  constexpr int NIT = (HY + 7) / 8;
  float4 vv[NIT];
  float ho[NIT][RS];  // lane 0: columns c - RS .. c - 1; lane 31: c + 4 .. c + 3 + RS
  const bool outer = lane == 0 || lane == 31;
  const int hc0 = lane == 0 ? c - RS : c + 4;
  // FROM_TB: T(r, c) = T_b(block(r, c)) read from the block temperatures (the expansion
  // fused into the first pass); the thread's columns' block indices are fixed
  const int nbx = (Lx + lb - 1) / lb;
  int bc[4] = {0, 0, 0, 0}, bh[RS];
  if (FROM_TB) {
#pragma unroll
    for (int j = 0; j < 4; ++j) bc[j] = cin ? (c + j) / lb : 0;
#pragma unroll
    for (int j = 0; j < RS; ++j) {
      const int cc = hc0 + j;
      bh[j] = (cc >= 0 && cc < Lx) ? cc / lb : 0;
    }
  }
#pragma unroll
  for (int t = 0; t < NIT; ++t) {
    const int y = wp + 8 * t;
    const int r = r0 - RS + y;
    const bool rin = y < HY && static_cast<unsigned>(r) < static_cast<unsigned>(Ly);
    vv[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (FROM_TB) {
      const float* tb = Tb + (rin ? ((r + row_base) / lb) * nbx : 0);
      if (rin && cin) vv[t] = make_float4(__ldg(tb + bc[0]), __ldg(tb + bc[1]), __ldg(tb + bc[2]), __ldg(tb + bc[3]));
#pragma unroll
      for (int j = 0; j < RS; ++j) {
        const int cc = hc0 + j;
        ho[t][j] = (outer && rin && cc >= 0 && cc < Lx) ? __ldg(tb + bh[j]) : 0.0f;
      }
    } else {
      const float* row = Tin + r * Lx;
      if (rin && cin) vv[t] = __ldg(reinterpret_cast<const float4*>(row + c));
#pragma unroll
      for (int j = 0; j < RS; ++j) {
        const int cc = hc0 + j;
        ho[t][j] = (outer && rin && cc >= 0 && cc < Lx) ? __ldg(row + cc) : 0.0f;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < NIT; ++t) {
    const int y = wp + 8 * t;
    if (y >= HY) break;  // warp-uniform
    const float4 v = vv[t];
    const Acc q[4] = {smooth_term<Acc>(v.x), smooth_term<Acc>(v.y), smooth_term<Acc>(v.z), smooth_term<Acc>(v.w)};
    Acc xl[RS], xr[RS];  // columns c - RS .. c - 1 and c + 4 .. c + 3 + RS
#pragma unroll
    for (int j = 0; j < RS; ++j) {
      xl[j] = __shfl_up_sync(0xffffffffu, q[4 - RS + j], 1);
      xr[j] = __shfl_down_sync(0xffffffffu, q[j], 1);
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < RS; ++j) xl[j] = smooth_term<Acc>(ho[t][j]);
    }
    if (lane == 31) {
#pragma unroll
      for (int j = 0; j < RS; ++j) xr[j] = smooth_term<Acc>(ho[t][j]);
    }
    auto x = [&](int k) -> Acc { return k < 0 ? xl[k + RS] : (k < 4 ? q[k] : xr[k - 4]); };
    Acc h[4];
    h[0] = x(-RS);
#pragma unroll
    for (int k = -RS + 1; k <= RS; ++k) h[0] += x(k);
#pragma unroll
    for (int i = 1; i < 4; ++i) h[i] = h[i - 1] + x(i + RS) - x(i - 1 - RS);
    Acc* hp = &H[y][4 * lane];
#pragma unroll
    for (int i = 0; i < 4; ++i) hp[i] = h[i];
  }
  __syncthreads();
  const int cc = threadIdx.x & (kWideCols - 1), hh = threadIdx.x >> 7;  // column, row half
  const int col = c0 + cc;
  if (col >= Lx) return;
  const int cl = col - RS > 0 ? col - RS : 0, cr = col + RS < Lx - 1 ? col + RS : Lx - 1;
  const int ncol = cr - cl + 1;
  constexpr int kRows = kWideRows / 2;
  const int yb = hh * kRows;
  float* out = Tout + (r0 + yb) * Lx + col;
  Acc sum = H[yb][cc];
#pragma unroll
  for (int d = 1; d < w; ++d) sum += H[yb + d][cc];
  const double full = static_cast<double>(w * ncol);
  const double yfull = __drcp_rn(full);  // the Markstein division of k_smooth_rs
#pragma unroll 4
  for (int k = 0; k < kRows; ++k) {
    if (k > 0) sum += H[yb + k + w - 1][cc] - H[yb + k - 1][cc];
    const int r = r0 + yb + k;
    if (r >= Ly) break;
    const int rg = r + row_base;
    const double a = smooth_value(sum) * 0x1p-40;
    double qd;
    if (rg - RS < 0 || rg + RS > Ly_g - 1) {
      const int ra = rg - RS > 0 ? rg - RS : 0, rb = rg + RS < Ly_g - 1 ? rg + RS : Ly_g - 1;
      qd = __ddiv_rn(a, static_cast<double>((rb - ra + 1) * ncol));
    } else {
      const double q0 = __dmul_rn(a, yfull);
      const double rem = __fma_rn(-full, q0, a);
      qd = __fma_rn(rem, yfull, q0);
    }
    out[k * Lx] = __double2float_rn(qd);
  }
}

// Per-gap records in ONE pass over the local sites (row-major, coalesced reads of mask /
// gid / phi / T): every gap site writes its whole 32-byte record at its id. The ids of a
// row's same-colour gaps are consecutive, so a warp's record stores are two contiguous runs
// of whole sectors (no read-modify-write). The buffer holds rows [lrow0, lrow0 + nrows)
// (global; the whole grid unless row slabs); neighbours outside those rows are left out —
// only ghost-row gaps, which are never updated, have any. T holds rows [trow0, trow1).
__global__ void __launch_bounds__(256) k_build_records(
    const int32_t* __restrict__ gid, const uint8_t* __restrict__ mask,
    const float* __restrict__ phi, const float* __restrict__ T, const float* __restrict__ binit,
    int64_t Lx, int64_t Ly, int64_t lrow0, int64_t nrows, int64_t trow0, int64_t trow1, int lb,
    GapRec* __restrict__ rec, float* __restrict__ ginit) {
  const int64_t lr = blockIdx.y;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= Lx) return;
  const int64_t i = lr * Lx + c;
  if (mask[i]) return;
  const int64_t r = lr + lrow0;  // global row
  GapRec R;
  R.site = static_cast<uint32_t>(r * Lx + c);  // global site index (Philox counter)
  const bool has[4] = {lr > 0, lr + 1 < nrows && r + 1 < Ly, c > 0, c + 1 < Lx};
  const int64_t off[4] = {-Lx, Lx, -1, 1};
  uint32_t flags = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int32_t v = 0;
    uint32_t ty = NB_NONE;
    if (has[k]) {
      const int64_t j = i + off[k];
      if (mask[j]) { ty = NB_KNOWN; v = __float_as_int(phi[j]); }
      else         { ty = NB_GAP;   v = gid[j]; }
    }
    flags |= ty << (2 * k);
    R.nb[k] = v;
  }
  R.flags = flags;
  R.beta = (r >= trow0 && r < trow1) ? __fdiv_rn(1.0f, T[(r - trow0) * Lx + c]) : 0.0f;
  const int64_t nbx = (Lx + lb - 1) / lb;
  const int64_t b = static_cast<int64_t>(static_cast<uint32_t>(r) / static_cast<uint32_t>(lb)) * nbx +
                    static_cast<uint32_t>(c) / static_cast<uint32_t>(lb);
  R.init = binit[b];
  const int32_t g = gid[i];
  ginit[g] = R.init;
  uint4* dst = reinterpret_cast<uint4*>(rec + g);
  dst[0] = make_uint4(R.site, __float_as_uint(R.beta), R.flags, __float_as_uint(R.init));
  dst[1] = make_uint4(static_cast<uint32_t>(R.nb[0]), static_cast<uint32_t>(R.nb[1]), static_cast<uint32_t>(R.nb[2]),
                      static_cast<uint32_t>(R.nb[3]));
}

// The record builder with streamed rows (Lx % 4 == 0, 16-byte aligned buffers): a thread
// owns 4 adjacent columns and walks kRowsPerWarp rows, keeping the rows above, at and below
// in registers (mask as 4 bytes, phi as float4, gid as int4) — every row is loaded once
// per column strip, all loads of a step are independent, and the west / east neighbours
// of the outer columns come from the adjacent lanes. Writes the same records as
// k_build_records.
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int k) { return (w >> (8 * k)) & 0xffu; }

__global__ void __launch_bounds__(256) k_build_records4(
    const int32_t* __restrict__ gid, const uint8_t* __restrict__ mask, const float* __restrict__ phi,
    const float* __restrict__ T, const float* __restrict__ binit, int64_t Lx64, int64_t Ly64, int64_t lrow064,
    int64_t nrows64, int64_t trow064, int64_t trow164, int lb, GapRec* __restrict__ rec, float* __restrict__ ginit) {
  // 32-bit index arithmetic (< 2^30 sites)
  const int Lx = static_cast<int>(Lx64), Ly = static_cast<int>(Ly64), lrow0 = static_cast<int>(lrow064);
  const int nrows = static_cast<int>(nrows64), trow0 = static_cast<int>(trow064), trow1 = static_cast<int>(trow164);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int c = blockIdx.x * 128 + 4 * lane;
  const bool cin = c < Lx;
  const int la = blockIdx.y * (8 * kRowsPerWarp) + wp * kRowsPerWarp;  // local rows
  const int lz = min(la + kRowsPerWarp, nrows);
  if (la >= nrows) return;  // warp-uniform
  const int nbx = (Lx + lb - 1) / lb;
  int bcol[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) bcol[j] = (c + j) / lb;
  auto ld = [&](int lr, uint32_t& m, float4& p, int4& g) {
    m = 0;
    p = make_float4(0.f, 0.f, 0.f, 0.f);
    g = make_int4(0, 0, 0, 0);
    if (cin && lr >= 0 && lr < nrows) {
      const int i = lr * Lx + c;
      m = *reinterpret_cast<const uint32_t*>(mask + i);
      p = *reinterpret_cast<const float4*>(phi + i);
      g = *reinterpret_cast<const int4*>(gid + i);
    }
  };
  uint32_t mu, mc, md;
  float4 pu, pc, pd;
  int4 gu, gc, gd;
  ld(la - 1, mu, pu, gu);
  ld(la, mc, pc, gc);
  for (int lr = la; lr < lz; ++lr) {
    const int r = lr + lrow0;  // global row
    const bool has_up = lr > 0, has_dn = lr + 1 < nrows && r + 1 < Ly;
    ld(has_dn ? lr + 1 : -1, md, pd, gd);
    float4 tv = make_float4(1.f, 1.f, 1.f, 1.f);
    const bool tin = cin && r >= trow0 && r < trow1;
    if (tin) tv = *reinterpret_cast<const float4*>(T + (r - trow0) * Lx + c);
    // west neighbour of column 0 (lane - 1's column 3), east neighbour of column 3 (lane + 1's 0)
    uint32_t mw = __shfl_up_sync(0xffffffffu, mc >> 24, 1);
    float pw = __shfl_up_sync(0xffffffffu, pc.w, 1);
    int gw = __shfl_up_sync(0xffffffffu, gc.w, 1);
    uint32_t me = __shfl_down_sync(0xffffffffu, mc & 0xffu, 1);
    float pe = __shfl_down_sync(0xffffffffu, pc.x, 1);
    int ge = __shfl_down_sync(0xffffffffu, gc.x, 1);
    const int i = lr * Lx + c;
    if (lane == 0 && cin && c > 0) { mw = mask[i - 1]; pw = phi[i - 1]; gw = gid[i - 1]; }
    if (lane == 31 && cin && c + 4 < Lx) { me = mask[i + 4]; pe = phi[i + 4]; ge = gid[i + 4]; }
    const int rb = r / lb;
    const float pcv[4] = {pc.x, pc.y, pc.z, pc.w}, puv[4] = {pu.x, pu.y, pu.z, pu.w}, pdv[4] = {pd.x, pd.y, pd.z, pd.w};
    const int gcv[4] = {gc.x, gc.y, gc.z, gc.w}, guv[4] = {gu.x, gu.y, gu.z, gu.w}, gdv[4] = {gd.x, gd.y, gd.z, gd.w};
    const float tvv[4] = {tv.x, tv.y, tv.z, tv.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!cin || byte_of(mc, j)) continue;
      // neighbours N, S, W, E: (present, known, phi, gid)
      const bool has[4] = {has_up, has_dn, c + j > 0, c + j + 1 < Lx};
      const uint32_t km[4] = {byte_of(mu, j), byte_of(md, j), j > 0 ? byte_of(mc, j - 1) : mw,
                              j < 3 ? byte_of(mc, j + 1) : me};
      const float kp[4] = {puv[j], pdv[j], j > 0 ? pcv[j - 1] : pw, j < 3 ? pcv[j + 1] : pe};
      const int kg[4] = {guv[j], gdv[j], j > 0 ? gcv[j - 1] : gw, j < 3 ? gcv[j + 1] : ge};
      uint32_t flags = 0, nb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t ty = NB_NONE, v = 0;
        if (has[k]) {
          if (km[k]) { ty = NB_KNOWN; v = __float_as_uint(kp[k]); }
          else       { ty = NB_GAP;   v = static_cast<uint32_t>(kg[k]); }
        }
        flags |= ty << (2 * k);
        nb[k] = v;
      }
      const float beta = tin ? __fdiv_rn(1.0f, tvv[j]) : 0.0f;
      const float init = binit[rb * nbx + bcol[j]];
      const int32_t g = gcv[j];
      ginit[g] = init;
      uint4* dst = reinterpret_cast<uint4*>(rec + g);
      dst[0] = make_uint4(static_cast<uint32_t>(r * Lx + c + j), __float_as_uint(beta), flags, __float_as_uint(init));
      dst[1] = make_uint4(nb[0], nb[1], nb[2], nb[3]);
    }
    mu = mc; pu = pc; gu = gc;
    mc = md; pc = pd; gc = gd;
  }
}

// ------------------------------------------------------------- a11: predict
__global__ void __launch_bounds__(256) k_predict(const float* __restrict__ z,
                                                 const uint8_t* __restrict__ mask,
                                                 const int32_t* __restrict__ gid,
                                                 const double* __restrict__ acc, int64_t n,
                                                 double denom, const DevScalars* __restrict__ sc,
                                                 int degenerate, float* __restrict__ out) {
  float zmin, zmax, s;
  range_params(sc, &zmin, &zmax, &s);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (mask[i]) { out[i] = z[i]; continue; }
    if (degenerate) { out[i] = zmin; continue; }
    const double mean = __ddiv_rn(acc[gid[i]], denom);
    const double dz = __dsub_rn(static_cast<double>(zmax), static_cast<double>(zmin));
    const double v = __dadd_rn(static_cast<double>(zmin),
                               __dmul_rn(dz, __ddiv_rn(mean, static_cast<double>(kTwoPiF))));
    out[i] = __double2float_rn(v);
  }
}

// The same, 4 sites per thread with 16-byte loads and stores (n % 4 == 0, aligned buffers).
__global__ void __launch_bounds__(256) k_predict4(const float* __restrict__ z,
                                                  const uint8_t* __restrict__ mask,
                                                  const int32_t* __restrict__ gid,
                                                  const double* __restrict__ acc, int64_t n,
                                                  double denom, const DevScalars* __restrict__ sc,
                                                  int degenerate, float* __restrict__ out) {
  float zmin, zmax, s;
  range_params(sc, &zmin, &zmax, &s);
  const double dz = __dsub_rn(static_cast<double>(zmax), static_cast<double>(zmin));
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n / 4; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t m = *reinterpret_cast<const uint32_t*>(mask + 4 * q);
    const float4 zv = __ldg(reinterpret_cast<const float4*>(z + 4 * q));
    const int4 gv = __ldg(reinterpret_cast<const int4*>(gid + 4 * q));
    const float zz[4] = {zv.x, zv.y, zv.z, zv.w};
    const int gg[4] = {gv.x, gv.y, gv.z, gv.w};
    float o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if ((m >> (8 * k)) & 0xffu) {
        o[k] = zz[k];
      } else if (degenerate) {
        o[k] = zmin;
      } else {
        const double mean = __ddiv_rn(acc[gg[k]], denom);
        o[k] = __double2float_rn(__dadd_rn(static_cast<double>(zmin),
                                           __dmul_rn(dz, __ddiv_rn(mean, static_cast<double>(kTwoPiF)))));
      }
    }
    *reinterpret_cast<float4*>(out + 4 * q) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void k_scatter_state(const float* __restrict__ phiK, const int32_t* __restrict__ gid,
                                const float* __restrict__ G, int64_t R, int64_t rr, int64_t n,
                                float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = gid[i];
    out[i] = g < 0 ? phiK[i] : G[static_cast<int64_t>(g) * R + rr];
  }
}

__global__ void k_scatter_acc(const int32_t* __restrict__ gid, const double* __restrict__ acc,
                              int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = gid[i];
    out[i] = g < 0 ? 0.0 : acc[g];
  }
}

inline int grid_for(int64_t work, int threads, int cap = 148 * 16) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

void launch_minmax_count(const float* z, const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t row_base,
                         DevScalars* sc, cudaStream_t st) {
  const int64_t n = Lx * Ly;
  const int g = grid_for((n + 15) / 16, 256);
  if (aligned16(z) && aligned16(mask))
    k_minmax_count<true><<<g, 256, 0, st>>>(z, mask, Lx, n, row_base, sc);
  else
    k_minmax_count<false><<<g, 256, 0, st>>>(z, mask, Lx, n, row_base, sc);
}

void launch_transform(const float* z, const uint8_t* mask, int64_t n, const DevScalars* sc,
                      float* phiK, cudaStream_t st) {
  const int g = grid_for((n + 3) / 4, 256);
  if (aligned16(z) && aligned16(phiK) && (reinterpret_cast<uintptr_t>(mask) & 3u) == 0)
    k_transform<true><<<g, 256, 0, st>>>(z, mask, n, sc, phiK);
  else
    k_transform<false><<<g, 256, 0, st>>>(z, mask, n, sc, phiK);
}

void launch_gap_rows(const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t row_base, int* rowcnt, int* rowoff,
                     cudaStream_t st) {
  k_row_counts<<<static_cast<unsigned>(Ly), 256, 0, st>>>(mask, Lx, Ly, row_base, rowcnt);
  k_scan_excl<<<1, 1024, 0, st>>>(rowcnt, 2 * Ly, rowoff);
}

void launch_gap_compact(const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t row_base, const int* rowoff,
                        int32_t* gid, cudaStream_t st) {
  if (Lx % 4 == 0 && aligned16(gid) && (reinterpret_cast<uintptr_t>(mask) & 3u) == 0) {
    k_row_compact4<<<static_cast<unsigned>((Ly + 7) / 8), 256, 0, st>>>(mask, Lx, Ly, row_base, rowoff, gid);
    return;
  }
  k_row_compact<<<static_cast<unsigned>(Ly), 256, 0, st>>>(mask, Lx, Ly, row_base, rowoff, gid);
}

void launch_gap_index(const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t row_base, int* rowcnt,
                      int* rowoff, int32_t* gid, cudaStream_t st) {
  launch_gap_rows(mask, Lx, Ly, row_base, rowcnt, rowoff, st);
  launch_gap_compact(mask, Lx, Ly, row_base, rowoff, gid, st);
}

void launch_block_stats(const float* phiK, const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t lrow0,
                        int64_t row0, int64_t row1, int lb, float q, long long* SB, long long* NB,
                        long long* SP, long long* NK, int64_t nblocks, DevScalars* sc, cudaStream_t st) {
  cudaMemsetAsync(SB, 0, sizeof(long long) * nblocks, st);
  cudaMemsetAsync(NB, 0, sizeof(long long) * nblocks, st);
  cudaMemsetAsync(SP, 0, sizeof(long long) * nblocks, st);
  cudaMemsetAsync(NK, 0, sizeof(long long) * nblocks, st);
  if (lb % 4 == 0 && Lx % 4 == 0 && aligned16(phiK) && (reinterpret_cast<uintptr_t>(mask) & 3u) == 0) {
    const int64_t tile0 = (row0 / kBs4Rows) * kBs4Rows;
    dim3 grid(static_cast<unsigned>((Lx + kBs4Cols - 1) / kBs4Cols),
              static_cast<unsigned>((row1 - tile0 + kBs4Rows - 1) / kBs4Rows));
    k_block_stats4<<<grid, 256, 0, st>>>(phiK, mask, Lx, Ly, lrow0, row0, row1, lb, q, SB, NB, SP, NK, sc);
    return;
  }
  const int64_t tile0 = (row0 / kTile) * kTile;
  dim3 grid(static_cast<unsigned>((Lx + kTile - 1) / kTile), static_cast<unsigned>((row1 - tile0 + kTile - 1) / kTile));
  k_block_stats<<<grid, 256, 0, st>>>(phiK, mask, Lx, Ly, lrow0, row0, row1, lb, q, SB, NB, SP, NK, sc);
}

void launch_block_T(const long long* SB, const long long* NB, const long long* SP,
                    const long long* NK, int64_t nblocks, const float* calT, const float* cale,
                    int K, float* Tb, DevScalars* sc, cudaStream_t st) {
  k_block_T<<<static_cast<unsigned>((nblocks + 255) / 256), 256, 0, st>>>(SB, NB, SP, NK, nblocks,
                                                                          calT, cale, K, Tb, sc);
}

void launch_median_fill(float* Tb, const long long* NB, int64_t nblocks, DevScalars* sc,
                        cudaStream_t st) {
  k_median_fill<<<1, 1024, 0, st>>>(Tb, NB, nblocks, sc);
}

void launch_expand(const float* Tb, int64_t Lx, int64_t trow0, int64_t trow1, int lb, float* T, cudaStream_t st) {
  k_expand<<<grid_for(Lx * (trow1 - trow0), 256), 256, 0, st>>>(Tb, Lx, trow0, trow1, lb, T);
}

template <int RS, int TY, bool F64>
static void smooth_rs(const float* Tin, const float* Tb, float* Tout, int64_t Lx, int64_t Ly, int64_t row_base,
                      int64_t Ly_g, int lb, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((Lx + kTile - 1) / kTile), static_cast<unsigned>((Ly + TY - 1) / TY));
  if (Tb)
    k_smooth_rs<RS, TY, true, F64><<<grid, 256, 0, st>>>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb);
  else
    k_smooth_rs<RS, TY, false, F64><<<grid, 256, 0, st>>>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb);
}

template <int RS>
static void smooth_rs_ty(const float* Tin, const float* Tb, float* Tout, int64_t Lx, int64_t Ly, int64_t row_base,
                         int64_t Ly_g, int lb, bool f64, cudaStream_t st) {
  if (RS <= 4 && Lx % 4 == 0 && (Tb || aligned16(Tin)) && aligned16(Tout) && !std::getenv("MPR_SST_NARROW")) {
    dim3 grid(static_cast<unsigned>((Lx + kWideCols - 1) / kWideCols), static_cast<unsigned>((Ly + kWideRows - 1) / kWideRows));
    constexpr int R4 = RS <= 4 ? RS : 4;
    if (Tb) {
      if (f64) k_smooth_wide<R4, true, true><<<grid, 256, 0, st>>>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb);
      else k_smooth_wide<R4, false, true><<<grid, 256, 0, st>>>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb);
    } else {
      if (f64) k_smooth_wide<R4, true, false><<<grid, 256, 0, st>>>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb);
      else k_smooth_wide<R4, false, false><<<grid, 256, 0, st>>>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb);
    }
    return;
  }
  // 32 x 64 tiles once the grid has >= 16 waves of them on 148 SMs, 32 x 32 below
  const bool tall = (Lx + kTile - 1) / kTile * ((Ly + 63) / 64) >= 148 * 16;
  if (f64) {
    if (tall) smooth_rs<RS, 64, true>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, st);
    else smooth_rs<RS, 32, true>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, st);
  } else {
    if (tall) smooth_rs<RS, 64, false>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, st);
    else smooth_rs<RS, 32, false>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, st);
  }
}

bool launch_smooth_specialised(const float* Tin, const float* Tb, float* Tout, int64_t Lx, int64_t Ly,
                               int64_t row_base, int64_t Ly_g, int rs, int lb, float Tmin, float Tmax, cudaStream_t st) {
  // exact fp64 window sums when every term is an integer-valued float and every sum < 2^53
  const double w = 2.0 * rs + 1.0;
  const bool f64 = Tmin >= 0x1p-17f && w * w * static_cast<double>(Tmax) < 8192.0;
  switch (rs) {
    case 1: smooth_rs_ty<1>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, f64, st); return true;
    case 2: smooth_rs_ty<2>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, f64, st); return true;
    case 3: smooth_rs_ty<3>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, f64, st); return true;
    case 4: smooth_rs_ty<4>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, f64, st); return true;
    case 5: smooth_rs_ty<5>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, f64, st); return true;
    case 6: smooth_rs_ty<6>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, f64, st); return true;
    case 7: smooth_rs_ty<7>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, f64, st); return true;
    case 8: smooth_rs_ty<8>(Tin, Tb, Tout, Lx, Ly, row_base, Ly_g, lb, f64, st); return true;
    default: return false;
  }
}

void launch_smooth(const float* Tin, float* Tout, int64_t Lx, int64_t Ly, int64_t row_base, int64_t Ly_g, int rs,
                   cudaStream_t st) {
  // 32 x 64 tiles once the grid has >= 16 waves of them on 148 SMs (C4 16384^2: 1.66 -> 1.16
  // ms per pass); 32 x 32 below, where more CTAs hide latency better (1024^2: 10.9 vs 13.6 us)
  const bool tall = (Lx + kTile - 1) / kTile * ((Ly + 63) / 64) >= 148 * 16;
  const int TY = tall ? 64 : 32;
  const int W = kTile + 2 * rs, HY = TY + 2 * rs;
  const size_t smem = sizeof(long long) * (static_cast<size_t>(HY) * W + static_cast<size_t>(HY) * kTile);
  const void* fn = tall ? reinterpret_cast<const void*>(k_smooth<64>) : reinterpret_cast<const void*>(k_smooth<32>);
  // > 48 KB of dynamic shared memory needs the opt-in, per device: set it on the calling
  // thread's current device whenever a large window asks for it (r_s >= 16)
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  dim3 grid(static_cast<unsigned>((Lx + kTile - 1) / kTile), static_cast<unsigned>((Ly + TY - 1) / TY));
  if (tall)
    k_smooth<64><<<grid, 256, smem, st>>>(Tin, Tout, Lx, Ly, row_base, Ly_g, rs);
  else
    k_smooth<32><<<grid, 256, smem, st>>>(Tin, Tout, Lx, Ly, row_base, Ly_g, rs);
}

void launch_block_init(const long long* SP, const long long* NK, int64_t nblocks, const DevScalars* sc,
                       float* binit, cudaStream_t st) {
  k_block_init<<<static_cast<unsigned>((nblocks + 255) / 256), 256, 0, st>>>(SP, NK, nblocks, sc, binit);
}

void launch_build_records(const int32_t* gid, const uint8_t* mask, const float* phiK,
                          const float* T, const float* binit, int64_t Lx, int64_t Ly, int64_t lrow0, int64_t lrow1,
                          int64_t trow0, int64_t trow1, int lb, int64_t P, GapRec* rec, float* ginit,
                          cudaStream_t st) {
  if (P == 0) return;
  const int64_t nrows = lrow1 - lrow0;
  if (Lx % 4 == 0 && aligned16(gid) && aligned16(phiK) && aligned16(T) && (reinterpret_cast<uintptr_t>(mask) & 3u) == 0) {
    dim3 grid(static_cast<unsigned>((Lx + 127) / 128), static_cast<unsigned>((nrows + 8 * kRowsPerWarp - 1) / (8 * kRowsPerWarp)));
    k_build_records4<<<grid, 256, 0, st>>>(gid, mask, phiK, T, binit, Lx, Ly, lrow0, nrows, trow0, trow1, lb, rec, ginit);
    return;
  }
  dim3 grid(static_cast<unsigned>((Lx + 255) / 256), static_cast<unsigned>(nrows));
  k_build_records<<<grid, 256, 0, st>>>(gid, mask, phiK, T, binit, Lx, Ly, lrow0, nrows, trow0, trow1, lb,
                                        rec, ginit);
}

void launch_predict(const float* z, const uint8_t* mask, const int32_t* gid, const double* acc,
                    int64_t n, double denom, const DevScalars* sc, int degenerate, float* out,
                    cudaStream_t st) {
  if (n % 4 == 0 && aligned16(z) && aligned16(gid) && aligned16(out) && (reinterpret_cast<uintptr_t>(mask) & 3u) == 0) {
    k_predict4<<<grid_for(n / 4, 256), 256, 0, st>>>(z, mask, gid, acc, n, denom, sc, degenerate, out);
    return;
  }
  k_predict<<<grid_for(n, 256), 256, 0, st>>>(z, mask, gid, acc, n, denom, sc, degenerate, out);
}

void launch_scatter_state(const float* phiK, const int32_t* gid, const float* G, int64_t R,
                          int64_t r, int64_t n, float* out, cudaStream_t st) {
  k_scatter_state<<<grid_for(n, 256), 256, 0, st>>>(phiK, gid, G, R, r, n, out);
}

void launch_scatter_acc(const int32_t* gid, const double* acc, int64_t n, double* out,
                        cudaStream_t st) {
  k_scatter_acc<<<grid_for(n, 256), 256, 0, st>>>(gid, acc, n, out);
}

// ---- double-checkerboard phase lists (row f3, ARITH §H): phase = 2*tile parity + colour
namespace {
__device__ __forceinline__ int dc_phase(uint32_t site, int64_t Lx, int lb) {
  const int64_t r = site / Lx, c = site - r * Lx;
  return static_cast<int>((((r / lb) + (c / lb)) & 1) * 2 + ((r + c) & 1));
}

__global__ void k_dc_count(const GapRec* __restrict__ rec, int64_t P, int64_t Lx, int lb,
                           unsigned long long* __restrict__ cnt) {
  unsigned long long c[4] = {0, 0, 0, 0};
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < P; g += (int64_t)gridDim.x * blockDim.x)
    ++c[dc_phase(rec[g].site, Lx, lb)];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned long long v = warp_sum_ull(c[k]);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&cnt[k], v);
  }
}

// Scatter gap ids into their phase segment; warp-aggregated cursors keep a warp's ids in
// order (coalesced state access in the sweep). The order inside a phase is free.
__global__ void k_dc_scatter(const GapRec* __restrict__ rec, int64_t P, int64_t Lx, int lb,
                             unsigned long long* __restrict__ cursor, uint32_t* __restrict__ list) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < P; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = base + threadIdx.x;
    const bool in = g < P;
    const int ph = in ? dc_phase(rec[g].site, Lx, lb) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, ph);
    const int leader = __ffs(peers) - 1;
    unsigned long long pos = 0;
    if (in && lane == leader) pos = atomicAdd(&cursor[ph], static_cast<unsigned long long>(__popc(peers)));
    pos = __shfl_sync(0xffffffffu, pos, leader);
    if (in) list[pos + __popc(peers & ((1u << lane) - 1u))] = static_cast<uint32_t>(g);
  }
}
}  // namespace

void launch_dc_count(const GapRec* rec, int64_t P, int64_t Lx, int lb, unsigned long long* cnt, cudaStream_t st) {
  cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), st);
  if (P > 0) k_dc_count<<<grid_for(P, 256), 256, 0, st>>>(rec, P, Lx, lb, cnt);
}

void launch_dc_scatter(const GapRec* rec, int64_t P, int64_t Lx, int lb, unsigned long long* cursor,
                       uint32_t* list, cudaStream_t st) {
  if (P > 0) k_dc_scatter<<<grid_for(P, 256), 256, 0, st>>>(rec, P, Lx, lb, cursor, list);
}

}  // namespace mpr
