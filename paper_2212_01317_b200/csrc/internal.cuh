// internal.cuh — context layout and kernel launchers of libmpr.so (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "mpr.h"

namespace mpr {

// Per-gap-site record, 32 bytes (one sector), read once per half-sweep per launch
// item and shared by all realizations of the batch.
//   site  : global row-major site index i = r*Lx + c (Philox counter x, ARITH §A)
//   beta  : 1/T_i (ARITH §F)
//   flags : 2 bits per neighbour k in (N, S, W, E): 0 none (outside the grid),
//           1 known (nb[k] holds the float bits of the frozen angle), 2 gap (nb[k]
//           holds the neighbour's gap id)
//   init  : BLOCK_MEAN initial angle (ARITH §G)
struct __align__(16) GapRec {
  uint32_t site;
  float beta;
  uint32_t flags;
  float init;
  int32_t nb[4];
};
static_assert(sizeof(GapRec) == 32, "GapRec must be one 32-byte sector");

enum NbType : uint32_t { NB_NONE = 0, NB_KNOWN = 1, NB_GAP = 2 };

// Device scalars written by the parameter kernels (one cudaMalloc).
struct DevScalars {
  int zmin_key, zmax_key;        // ordered-int keys (device_math.cuh)
  int bad_sample;                // non-finite known value seen
  int pad0;
  unsigned long long n_known;    // samples
  unsigned long long n_gap[2];   // gaps by colour (0 = A: (r+c) even)
  unsigned long long n_avail;    // blocks with >= 1 sample bond
  unsigned long long n_fallback; // blocks given the median
  long long sum_SB;              // sum over blocks of SB (known-known bond cos, 2^32)
  long long sum_SP;              // sum of llrint(phi*2^28) over samples
  long long sum_NK;              // samples (again, as int64 for the global mean)
  long long sum_SB2;             // sum over sample bonds of llrint(fp32(b*b) * 2^32) (R22)
  long long sum_NB;              // sample bonds (N_SP of Eq.(2) over the whole grid)
  float median_T;
  float pad1;
};

// ---- launchers (params.cu) ----
// Row-slab convention: a local buffer of `Ly` rows whose row 0 is the global row `row_base`
// (row_base = 0 and Ly = the grid's rows outside row-slab mode); colours and Philox site
// counters are global.
void launch_minmax_count(const float* z, const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t row_base,
                         DevScalars* sc, cudaStream_t st);
void launch_transform(const float* z, const uint8_t* mask, int64_t n, const DevScalars* sc,
                      float* phiK, cudaStream_t st);
// gap ids in (colour, local row, column) order: per-row counts + exclusive scan, then the
// compaction (gid per site); the records (site, neighbours, beta, init) are written whole by
// launch_build_records once the temperatures exist
void launch_gap_rows(const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t row_base, int* rowcnt, int* rowoff,
                     cudaStream_t st);
void launch_gap_compact(const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t row_base, const int* rowoff,
                        int32_t* gid, cudaStream_t st);
void launch_gap_index(const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t row_base, int* rowcnt,
                      int* rowoff, int32_t* gid, cudaStream_t st);
// block sums of the own rows [row0, row1) (global) of a buffer starting at global row lrow0
// (also adds the squared sample-bond cosines to sc->sum_SB2: the derived slope tolerance, R22)
void launch_block_stats(const float* phiK, const uint8_t* mask, int64_t Lx, int64_t Ly, int64_t lrow0,
                        int64_t row0, int64_t row1, int lb, float q, long long* SB, long long* NB,
                        long long* SP, long long* NK, int64_t nblocks, DevScalars* sc, cudaStream_t st);
void launch_block_T(const long long* SB, const long long* NB, const long long* SP,
                    const long long* NK, int64_t nblocks, const float* calT, const float* cale,
                    int K, float* Tb, DevScalars* sc, cudaStream_t st);
void launch_median_fill(float* Tb, const long long* NB, int64_t nblocks, DevScalars* sc,
                        cudaStream_t st);
void launch_expand(const float* Tb, int64_t Lx, int64_t trow0, int64_t trow1, int lb, float* T, cudaStream_t st);
void launch_smooth(const float* Tin, float* Tout, int64_t Lx, int64_t Ly, int64_t row_base, int64_t Ly_g, int rs,
                   cudaStream_t st);
// The specialised pass for r_s = 1..8 (false: not specialised, use launch_smooth). Tb non-null:
// the input is the expansion of the block temperatures (first pass, Tin unused).
// Tmin / Tmax: the calibration table's range (every T of the field lies in it; they decide
// whether the exact window sums can be formed in fp64).
bool launch_smooth_specialised(const float* Tin, const float* Tb, float* Tout, int64_t Lx, int64_t Ly,
                               int64_t row_base, int64_t Ly_g, int rs, int lb, float Tmin, float Tmax,
                               cudaStream_t st);
// BLOCK_MEAN initial angle per block (ARITH §G), after launch_block_T (global sample sums)
void launch_block_init(const long long* SP, const long long* NK, int64_t nblocks, const DevScalars* sc,
                       float* binit, cudaStream_t st);
void launch_build_records(const int32_t* gid, const uint8_t* mask, const float* phiK,
                          const float* T, const float* binit, int64_t Lx, int64_t Ly, int64_t lrow0, int64_t lrow1,
                          int64_t trow0, int64_t trow1, int lb, int64_t P, GapRec* rec, float* ginit,
                          cudaStream_t st);
void launch_predict(const float* z, const uint8_t* mask, const int32_t* gid, const double* acc,
                    int64_t n, double denom, const DevScalars* sc, int degenerate, float* out,
                    cudaStream_t st);
void launch_scatter_state(const float* phiK, const int32_t* gid, const float* G, int64_t R,
                          int64_t r, int64_t n, float* out, cudaStream_t st);
void launch_scatter_acc(const int32_t* gid, const double* acc, int64_t n, double* out,
                        cudaStream_t st);

// double-checkerboard phase lists (row f3): counts per phase (2*tile parity + colour),
// then a scatter of the gap ids into [cursor[p], ...) segments of `list`
void launch_dc_count(const GapRec* rec, int64_t P, int64_t Lx, int lb, unsigned long long* cnt, cudaStream_t st);
void launch_dc_scatter(const GapRec* rec, int64_t P, int64_t Lx, int lb, unsigned long long* cursor,
                       uint32_t* list, cudaStream_t st);

// ---- launchers (sweep.cu) ----
struct SweepArgs {
  const GapRec* rec;
  float* G;          // state, [P][R] floats (gap-site major, realization minor)
  float* A;          // accumulator of the last n_avg sweeps, same layout (nullable)
  int64_t g_begin;   // first gap id of this colour
  int64_t g_count;   // gap sites of this colour (or of the list)
  const uint32_t* glist;  // nullable: gap ids of this phase (DC order), else the range
  int64_t P;         // gap ids allocated in G (G holds P * R floats)
  int R;             // realization stride of the batch (even)
  int npairs;        // realization pairs in the batch
  uint32_t pair_base;// global pair index of pair 0 (= m_base / 2)
  uint32_t sweep;    // 1-based sweep index s
  uint32_t k0, k1;   // Philox key
  uint32_t rk0[10], rk1[10];  // its round keys k + i * (0x9E3779B9, 0xBB67AE85), filled by
                              // launch_sweep_half: kernel-parameter (constant-bank) operands
  float q, J;
  int is_b;          // colour B half-sweep
  int accumulate;    // add the new state to A (fixed window)
  const int* win_lo; // nullable: adaptive protocol, realization r accumulates at sweeps
  const int* win_hi; //           win_lo[r] < s <= win_hi[r] and stops after win_hi[r]
  long long* energy; // nullable: per-realization fixed-point bond sums (ARITH §J) for
                     // this sweep, stride energy_stride
  int64_t energy_stride;
  int r_valid_lo, r_valid_hi;  // realizations [lo, hi) of the batch contribute energy
  unsigned long long* fstats;  // nullable: filter kernels add [0] queued pairs, [1] live pairs
};
int sweep_grid_size(int device, int variant);
// Variant 40's premises on this device (sweep.cu k_filter_check, run once per device):
// err[0] = the SFU sine's largest error against ARITH §B2's sine over every argument the
// filter sees, err[1] = the largest exp_spec(x) * 2^24 for x in [-80, -17]. Returns 1 when
// err[0] <= the bound's allowance and err[1] < 1 (the filter may run), else 0.
int sfu_filter_check(int device, double* err);
// Row f3 with shared-memory tiles: one launch updates every l_b tile of parity
// tau, both colours inside the tile (= the DC phases (tau, A), (tau, B)). dc_tile_chunk: the
// realizations per CTA for this l_b and batch (0: the tile does not fit shared memory).
int dc_tile_chunk(int lb, int R);
void launch_sweep_dc_tiles(const SweepArgs& s, const int32_t* gid, const float* phiK, const float* T, int64_t Lx,
                           int64_t Ly, int lb, int tau, int Rc, cudaStream_t st);
// grid: CTAs of one resident wave (sweep_grid_size); waves_forced > 0 fixes the number of
// resident waves per launch (else ~16 items per thread, 1-32 waves)
void launch_sweep_half(const SweepArgs& a, int grid, int variant, cudaStream_t st, int waves_forced = 0);
void launch_init_states(const GapRec* rec, const float* ginit, float* G, float* A, int64_t P, int R, int npairs,
                        uint32_t pair_base, int random_init, uint32_t k0, uint32_t k1,
                        cudaStream_t st);
// Adaptive protocol (row f1, ARITH §K) decided on the device: after sweep s, every
// undecided realization r < r_hi runs the slope test on its energies of sweeps
// s-n_fit+1 .. s (check) or is forced (forced), exactly as the host test would. A decided
// realization gets eq[r] = +-s and the averaging window (s, s + n_avg] in win_lo/win_hi;
// status[0] counts the undecided realizations, status[1] is the largest window end.
struct AdaptiveCheckArgs {
  const long long* energy;  // [R][energy_stride] fixed-point bond sums (ARITH §J)
  int64_t energy_stride;
  long long sum_known_fx;   // fixed-point sum of the known-known bonds
  double n_bonds;           // N_bonds of ARITH §J
  int s, n_fit, n_avg, check, forced, r_hi;
  double slope_tol;
  int* win_lo;
  int* win_hi;
  int* eq;
  int* status;
};
void launch_adaptive_check(const AdaptiveCheckArgs& a, cudaStream_t st);
void launch_acc_reduce(const float* X, int64_t g_begin, int64_t g_count, int R, int r_lo, int r_hi,
                       double* acc, cudaStream_t st);

// ---- calib.cu (row f2) ----
// Sweeps K*reps unconditional lattices (n_eq + n_meas sweeps); fx_host receives the
// fixed-point energy of lattice l = k*reps + rep after sweep s at [(s-1)*K*reps + l].
cudaError_t run_calibration(const float* T_host, int K, int L, float q, int n_eq, int n_meas, int reps,
                            uint64_t seed, long long* fx_host, cudaStream_t st);

}  // namespace mpr
