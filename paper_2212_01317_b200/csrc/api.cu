// api.cu — the C-ABI of libmpr.so (include/mpr.h): context state machine, device
// memory ownership, stage orchestration, the realization-batch loop of the conditional
// simulation and the multi-rank decompositions of SURVEY §8(e) (realization shards and
// row slabs, through the Comm transport of comm.cuh). All arithmetic happens in the
// kernels of params.cu and sweep.cu; this file only allocates, launches, copies and
// issues collectives.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "comm.cuh"
#include "internal.cuh"
#include "mpr.h"

using namespace mpr;

namespace {

// Grow-only device buffer.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t b) {
    if (b <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (b == 0) b = 16;
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

enum Stage { ST_INIT = 0, ST_DATA = 1, ST_PARAMS = 2, ST_SIM = 3 };

// Everything a realization batch's launch sequence depends on (CUDA graph cache key).
struct BatchKey {
  int64_t P, PA;
  int Rb;
  uint32_t pair_base;
  int32_t sweeps;
  uint32_t k0, k1;
  int n_avg, init, r_lo, r_hi, timing, variant, order, defer;
  float q, J;
  void *G, *A, *rec, *acc;
  long long* energy;
  // DC order: the phase segments baked into the captured launches (a new mask with the same
  // P and PA can have other phase boundaries)
  void* dclist;
  int64_t dc_off[5];
  int dc_rc;  // DC with shared-memory tiles: realizations per tile CTA (0: the phase lists)
  // the other buffers the captured launches read (a realloc can hand back an old address)
  void *ginit, *gid, *phiK, *T;
  // own gap-id ranges per colour (row slabs: a sub-range of the local ids)
  int64_t own[2][2];
};

struct GraphEntry {
  BatchKey key{};
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
};

// Contiguous, pair-aligned realization range of `rank` (one Philox call serves ids 2k and
// 2k + 1, ARITH §A); the ranges cover [0, M) once and differ by at most one pair.
void shard_range(int64_t M, int world, int rank, int64_t* m0, int64_t* m1) {
  const int64_t npairs = (M + 1) / 2;
  const int64_t p0 = rank * npairs / world, p1 = (rank + 1) * npairs / world;
  *m0 = std::min<int64_t>(2 * p0, M);
  *m1 = std::min<int64_t>(2 * p1, M);
}

// Rows [r0, r1) of row slab `rank`.
void row_range(int64_t Ly, int world, int rank, int64_t* r0, int64_t* r1) {
  *r0 = rank * Ly / world;
  *r1 = (rank + 1) * Ly / world;
}

}  // namespace

struct mpr_ctx {
  mpr_config cfg{};
  std::vector<float> calT, cale;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int stage = ST_INIT;
  std::string err;
  int sweep_grid = 0;
  int sweep_variant = 33;  // kernel variant (MPR_SWEEP_VARIANT, tuning only; sweep.cu)
  int sweep_waves = 0;     // resident waves per half-sweep launch (MPR_SWEEP_WAVES; 0 = auto)
  // MPR_FILTER_STATS=1: the filter kernels count their queued (exact-path) and all live
  // pairs into fstats[0..1] (one atomic per warp and launch; tests and bench only)
  DBuf fstats;
  // multi-rank
  std::unique_ptr<Comm> comm;
  int rank = 0, world = 1;
  bool rows = false;       // MPR_SHARD_ROWS with world > 1: slab-local layout + halos
  bool shards = false;     // MPR_SHARD_REALIZATIONS with world > 1: id ranges + reduction
  // row slabs: the halo exchange on its own stream, overlapped with the interior rows
  int halo_overlap = 1;    // MPR_HALO_OVERLAP=0: exchange in line after each half-sweep
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;
  int64_t comm_calls = 0;
  // problem (global)
  int64_t Lx = 0, Ly = 0;
  int64_t P_glob = 0, PA_glob = 0, n_known = 0;
  float zmin = 0, zmax = 0;
  int degenerate = 0;
  int64_t nbx = 0, nby = 0, nblocks = 0;
  int64_t n_fallback = 0;
  float median_T = 0;
  long long sum_SB_fx = 0;  // fixed-point bond sum of the known-known bonds (ARITH §J)
  long long sum_SB2_fx = 0; // fixed-point sum of their squared cosines (reading R22)
  long long n_sample_bonds = 0;
  // this rank's rows: own [row0, row1); local z/mask/phi/gid rows [lrow0, lrow1) (own + one
  // ghost row per side); local temperature rows [trow0, trow1) (own + the smoothing halo)
  int64_t row0 = 0, row1 = 0, lrow0 = 0, lrow1 = 0, trow0 = 0, trow1 = 0;
  int64_t n = 0;            // local sites (lrow1 - lrow0) * Lx
  int64_t nT = 0;           // local temperature sites
  // local gap ids: (colour, local row, column) order; P of them, PA of colour A
  int64_t P = 0, PA = 0;
  int64_t own[2][2] = {{0, 0}, {0, 0}};      // own gap ids of colour c: [own[c][0], own[c][1])
  int64_t ghost[2][2][2] = {};               // ghost row side s (0 up, 1 down), colour c: [b, e)
  int64_t bnd[2][2][2] = {};                 // own boundary row side s (0 first, 1 last), colour c
  // simulation bookkeeping
  int64_t M_total = 0, sweeps = 0, batch = 0, last_m_base = 0, last_R = 0, m_begin = 0, m_end = 0;
  int64_t split_min_P = int64_t(1) << 21;  // choose_batch's 4k + 2 split threshold (MPR_SPLIT_MIN_P)
  int64_t batch_key_P = -1, batch_key_R = -1, batch_cached = 0;
  int64_t launches = 0, total_launches = 0;
  int timing = 0;
  int64_t sweep_launches = 0;
  double sweep_ms = 0.0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> ev_pool;  // row slabs: events around each half-sweep kernel
  cudaEvent_t ev_check = nullptr;  // adaptive protocol: status copy of the last device check
  // CUDA graphs of the per-batch launch sequence (replayed when the key repeats)
  int use_graphs = 1;
  int slab_graphs = 0;  // MPR_SLAB_GRAPHS: also capture row-slab batches (NCCL halos inside)
  // MPR_DC_TILED=1: DC order on the paper's shared-memory tiles (k_sweep_dc_tile) instead of
  // the phase lists. Bit-identical; measured 2.6-4.5x slower at C2 (M = 100: 12.4-21.7 ms of
  // sweeps against 4.8 ms; profiles/r02_summary.md), so the lists are the default DC path.
  int dc_tiled = 0;
  std::vector<GraphEntry> graphs = std::vector<GraphEntry>(8);
  size_t graph_next = 0;
  int energy_enabled = 0;
  // ordered (deterministic) multi-rank reduction: simulate_range keeps the batch states and
  // mpr_accumulate_states adds them later (mpr_set_deferred_reduce)
  int defer_reduce = 0;
  int pending_reduce = 0, pending_Rb = 0, pending_r_lo = 0, pending_r_hi = 0;
  int64_t energy_M = 0, energy_S = 0;
  double last_slope_tol = 0.0;  // the slope tolerance the last adaptive run used
  std::vector<int> rowoff_h, rowcnt_h;  // host copies of the gap-id row offsets (row slabs)
  // device memory
  DBuf z, mask, phiK, scal, calTd, caled, rowcnt, rowoff, gid, rec, bstats, Tb, T, T2, G, A, acc,
      energy, out, tmp, win, dclist, dccnt, ginit;
  int64_t dc_off[5] = {0, 0, 0, 0, 0};  // DC phase segments of dclist (row f3)
  DevScalars* hsc = nullptr;  // pinned host mirror of the device scalars
};

namespace {

mpr_status fail(mpr_ctx* c, mpr_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

mpr_status cuda_fail(mpr_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(c, MPR_ERR_OOM, std::string(where) + ": out of device memory");
  }
  return fail(c, MPR_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr, where)                                 \
  do {                                                  \
    cudaError_t e_ = (expr);                            \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, where); \
  } while (0)

mpr_status check_launch(mpr_ctx* c, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(c, e, where);
  return MPR_OK;
}

#define CKL(where)                              \
  do {                                          \
    mpr_status s_ = check_launch(c, where);     \
    if (s_ != MPR_OK) return s_;                \
    ++c->total_launches;                        \
  } while (0)

// A collective through the context's communicator; errors carry the transport's message.
#define CKC(expr, where)                                                        \
  do {                                                                          \
    mpr_status s_ = (expr);                                                     \
    ++c->comm_calls;                                                            \
    if (s_ != MPR_OK) return fail(c, s_, std::string(where) + ": " + c->comm->err); \
  } while (0)

// Makes the context's device current for the duration of a call and restores the caller's
// current device afterwards (the library must not move e.g. torch's current device).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define SET_DEVICE(c)                                                     \
  DeviceGuard dev_guard_((c)->device);                                   \
  if (dev_guard_.err != cudaSuccess) return cuda_fail(c, dev_guard_.err, "set device")

mpr_status validate_cfg(const mpr_config* cfg, std::string& why) {
  if (!cfg) { why = "cfg is NULL"; return MPR_ERR_INVALID_ARG; }
  if (!(cfg->J > 0.0f) || !std::isfinite(cfg->J)) { why = "J must be finite and > 0"; return MPR_ERR_INVALID_ARG; }
  if (!(cfg->q > 0.0f && cfg->q <= 0.5f)) { why = "q must be in (0, 1/2]"; return MPR_ERR_INVALID_ARG; }
  if (cfg->l_b < 2) { why = "l_b must be >= 2"; return MPR_ERR_INVALID_ARG; }
  if (cfg->r_s < 0 || cfg->r_s > 16) { why = "r_s must be in [0, 16]"; return MPR_ERR_INVALID_ARG; }
  if (cfg->n_s < 0 || cfg->n_s > 1024) { why = "n_s must be in [0, 1024]"; return MPR_ERR_INVALID_ARG; }
  if (cfg->init != MPR_INIT_BLOCK_MEAN && cfg->init != MPR_INIT_RANDOM) { why = "init must be BLOCK_MEAN or RANDOM"; return MPR_ERR_INVALID_ARG; }
  if (cfg->n_avg < 1) { why = "n_avg must be >= 1"; return MPR_ERR_INVALID_ARG; }
  if (cfg->max_batch < 0) { why = "max_batch must be >= 0"; return MPR_ERR_INVALID_ARG; }
  if (cfg->order != MPR_ORDER_SC && cfg->order != MPR_ORDER_DC) { why = "order must be SC or DC"; return MPR_ERR_INVALID_ARG; }
  if (cfg->shard != MPR_SHARD_REALIZATIONS && cfg->shard != MPR_SHARD_ROWS) { why = "shard must be REALIZATIONS or ROWS"; return MPR_ERR_INVALID_ARG; }
  if (cfg->nccl_comm && cfg->group) { why = "nccl_comm and group are exclusive"; return MPR_ERR_INVALID_ARG; }
  if (cfg->shard == MPR_SHARD_ROWS && cfg->order != MPR_ORDER_SC && (cfg->nccl_comm || cfg->group)) {
    why = "row slabs need the SC order";
    return MPR_ERR_INVALID_ARG;
  }
  if (!cfg->calib_T || !cfg->calib_e || cfg->calib_n < 2 || cfg->calib_n > 256) {
    why = "calibration table must have 2..256 points";
    return MPR_ERR_INVALID_ARG;
  }
  // ARITH §E: a smoothing window sum of (2 r_s + 1)^2 terms llrint(T * 2^40) stays below
  // 2^63 iff (2 r_s + 1)^2 * T_max < 2^23 (T never exceeds the table's last T)
  {
    const double w = 2.0 * cfg->r_s + 1.0;
    const float Tmax = cfg->calib_T[cfg->calib_n - 1];
    if (cfg->n_s > 0 && std::isfinite(Tmax) && w * w * static_cast<double>(Tmax) >= 8388608.0) {
      why = "calibration T_max * (2 r_s + 1)^2 must be < 2^23 (ARITH §E window-sum bound)";
      return MPR_ERR_INVALID_ARG;
    }
  }
  for (int k = 0; k < cfg->calib_n; ++k) {
    const float T = cfg->calib_T[k], e = cfg->calib_e[k];
    if (!std::isfinite(T) || !std::isfinite(e) || !(T > 0.0f) || T > 1e4f) {
      why = "calibration table: T must be finite, in (0, 1e4]";
      return MPR_ERR_INVALID_ARG;
    }
    if (k > 0 && !(T > cfg->calib_T[k - 1] && e > cfg->calib_e[k - 1])) {
      why = "calibration table: T and e must be strictly increasing";
      return MPR_ERR_INVALID_ARG;
    }
  }
  return MPR_OK;
}

void set_scalars_init(DevScalars* h) {
  std::memset(h, 0, sizeof(*h));
  h->zmin_key = 0x7fffffff;
  h->zmax_key = static_cast<int>(0x80000000u);
}

// Inverse of the ordered-int key of device_math.cuh (host side).
float key_to_float(int k) {
  const int b = k >= 0 ? k : (k ^ 0x7fffffff);
  float f;
  std::memcpy(&f, &b, sizeof f);
  return f;
}

// e = (-(double)E_fx * 2^-32) / N_bonds  (ARITH §J)
double energy_from_fx(const mpr_ctx* c, long long E_fx) {
  const double nb = static_cast<double>(2 * c->Lx * c->Ly - c->Lx - c->Ly);
  return (-static_cast<double>(E_fx) * 0x1p-32) / nb;
}

// Reading R22: the slope tolerance of the equilibrium test derived from the data —
// the standard error of the sample specific energy e_s (Eq.(2)), spread over
// the n_fit-sweep fit window: tau = SE(e_s) / n_fit with SE(e_s)^2 = var(b) / N_SP over the
// sample bonds' cosines b (exact fixed-point sums S1 = sum llrint(b 2^32), S2 = sum llrint(b^2
// 2^32)). A drift below it over the window is smaller than the uncertainty of the energy the
// temperatures were matched to. fp64, in this order (the oracle's oracle_derived_slope_tol).
double derived_slope_tol(long long S1, long long S2, long long N, int n_fit) {
  if (N < 1) return 0.0;
  const double n = static_cast<double>(N);
  const double mean = (static_cast<double>(S1) * 0x1p-32) / n;
  const double m2 = (static_cast<double>(S2) * 0x1p-32) / n;
  double var = m2 - mean * mean;
  if (var < 0.0) var = 0.0;
  return std::sqrt(var / n) / static_cast<double>(n_fit);
}

// ---- row slabs: neighbour exchange of whole local rows (z / mask halos) -------------
// Row `r` (global) of a row-major local array with local row 0 = lrow0.
template <class T>
T* local_row(const mpr_ctx* c, T* base, int64_t r) {
  return base + (r - c->lrow0) * c->Lx;
}

// The first own row goes up (it is the upper neighbour's lower ghost row), the last own
// row goes down; the ghost rows come back from the neighbours.
template <class T>
mpr_status exchange_rows(mpr_ctx* c, T* base, CommType t) {
  std::vector<P2P> sends, recvs;
  const size_t cnt = static_cast<size_t>(c->Lx);
  if (c->rank > 0) {
    sends.push_back({c->rank - 1, local_row(c, base, c->row0), cnt});
    recvs.push_back({c->rank - 1, local_row(c, base, c->row0 - 1), cnt});
  }
  if (c->rank < c->world - 1) {
    sends.push_back({c->rank + 1, local_row(c, base, c->row1 - 1), cnt});
    recvs.push_back({c->rank + 1, local_row(c, base, c->row1), cnt});
  }
  CKC(c->comm->exchange(sends, recvs, t, c->stream), "halo rows");
  return MPR_OK;
}

// After a colour-`col` half-sweep: the colour's states of the first and last own rows go
// to the neighbours' ghost rows (gap-site major, realization minor: each row's colour-c
// states are one contiguous run of R floats per gap). SURVEY §8(e) 2.
mpr_status exchange_halo(mpr_ctx* c, int col, int R, cudaStream_t stream) {
  std::vector<P2P> sends, recvs;
  float* G = c->G.as<float>();
  auto seg = [&](const int64_t (&r)[2]) { return static_cast<size_t>((r[1] - r[0]) * R); };
  if (c->rank > 0) {
    sends.push_back({c->rank - 1, G + c->bnd[0][col][0] * R, seg(c->bnd[0][col])});
    recvs.push_back({c->rank - 1, G + c->ghost[0][col][0] * R, seg(c->ghost[0][col])});
  }
  if (c->rank < c->world - 1) {
    sends.push_back({c->rank + 1, G + c->bnd[1][col][0] * R, seg(c->bnd[1][col])});
    recvs.push_back({c->rank + 1, G + c->ghost[1][col][0] * R, seg(c->ghost[1][col])});
  }
  CKC(c->comm->exchange(sends, recvs, CT_F32, stream), "halo exchange");
  return MPR_OK;
}

// Own, ghost and boundary gap-id ranges from the host copy of the per-row colour offsets.
void slab_ranges(mpr_ctx* c) {
  const int64_t nl = c->lrow1 - c->lrow0;
  auto off = [&](int col, int64_t r) -> int64_t {  // first id of colour col in global row r
    const int64_t lr = r - c->lrow0;
    if (lr >= nl) return col == 0 ? c->PA : c->P;
    return c->rowoff_h[static_cast<size_t>(col * nl + lr)];
  };
  for (int col = 0; col < 2; ++col) {
    c->own[col][0] = off(col, c->row0);
    c->own[col][1] = off(col, c->row1);
    c->ghost[0][col][0] = off(col, c->lrow0);
    c->ghost[0][col][1] = off(col, c->row0);  // empty when lrow0 == row0
    c->ghost[1][col][0] = off(col, c->row1);
    c->ghost[1][col][1] = off(col, c->lrow1);  // empty when lrow1 == row1
    c->bnd[0][col][0] = off(col, c->row0);
    c->bnd[0][col][1] = off(col, c->row0 + 1);
    c->bnd[1][col][0] = off(col, c->row1 - 1);
    c->bnd[1][col][1] = off(col, c->row1);
  }
}

mpr_status stage_data(mpr_ctx* c) {
  cudaStream_t st = c->stream;
  if (c->rows) {  // ghost rows of z and mask from the neighbours (cross-slab bonds, sweep)
    mpr_status s = exchange_rows(c, c->z.as<float>(), CT_F32);
    if (s != MPR_OK) return s;
    s = exchange_rows(c, c->mask.as<uint8_t>(), CT_U8);
    if (s != MPR_OK) return s;
  }
  set_scalars_init(c->hsc);
  CK(cudaMemcpyAsync(c->scal.p, c->hsc, sizeof(DevScalars), cudaMemcpyHostToDevice, st), "scalars upload");
  // a1 over the OWN rows (each sample counted by exactly one rank)
  launch_minmax_count(local_row(c, c->z.as<float>(), c->row0), local_row(c, c->mask.as<uint8_t>(), c->row0), c->Lx,
                      c->row1 - c->row0, c->row0, c->scal.as<DevScalars>(), st);
  CKL("minmax_count");
  if (c->rows) {  // global extrema and counts (exact: min/max of keys, integer sums)
    DevScalars* d = c->scal.as<DevScalars>();
    CKC(c->comm->allreduce(&d->zmin_key, 1, CT_I32, OP_MIN, st), "allreduce z_min");
    CKC(c->comm->allreduce(&d->zmax_key, 1, CT_I32, OP_MAX, st), "allreduce z_max");
    CKC(c->comm->allreduce(&d->bad_sample, 1, CT_I32, OP_MAX, st), "allreduce flags");
    CKC(c->comm->allreduce(&d->n_known, 3, CT_U64, OP_SUM, st), "allreduce counts");
  }
  CK(cudaMemcpyAsync(c->hsc, c->scal.p, sizeof(DevScalars), cudaMemcpyDeviceToHost, st), "scalars download");
  CK(cudaStreamSynchronize(st), "minmax_count sync");
  if (c->hsc->bad_sample) return fail(c, MPR_ERR_INVALID_ARG, "non-finite value at a known sample");
  c->n_known = static_cast<int64_t>(c->hsc->n_known);
  if (c->n_known < 2) return fail(c, MPR_ERR_TOO_FEW_SAMPLES, "fewer than 2 known samples");
  c->PA_glob = static_cast<int64_t>(c->hsc->n_gap[0]);
  c->P_glob = c->PA_glob + static_cast<int64_t>(c->hsc->n_gap[1]);
  c->zmin = key_to_float(c->hsc->zmin_key) + 0.0f;
  c->zmax = key_to_float(c->hsc->zmax_key) + 0.0f;
  c->degenerate = (c->zmin == c->zmax);
  const int64_t n = c->n;
  const int64_t nl = c->lrow1 - c->lrow0;
  CK(c->phiK.ensure(sizeof(float) * n), "alloc phi");
  launch_transform(c->z.as<float>(), c->mask.as<uint8_t>(), n, c->scal.as<DevScalars>(), c->phiK.as<float>(), st);
  CKL("transform");
  CK(c->gid.ensure(sizeof(int32_t) * n), "alloc gid");
  CK(c->rowcnt.ensure(sizeof(int) * 2 * nl), "alloc rowcnt");
  CK(c->rowoff.ensure(sizeof(int) * 2 * nl), "alloc rowoff");
  if (!c->rows) {
    c->PA = c->PA_glob;
    c->P = c->P_glob;
  } else {  // local ids cover the ghost rows too: count them first
    launch_gap_rows(c->mask.as<uint8_t>(), c->Lx, nl, c->lrow0, c->rowcnt.as<int>(), c->rowoff.as<int>(), st);
    c->total_launches += 2;
    c->rowoff_h.resize(static_cast<size_t>(2 * nl));
    c->rowcnt_h.resize(static_cast<size_t>(2 * nl));
    CK(cudaMemcpyAsync(c->rowoff_h.data(), c->rowoff.p, sizeof(int) * 2 * nl, cudaMemcpyDeviceToHost, st), "D2H rowoff");
    CK(cudaMemcpyAsync(c->rowcnt_h.data(), c->rowcnt.p, sizeof(int) * 2 * nl, cudaMemcpyDeviceToHost, st), "D2H rowcnt");
    CK(cudaStreamSynchronize(st), "gap rows sync");
    c->PA = c->rowoff_h[static_cast<size_t>(nl)];
    c->P = c->rowoff_h[static_cast<size_t>(2 * nl - 1)] + c->rowcnt_h[static_cast<size_t>(2 * nl - 1)];
  }
  CK(c->rec.ensure(sizeof(GapRec) * std::max<int64_t>(c->P, 1)), "alloc records");
  CK(c->ginit.ensure(sizeof(float) * std::max<int64_t>(c->P, 1)), "alloc init angles");
  if (!c->rows) {
    launch_gap_index(c->mask.as<uint8_t>(), c->Lx, nl, 0, c->rowcnt.as<int>(), c->rowoff.as<int>(), c->gid.as<int32_t>(),
                     st);
    c->total_launches += 3;
    c->own[0][0] = 0; c->own[0][1] = c->PA;
    c->own[1][0] = c->PA; c->own[1][1] = c->P;
  } else {
    launch_gap_compact(c->mask.as<uint8_t>(), c->Lx, nl, c->lrow0, c->rowoff.as<int>(), c->gid.as<int32_t>(), st);
    CKL("gap_compact");
    slab_ranges(c);
  }
  // no final sync: the caller's buffers were copied before the min/max sync above, and
  // the gap-index kernels only touch context buffers (stream-ordered before later calls)
  c->stage = ST_DATA;
  c->pending_reduce = 0;
  c->M_total = 0;
  return MPR_OK;
}

mpr_status check_dims(mpr_ctx* c, int64_t Lx, int64_t Ly) {
  if (Lx < 2 || Ly < 2) return fail(c, MPR_ERR_INVALID_ARG, "Lx and Ly must be >= 2");
  // ARITH §E/§J: with Lx*Ly <= 2^30 every int64 fixed-point sum stays below 2^63 (the grid
  // energy and a one-block SB have < 2^31 bonds of magnitude <= 2^32; SP < 2^30 * 2^31)
  if (Lx > (int64_t(1) << 30) || Ly > (int64_t(1) << 30) || Lx * Ly > (int64_t(1) << 30))
    return fail(c, MPR_ERR_INVALID_ARG, "Lx*Ly must be <= 2^30 (ARITH §E fixed-point bounds)");
  if (c->rows && Ly < c->world) return fail(c, MPR_ERR_INVALID_ARG, "row slabs need Ly >= world");
  return MPR_OK;
}

// Geometry of this rank's slab and the local buffers (whole grid unless row slabs).
mpr_status alloc_inputs(mpr_ctx* c, int64_t Lx, int64_t Ly) {
  c->Lx = Lx;
  c->Ly = Ly;
  if (c->rows) {
    row_range(Ly, c->world, c->rank, &c->row0, &c->row1);
    c->lrow0 = std::max<int64_t>(c->row0 - 1, 0);
    c->lrow1 = std::min<int64_t>(c->row1 + 1, Ly);
    // a temperature halo of r_s * n_s rows (at least the ghost row): after n_s passes the
    // clipped-window error of the halo's inner edge has moved r_s * n_s rows, not into the slab
    const int64_t H = std::max<int64_t>(static_cast<int64_t>(c->cfg.r_s) * c->cfg.n_s, 1);
    c->trow0 = std::max<int64_t>(c->row0 - H, 0);
    c->trow1 = std::min<int64_t>(c->row1 + H, Ly);
  } else {
    c->row0 = c->lrow0 = c->trow0 = 0;
    c->row1 = c->lrow1 = c->trow1 = Ly;
  }
  c->n = (c->lrow1 - c->lrow0) * Lx;
  c->nT = (c->trow1 - c->trow0) * Lx;
  c->stage = ST_INIT;
  CK(c->z.ensure(sizeof(float) * c->n), "alloc z");
  CK(c->mask.ensure(c->n), "alloc mask");
  return MPR_OK;
}

int64_t choose_batch(mpr_ctx* c, int64_t M_span) {
  int64_t R = M_span + (M_span & 1);
  if (R > 1024) R = 1024;
  if (c->cfg.max_batch > 0) {
    int64_t mb = c->cfg.max_batch + (c->cfg.max_batch & 1);
    R = std::min(R, std::max<int64_t>(mb, 2));
  }
  // cudaMemGetInfo is slow (driver round trip): reuse the last answer for the same shape
  if (c->batch_key_P == c->P && c->batch_key_R == R && c->batch_cached > 0) return c->batch_cached;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const double per_r = 4.0 * static_cast<double>(std::max<int64_t>(c->P, 1)) * (c->cfg.n_avg > 1 ? 2.0 : 1.0);
  const double budget = 0.6 * static_cast<double>(fr + c->G.bytes + c->A.bytes);
  int64_t cap = static_cast<int64_t>(budget / per_r);
  // the sweep kernel indexes the state with 32-bit element offsets: P * R < 2^31
  cap = std::min<int64_t>(cap, ((int64_t(1) << 31) - 1) / std::max<int64_t>(c->P, 1));
  cap -= cap & 1;
  if (cap < 2) cap = 2;
  int64_t B = std::min(R, cap);
  // The default sweep kernel (variants 22, 28) moves two realization pairs per thread and
  // needs an even pair count per batch: split R = 4k + 2 as 4k + 2 (e.g. M = 10 -> 8 + 2;
  // the 2-realization batch runs the one-pair kernel). Only for large grids: a separate 2-realization batch costs a full launch sequence,
  // which small, latency-bound problems do not win back (256^2..1024^2, M = 10: measured
  // 0.36 -> 0.50 ms and 1.25 -> 1.39 ms when split; 16384^2: 3.85 -> 3.40 ms / half-sweep).
  // (A 5-pair-per-thread kernel running R = 10 as one batch with float2 moves was measured
  // slower at C4: 3.65 ms per half-sweep against 2.21 + 0.78 ms for 8 + 2; dropped.)
  if ((c->sweep_variant == 22 || c->sweep_variant == 28 || c->sweep_variant == 33 || c->sweep_variant == 40) && B % 4 == 2 && B > 2 &&
      c->P >= c->split_min_P)
    B -= 2;
  c->batch_key_P = c->P;
  c->batch_key_R = R;
  c->batch_cached = B;
  return c->batch_cached;
}

}  // namespace

extern "C" {

const char* mpr_version(void) { return "libmpr 0.2 (sm_100a, LE-MPR / SV-MPR arXiv 2212.01317)"; }

int mpr_filter_check(int device, double* err_out) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    return 0;
  }
  return sfu_filter_check(device, err_out);
}

void mpr_config_default(mpr_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->device = 0;
  cfg->stream = nullptr;
  cfg->J = 1.0f;
  cfg->q = 0.5f;
  cfg->l_b = 32;
  cfg->r_s = 2;
  cfg->n_s = 5;
  cfg->init = MPR_INIT_BLOCK_MEAN;
  cfg->n_avg = 1;
  cfg->max_batch = 0;
  cfg->shard = MPR_SHARD_REALIZATIONS;
}

mpr_status mpr_init(const mpr_config* cfg, mpr_ctx** out) {
  if (!out) return MPR_ERR_INVALID_ARG;
  *out = nullptr;
  std::string why;
  mpr_status s = validate_cfg(cfg, why);
  if (s != MPR_OK) {
    std::fprintf(stderr, "mpr_init: %s\n", why.c_str());
    return s;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    std::fprintf(stderr, "mpr_init: no CUDA device\n");
    return MPR_ERR_CUDA;
  }
  if (cfg->device < 0 || cfg->device >= ndev) return MPR_ERR_INVALID_ARG;
  mpr_ctx* c = new mpr_ctx();
  c->cfg = *cfg;
  c->device = cfg->device;
  c->calT.assign(cfg->calib_T, cfg->calib_T + cfg->calib_n);
  c->cale.assign(cfg->calib_e, cfg->calib_e + cfg->calib_n);
  c->cfg.calib_T = c->calT.data();
  c->cfg.calib_e = c->cale.data();
  DeviceGuard dev_guard(c->device);
  cudaError_t e = dev_guard.err;
  if (e == cudaSuccess) {
    if (cfg->stream) {
      c->stream = static_cast<cudaStream_t>(cfg->stream);
    } else {
      e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
      c->own_stream = true;
    }
  }
  if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&c->hsc), sizeof(DevScalars));
  if (e == cudaSuccess) e = c->scal.ensure(sizeof(DevScalars));
  if (e == cudaSuccess) e = c->calTd.ensure(sizeof(float) * c->calT.size());
  if (e == cudaSuccess) e = c->caled.ensure(sizeof(float) * c->cale.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(c->calTd.p, c->calT.data(), sizeof(float) * c->calT.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(c->caled.p, c->cale.data(), sizeof(float) * c->cale.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "mpr_init: %s\n", cudaGetErrorString(e));
    mpr_destroy(c);
    return e == cudaErrorMemoryAllocation ? MPR_ERR_OOM : MPR_ERR_CUDA;
  }
  if (cfg->nccl_comm || cfg->group) {
    Comm* cm = cfg->nccl_comm ? make_nccl_comm(cfg->nccl_comm, c->device, why)
                              : make_group_comm(cfg->group, cfg->group_rank, why);
    if (!cm) {
      std::fprintf(stderr, "mpr_init: %s\n", why.c_str());
      mpr_destroy(c);
      return cfg->nccl_comm ? MPR_ERR_NCCL : MPR_ERR_INVALID_ARG;
    }
    c->comm.reset(cm);
    c->rank = cm->rank;
    c->world = cm->world;
  }
  // MPR_FORCE_COMM=1 (tests): the multi-rank code paths even at world size 1, so that a
  // single GPU runs the transport's collectives for real
  const char* fc = std::getenv("MPR_FORCE_COMM");
  const bool multi = c->comm && (c->world > 1 || (fc && std::atoi(fc)));
  c->rows = multi && cfg->shard == MPR_SHARD_ROWS;
  c->shards = multi && cfg->shard == MPR_SHARD_REALIZATIONS;
  if (const char* v = std::getenv("MPR_HALO_OVERLAP")) c->halo_overlap = std::atoi(v) ? 1 : 0;
  if (c->rows) {
    e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_bnd, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      std::fprintf(stderr, "mpr_init: %s\n", cudaGetErrorString(e));
      mpr_destroy(c);
      return MPR_ERR_CUDA;
    }
  }
  if (const char* v = std::getenv("MPR_SWEEP_VARIANT")) c->sweep_variant = std::atoi(v);
  if (const char* v = std::getenv("MPR_SWEEP_WAVES")) c->sweep_waves = std::max(0, std::atoi(v));
  // the SFU-filtered kernel (variant 40, opt-in: measured slower) only where
  // its error bound was verified on this device; otherwise the exact kernel 28
  if ((c->sweep_variant == 40 || c->sweep_variant == 41) && !sfu_filter_check(c->device, nullptr)) {
    std::fprintf(stderr, "mpr_init: SFU filter check failed on device %d, using sweep variant 33\n", c->device);
    c->sweep_variant = 33;
  }
  if (const char* v = std::getenv("MPR_FILTER_STATS"))
    if (std::atoi(v)) {
      if (c->fstats.ensure(2 * sizeof(unsigned long long)) != cudaSuccess ||
          cudaMemset(c->fstats.p, 0, 2 * sizeof(unsigned long long)) != cudaSuccess) {
        mpr_destroy(c);
        return MPR_ERR_CUDA;
      }
    }
  if (const char* v = std::getenv("MPR_NO_GRAPHS")) c->use_graphs = std::atoi(v) ? 0 : 1;
  if (const char* v = std::getenv("MPR_SLAB_GRAPHS")) c->slab_graphs = std::atoi(v) ? 1 : 0;
  if (const char* v = std::getenv("MPR_DC_TILED")) c->dc_tiled = std::atoi(v) ? 1 : 0;
  if (const char* v = std::getenv("MPR_SPLIT_MIN_P")) c->split_min_P = std::atoll(v);
  c->sweep_grid = sweep_grid_size(c->device, c->sweep_variant);
  *out = c;
  return MPR_OK;
}

void mpr_destroy(mpr_ctx* c) {
  if (!c) return;
  DeviceGuard dev_guard(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  DBuf* bufs[] = {&c->z, &c->mask, &c->phiK, &c->scal, &c->calTd, &c->caled, &c->rowcnt, &c->rowoff,
                  &c->gid, &c->rec, &c->bstats, &c->Tb, &c->T, &c->T2, &c->G, &c->A, &c->acc,
                  &c->energy, &c->out, &c->tmp, &c->win, &c->dclist, &c->dccnt, &c->ginit, &c->fstats};
  for (DBuf* b : bufs) b->release();
  if (c->hsc) cudaFreeHost(c->hsc);
  for (auto& e : c->graphs)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (cudaEvent_t ev : c->ev_pool) cudaEventDestroy(ev);
  if (c->ev_check) cudaEventDestroy(c->ev_check);
  if (c->ev_bnd) cudaEventDestroy(c->ev_bnd);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->comm_stream) {
    cudaStreamSynchronize(c->comm_stream);
    cudaStreamDestroy(c->comm_stream);
  }
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* mpr_last_error(const mpr_ctx* c) { return c ? c->err.c_str() : "NULL context"; }

mpr_status mpr_set_data(mpr_ctx* c, const float* grid, const uint8_t* mask, int64_t Lx, int64_t Ly) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (!grid || !mask) return fail(c, MPR_ERR_INVALID_ARG, "grid and mask must be non-NULL");
  mpr_status s = check_dims(c, Lx, Ly);
  if (s != MPR_OK) return s;
  SET_DEVICE(c);
  s = alloc_inputs(c, Lx, Ly);
  if (s != MPR_OK) return s;
  // the own rows only (the whole grid unless row slabs); ghost rows come from the neighbours
  const int64_t off = c->row0 * Lx, cnt = (c->row1 - c->row0) * Lx;
  CK(cudaMemcpyAsync(local_row(c, c->z.as<float>(), c->row0), grid + off, sizeof(float) * cnt, cudaMemcpyHostToDevice,
                     c->stream), "H2D grid");
  CK(cudaMemcpyAsync(local_row(c, c->mask.as<uint8_t>(), c->row0), mask + off, cnt, cudaMemcpyHostToDevice, c->stream),
     "H2D mask");
  return stage_data(c);
}

mpr_status mpr_set_data_device(mpr_ctx* c, const float* grid, const uint8_t* mask, int64_t Lx, int64_t Ly) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (!grid || !mask) return fail(c, MPR_ERR_INVALID_ARG, "grid and mask must be non-NULL");
  mpr_status s = check_dims(c, Lx, Ly);
  if (s != MPR_OK) return s;
  SET_DEVICE(c);
  s = alloc_inputs(c, Lx, Ly);
  if (s != MPR_OK) return s;
  // row slabs: the device pointers hold the own rows only
  const int64_t cnt = (c->row1 - c->row0) * Lx;
  CK(cudaMemcpyAsync(local_row(c, c->z.as<float>(), c->row0), grid, sizeof(float) * cnt, cudaMemcpyDeviceToDevice,
                     c->stream), "D2D grid");
  CK(cudaMemcpyAsync(local_row(c, c->mask.as<uint8_t>(), c->row0), mask, cnt, cudaMemcpyDeviceToDevice, c->stream),
     "D2D mask");
  return stage_data(c);
}

mpr_status mpr_estimate_local_params(mpr_ctx* c, float* T_out) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (c->stage < ST_DATA) return fail(c, MPR_ERR_STATE, "estimate_local_params before set_data");
  SET_DEVICE(c);
  cudaStream_t st = c->stream;
  const int lb = c->cfg.l_b;
  c->nbx = (c->Lx + lb - 1) / lb;
  c->nby = (c->Ly + lb - 1) / lb;
  c->nblocks = c->nbx * c->nby;
  CK(c->bstats.ensure(sizeof(long long) * 4 * c->nblocks), "alloc block stats");
  CK(c->Tb.ensure(sizeof(float) * 2 * c->nblocks), "alloc Tb");  // T_b, then the blocks' init angles
  CK(c->T.ensure(sizeof(float) * c->nT), "alloc T");
  if (c->cfg.n_s > 0) CK(c->T2.ensure(sizeof(float) * c->nT), "alloc T2");
  long long* SB = c->bstats.as<long long>();
  long long* NB = SB + c->nblocks;
  long long* SP = NB + c->nblocks;
  long long* NK = SP + c->nblocks;
  DevScalars* dsc = c->scal.as<DevScalars>();
  // reset the parameter-stage scalars (n_avail .. median_T)
  const size_t off = offsetof(DevScalars, n_avail);
  CK(cudaMemsetAsync(reinterpret_cast<char*>(dsc) + off, 0, sizeof(DevScalars) - off, st), "reset scalars");
  // a3 over the own rows (a bond belongs to the block of its left/top end: the rank owning
  // that end counts it; a down bond of the last own row reads the lower ghost row)
  launch_block_stats(c->phiK.as<float>(), c->mask.as<uint8_t>(), c->Lx, c->Ly, c->lrow0, c->row0, c->row1, lb,
                     c->cfg.q, SB, NB, SP, NK, c->nblocks, dsc, st);
  CKL("block_stats");
  // row slabs: every rank's partial block sums -> the global ones on every rank (exact int64)
  if (c->rows) {
    CKC(c->comm->allreduce(SB, static_cast<size_t>(4 * c->nblocks), CT_I64, OP_SUM, st), "allreduce block sums");
    CKC(c->comm->allreduce(&dsc->sum_SB2, 1, CT_I64, OP_SUM, st), "allreduce squared bond sum");
  }
  launch_block_T(SB, NB, SP, NK, c->nblocks, c->calTd.as<float>(), c->caled.as<float>(),
                 static_cast<int>(c->calT.size()), c->Tb.as<float>(), dsc, st);
  CKL("block_T");
  launch_median_fill(c->Tb.as<float>(), NB, c->nblocks, dsc, st);
  CKL("median_fill");
  float* binit = c->Tb.as<float>() + c->nblocks;
  launch_block_init(SP, NK, c->nblocks, dsc, binit, st);
  CKL("block_init");
  // a5 on the local temperature rows [trow0, trow1) (the whole grid unless row slabs). With a
  // specialised radius the first pass reads the block temperatures directly (no expanded
  // field is written); otherwise expand, then the generic passes.
  const int64_t nTr = c->trow1 - c->trow0;
  int k0 = 0;
  const float Tmin = c->calT.front(), Tmax = c->calT.back();
  if (c->cfg.n_s > 0 && launch_smooth_specialised(nullptr, c->Tb.as<float>(), c->T.as<float>(), c->Lx, nTr, c->trow0,
                                                  c->Ly, c->cfg.r_s, lb, Tmin, Tmax, st)) {
    CKL("smooth (from T_b)");
    k0 = 1;
  } else {
    launch_expand(c->Tb.as<float>(), c->Lx, c->trow0, c->trow1, lb, c->T.as<float>(), st);
    CKL("expand");
  }
  for (int k = k0; k < c->cfg.n_s; ++k) {
    if (!launch_smooth_specialised(c->T.as<float>(), nullptr, c->T2.as<float>(), c->Lx, nTr, c->trow0, c->Ly,
                                   c->cfg.r_s, lb, Tmin, Tmax, st))
      launch_smooth(c->T.as<float>(), c->T2.as<float>(), c->Lx, nTr, c->trow0, c->Ly, c->cfg.r_s, st);
    CKL("smooth");
    std::swap(c->T, c->T2);
  }
  launch_build_records(c->gid.as<int32_t>(), c->mask.as<uint8_t>(), c->phiK.as<float>(), c->T.as<float>(), binit,
                       c->Lx, c->Ly, c->lrow0, c->lrow1, c->trow0, c->trow1, lb, c->P, c->rec.as<GapRec>(),
                       c->ginit.as<float>(), st);
  CKL("build_records");
  CK(cudaMemcpyAsync(c->hsc, c->scal.p, sizeof(DevScalars), cudaMemcpyDeviceToHost, st), "scalars download");
  if (T_out)
    CK(cudaMemcpyAsync(T_out + c->row0 * c->Lx, c->T.as<float>() + (c->row0 - c->trow0) * c->Lx,
                       sizeof(float) * (c->row1 - c->row0) * c->Lx, cudaMemcpyDeviceToHost, st), "D2H T");
  CK(cudaStreamSynchronize(st), "estimate_local_params sync");
  c->n_fallback = static_cast<int64_t>(c->hsc->n_fallback);
  c->median_T = c->hsc->median_T;
  c->sum_SB_fx = c->hsc->sum_SB;
  c->sum_SB2_fx = c->hsc->sum_SB2;
  c->n_sample_bonds = c->hsc->sum_NB;
  if (c->hsc->n_avail == 0 && !c->degenerate)
    return fail(c, MPR_ERR_NO_SAMPLE_BONDS, "no block has a sample-sample bond (PAPER.md:108)");
  if (c->cfg.order == MPR_ORDER_DC && c->P > 0) {
    // phase lists of the double checkerboard (row f3): count, offsets, scatter
    CK(c->dccnt.ensure(4 * sizeof(unsigned long long)), "alloc dc counts");
    CK(c->dclist.ensure(sizeof(uint32_t) * c->P), "alloc dc list");
    unsigned long long cnt[4];
    launch_dc_count(c->rec.as<GapRec>(), c->P, c->Lx, lb, c->dccnt.as<unsigned long long>(), st);
    CKL("dc_count");
    CK(cudaMemcpyAsync(cnt, c->dccnt.p, sizeof cnt, cudaMemcpyDeviceToHost, st), "D2H dc counts");
    CK(cudaStreamSynchronize(st), "dc sync");
    c->dc_off[0] = 0;
    for (int p = 0; p < 4; ++p) c->dc_off[p + 1] = c->dc_off[p] + static_cast<int64_t>(cnt[p]);
    unsigned long long cur[4] = {0, static_cast<unsigned long long>(c->dc_off[1]),
                                 static_cast<unsigned long long>(c->dc_off[2]),
                                 static_cast<unsigned long long>(c->dc_off[3])};
    CK(cudaMemcpyAsync(c->dccnt.p, cur, sizeof cur, cudaMemcpyHostToDevice, st), "H2D dc cursors");
    launch_dc_scatter(c->rec.as<GapRec>(), c->P, c->Lx, lb, c->dccnt.as<unsigned long long>(),
                      c->dclist.as<uint32_t>(), st);
    CKL("dc_scatter");
    CK(cudaStreamSynchronize(st), "dc sync");
  }
  c->stage = ST_PARAMS;
  c->M_total = 0;
  return MPR_OK;
}

mpr_status mpr_set_energy_trace(mpr_ctx* c, int enable) {
  if (!c) return MPR_ERR_INVALID_ARG;
  c->energy_enabled = enable ? 1 : 0;
  return MPR_OK;
}

mpr_status mpr_set_kernel_timing(mpr_ctx* c, int enable) {
  if (!c) return MPR_ERR_INVALID_ARG;
  c->timing = enable ? 1 : 0;
  c->sweep_ms = 0.0;
  c->sweep_launches = 0;
  return MPR_OK;
}

mpr_status mpr_reset_accumulator(mpr_ctx* c) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (c->stage < ST_PARAMS) return fail(c, MPR_ERR_STATE, "reset_accumulator before estimate_local_params");
  SET_DEVICE(c);
  CK(c->acc.ensure(sizeof(double) * std::max<int64_t>(c->P, 1)), "alloc acc");
  CK(cudaMemsetAsync(c->acc.p, 0, sizeof(double) * std::max<int64_t>(c->P, 1), c->stream), "zero acc");
  c->M_total = 0;
  c->energy_M = 0;
  c->stage = ST_PARAMS;
  return MPR_OK;
}

// Row slabs: the half-sweep kernel's own device time (events around the launch; the
// batch-level events would also include the halo collectives).
static mpr_status slab_timing_event(mpr_ctx* c, size_t k, cudaEvent_t* ev) {
  while (c->ev_pool.size() <= k) {
    cudaEvent_t e = nullptr;
    CK(cudaEventCreate(&e), "event");
    c->ev_pool.push_back(e);
  }
  *ev = c->ev_pool[k];
  return MPR_OK;
}

// One SC colour half-sweep over this rank's gap sites of `colour` (a carries the batch, the
// sweep and the accumulation flags): one launch over the colour's own id range, or — row
// slabs — the update of the own rows followed by the halo exchange of this colour. With
// halo_overlap (and >= 3 own rows) the two boundary rows go first, their exchange runs on
// the comm stream while the interior rows update, and the context stream waits for it
// before the next half-sweep (which reads this colour's ghost rows). The interior does not
// touch this colour's ghost rows and the exchange does not touch the other colour, so the
// overlap changes no bit. timing: CUDA events around every launch (kernel time only).
static mpr_status sc_half_sweep(mpr_ctx* c, SweepArgs& a, int colour, int variant, bool timing, unsigned ev_flags,
                                size_t* evk, int64_t* nsweep) {
  cudaStream_t st = c->stream;
  a.is_b = colour;
  auto sweep_range = [&](int64_t g0, int64_t g1) -> mpr_status {
    if (g1 <= g0) return MPR_OK;
    a.g_begin = g0;
    a.g_count = g1 - g0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) {
      mpr_status se = slab_timing_event(c, (*evk)++, &e0);
      if (se == MPR_OK) se = slab_timing_event(c, (*evk)++, &e1);
      if (se != MPR_OK) return se;
      CK(cudaEventRecordWithFlags(e0, st, ev_flags), "event record");
    }
    launch_sweep_half(a, c->sweep_grid, variant, st, c->sweep_waves);
    CKL("sweep_half");
    if (timing) CK(cudaEventRecordWithFlags(e1, st, ev_flags), "event record");
    ++c->launches;
    if (nsweep) ++*nsweep;
    return MPR_OK;
  };
  mpr_status sr = MPR_OK;
  if (c->rows && c->halo_overlap && c->row1 - c->row0 >= 3) {
    sr = sweep_range(c->bnd[0][colour][0], c->bnd[0][colour][1]);
    if (sr == MPR_OK) sr = sweep_range(c->bnd[1][colour][0], c->bnd[1][colour][1]);
    if (sr != MPR_OK) return sr;
    CK(cudaEventRecord(c->ev_bnd, st), "event record");
    sr = sweep_range(c->bnd[0][colour][1], c->bnd[1][colour][0]);
    if (sr != MPR_OK) return sr;
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_bnd, 0), "comm stream wait");
    sr = exchange_halo(c, colour, a.R, c->comm_stream);
    if (sr != MPR_OK) return sr;
    CK(cudaEventRecord(c->ev_halo, c->comm_stream), "event record");
    CK(cudaStreamWaitEvent(st, c->ev_halo, 0), "stream wait halo");
    return MPR_OK;
  }
  sr = sweep_range(c->own[colour][0], c->own[colour][1]);
  if (sr != MPR_OK) return sr;
  if (c->rows) return exchange_halo(c, colour, a.R, st);
  return MPR_OK;
}

// One realization batch: init, 2*S half-sweeps (bracketed by the timing events; row slabs:
// each followed by the halo exchange of its colour), and the realization sum into the
// accumulator. Issued directly or captured into a CUDA graph.
static mpr_status issue_batch(mpr_ctx* c, const BatchKey& k, int64_t* nsweep, bool capturing) {
  // inside a stream capture the timing events must be external record nodes
  const unsigned ev_flags = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
  cudaStream_t st = c->stream;
  const bool avg = k.n_avg > 1;
  const int npairs = k.Rb / 2;
  // every local gap (ghost rows too: initial states are a pure function of the global ids,
  // so the ghost rows need no exchange before the first half-sweep)
  launch_init_states(c->rec.as<GapRec>(), c->ginit.as<float>(), c->G.as<float>(), avg ? c->A.as<float>() : nullptr, k.P,
                     k.Rb, npairs,
                     k.pair_base, k.init == MPR_INIT_RANDOM, k.k0, k.k1, st);
  CKL("init_states");
  ++c->launches;
  SweepArgs a{};
  a.rec = c->rec.as<GapRec>();
  a.G = c->G.as<float>();
  a.P = c->P;
  a.A = avg ? c->A.as<float>() : nullptr;
  a.R = k.Rb;
  a.npairs = npairs;
  a.pair_base = k.pair_base;
  a.k0 = k.k0;
  a.k1 = k.k1;
  a.q = k.q;
  a.J = k.J;
  a.r_valid_lo = k.r_lo;
  a.r_valid_hi = k.r_hi;
  a.energy_stride = k.sweeps;
  a.fstats = c->fstats.as<unsigned long long>();
  *nsweep = 0;
  const bool per_launch_timing = k.timing && c->rows;
  size_t evk = 0;
  if (k.timing && !c->rows) CK(cudaEventRecordWithFlags(c->ev0, st, ev_flags), "event record");
  for (int32_t s = 1; s <= k.sweeps; ++s) {
    a.sweep = static_cast<uint32_t>(s);
    a.accumulate = avg && (s > k.sweeps - k.n_avg);
    a.energy = k.energy ? k.energy + (s - 1) : nullptr;
    if (k.dc_rc > 0) {  // DC on shared-memory tiles: one launch per tile parity (both colours)
      for (int tau = 0; tau < 2; ++tau) {
        launch_sweep_dc_tiles(a, c->gid.as<int32_t>(), c->phiK.as<float>(), c->T.as<float>(), c->Lx, c->Ly,
                              c->cfg.l_b, tau, k.dc_rc, st);
        CKL("sweep_dc_tiles");
        ++c->launches;
        ++*nsweep;
      }
      continue;
    }
    // SC: colour A then B (contiguous gap-id ranges); DC: (even tiles A, B), (odd tiles A, B)
    const int nphase = k.order == MPR_ORDER_DC ? 4 : 2;
    for (int ph = 0; ph < nphase; ++ph) {
      const int colour = ph & 1;
      a.is_b = colour;
      if (k.order == MPR_ORDER_DC) {
        a.glist = c->dclist.as<uint32_t>() + c->dc_off[ph];
        a.g_begin = 0;
        a.g_count = c->dc_off[ph + 1] - c->dc_off[ph];
        if (a.g_count > 0) {
          launch_sweep_half(a, c->sweep_grid, k.variant, st, c->sweep_waves);
          CKL("sweep_half");
          ++c->launches;
          ++*nsweep;
        }
        continue;
      }
      a.glist = nullptr;
      mpr_status sr = sc_half_sweep(c, a, colour, k.variant, per_launch_timing, ev_flags, &evk, nsweep);
      if (sr != MPR_OK) return sr;
    }
  }
  if (k.timing && !c->rows) CK(cudaEventRecordWithFlags(c->ev1, st, ev_flags), "event record");
  if (!k.defer) {
    // the realization sum over the own gap ids (one contiguous range unless row slabs)
    const float* X = avg ? c->A.as<float>() : c->G.as<float>();
    if (k.own[0][1] == k.own[1][0]) {
      launch_acc_reduce(X, k.own[0][0], k.own[1][1] - k.own[0][0], k.Rb, k.r_lo, k.r_hi, c->acc.as<double>(), st);
      CKL("acc_reduce");
      ++c->launches;
    } else {
      for (int col = 0; col < 2; ++col) {
        launch_acc_reduce(X, k.own[col][0], k.own[col][1] - k.own[col][0], k.Rb, k.r_lo, k.r_hi, c->acc.as<double>(),
                          st);
        CKL("acc_reduce");
        ++c->launches;
      }
    }
  }
  return MPR_OK;
}

mpr_status mpr_simulate_range(mpr_ctx* c, int64_t M, int32_t sweeps, uint64_t seed, int64_t m_begin,
                              int64_t m_end) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (c->stage < ST_PARAMS) return fail(c, MPR_ERR_STATE, "simulate before estimate_local_params");
  if (M < 1 || sweeps < 1) return fail(c, MPR_ERR_INVALID_ARG, "M and sweeps must be >= 1");
  if (c->cfg.n_avg > sweeps) return fail(c, MPR_ERR_INVALID_ARG, "n_avg must be <= sweeps");
  if (m_begin < 0 || m_end > M || m_begin > m_end) return fail(c, MPR_ERR_INVALID_ARG, "bad realization range");
  if (M >= (int64_t(1) << 32)) return fail(c, MPR_ERR_INVALID_ARG, "M too large");
  if (c->rows && c->defer_reduce) return fail(c, MPR_ERR_INVALID_ARG, "row slabs do not defer the reduction");
  if (!c->acc.p) {
    mpr_status s = mpr_reset_accumulator(c);
    if (s != MPR_OK) return s;
  }
  SET_DEVICE(c);
  cudaStream_t st = c->stream;
  c->M_total = M;
  c->sweeps = sweeps;
  c->launches = 0;
  c->m_begin = m_begin;
  c->m_end = m_end;
  const uint32_t k0 = static_cast<uint32_t>(seed & 0xffffffffu), k1 = static_cast<uint32_t>(seed >> 32);
  if (c->energy_enabled && c->cfg.order != MPR_ORDER_SC)
    return fail(c, MPR_ERR_INVALID_ARG, "the fused energy trace needs the SC order");
  if (c->energy_enabled) {
    if (c->energy_M != M || c->energy_S != sweeps) {
      CK(c->energy.ensure(sizeof(long long) * M * sweeps), "alloc energy");
      CK(cudaMemsetAsync(c->energy.p, 0, sizeof(long long) * M * sweeps, st), "zero energy");
      c->energy_M = M;
      c->energy_S = sweeps;
    }
  }
  if (c->degenerate || c->P_glob == 0 || m_begin == m_end) {
    c->stage = ST_SIM;
    return MPR_OK;
  }
  const int64_t mb0 = m_begin & ~int64_t(1);
  const int64_t R = choose_batch(c, m_end - mb0);
  if (c->defer_reduce && R < m_end - mb0)
    return fail(c, MPR_ERR_INVALID_ARG, "deferred reduce: the realization range must fit one batch");
  if (c->pending_reduce) return fail(c, MPR_ERR_STATE, "deferred states not accumulated yet");
  c->batch = R;
  const bool avg = c->cfg.n_avg > 1;
  CK(c->G.ensure(sizeof(float) * std::max<int64_t>(c->P, 1) * R), "alloc state");
  if (avg) CK(c->A.ensure(sizeof(float) * std::max<int64_t>(c->P, 1) * R), "alloc accumulator state");
  // row slabs capture their batches only with a stream-ordered transport, on request
  const bool graphs = c->use_graphs && (!c->rows || (c->comm->stream_ordered() && c->slab_graphs));
  for (int64_t mb = mb0; mb < m_end; mb += R) {
    const int64_t span = std::min<int64_t>(R, m_end - mb);
    const int Rb = static_cast<int>(span + (span & 1));
    const uint32_t pair_base = static_cast<uint32_t>(mb / 2);
    const int r_lo = static_cast<int>(std::max<int64_t>(m_begin - mb, 0));
    const int r_hi = static_cast<int>(std::min<int64_t>(m_end - mb, Rb));
    if (c->timing && !c->ev0) {
      CK(cudaEventCreate(&c->ev0), "event");
      CK(cudaEventCreate(&c->ev1), "event");
    }
    BatchKey key{};
    key.P = c->P; key.PA = c->PA; key.Rb = Rb; key.pair_base = pair_base; key.sweeps = sweeps;
    key.k0 = k0; key.k1 = k1; key.n_avg = c->cfg.n_avg; key.init = c->cfg.init; key.r_lo = r_lo; key.r_hi = r_hi;
    key.timing = c->timing; key.variant = c->sweep_variant; key.q = c->cfg.q; key.J = c->cfg.J;
    key.order = c->cfg.order;
    key.defer = c->defer_reduce;
    key.G = c->G.p; key.A = c->A.p; key.rec = c->rec.p; key.acc = c->acc.p;
    key.ginit = c->ginit.p; key.gid = c->gid.p; key.phiK = c->phiK.p; key.T = c->T.p;
    key.energy = c->energy_enabled ? c->energy.as<long long>() + mb * sweeps : nullptr;
    if (c->cfg.order == MPR_ORDER_DC) {
      key.dclist = c->dclist.p;
      for (int k = 0; k < 5; ++k) key.dc_off[k] = c->dc_off[k];
      key.dc_rc = c->dc_tiled ? dc_tile_chunk(c->cfg.l_b, Rb) : 0;
    }
    for (int col = 0; col < 2; ++col)
      for (int e = 0; e < 2; ++e) key.own[col][e] = c->own[col][e];
    int64_t nsweep_launch = 0;
    if (graphs) {
      cudaGraphExec_t exec = nullptr;
      for (auto& e : c->graphs)
        if (e.exec && std::memcmp(&e.key, &key, sizeof key) == 0) exec = e.exec;
      if (!exec) {
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
        const int64_t l0 = c->launches, t0 = c->total_launches;  // capture launches nothing
        mpr_status sb = issue_batch(c, key, &nsweep_launch, true);
        c->launches = l0;
        c->total_launches = t0;
        cudaGraph_t graph = nullptr;
        cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (sb != MPR_OK) { if (graph) cudaGraphDestroy(graph); return sb; }
        CK(ce, "end capture");
        ce = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(ce, "graph instantiate");
        GraphEntry& slot = c->graphs[c->graph_next++ % c->graphs.size()];
        if (slot.exec) cudaGraphExecDestroy(slot.exec);
        std::memcpy(&slot.key, &key, sizeof key);  // bytewise (padding included) for memcmp
        slot.exec = exec;
        slot.launches = nsweep_launch;
      } else {
        for (auto& e : c->graphs)
          if (e.exec == exec) nsweep_launch = e.launches;
      }
      CK(cudaGraphLaunch(exec, st), "graph launch");
      const int64_t nacc = key.defer ? 0 : (key.own[0][1] == key.own[1][0] ? 1 : 2);
      c->launches += nsweep_launch + 1 + nacc;
      c->total_launches += nsweep_launch + 1 + nacc;
    } else {
      mpr_status sb = issue_batch(c, key, &nsweep_launch, false);
      if (sb != MPR_OK) return sb;
    }
    if (c->timing) {
      if (!c->rows) {
        CK(cudaEventSynchronize(c->ev1), "event sync");
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event elapsed");
        c->sweep_ms += ms;
      } else {
        CK(cudaStreamSynchronize(st), "timing sync");
        for (int64_t k = 0; k < nsweep_launch; ++k) {
          float ms = 0.0f;
          CK(cudaEventElapsedTime(&ms, c->ev_pool[2 * k], c->ev_pool[2 * k + 1]), "event elapsed");
          c->sweep_ms += ms;
        }
      }
      c->sweep_launches += nsweep_launch;
    }
    c->last_m_base = mb;
    c->last_R = Rb;
    if (key.defer) {
      c->pending_reduce = 1;
      c->pending_Rb = Rb;
      c->pending_r_lo = r_lo;
      c->pending_r_hi = r_hi;
    }
  }
  CK(cudaStreamSynchronize(st), "simulate sync");
  c->stage = ST_SIM;
  return MPR_OK;
}

mpr_status mpr_set_deferred_reduce(mpr_ctx* c, int enable) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (c->pending_reduce) return fail(c, MPR_ERR_STATE, "deferred states not accumulated yet");
  c->defer_reduce = enable ? 1 : 0;
  return MPR_OK;
}

mpr_status mpr_accumulate_states(mpr_ctx* c) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (!c->pending_reduce) return fail(c, MPR_ERR_STATE, "no deferred states (simulate_range with deferred reduce)");
  SET_DEVICE(c);
  const bool avg = c->cfg.n_avg > 1;
  launch_acc_reduce(avg ? c->A.as<float>() : c->G.as<float>(), 0, c->P, c->pending_Rb, c->pending_r_lo,
                    c->pending_r_hi, c->acc.as<double>(), c->stream);
  CKL("acc_reduce");
  c->pending_reduce = 0;
  CK(cudaStreamSynchronize(c->stream), "accumulate sync");
  return MPR_OK;
}

// Realization shards: this rank's range, then the sum over ranks — one
// all-reduce of the fp64 accumulator, or the rank-ordered chain (bit-identical to one GPU).
static mpr_status simulate_realization_shards(mpr_ctx* c, int64_t M, int32_t sweeps, uint64_t seed) {
  int64_t m0 = 0, m1 = 0;
  shard_range(M, c->world, c->rank, &m0, &m1);
  cudaStream_t st = c->stream;
  const size_t nP = static_cast<size_t>(std::max<int64_t>(c->P, 1));
  double* acc = c->acc.as<double>();
  mpr_status s = MPR_OK;
  if (c->cfg.ordered_reduce) {
    const int prev = c->defer_reduce;
    c->defer_reduce = 1;
    s = mpr_simulate_range(c, M, sweeps, seed, m0, m1);
    c->defer_reduce = prev;
    if (s != MPR_OK) return s;
    SET_DEVICE(c);
    if (c->rank > 0) CKC(c->comm->exchange({}, {{c->rank - 1, acc, nP}}, CT_F64, st), "ordered reduce recv");
    if (c->pending_reduce) {
      s = mpr_accumulate_states(c);
      if (s != MPR_OK) return s;
    }
    if (c->rank < c->world - 1) CKC(c->comm->exchange({{c->rank + 1, acc, nP}}, {}, CT_F64, st), "ordered reduce send");
    CKC(c->comm->broadcast(acc, nP, CT_F64, c->world - 1, st), "ordered reduce broadcast");
  } else {
    s = mpr_simulate_range(c, M, sweeps, seed, m0, m1);
    if (s != MPR_OK) return s;
    SET_DEVICE(c);
    CKC(c->comm->allreduce(acc, nP, CT_F64, OP_SUM, st), "allreduce accumulator");
  }
  CK(cudaStreamSynchronize(st), "shard reduce sync");
  c->m_begin = m0;
  c->m_end = m1;
  c->M_total = M;
  return MPR_OK;
}

mpr_status mpr_simulate(mpr_ctx* c, int64_t M, int32_t sweeps, uint64_t seed) {
  mpr_status s = mpr_reset_accumulator(c);
  if (s != MPR_OK) return s;
  if (c->shards) {
    if (M < 1 || sweeps < 1) return fail(c, MPR_ERR_INVALID_ARG, "M and sweeps must be >= 1");
    s = simulate_realization_shards(c, M, sweeps, seed);
  } else {
    s = mpr_simulate_range(c, M, sweeps, seed, 0, M);
  }
  if (s != MPR_OK) return s;
  // the energy trace: every rank summed its own sites (row slabs) or realizations (shards)
  if ((c->rows || c->shards) && c->energy_enabled && c->energy_M > 0) {
    SET_DEVICE(c);
    CKC(c->comm->allreduce(c->energy.p, static_cast<size_t>(c->energy_M * c->energy_S), CT_I64, OP_SUM, c->stream),
        "allreduce energy");
    CK(cudaStreamSynchronize(c->stream), "energy sync");
  }
  return MPR_OK;
}

// Row f1 (ARITH §K): every realization sweeps until its energy trace passes
// the slope test at a check sweep, then averages n_avg more sweeps. The sweeps run on the
// device for the whole batch; at check sweeps the host reads the fixed-point energies,
// decides, and uploads the per-realization accumulation windows. Realization shards: each
// rank runs its range; the accumulators and s_eq are summed over the ranks.
mpr_status mpr_simulate_adaptive(mpr_ctx* c, int64_t M, uint64_t seed, int32_t n_fit, int32_t n_f,
                                 int32_t max_sweeps, double slope_tol, int32_t* s_eq_out) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (!std::isfinite(slope_tol)) return fail(c, MPR_ERR_INVALID_ARG, "slope_tol must be finite");
  if (c->stage < ST_PARAMS) return fail(c, MPR_ERR_STATE, "simulate before estimate_local_params");
  const int n_avg = c->cfg.n_avg;
  if (M < 1 || n_fit < 3 || n_f < 1 || max_sweeps < n_avg + 1 || M >= (int64_t(1) << 32))
    return fail(c, MPR_ERR_INVALID_ARG, "need M >= 1, n_fit >= 3, n_f >= 1, max_sweeps > n_avg");
  // slope_tol < 0: the tolerance derived from the sample energy's standard error (R22)
  if (slope_tol < 0.0) slope_tol = derived_slope_tol(c->sum_SB_fx, c->sum_SB2_fx, c->n_sample_bonds, n_fit);
  c->last_slope_tol = slope_tol;
  if (c->cfg.order != MPR_ORDER_SC)
    return fail(c, MPR_ERR_INVALID_ARG, "the adaptive protocol needs the SC order (fused energy)");
  mpr_status st0 = mpr_reset_accumulator(c);
  if (st0 != MPR_OK) return st0;
  SET_DEVICE(c);
  cudaStream_t st = c->stream;
  c->M_total = M;
  c->sweeps = max_sweeps;
  c->launches = 0;
  int64_t m0 = 0, m1 = M;
  const bool sharded = c->shards;
  if (sharded) shard_range(M, c->world, c->rank, &m0, &m1);
  c->m_begin = m0;
  c->m_end = m1;
  if (c->degenerate || c->P == 0) {
    if (s_eq_out)
      for (int64_t m = 0; m < M; ++m) s_eq_out[m] = 0;
    c->stage = ST_SIM;
    return MPR_OK;
  }
  std::vector<int32_t> s_eq_all(static_cast<size_t>(sharded ? M : 0), 0);
  const uint32_t k0 = static_cast<uint32_t>(seed & 0xffffffffu), k1 = static_cast<uint32_t>(seed >> 32);
  const int64_t R = choose_batch(c, std::max<int64_t>(m1 - m0, 2));
  CK(c->G.ensure(sizeof(float) * c->P * R), "alloc state");
  CK(c->A.ensure(sizeof(float) * c->P * R), "alloc accumulator state");
  // row slabs: every rank's kernels sum the bonds of its own sites (a partial energy); the
  // check reads the sum over the ranks, re-formed from the partials before each check
  CK(c->energy.ensure(sizeof(long long) * R * max_sweeps * (c->rows ? 2 : 1)), "alloc energy");
  long long* e_part = c->energy.as<long long>();
  long long* e_glob = c->rows ? e_part + R * max_sweeps : e_part;
  CK(c->win.ensure(sizeof(int) * 2 * R), "alloc windows");
  // Decisions are taken on the device (k_adaptive_check, ARITH §K bit for bit), so the host
  // never stalls the GPU for a check: it reads the device status (undecided count, last
  // window end) one check late from pinned memory, while the next n_f sweeps are already
  // queued. Sweeps issued after every realization finished are no-ops (frozen pairs).
  CK(c->tmp.ensure(sizeof(int) * (R + 2)), "alloc decisions");
  int* eq_d = c->tmp.as<int>();
  int* status_d = eq_d + R;
  int* hbuf = nullptr;  // pinned: [0, 2*R) windows; [2R, 2R+2) status; [2R+2, 3R+2) decisions
  CK(cudaMallocHost(reinterpret_cast<void**>(&hbuf), sizeof(int) * (3 * R + 2)), "pinned staging");
  struct PinnedFree {
    void* p;
    ~PinnedFree() { if (p) cudaFreeHost(p); }
  } hbuf_free{hbuf};
  int* win = hbuf;
  volatile int* status_h = hbuf + 2 * R;
  int* eq_h = hbuf + 2 * R + 2;
  if (!c->ev_check) CK(cudaEventCreateWithFlags(&c->ev_check, cudaEventDisableTiming), "event");
  for (int64_t mb = m0; mb < m1; mb += R) {
    const int64_t span = std::min<int64_t>(R, m1 - mb);
    const int Rb = static_cast<int>(span + (span & 1));
    const int r_hi = static_cast<int>(span);
    // windows: (lo, hi] accumulates; hi = INT_MAX while undecided; the pad realization
    // (odd M) is "done" from the start
    for (int r = 0; r < Rb; ++r) {
      win[r] = r < r_hi ? INT32_MAX : 0;
      win[Rb + r] = r < r_hi ? INT32_MAX : 0;
    }
    status_h[0] = r_hi;
    status_h[1] = 0;
    CK(cudaMemcpyAsync(c->win.p, win, sizeof(int) * 2 * Rb, cudaMemcpyHostToDevice, st), "H2D windows");
    CK(cudaMemcpyAsync(status_d, const_cast<int*>(status_h), sizeof(int) * 2, cudaMemcpyHostToDevice, st),
       "H2D status");
    CK(cudaMemsetAsync(eq_d, 0, sizeof(int) * Rb, st), "zero decisions");
    CK(cudaMemsetAsync(e_part, 0, sizeof(long long) * Rb * max_sweeps, st), "zero energy");
    CK(cudaStreamSynchronize(st), "adaptive batch start");  // the pinned windows are reused below
    launch_init_states(c->rec.as<GapRec>(), c->ginit.as<float>(), c->G.as<float>(), c->A.as<float>(), c->P, Rb, Rb / 2,
                       static_cast<uint32_t>(mb / 2), c->cfg.init == MPR_INIT_RANDOM, k0, k1, st);
    CKL("init_states");
    ++c->launches;
    SweepArgs a{};
    a.rec = c->rec.as<GapRec>();
    a.G = c->G.as<float>();
    a.P = c->P;
    a.A = c->A.as<float>();
    a.R = Rb;
    a.npairs = Rb / 2;
    a.pair_base = static_cast<uint32_t>(mb / 2);
    a.k0 = k0;
    a.k1 = k1;
    a.q = c->cfg.q;
    a.J = c->cfg.J;
    a.fstats = c->fstats.as<unsigned long long>();
    a.win_lo = c->win.as<int>();
    a.win_hi = c->win.as<int>() + Rb;
    a.energy_stride = max_sweeps;
    a.r_valid_lo = 0;
    a.r_valid_hi = r_hi;
    AdaptiveCheckArgs ca{};
    ca.energy = e_glob;
    ca.energy_stride = max_sweeps;
    ca.sum_known_fx = c->sum_SB_fx;
    ca.n_bonds = static_cast<double>(2 * c->Lx * c->Ly - c->Lx - c->Ly);
    ca.n_fit = n_fit;
    ca.n_avg = n_avg;
    ca.r_hi = r_hi;
    ca.slope_tol = slope_tol;
    ca.win_lo = c->win.as<int>();
    ca.win_hi = c->win.as<int>() + Rb;
    ca.eq = eq_d;
    ca.status = status_d;
    bool status_pending = false;  // a status copy is in flight behind ev_check
    int stop_all = INT32_MAX;     // known once the device reports no undecided realization
    for (int32_t s = 1; s <= max_sweeps && s <= stop_all; ++s) {
      a.sweep = static_cast<uint32_t>(s);
      a.energy = e_part + (s - 1);
      for (int colour = 0; colour < 2; ++colour) {
        size_t evk = 0;
        mpr_status sr = sc_half_sweep(c, a, colour, c->sweep_variant, false, 0u, &evk, nullptr);
        if (sr != MPR_OK) return sr;
      }
      const bool check = s >= n_fit + n_f && (s - n_fit) % n_f == 0 && s + n_avg <= max_sweeps;
      const bool forced = s == max_sweeps - n_avg;
      if (check || forced) {
        // the previous check's status: its copy was issued n_f sweeps ago, so waiting for it
        // leaves n_f sweeps of queued work on the GPU (no bubble) and bounds how far the
        // host runs ahead of the decisions (at most n_f no-op sweeps after the last one)
        if (status_pending) {
          CK(cudaEventSynchronize(c->ev_check), "status wait");
          status_pending = false;
          if (status_h[0] == 0) stop_all = status_h[1];
        }
        if (stop_all != INT32_MAX) continue;
        if (c->rows) {  // the whole-grid energies of every realization so far (exact int64 sums)
          CK(cudaMemcpyAsync(e_glob, e_part, sizeof(long long) * Rb * max_sweeps, cudaMemcpyDeviceToDevice, st),
             "copy energies");
          CKC(c->comm->allreduce(e_glob, static_cast<size_t>(Rb) * max_sweeps, CT_I64, OP_SUM, st), "allreduce energies");
        }
        ca.s = s;
        ca.check = check;
        ca.forced = forced;
        launch_adaptive_check(ca, st);
        CKL("adaptive_check");
        ++c->launches;
        if (!status_pending) {
          CK(cudaMemcpyAsync(const_cast<int*>(status_h), status_d, sizeof(int) * 2, cudaMemcpyDeviceToHost, st),
             "D2H status");
          CK(cudaEventRecord(c->ev_check, st), "event record");
          status_pending = true;
        }
      }
    }
    CK(cudaMemcpyAsync(eq_h, eq_d, sizeof(int) * Rb, cudaMemcpyDeviceToHost, st), "D2H decisions");
    for (int col = 0; col < 2; ++col) {  // the own gap ids (one range unless row slabs)
      const int64_t g0 = col == 0 ? c->own[0][0] : c->own[1][0];
      const int64_t g1 = (col == 0 && c->own[0][1] == c->own[1][0]) ? c->own[1][1] : c->own[col][1];
      launch_acc_reduce(c->A.as<float>(), g0, g1 - g0, Rb, 0, r_hi, c->acc.as<double>(), st);
      CKL("acc_reduce");
      ++c->launches;
      if (c->own[0][1] == c->own[1][0]) break;
    }
    CK(cudaStreamSynchronize(st), "adaptive sync");
    for (int r = 0; r < r_hi; ++r) {
      if (sharded) s_eq_all[static_cast<size_t>(mb + r)] = eq_h[r];
      else if (s_eq_out) s_eq_out[mb + r] = eq_h[r];
    }
    c->last_m_base = mb;
    c->last_R = Rb;
  }
  if (sharded) {  // accumulators and decisions of every rank (zeros outside a rank's range)
    CKC(c->comm->allreduce(c->acc.p, static_cast<size_t>(c->P), CT_F64, OP_SUM, st), "allreduce accumulator");
    CK(c->tmp.ensure(sizeof(int32_t) * static_cast<size_t>(M)), "alloc s_eq");
    CK(cudaMemcpyAsync(c->tmp.p, s_eq_all.data(), sizeof(int32_t) * M, cudaMemcpyHostToDevice, st), "H2D s_eq");
    CKC(c->comm->allreduce(c->tmp.p, static_cast<size_t>(M), CT_I32, OP_SUM, st), "allreduce s_eq");
    CK(cudaMemcpyAsync(s_eq_all.data(), c->tmp.p, sizeof(int32_t) * M, cudaMemcpyDeviceToHost, st), "D2H s_eq");
    CK(cudaStreamSynchronize(st), "adaptive reduce sync");
    if (s_eq_out) std::memcpy(s_eq_out, s_eq_all.data(), sizeof(int32_t) * M);
  }
  c->batch = R;
  c->stage = ST_SIM;
  return MPR_OK;
}

mpr_status mpr_sync(mpr_ctx* c) {
  if (!c) return MPR_ERR_INVALID_ARG;
  SET_DEVICE(c);
  CK(cudaStreamSynchronize(c->stream), "sync");
  return MPR_OK;
}

mpr_status mpr_build_calibration(mpr_ctx* c, const float* T, int32_t K, int32_t L, float q, int32_t n_eq,
                                 int32_t n_meas, int32_t reps, uint64_t seed, float* e_out, double* e_raw_out) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (!T || !e_out || K < 2 || L < 2 || n_eq < 0 || n_meas < 1 || reps < 1 || !(q > 0.0f && q <= 0.5f))
    return fail(c, MPR_ERR_INVALID_ARG, "bad calibration arguments");
  for (int k = 0; k < K; ++k)
    if (!(T[k] > 0.0f) || !std::isfinite(T[k]) || (k > 0 && !(T[k] > T[k - 1])))
      return fail(c, MPR_ERR_INVALID_ARG, "calibration temperatures must be positive and increasing");
  SET_DEVICE(c);
  const int nlat = K * reps, S = n_eq + n_meas;
  std::vector<long long> fx(static_cast<size_t>(nlat) * S);
  CK(run_calibration(T, K, L, q, n_eq, n_meas, reps, seed, fx.data(), c->stream), "calibration sweeps");
  // mean energy of each lattice over the measurement sweeps, then over replicas (fp64,
  // in sweep / replica order)
  const double nb = static_cast<double>(2 * static_cast<int64_t>(L) * L - L - L);
  std::vector<double> raw(static_cast<size_t>(K));
  for (int k = 0; k < K; ++k) {
    double rsum = 0.0;
    for (int r = 0; r < reps; ++r) {
      double sum = 0.0;
      for (int s = n_eq + 1; s <= S; ++s) {
        const long long E = fx[static_cast<size_t>(s - 1) * nlat + k * reps + r];
        sum = sum + (-static_cast<double>(E) * 0x1p-32) / nb;
      }
      rsum = rsum + sum / static_cast<double>(n_meas);
    }
    raw[k] = rsum / static_cast<double>(reps);
  }
  // pool adjacent violators (non-decreasing), then strictly increasing in fp32
  std::vector<double> val, wt;
  std::vector<int> len;
  for (int k = 0; k < K; ++k) {
    val.push_back(raw[k]);
    wt.push_back(1.0);
    len.push_back(1);
    while (val.size() > 1 && val[val.size() - 2] > val.back()) {
      const double v2 = val.back(), w2 = wt.back();
      const int l2 = len.back();
      val.pop_back(); wt.pop_back(); len.pop_back();
      const double v1 = val.back(), w1 = wt.back();
      const int l1 = len.back();
      val.pop_back(); wt.pop_back(); len.pop_back();
      val.push_back((v1 * w1 + v2 * w2) / (w1 + w2));
      wt.push_back(w1 + w2);
      len.push_back(l1 + l2);
    }
  }
  int k = 0;
  for (size_t b = 0; b < val.size(); ++b)
    for (int t = 0; t < len[b]; ++t) e_out[k++] = static_cast<float>(val[b]);
  for (k = 1; k < K; ++k)
    if (e_out[k] <= e_out[k - 1]) e_out[k] = std::nextafter(e_out[k - 1], 1.0f);
  if (e_raw_out)
    for (k = 0; k < K; ++k) e_raw_out[k] = raw[k];
  return MPR_OK;
}

mpr_status mpr_accumulator_device(mpr_ctx* c, double** acc_dev, int64_t* n) {
  if (!c || !acc_dev || !n) return MPR_ERR_INVALID_ARG;
  if (c->stage < ST_PARAMS || !c->acc.p) return fail(c, MPR_ERR_STATE, "no accumulator yet");
  *acc_dev = c->acc.as<double>();
  *n = c->P;
  return MPR_OK;
}

// a11 over the own rows into out_rows_dev ((row1 - row0) x Lx floats).
static mpr_status predict_own_rows(mpr_ctx* c, float* out_rows_dev) {
  if (c->stage < ST_SIM || c->M_total < 1) return fail(c, MPR_ERR_STATE, "predict before simulate");
  const double denom = static_cast<double>(c->M_total * static_cast<int64_t>(c->cfg.n_avg));
  launch_predict(local_row(c, c->z.as<float>(), c->row0), local_row(c, c->mask.as<uint8_t>(), c->row0),
                 local_row(c, c->gid.as<int32_t>(), c->row0), c->acc.as<double>(), (c->row1 - c->row0) * c->Lx, denom,
                 c->scal.as<DevScalars>(), c->degenerate, out_rows_dev, c->stream);
  CKL("predict");
  return MPR_OK;
}

// The whole prediction into out_dev (Lx*Ly floats): row slabs all-gather their rows.
static mpr_status predict_all(mpr_ctx* c, float* out_dev) {
  mpr_status s = predict_own_rows(c, out_dev + c->row0 * c->Lx);
  if (s != MPR_OK || !c->rows) return s;
  std::vector<size_t> counts(static_cast<size_t>(c->world)), displs(static_cast<size_t>(c->world));
  for (int w = 0; w < c->world; ++w) {
    int64_t r0 = 0, r1 = 0;
    row_range(c->Ly, c->world, w, &r0, &r1);
    counts[static_cast<size_t>(w)] = static_cast<size_t>((r1 - r0) * c->Lx);
    displs[static_cast<size_t>(w)] = static_cast<size_t>(r0 * c->Lx);
  }
  CKC(c->comm->allgatherv(out_dev + c->row0 * c->Lx, out_dev, counts, displs, CT_F32, c->stream),
      "allgather predictions");
  return MPR_OK;
}

mpr_status mpr_predict(mpr_ctx* c, float* out) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (!out) return fail(c, MPR_ERR_INVALID_ARG, "out is NULL");
  SET_DEVICE(c);
  const int64_t total = c->Lx * c->Ly;
  CK(c->out.ensure(sizeof(float) * total), "alloc out");
  mpr_status s = predict_all(c, c->out.as<float>());
  if (s != MPR_OK) return s;
  CK(cudaMemcpyAsync(out, c->out.p, sizeof(float) * total, cudaMemcpyDeviceToHost, c->stream), "D2H out");
  CK(cudaStreamSynchronize(c->stream), "predict sync");
  return MPR_OK;
}

mpr_status mpr_predict_device(mpr_ctx* c, float* out_dev) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (!out_dev) return fail(c, MPR_ERR_INVALID_ARG, "out is NULL");
  SET_DEVICE(c);
  mpr_status s = predict_all(c, out_dev);
  if (s != MPR_OK) return s;
  CK(cudaStreamSynchronize(c->stream), "predict sync");
  return MPR_OK;
}

mpr_status mpr_predict_rows(mpr_ctx* c, float* out_rows) {
  if (!c) return MPR_ERR_INVALID_ARG;
  if (!out_rows) return fail(c, MPR_ERR_INVALID_ARG, "out is NULL");
  SET_DEVICE(c);
  const int64_t cnt = (c->row1 - c->row0) * c->Lx;
  CK(c->out.ensure(sizeof(float) * std::max<int64_t>(cnt, 1)), "alloc out");
  mpr_status s = predict_own_rows(c, c->out.as<float>());
  if (s != MPR_OK) return s;
  CK(cudaMemcpyAsync(out_rows, c->out.p, sizeof(float) * cnt, cudaMemcpyDeviceToHost, c->stream), "D2H out");
  CK(cudaStreamSynchronize(c->stream), "predict sync");
  return MPR_OK;
}

mpr_status mpr_get_info(mpr_ctx* c, mpr_info* info) {
  if (!c || !info) return MPR_ERR_INVALID_ARG;
  std::memset(info, 0, sizeof(*info));
  info->Lx = c->Lx;
  info->Ly = c->Ly;
  info->n_samples = c->n_known;
  info->n_gaps = c->P_glob;
  info->n_gaps_a = c->PA_glob;
  info->z_min = c->zmin;
  info->z_max = c->zmax;
  info->degenerate_range = c->degenerate;
  info->n_blocks = c->nblocks;
  info->n_blocks_fallback = c->n_fallback;
  info->median_T = c->median_T;
  info->M = c->M_total;
  info->sweeps = c->sweeps;
  info->batch = c->batch;
  info->kernel_launches = c->launches;
  info->total_launches = c->total_launches;
  info->sweep_launches = c->sweep_launches;
  info->sweep_ms = c->sweep_ms;
  info->last_m_base = c->last_m_base;
  info->last_batch = c->last_R;
  info->sweep_variant = c->sweep_variant;
  info->rank = c->rank;
  info->world = c->world;
  info->shard = c->cfg.shard;
  info->row_begin = c->row0;
  info->row_end = c->row1;
  info->m_begin = c->m_begin;
  info->m_end = c->m_end;
  info->n_gaps_local = c->P;
  info->comm_calls = c->comm_calls;
  info->slope_tol = c->last_slope_tol;
  info->sample_bonds = c->n_sample_bonds;
  info->filter_exact_pairs = info->filter_pairs = -1;
  if (c->fstats.p) {
    unsigned long long h[2] = {0, 0};
    CK(cudaStreamSynchronize(c->stream), "filter stats sync");
    CK(cudaMemcpy(h, c->fstats.p, sizeof(h), cudaMemcpyDeviceToHost), "filter stats");
    info->filter_exact_pairs = static_cast<int64_t>(h[0]);
    info->filter_pairs = static_cast<int64_t>(h[1]);
  }
  return MPR_OK;
}

mpr_status mpr_debug_get(mpr_ctx* c, mpr_buffer which, int64_t index, void* host_out) {
  if (!c || !host_out) return MPR_ERR_INVALID_ARG;
  SET_DEVICE(c);
  cudaStream_t st = c->stream;
  // the Lx*Ly buffers: the own rows, at their offsets of the (whole-grid) host buffer
  const int64_t own = (c->row1 - c->row0) * c->Lx, hoff = c->row0 * c->Lx;
  switch (which) {
    case MPR_BUF_PHI_KNOWN:
      if (c->stage < ST_DATA) return fail(c, MPR_ERR_STATE, "no data");
      CK(cudaMemcpyAsync(static_cast<float*>(host_out) + hoff, local_row(c, c->phiK.as<float>(), c->row0),
                         sizeof(float) * own, cudaMemcpyDeviceToHost, st), "D2H");
      break;
    case MPR_BUF_T:
      if (c->stage < ST_PARAMS) return fail(c, MPR_ERR_STATE, "no parameters");
      CK(cudaMemcpyAsync(static_cast<float*>(host_out) + hoff, c->T.as<float>() + (c->row0 - c->trow0) * c->Lx,
                         sizeof(float) * own, cudaMemcpyDeviceToHost, st), "D2H");
      break;
    case MPR_BUF_BLOCK_T:
      if (c->stage < ST_PARAMS) return fail(c, MPR_ERR_STATE, "no parameters");
      CK(cudaMemcpyAsync(host_out, c->Tb.p, sizeof(float) * c->nblocks, cudaMemcpyDeviceToHost, st), "D2H");
      break;
    case MPR_BUF_BLOCK_STATS:
      if (c->stage < ST_PARAMS) return fail(c, MPR_ERR_STATE, "no parameters");
      CK(cudaMemcpyAsync(host_out, c->bstats.p, sizeof(long long) * 4 * c->nblocks, cudaMemcpyDeviceToHost, st),
         "D2H");
      break;
    case MPR_BUF_STATE: {
      if (c->stage < ST_SIM || !c->G.p || c->last_R == 0) return fail(c, MPR_ERR_STATE, "no state");
      const int64_t r = index - c->last_m_base;
      if (r < 0 || r >= c->last_R) return fail(c, MPR_ERR_INVALID_ARG, "realization not in the last batch");
      CK(c->tmp.ensure(sizeof(double) * std::max<int64_t>(own, 1)), "alloc tmp");
      launch_scatter_state(local_row(c, c->phiK.as<float>(), c->row0), local_row(c, c->gid.as<int32_t>(), c->row0),
                           c->G.as<float>(), c->last_R, r, own, c->tmp.as<float>(), st);
      CKL("scatter_state");
      CK(cudaMemcpyAsync(static_cast<float*>(host_out) + hoff, c->tmp.p, sizeof(float) * own, cudaMemcpyDeviceToHost,
                         st), "D2H");
      break;
    }
    case MPR_BUF_ACC:
      if (c->stage < ST_PARAMS || !c->acc.p) return fail(c, MPR_ERR_STATE, "no accumulator");
      CK(c->tmp.ensure(sizeof(double) * std::max<int64_t>(own, 1)), "alloc tmp");
      launch_scatter_acc(local_row(c, c->gid.as<int32_t>(), c->row0), c->acc.as<double>(), own, c->tmp.as<double>(),
                         st);
      CKL("scatter_acc");
      CK(cudaMemcpyAsync(static_cast<double*>(host_out) + hoff, c->tmp.p, sizeof(double) * own,
                         cudaMemcpyDeviceToHost, st), "D2H");
      break;
    case MPR_BUF_ENERGY: {
      if (!c->energy_enabled || c->energy_M == 0) return fail(c, MPR_ERR_STATE, "energy trace not enabled");
      const int64_t cnt = c->energy_M * c->energy_S;
      // the int64 fixed-point sums have the size of the doubles they become: copy in place
      CK(cudaMemcpyAsync(host_out, c->energy.p, sizeof(long long) * cnt, cudaMemcpyDeviceToHost, st), "D2H");
      CK(cudaStreamSynchronize(st), "debug sync");
      long long* fx = static_cast<long long*>(host_out);
      double* e = static_cast<double*>(host_out);
      for (int64_t k = 0; k < cnt; ++k) e[k] = energy_from_fx(c, c->sum_SB_fx + fx[k]);
      return MPR_OK;
    }
    default:
      return fail(c, MPR_ERR_INVALID_ARG, "unknown buffer");
  }
  CK(cudaStreamSynchronize(st), "debug sync");
  return MPR_OK;
}

}  // extern "C"
