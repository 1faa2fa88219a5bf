/*
 * mpr.h — C-ABI of libmpr.so, the B200 (sm_100a) LE-MPR gap filler.
 *
 * Method: Lach & Zukovic, "Fast gap-filling of massive data by local-equilibrium
 * conditional simulations on GPU", arXiv 2212.01317. The library runs
 * the paper's SV-MPR hot path (the north star's "LE-MPR"): data -> spin transform
 * (PAPER.md:85), block sample energies and energy-matched block temperatures with
 * the median fallback (Eq.(2)), SST smoothing
 * (PAPER.md:124), conditional checkerboard Metropolis over the gap sites with the
 * samples frozen, and the back-transformed conditional mean
 * (PAPER.md:95). MPR (uniform T) is l_b >= max(Lx, Ly); BST is n_s = 0.
 * Every floating-point step that feeds a decision follows docs/ARITH.md.
 *
 * Conventions shared by every call:
 *  - Grids are row-major, Ly rows x Lx columns, element (r, c) at index r*Lx + c.
 *  - mask[i] != 0 marks a known sample (the set G_S of PAPER.md:80); mask[i] == 0 a
 *    gap (G_P). grid[i] at a gap is never read (it may be NaN).
 *  - Host pointers are borrowed for the duration of the call only; the library
 *    copies in and out and never frees caller memory. Device pointers ("_device"
 *    variants) must be device memory of ctx's device, valid until the call returns
 *    on the host (all work is stream-ordered on the context stream and the calls
 *    synchronise that stream before returning unless stated otherwise).
 *  - Call order: mpr_init -> mpr_set_data -> mpr_estimate_local_params ->
 *    mpr_simulate (or mpr_simulate_range, any number of times) -> mpr_predict.
 *    Re-calling an earlier stage invalidates the later ones; out-of-order calls
 *    return MPR_ERR_STATE.
 *  - Every call returns a status; on failure mpr_last_error(ctx) holds one line.
 *  - A context is single-owner (not thread-safe); distinct contexts are independent
 *    and may be driven concurrently from different host threads.
 *  - Each call makes ctx's device current while it runs and restores the calling
 *    thread's current device before returning.
 */
#ifndef MPR_H_
#define MPR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpr_ctx mpr_ctx;
typedef struct mpr_group mpr_group;  /* in-process communicator (mpr_group_create)      */

typedef enum {
  MPR_OK = 0,
  MPR_ERR_INVALID_ARG = 1,      /* bad size, parameter, table or non-finite sample   */
  MPR_ERR_STATE = 2,            /* call out of order                                 */
  MPR_ERR_TOO_FEW_SAMPLES = 3,  /* fewer than 2 known sites                          */
  MPR_ERR_NO_SAMPLE_BONDS = 4,  /* no block has a sample-sample bond  */
  MPR_ERR_CUDA = 5,             /* a CUDA runtime error; message in mpr_last_error   */
  MPR_ERR_OOM = 6,              /* device allocation failed                          */
  MPR_ERR_NCCL = 7              /* an NCCL call failed (or libnccl.so.2 is missing)  */
} mpr_status;

typedef enum { MPR_INIT_BLOCK_MEAN = 0, MPR_INIT_RANDOM = 1 } mpr_init_mode;

/* How a multi-rank context splits the work (the paper itself is single-GPU,
 * PAPER.md:192). With a communicator (nccl_comm or group) every rank makes the same calls
 * with the same arguments (SPMD):
 *  MPR_SHARD_REALIZATIONS: every rank holds the whole problem and computes the (exact,
 *    deterministic) parameter stage itself; mpr_simulate runs the rank's contiguous,
 *    pair-aligned range of the global realization ids (rank w of W: pairs
 *    [w*ceil(M/2)/W, (w+1)*ceil(M/2)/W)) and sums the fp64 accumulators with one
 *    all-reduce (or the rank-ordered chain when ordered_reduce = 1: bit-identical to one
 *    GPU). Weak or strong scaling over independent chains.
 *  MPR_SHARD_ROWS: the grid is split into row slabs, rank w owning rows
 *    [w*Ly/W, (w+1)*Ly/W); a rank's device memory holds only its rows plus one ghost row
 *    per side (and max(r_s*n_s, 1) rows of temperature halo), so grids larger than one
 *    GPU fit. The parameter stage is distributed and exact: (z_min, z_max) and counts by
 *    all-reduce, the ghost rows of z / mask by neighbour exchange (cross-slab bonds), the
 *    block sums (ARITH §E, exact int64) by all-reduce so every rank holds every T_b and
 *    takes the same lower median, the smoothing halo recomputed locally from T_b. Every
 *    colour half-sweep is followed by the exchange of the colour's boundary-row states
 *    with the two neighbours (stream ordered with NCCL: no host synchronisation). The
 *    chains are bit-identical to one GPU (global (site, sweep, realization) Philox
 *    counters). */
typedef enum { MPR_SHARD_REALIZATIONS = 0, MPR_SHARD_ROWS = 1 } mpr_shard;

typedef struct {
  int device;        /* CUDA device ordinal                                           */
  void *stream;      /* cudaStream_t to run on (e.g. torch's current stream); NULL =>
                        the library creates its own non-blocking stream                */
  float J;           /* coupling J > 0 of Eq.(1); default 1           */
  float q;           /* modification parameter, 0 < q <= 1/2; default .5 */
  int l_b;           /* block side (l_b = 32 in Table 2); >= 2            */
  int r_s;           /* smoothing radius (unstated; R8); >= 0   */
  int n_s;           /* smoothing passes (n_s = 5); 0 => BST              */
  int init;          /* mpr_init_mode                                   */
  int n_avg;         /* sweeps averaged at the end of each realization (>= 1)          */
  const float *calib_T;  /* calibration table T_k, strictly increasing, 0 < T <= 1e4;
                            with n_s > 0 also T_max * (2 r_s + 1)^2 < 2^23 (ARITH §E)  */
  const float *calib_e;  /* e_k = e(T_k), strictly increasing (host pointers, copied)  */
  int calib_n;           /* K >= 2                                                     */
  int64_t max_batch;     /* max realizations simulated concurrently (0 => automatic)  */
  int order;             /* mpr_order: update order of a sweep (ARITH §H)              */
  /* ---- multi-rank; all zero => one GPU ---------------------- */
  void *nccl_comm;       /* ncclComm_t of this rank (made with mpr_nccl_comm_init, so it
                            belongs to the process's libnccl.so.2); not owned. Its device
                            must be cfg.device. NULL => no NCCL                          */
  mpr_group *group;      /* in-process communicator instead of NCCL (W contexts of one
                            process, each driven by its own host thread; host-synchronous
                            collectives); exclusive with nccl_comm                       */
  int group_rank;        /* this context's rank in `group`                               */
  int shard;             /* mpr_shard                                                    */
  int ordered_reduce;    /* MPR_SHARD_REALIZATIONS: 1 => the accumulator travels rank 0 ->
                            W-1, each adding its realizations in ascending order, then a
                            broadcast: bit-identical to one GPU (the realization shard must
                            fit one launch batch)                                        */
} mpr_config;

/* MPR_ORDER_SC: single checkerboard, colour A then B.
 * MPR_ORDER_DC: double checkerboard (row f3): even l_b-tiles (A, B),
 * then odd tiles (A, B). DC supports mpr_simulate / mpr_simulate_range only (the fused
 * energy trace, the adaptive protocol and row slabs need the SC order: INVALID_ARG). */
typedef enum { MPR_ORDER_SC = 0, MPR_ORDER_DC = 1 } mpr_order;

/* Fill *cfg with the defaults above (calibration pointers NULL: the caller must set
 * them; the Python binding loads the shipped table). */
void mpr_config_default(mpr_config *cfg);

/* ---- communicators ----------------------------------------------------------------
 * NCCL (one process per GPU): rank 0 calls mpr_nccl_unique_id, the id (128 bytes) is sent
 * to every rank out of band (e.g. a torch.distributed broadcast), and each rank calls
 * mpr_nccl_comm_init with its device. libnccl.so.2 is resolved at run time (the copy the
 * process already loaded, if any); without it these calls return MPR_ERR_NCCL. The
 * communicator outlives every context that uses it; release with mpr_nccl_comm_destroy.
 * In-process group: mpr_group_create(W) once, then W contexts with cfg.group = g and
 * cfg.group_rank = 0..W-1, each driven by its own host thread (a rank blocks in a
 * collective until all W have arrived; 600 s timeout, MPR_GROUP_TIMEOUT_S). Destroy the
 * group after its contexts. */
#define MPR_NCCL_UNIQUE_ID_BYTES 128
mpr_status mpr_nccl_unique_id(void *id_out);
mpr_status mpr_nccl_comm_init(int world, int rank, const void *id, int device, void **comm_out);
mpr_status mpr_nccl_comm_destroy(void *comm);
mpr_status mpr_group_create(int world, mpr_group **out);
void mpr_group_destroy(mpr_group *g);

/* Create a context on cfg->device. Validates cfg (INVALID_ARG) and copies the table.
 * Ownership of *out passes to the caller; release with mpr_destroy. */
mpr_status mpr_init(const mpr_config *cfg, mpr_ctx **out);

/* Release every device and host resource of ctx (NULL is a no-op). */
void mpr_destroy(mpr_ctx *ctx);

/* One-line description of the last failure on ctx ("" if none). Owned by ctx. */
const char *mpr_last_error(const mpr_ctx *ctx);

/* Stage a problem: grid (float32, Lx*Ly) and mask (uint8, Lx*Ly), host memory: the WHOLE
 * grid on every rank (SPMD); with MPR_SHARD_ROWS a rank copies only its own rows to the
 * device and receives its ghost rows from the neighbouring ranks.
 * Computes z_min/z_max over the samples and the spin angles phi = 2pi(z - z_min)/
 * (z_max - z_min) at the samples (ARITH §D), and builds the gap-site
 * index. Errors: Lx < 2 or Ly < 2 or Lx*Ly > 2^30 (the bound under which every int64
 * fixed-point sum of ARITH §E/§J fits) or a non-finite sample ->
 * INVALID_ARG; fewer than 2 samples -> TOO_FEW_SAMPLES. z_max == z_min is not an
 * error: the DEGENERATE_RANGE flag is set, simulate is a no-op and predict fills
 * the gaps with z_min. */
mpr_status mpr_set_data(mpr_ctx *ctx, const float *grid, const uint8_t *mask, int64_t Lx, int64_t Ly);

/* Same as mpr_set_data with device pointers (a device-to-device copy into the context).
 * With MPR_SHARD_ROWS the pointers hold the rank's OWN rows only ((row_end - row_begin)
 * x Lx, rows as in mpr_info), so no device ever holds the whole grid. Lx, Ly are the
 * global sizes. Both calls return once the inputs are copied and the sample counts are
 * known; the gap-site index may still be building on the context stream (later calls
 * are ordered after it). */
mpr_status mpr_set_data_device(mpr_ctx *ctx, const float *grid_dev, const uint8_t *mask_dev,
                               int64_t Lx, int64_t Ly);

/* Local parameter field: block sample energies e_b (Eq.(2) per
 * block; a bond belongs to the block of its left/top end), block temperatures by
 * energy matching (table inversion), the lower-median fallback for blocks without
 * sample bonds, expansion to sites and n_s smoothing passes of radius r_s.
 * T_out (nullable, host, Lx*Ly floats) receives the per-site temperature field (with
 * MPR_SHARD_ROWS: the rank's own rows, written at their offsets; other rows untouched).
 * Errors: NO_SAMPLE_BONDS when no block has a sample-sample bond. */
mpr_status mpr_estimate_local_params(mpr_ctx *ctx, float *T_out);

/* Conditional simulation (ARITH §G-H): realizations
 * m = 0..M-1 (global ids), each initialised (BLOCK_MEAN or RANDOM) and swept
 * `sweeps` times (colour A = (r+c) even, then B) with the Philox stream keyed by
 * `seed`; the last n_avg sweeps of every realization are accumulated for the
 * conditional mean. Replaces any previous accumulation. Multi-rank: see mpr_shard (the
 * reduction over ranks happens inside this call). Errors: M < 1, sweeps < 1,
 * n_avg > sweeps -> INVALID_ARG. */
mpr_status mpr_simulate(mpr_ctx *ctx, int64_t M, int32_t sweeps, uint64_t seed);

/* Adaptive equilibration (n_fit = 20 "memory length of the energy time
 * series", n_f = 5 "frequency of verification"; test of ARITH §K, reading R20): every
 * realization sweeps until, at a check sweep s = n_fit + k*n_f, the least-squares slope
 * of its last n_fit whole-grid energies (ARITH §J, exact fixed point) is >=
 * -max(2 sigma / n_fit, slope_tol); it then averages the next n_avg sweeps and stops.
 * slope_tol (energy per sweep; 0 = SPEC's rule) is SPEC's configurable tolerance; a
 * negative slope_tol asks for the tolerance derived from the data (reading R22):
 * SE(e_s) / n_fit, the standard error of the sample specific energy of Eq.(2) over the sample
 * bonds' cosines, spread over the fit window (mpr_info.slope_tol reports the value used).
 * No check passes before max_sweeps - n_avg => equilibrium is declared there (returned
 * negated). s_eq_out (nullable, host, M int32) receives each realization's equilibrium
 * sweep. Replaces any previous accumulation; predict as after mpr_simulate. The test
 * runs on the device after each check sweep (fp64, ARITH §K operation order); the host
 * trails one check behind, so sweeps issued after the last realization finished are
 * no-ops. Realization shards: each rank runs its id range; the accumulators and s_eq are
 * summed over the ranks (every rank gets all M decisions). Row slabs: every rank sweeps
 * its rows for all M; the per-rank partial energies are summed over the ranks before each
 * device-side check, so every rank takes the same decisions. Errors: M < 1, n_fit < 3,
 * n_f < 1, max_sweeps <= n_avg, non-finite slope_tol -> INVALID_ARG. */
mpr_status mpr_simulate_adaptive(mpr_ctx *ctx, int64_t M, uint64_t seed, int32_t n_fit, int32_t n_f,
                                 int32_t max_sweeps, double slope_tol, int32_t *s_eq_out);

/* Calibration curve e(T) on the GPU (row f2; the T <-> e relation the energy matching of
 * PAPER.md:90 inverts, construction deferred to [mz-dth18]; reading R2):
 * for each of the K increasing temperatures T (host), `reps` replicas of an open L x L
 * lattice, every site free, start ordered (phi = pi) and run n_eq + n_meas checkerboard
 * sweeps of symmetric local moves phi' = phi + min(2pi, 3 sqrt T)(2u - 1) (rejected outside
 * [0, 2pi]; Philox counter (site, sweep, replica, tag 3)); e_raw[k] = mean over replicas
 * of the mean whole-grid energy (ARITH §J) over the measurement sweeps; e_out (host, K
 * floats) = its pool-adjacent-violators fit rounded to fp32 and made strictly increasing
 * (ties split by one ulp) — usable directly as mpr_config.calib_e. e_raw_out nullable.
 * Uses ctx's device and stream; does not touch the context's problem state. */
mpr_status mpr_build_calibration(mpr_ctx *ctx, const float *T, int32_t K, int32_t L, float q, int32_t n_eq,
                                 int32_t n_meas, int32_t reps, uint64_t seed, float *e_out, double *e_raw_out);

/* Building block below mpr_simulate (no collective of its own): simulate global
 * realization ids [m_begin, m_end) of an M-realization run and ADD them to the
 * accumulator (reset it first with mpr_reset_accumulator). Summing the accumulators of
 * ranks that ran disjoint ranges (mpr_accumulator_device + an external all-reduce) equals
 * the single-call mpr_simulate(M) up to fp64 summation order. With MPR_SHARD_ROWS every
 * rank must call it with the same range (the halo exchanges run inside); the energy
 * trace is then per-rank partial (mpr_simulate sums it). */
mpr_status mpr_reset_accumulator(mpr_ctx *ctx);
mpr_status mpr_simulate_range(mpr_ctx *ctx, int64_t M, int32_t sweeps, uint64_t seed,
                              int64_t m_begin, int64_t m_end);

/* Ordered (deterministic) multi-rank reduction. With the deferred reduce enabled,
 * mpr_simulate_range keeps the final states of its realizations (the range must fit one
 * launch batch, else INVALID_ARG) instead of adding them to the accumulator;
 * mpr_accumulate_states then adds them, realizations in ascending order, to whatever the
 * accumulator holds at that moment. Chaining the ranks in rank order is then bit-identical
 * to one GPU: each rank receives the accumulator of the ranks before it (for example
 * NCCL recv into mpr_accumulator_device), accumulates its own realizations, and sends the
 * result on; the last rank broadcasts it (mpr_config.ordered_reduce does exactly this
 * inside mpr_simulate). The adaptive protocol ignores the setting; row slabs reject it.
 * A pending deferred batch blocks further simulate calls (STATE) until it is
 * accumulated; set_data drops it. */
mpr_status mpr_set_deferred_reduce(mpr_ctx *ctx, int enable);
mpr_status mpr_accumulate_states(mpr_ctx *ctx);

/* Device view of the per-gap-site accumulator (double, *n entries, gap-site order)
 * so an external collective (NCCL all-reduce) can sum it in place across ranks. The
 * pointer stays owned by ctx and valid until the next set_data/destroy. */
mpr_status mpr_accumulator_device(mpr_ctx *ctx, double **acc_dev, int64_t *n);

/* Wait for all work queued on the context stream. */
mpr_status mpr_sync(mpr_ctx *ctx);

/* Predictions (ARITH §I): known sites return the input bitwise, gaps
 * z_min + (z_max - z_min) * mean_phi / 2pi. out: host, Lx*Ly floats, caller-owned; every
 * rank receives the whole grid (MPR_SHARD_ROWS: the slabs' rows are all-gathered).
 * mpr_predict_device: the same into device memory (Lx*Ly floats). mpr_predict_rows: the
 * rank's own rows only (MPR_SHARD_ROWS: (row_end - row_begin) x Lx floats, host; the
 * whole grid otherwise): no rank ever holds the whole prediction. */
mpr_status mpr_predict(mpr_ctx *ctx, float *out);
mpr_status mpr_predict_device(mpr_ctx *ctx, float *out_dev);
mpr_status mpr_predict_rows(mpr_ctx *ctx, float *out_rows);

/* ---- diagnostics / test hooks -------------------------------------------- */
typedef struct {
  int64_t Lx, Ly, n_samples, n_gaps, n_gaps_a;  /* n_gaps_a: colour-A gap sites      */
  float z_min, z_max;
  int degenerate_range;                          /* z_max == z_min                  */
  int64_t n_blocks, n_blocks_fallback;           /* blocks given the median         */
  float median_T;
  int64_t M, sweeps;                             /* last simulate call              */
  int64_t batch;                                 /* realizations per launch batch   */
  int64_t kernel_launches;                       /* kernels launched by the last
                                                    simulate call                   */
  int64_t total_launches;                        /* kernels launched since mpr_init */
  int64_t sweep_launches;                        /* half-sweep kernels timed        */
  double sweep_ms;                               /* device time of those launches
                                                    (CUDA events on the context
                                                    stream; needs kernel timing)    */
  int64_t last_m_base, last_batch;               /* realizations [last_m_base,
                                                    last_m_base + last_batch) are in
                                                    the state buffer (MPR_BUF_STATE)*/
  int32_t sweep_variant;                         /* half-sweep kernel variant in use
                                                    (MPR_SWEEP_VARIANT; 33 default:
                                                    two realization pairs per thread,
                                                    interleaved (28 for energy
                                                    sweeps, 13 for odd pair counts);
                                                    40/41: the SFU-filtered forms,
                                                    opt-in, 33 when mpr_filter_check
                                                    fails)                          */
  int32_t rank, world, shard;                    /* multi-rank layout                */
  int64_t row_begin, row_end;                    /* own rows (whole grid unless
                                                    MPR_SHARD_ROWS)                 */
  int64_t m_begin, m_end;                        /* own realizations of the last
                                                    simulate call                   */
  int64_t n_gaps_local;                          /* gap sites held by this rank
                                                    (own + ghost rows)              */
  int64_t comm_calls;                            /* collectives issued since init    */
  double slope_tol;                              /* slope tolerance of the last
                                                    adaptive run (derived: R22)     */
  int64_t sample_bonds;                          /* N_SP: sample-sample bonds        */
  int64_t filter_exact_pairs, filter_pairs;      /* variant 40/41 with
                                                    MPR_FILTER_STATS=1: realization
                                                    pairs sent to the exact path / all
                                                    pairs updated since mpr_init
                                                    (-1: not counted)               */
} mpr_info;
mpr_status mpr_get_info(mpr_ctx *ctx, mpr_info *info);

/* Buffers for tests (with MPR_SHARD_ROWS the Lx*Ly buffers get the rank's own rows at
 * their offsets, other rows untouched; the block buffers and the energy are global): */
typedef enum {
  MPR_BUF_PHI_KNOWN = 0,  /* float, Lx*Ly: angles at samples, 0 at gaps          */
  MPR_BUF_T = 1,          /* float, Lx*Ly: temperature field                      */
  MPR_BUF_BLOCK_T = 2,    /* float, n_blocks: block temperatures after fallback   */
  MPR_BUF_BLOCK_STATS = 3,/* int64, 4*n_blocks: SB, NB, SP, NK (ARITH §E)         */
  MPR_BUF_STATE = 4,      /* float, Lx*Ly per realization: dense angles of the
                             realizations of the LAST simulate batch (index arg)  */
  MPR_BUF_ACC = 5,        /* double, Lx*Ly: accumulator scattered to sites (0 at
                             samples)                                             */
  MPR_BUF_ENERGY = 6      /* double, M*sweeps: whole-grid specific energy after
                             each sweep (only if mpr_set_energy_trace(ctx, 1))    */
} mpr_buffer;
mpr_status mpr_debug_get(mpr_ctx *ctx, mpr_buffer which, int64_t index, void *host_out);

/* Enable (1) / disable (0) the fused whole-grid energy trace (ARITH §J). */
mpr_status mpr_set_energy_trace(mpr_ctx *ctx, int enable);

/* Enable (1) / disable (0) CUDA-event timing of the half-sweep kernels: events are
 * recorded on the context stream around each batch's sweep loop and summed into
 * mpr_info.sweep_ms / sweep_launches (reset by enabling again). */
mpr_status mpr_set_kernel_timing(mpr_ctx *ctx, int enable);

/* Library version string. */
const char *mpr_version(void);

/* Premises of the SFU rejection filter of the opt-in half-sweep kernel (variant 40,
 * DESIGN.md §7), measured on `device` over every argument the filter can see (run once
 * per device and process, a few ms):
 *   err_out[0] = max |y * S(fl(y*y)) - sin_SFU(y)| over every fp32 |y| <= 3.2, where S is
 *                ARITH §B2's sine polynomial (the product-form dE of PAPER.md Eq.(1)); the
 *                filter's bound B assumes <= 4e-6;
 *   err_out[1] = max exp_spec(x) * 2^24 over every fp32 x in [-80, -17] (must be < 1:
 *                such a Metropolis step, accepts only when u(w) = 0).
 * err_out: 2 doubles, host, borrowed; may be NULL. Returns 1 when both premises hold (a
 * context asking for variant 40 runs it), 0 otherwise (mpr_init falls back to the exact
 * kernel 33) or when no device is usable. */
int mpr_filter_check(int device, double *err_out);

#ifdef __cplusplus
}
#endif
#endif /* MPR_H_ */
