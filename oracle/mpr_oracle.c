/*
 * mpr_oracle.c — plain, slow, obviously-correct CPU oracle for the LE-MPR
 * (SV-MPR) conditional simulation of Lach & Zukovic, arXiv 2212.01317.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2212_01317_b200/) never links, imports or executes it, and this file
 * shares no code, header, table or constant generator with the CUDA path: both
 * follow the text of docs/ARITH.md independently.
 *
 * Every function cites the passage it follows: "P:<line>" is /root/reference/PAPER.md,
 * "ARITH §X" is docs/ARITH.md. Build: gcc -O2 -ffp-contract=off -fno-fast-math.
 *
 * Parity status: every function is pinned by a
 * `-m "not gpu"` test against something other than itself (KAT vectors, libm,
 * closed forms, hand lattices, quadrature, brute force) EXCEPT the local-equilibrium
 * chain with coupled gap sites under a spatially varying T, which has no Gibbs
 * measure ("actually non-equilibrium"): parity unpinned beyond the invariants
 * and the uniform-T / isolated-site special cases.
 *
 * Integer bounds (ARITH §E, §J): inputs with Lx*Ly <= 2^30 and (2 r_s + 1)^2 * T_max < 2^23
 * (the limits mpr_set_data / mpr_init enforce) keep every int64 fixed-point sum below 2^63.
 *
 * Two builds of this one file: liboracle.so (single thread: parity) and liboracle_omp.so
 * (-fopenmp: the same-colour rows of a half-sweep and the rows of a smoothing pass split
 * over threads; used only to time the oracle on all host cores). Their results are
 * bit-identical (test_openmp_build_bit_identical).
 */

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Threads of the OpenMP build (returns the count in use; 1 in the plain build). */
int oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

#define TWO_PI_F 0x1.921fb6p+2f

/* ---------------------------------------------------------------- ARITH §A */
/* Philox4x32-10 (Salmon et al. 2011), written out round by round. */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u(w) = (w >> 8) * 2^-24  (ARITH §A) */
float oracle_uniform(uint32_t w) { return (float)(w >> 8) * 0x1p-24f; }

/* The two words (wa, wb) of realization m at site i, sweep s (ARITH §A). */
static void sweep_words(uint32_t site, uint32_t sweep, int64_t m, uint64_t seed,
                        uint32_t *wa, uint32_t *wb)
{
    uint32_t ctr[4] = {site, sweep, (uint32_t)(m >> 1), 2u};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    if ((m & 1) == 0) { *wa = w[0]; *wb = w[1]; }
    else              { *wa = w[2]; *wb = w[3]; }
}

/* ---------------------------------------------------------------- ARITH §B */
float oracle_cos_spec(float x)
{
    float t = x * x;
    float p = 0x1.e0c79cp-30f;
    p = fmaf(p, t, -0x1.2392p-22f);
    p = fmaf(p, t, 0x1.9fb7a2p-16f);
    p = fmaf(p, t, -0x1.6c12aep-10f);
    p = fmaf(p, t, 0x1.555536p-5f);
    p = fmaf(p, t, -0.5f);
    p = fmaf(p, t, 1.0f);
    return p;
}

/* --------------------------------------------------------------- ARITH §B2 */
/* sin_spec(x) = x * S(x*x) for x in [-pi_f, pi_f]: odd polynomial of degree 11 whose
 * even part S is evaluated by Horner in fp32 fmaf (coefficients frozen in ARITH §B2). */
float oracle_sin_poly(float t)
{
    float p = -0x1.610f4ap-26f;
    p = fmaf(p, t, 0x1.6b1478p-19f);
    p = fmaf(p, t, -0x1.9f8a18p-13f);
    p = fmaf(p, t, 0x1.110ba2p-7f);
    p = fmaf(p, t, -0x1.55550cp-3f);
    p = fmaf(p, t, 1.0f);
    return p;
}

float oracle_sin_spec(float x)
{
    return x * oracle_sin_poly(x * x);
}

/* q = 1/2 (h = 1/4): x * S4(x*x) with S4's coefficients c_k * 2^-(4k+2), i.e.
 * (x/4) * S((x/4)^2) with the power-of-two scalings folded in (ARITH §B2). */
float oracle_sin_poly_quarter(float t)
{
    float p = -0x1.610f4ap-48f;
    p = fmaf(p, t, 0x1.6b1478p-37f);
    p = fmaf(p, t, -0x1.9f8a18p-27f);
    p = fmaf(p, t, 0x1.110ba2p-17f);
    p = fmaf(p, t, -0x1.55550cp-9f);
    p = fmaf(p, t, 0x1p-2f);
    return p;
}

/* ---------------------------------------------------------------- ARITH §C */
float oracle_exp_spec(float x)
{
    if (x < -80.0f) return 0.0f;
    float n = rintf(x * 0x1.715476p+0f);
    float f = fmaf(-n, 0x1.62e430p-1f, x);
    f = fmaf(-n, -0x1.05c610p-29f, f);
    float p = 0x1.6ac2a0p-10f;
    p = fmaf(p, f, 0x1.126e38p-7f);
    p = fmaf(p, f, 0x1.555890p-5f);
    p = fmaf(p, f, 0x1.555408p-3f);
    p = fmaf(p, f, 0x1.fffffap-2f);
    p = fmaf(p, f, 1.0f);
    p = fmaf(p, f, 1.0f);
    int ni = (int)n;
    union { uint32_t u; float f; } s;
    s.u = (uint32_t)(ni + 127) << 23;
    return p * s.f;
}

/* Bond energy -J cos[q(phi_i - phi_j)] of Eq.(1), with cos_spec. */
float oracle_bond_energy(float phi_i, float phi_j, float q, float J)
{
    return -(J * oracle_cos_spec(q * (phi_i - phi_j)));
}

/* ---------------------------------------------------------------- ARITH §D */
/* Linear map of the data to spin angles in [0, 2pi]. Returns 1 when the
 * sample range is degenerate (z_max == z_min), 0 otherwise, -1 with fewer than 2 samples.
 * phi is written at known sites only (gaps set to 0). */
int oracle_transform(const float *z, const uint8_t *mask, int64_t n,
                     float *zmin_out, float *zmax_out, float *phi)
{
    int64_t N = 0;
    float zmin = 0.0f, zmax = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        if (!mask[i]) continue;
        if (N == 0 || z[i] < zmin) zmin = z[i];
        if (N == 0 || z[i] > zmax) zmax = z[i];
        ++N;
    }
    zmin = zmin + 0.0f;   /* ARITH §D: -0 becomes +0 */
    zmax = zmax + 0.0f;
    *zmin_out = zmin; *zmax_out = zmax;
    if (N < 2) return -1;   /* fewer than 2 samples: rejected */
    int degenerate = (zmax == zmin);
    float range = zmax - zmin;
    float s = degenerate ? 0.0f : TWO_PI_F / range;
    for (int64_t i = 0; i < n; ++i) {
        if (!mask[i]) { phi[i] = 0.0f; continue; }
        float v = (z[i] - zmin) * s;
        phi[i] = fminf(v, TWO_PI_F);
    }
    return degenerate;
}

/* ------------------------------------------------- Eq.(2), P:91-95 (global) */
/* Sample specific energy e_s = -(1/N_SP) sum over sample-sample NN pairs of
 * cos[q(phi_i - phi_j)], each unordered pair counted once (reading R3).
 * Computed in fp64 with libm cos: the plain definition. */
double oracle_sample_specific_energy(const float *phi, const uint8_t *mask, int Lx, int Ly,
                                     float q, int64_t *nsp_out)
{
    double sum = 0.0;
    int64_t nsp = 0;
    for (int r = 0; r < Ly; ++r)
        for (int c = 0; c < Lx; ++c) {
            int64_t i = (int64_t)r * Lx + c;
            if (!mask[i]) continue;
            if (c + 1 < Lx && mask[i + 1]) {
                sum += cos((double)q * ((double)phi[i] - (double)phi[i + 1]));
                ++nsp;
            }
            if (r + 1 < Ly && mask[i + Lx]) {
                sum += cos((double)q * ((double)phi[i] - (double)phi[i + Lx]));
                ++nsp;
            }
        }
    *nsp_out = nsp;
    return nsp ? -sum / (double)nsp : 0.0;
}

/* Whole-grid specific energy (all bonds), P:90 / P:249; ARITH §J (fp64, libm). */
double oracle_grid_specific_energy(const float *phi, int Lx, int Ly, float q)
{
    double sum = 0.0;
    int64_t nb = 0;
    for (int r = 0; r < Ly; ++r)
        for (int c = 0; c < Lx; ++c) {
            int64_t i = (int64_t)r * Lx + c;
            if (c + 1 < Lx) { sum += cos((double)q * ((double)phi[i] - (double)phi[i + 1])); ++nb; }
            if (r + 1 < Ly) { sum += cos((double)q * ((double)phi[i] - (double)phi[i + Lx])); ++nb; }
        }
    return nb ? -sum / (double)nb : 0.0;
}

/* ------------------------------------------------- ARITH §E-F, P:108 (BST) */
/* Block-specific bond sums. A bond (i, right/down j) with both ends known is
 * attributed to block(i) (reading R4 of P:108). Arrays are nby*nbx. */
void oracle_block_stats(const float *phi, const uint8_t *mask, int Lx, int Ly, int lb, float q,
                        int64_t *SB, int64_t *NB, int64_t *SP, int64_t *NK)
{
    int nbx = (Lx + lb - 1) / lb, nby = (Ly + lb - 1) / lb;
    for (int b = 0; b < nbx * nby; ++b) { SB[b] = 0; NB[b] = 0; SP[b] = 0; NK[b] = 0; }
    for (int r = 0; r < Ly; ++r)
        for (int c = 0; c < Lx; ++c) {
            int64_t i = (int64_t)r * Lx + c;
            if (!mask[i]) continue;
            int b = (r / lb) * nbx + (c / lb);
            SP[b] += llrintf(phi[i] * 0x1p28f);
            NK[b] += 1;
            if (c + 1 < Lx && mask[i + 1]) {
                float bond = oracle_cos_spec(q * (phi[i] - phi[i + 1]));
                SB[b] += llrintf(bond * 0x1p32f);
                NB[b] += 1;
            }
            if (r + 1 < Ly && mask[i + Lx]) {
                float bond = oracle_cos_spec(q * (phi[i] - phi[i + Lx]));
                SB[b] += llrintf(bond * 0x1p32f);
                NB[b] += 1;
            }
        }
}

/* e_b from the exact fixed-point sum (ARITH §F). */
float oracle_block_energy(int64_t SB, int64_t NB)
{
    return (float)((-(double)SB * 0x1p-32) / (double)NB);
}

/* Energy matching: T such that e(T) = e_s, by piecewise-linear inversion of
 * the calibration table with clamping (ARITH §F). */
float oracle_estimate_temperature(float e, const float *Tk, const float *ek, int K)
{
    if (e <= ek[0]) return Tk[0];
    if (e >= ek[K - 1]) return Tk[K - 1];
    int k = 0;
    for (int j = 0; j < K; ++j)
        if (ek[j] <= e) k = j;
    float w = (e - ek[k]) / (ek[k + 1] - ek[k]);
    return Tk[k] + w * (Tk[k + 1] - Tk[k]);
}

static int cmp_float(const void *a, const void *b)
{
    float x = *(const float *)a, y = *(const float *)b;
    return (x > y) - (x < y);
}

/* Lower median of v[0..n-1] (reading R7), by sorting a copy. */
float oracle_lower_median(const float *v, int64_t n)
{
    float *c = (float *)malloc(sizeof(float) * (size_t)n);
    memcpy(c, v, sizeof(float) * (size_t)n);
    qsort(c, (size_t)n, sizeof(float), cmp_float);
    float m = c[(n - 1) / 2];
    free(c);
    return m;
}

/* Block temperatures with the median fallback for blocks without sample bonds,
 * P:108. Returns the number of available blocks (0 => no sample bonds anywhere). */
int64_t oracle_block_temperatures(const int64_t *SB, const int64_t *NB, int64_t nblocks,
                                  const float *Tk, const float *ek, int K, float *Tb)
{
    float *avail = (float *)malloc(sizeof(float) * (size_t)(nblocks > 0 ? nblocks : 1));
    int64_t na = 0;
    for (int64_t b = 0; b < nblocks; ++b) {
        if (NB[b] > 0) {
            Tb[b] = oracle_estimate_temperature(oracle_block_energy(SB[b], NB[b]), Tk, ek, K);
            avail[na++] = Tb[b];
        }
    }
    if (na > 0) {
        float med = oracle_lower_median(avail, na);
        for (int64_t b = 0; b < nblocks; ++b)
            if (NB[b] == 0) Tb[b] = med;
    }
    free(avail);
    return na;
}

/* Step field T(r,c) = T_b(block(r,c)). */
void oracle_expand(const float *Tb, int Lx, int Ly, int lb, float *T)
{
    int nbx = (Lx + lb - 1) / lb;
    for (int r = 0; r < Ly; ++r)
        for (int c = 0; c < Lx; ++c)
            T[(int64_t)r * Lx + c] = Tb[(r / lb) * nbx + (c / lb)];
}

/* SST: n_s passes of the clipped (2 r_s + 1)^2 window mean, P:124 (ARITH §F).
 * Direct 2-D window loop per site, exact int64 sums. */
void oracle_smooth(float *T, int Lx, int Ly, int rs, int ns)
{
    int64_t n = (int64_t)Lx * Ly;
    float *out = (float *)malloc(sizeof(float) * (size_t)n);
    for (int pass = 0; pass < ns; ++pass) {
#pragma omp parallel for schedule(static)
        for (int r = 0; r < Ly; ++r)
            for (int c = 0; c < Lx; ++c) {
                int r0 = r - rs < 0 ? 0 : r - rs, r1 = r + rs > Ly - 1 ? Ly - 1 : r + rs;
                int c0 = c - rs < 0 ? 0 : c - rs, c1 = c + rs > Lx - 1 ? Lx - 1 : c + rs;
                int64_t W = 0;
                for (int rr = r0; rr <= r1; ++rr)
                    for (int cc = c0; cc <= c1; ++cc)
                        W += llrintf(T[(int64_t)rr * Lx + cc] * 0x1p40f);
                int64_t cnt = (int64_t)(r1 - r0 + 1) * (c1 - c0 + 1);
                out[(int64_t)r * Lx + c] = (float)(((double)W * 0x1p-40) / (double)cnt);
            }
        memcpy(T, out, sizeof(float) * (size_t)n);
    }
    free(out);
}

/* ------------------------------------------------------ ARITH §G */
/* The one definition of both initial angles (ARITH §G), shared by oracle_init and
 * oracle_simulate_window so the two cannot drift apart.
 * RANDOM: phi = u(w) * TWO_PI_F with w the INIT word of realization m at global site
 * `site`: Philox counter (site, sweep 0, m >> 1, tag 1), word w0 for even m, w2 for odd m
 * (ARITH §A). The angle is uniform on [0, 2pi) (pinned by test_random_init_*). */
static float init_angle_random(uint32_t site, int64_t m, uint64_t seed)
{
    uint32_t ctr[4] = {site, 0u, (uint32_t)(m >> 1), 1u};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    return oracle_uniform((m & 1) ? w[2] : w[0]) * TWO_PI_F;
}

/* BLOCK_MEAN: the mean known angle of block b, (float)((double)SP_b 2^-28 / NK_b), or the
 * global sample mean gmean when the block has no sample. */
static float init_angle_block_mean(int64_t SP_b, int64_t NK_b, float gmean)
{
    return NK_b ? (float)(((double)SP_b * 0x1p-28) / (double)NK_b) : gmean;
}

static float global_mean_angle(const int64_t *SP, const int64_t *NK, int64_t nblocks)
{
    int64_t spg = 0, nkg = 0;
    for (int64_t b = 0; b < nblocks; ++b) { spg += SP[b]; nkg += NK[b]; }
    return nkg ? (float)(((double)spg * 0x1p-28) / (double)nkg) : 0.0f;
}

/* init_mode 0 = BLOCK_MEAN, 1 = RANDOM. phi holds known angles; gaps are written. */
void oracle_init(float *phi, const uint8_t *mask, int Lx, int Ly, int lb,
                 const int64_t *SP, const int64_t *NK, int init_mode, int64_t m, uint64_t seed)
{
    int nbx = (Lx + lb - 1) / lb, nby = (Ly + lb - 1) / lb;
    float gmean = global_mean_angle(SP, NK, (int64_t)nbx * nby);
    for (int r = 0; r < Ly; ++r)
        for (int c = 0; c < Lx; ++c) {
            int64_t i = (int64_t)r * Lx + c;
            if (mask[i]) continue;
            if (init_mode == 0) {
                int b = (r / lb) * nbx + (c / lb);
                phi[i] = init_angle_block_mean(SP[b], NK[b], gmean);
            } else {
                phi[i] = init_angle_random((uint32_t)i, m, seed);
            }
        }
}

/* ------------------------------------------------ ARITH §H */
/* Energy change dE = E(phi') - E(phi) of moving site (r,c) to angle prop, with
 * E = -J sum_j cos[q(phi - phi_j)] over its in-grid neighbours (Eq.(1)).
 * ARITH §H evaluates it through the identity cos A - cos B = 2 sin((B-A)/2) sin((A+B)/2):
 *   dE = 2J * sin[q(phi' - phi)/2] * sum_j sin[q((phi' + phi)/2 - phi_j)]
 * (SURVEY §8(c.2) option (ii); reading R19 in DESIGN.md), in this exact fp32 order:
 *   h = q/2;  d = phi' - phi;  a0 = h * d;  S1 = a0 * S(a0*a0);  s = phi' + phi;  Sig = +0
 *   for j in N, S, W, E inside the grid:  x = fma(-2, phi_j, s);  a = h * x;
 *                                         Sig = fma(a, S(a*a), Sig)
 *   dE = (2J) * (S1 * Sig)
 * For q = 1/2 the products by h = 1/4 are folded into the polynomial (S4, ARITH §B2):
 *   S1 = d * S4(d*d);  Sig = fma(x, S4(x*x), Sig).
 * h, 2J and 2 phi_j are exact power-of-two scalings. */
float oracle_delta_energy(const float *phi, int Lx, int Ly, int r, int c, float prop, float q, float J)
{
    float cur = phi[(int64_t)r * Lx + c];
    const int quarter = (q == 0.5f);  /* ARITH §B2: the folded form for q = 1/2 */
    float h = q * 0.5f;
    float d = prop - cur;
    float S1;
    if (quarter) {
        S1 = d * oracle_sin_poly_quarter(d * d);
    } else {
        float a0 = h * d;
        S1 = a0 * oracle_sin_poly(a0 * a0);
    }
    float s = prop + cur;
    float sig = +0.0f;
    int nr[4] = {r - 1, r + 1, r, r};
    int nc[4] = {c, c, c - 1, c + 1};
    for (int k = 0; k < 4; ++k) {
        if (nr[k] < 0 || nr[k] >= Ly || nc[k] < 0 || nc[k] >= Lx) continue;
        float pj = phi[(int64_t)nr[k] * Lx + nc[k]];
        float x = fmaf(-2.0f, pj, s);
        if (quarter) {
            sig = fmaf(x, oracle_sin_poly_quarter(x * x), sig);
        } else {
            float a = h * x;
            sig = fmaf(a, oracle_sin_poly(a * a), sig);
        }
    }
    return (2.0f * J) * (S1 * sig);
}

/* The direct form, sum of the bond cosines in the order N, S, W, E: used by the calibration
 * recipe (ARITH §H, last paragraph), whose table predates the product form. */
float oracle_delta_energy_direct(const float *phi, int Lx, int Ly, int r, int c, float prop, float q, float J)
{
    float cur = phi[(int64_t)r * Lx + c];
    float s_cur = +0.0f, s_new = +0.0f;
    int nr[4] = {r - 1, r + 1, r, r};
    int nc[4] = {c, c, c - 1, c + 1};
    for (int k = 0; k < 4; ++k) {
        if (nr[k] < 0 || nr[k] >= Ly || nc[k] < 0 || nc[k] >= Lx) continue;
        float pj = phi[(int64_t)nr[k] * Lx + nc[k]];
        s_cur = s_cur + oracle_cos_spec(q * (cur - pj));
        s_new = s_new + oracle_cos_spec(q * (prop - pj));
    }
    return J * (s_cur - s_new);
}

/* One Metropolis update of gap site (r,c) with the uniform independence proposal
 * phi' ~ U[0, 2pi) (reading R1) and acceptance min(1, exp(-dE/T)), T = 1/beta
 * (P:85); returns 1 if accepted. */
static int update_site_ctr(float *phi, int Lx, int Ly, int r, int c, uint32_t ctr_site, float beta,
                           float q, float J, uint32_t sweep, int64_t m, uint64_t seed)
{
    int64_t i = (int64_t)r * Lx + c;
    uint32_t wa, wb;
    sweep_words(ctr_site, sweep, m, seed, &wa, &wb);
    float prop = oracle_uniform(wa) * TWO_PI_F;
    float dE = oracle_delta_energy(phi, Lx, Ly, r, c, prop, q, J);
    int accept = (dE <= 0.0f) || (oracle_uniform(wb) < oracle_exp_spec(-(dE * beta)));
    if (accept) phi[i] = prop;
    return accept;
}

static int update_site(float *phi, int Lx, int Ly, int r, int c, float beta, float q, float J,
                       uint32_t sweep, int64_t m, uint64_t seed)
{
    return update_site_ctr(phi, Lx, Ly, r, c, (uint32_t)((int64_t)r * Lx + c), beta, q, J, sweep, m, seed);
}

/* Realization m of a CROP [r_off, r_off+wLy) x [c_off, c_off+wLx) of an Lx_g x Ly_g grid
 * (test device for full-size sampled parity): gaps initialised from the GLOBAL block sums
 * (BLOCK_MEAN) or the global-site Philox counter (RANDOM), then S sweeps whose colour and
 * Philox counters use global coordinates. The crop edge acts as an open boundary, so sites
 * within 2S+1 of an inner crop edge are not exact; the caller compares only the interior
 * (information moves one site per half-sweep). phi0/mask/beta are crop arrays. */
void oracle_simulate_window(const float *phi0, const uint8_t *mask, const float *beta, int wLx, int wLy,
                            int r_off, int c_off, int Lx_g, int Ly_g, int lb, const int64_t *SP_g,
                            const int64_t *NK_g, int init_mode, float q, float J, int64_t m, int S,
                            uint64_t seed, float *phi)
{
    int nbx = (Lx_g + lb - 1) / lb, nby = (Ly_g + lb - 1) / lb;
    float gmean = global_mean_angle(SP_g, NK_g, (int64_t)nbx * nby);
    memcpy(phi, phi0, sizeof(float) * (size_t)wLx * (size_t)wLy);
    for (int r = 0; r < wLy; ++r)
        for (int c = 0; c < wLx; ++c) {
            int64_t i = (int64_t)r * wLx + c;
            if (mask[i]) continue;
            int rg = r + r_off, cg = c + c_off;
            if (init_mode == 0) {
                int b = (rg / lb) * nbx + (cg / lb);
                phi[i] = init_angle_block_mean(SP_g[b], NK_g[b], gmean);
            } else {
                phi[i] = init_angle_random((uint32_t)((int64_t)rg * Lx_g + cg), m, seed);
            }
        }
    for (int s = 1; s <= S; ++s)
        for (int colour = 0; colour < 2; ++colour)
            for (int r = 0; r < wLy; ++r)
                for (int c = 0; c < wLx; ++c) {
                    int64_t i = (int64_t)r * wLx + c;
                    int rg = r + r_off, cg = c + c_off;
                    if (((rg + cg) & 1) != colour || mask[i]) continue;
                    update_site_ctr(phi, wLx, wLy, r, c, (uint32_t)((int64_t)rg * Lx_g + cg), beta[i], q, J,
                                    (uint32_t)s, m, seed);
                }
}

/* One checkerboard sweep (colour A = (r+c) even, then B) over the gap sites of one
 * realization. reverse != 0 visits each colour's sites in reverse order (parity
 * safety test: the result must not depend on the order). Returns #accepted.
 * The sites of one colour are independent (each reads only other-colour neighbours,
 * P:119), so the timing build (liboracle_omp.so, -fopenmp) splits a colour's rows over
 * threads; without -fopenmp the pragma is ignored. Both builds give the same bits. */
int64_t oracle_sweep(float *phi, const uint8_t *mask, const float *beta, int Lx, int Ly,
                     float q, float J, uint32_t sweep, int64_t m, uint64_t seed, int reverse)
{
    int64_t acc = 0;
    for (int colour = 0; colour < 2; ++colour) {
#pragma omp parallel for schedule(static) reduction(+ : acc)
        for (int t = 0; t < Ly; ++t) {
            int r = reverse ? Ly - 1 - t : t;
            for (int u = 0; u < Lx; ++u) {
                int c = reverse ? Lx - 1 - u : u;
                int64_t i = (int64_t)r * Lx + c;
                if (((r + c) & 1) != colour || mask[i]) continue;
                acc += update_site(phi, Lx, Ly, r, c, beta[i], q, J, sweep, m, seed);
            }
        }
    }
    return acc;
}

/* Double-checkerboard sweep (row f3; "first only the even (odd) numbered
 * tiles are updated in parallel and then only the odd (even) tiles", tiles = the l_b x l_b
 * blocks of the temperature estimate): phases (even tiles, A), (even tiles, B),
 * (odd tiles, A), (odd tiles, B); tile parity = (r/l_b + c/l_b) mod 2 (ARITH §H). */
int64_t oracle_sweep_dc(float *phi, const uint8_t *mask, const float *beta, int Lx, int Ly, float q,
                        float J, uint32_t sweep, int64_t m, uint64_t seed, int lb)
{
    int64_t acc = 0;
    for (int tile = 0; tile < 2; ++tile)
        for (int colour = 0; colour < 2; ++colour)
            for (int r = 0; r < Ly; ++r)
                for (int c = 0; c < Lx; ++c) {
                    int64_t i = (int64_t)r * Lx + c;
                    if (((r + c) & 1) != colour || mask[i]) continue;
                    if (((r / lb + c / lb) & 1) != tile) continue;
                    acc += update_site(phi, Lx, Ly, r, c, beta[i], q, J, sweep, m, seed);
                }
    return acc;
}

/* One colour half of sweep `sweep` restricted to rows [r0, r1) (a row slab of the
 * checkerboard update): the gap sites of that colour in those rows, in row-major
 * order. Returns #accepted. */
int64_t oracle_half_sweep_rows(float *phi, const uint8_t *mask, const float *beta, int Lx, int Ly,
                               float q, float J, uint32_t sweep, int64_t m, uint64_t seed,
                               int colour, int r0, int r1)
{
    int64_t acc = 0;
    for (int r = r0; r < r1; ++r)
        for (int c = 0; c < Lx; ++c) {
            int64_t i = (int64_t)r * Lx + c;
            if (((r + c) & 1) != colour || mask[i]) continue;
            acc += update_site(phi, Lx, Ly, r, c, beta[i], q, J, sweep, m, seed);
        }
    return acc;
}

/* Sweeps s_begin..s_end-1 of realization m on a given beta field; adds phi after
 * every sweep to sum_phi (fp64, per site) and returns #accepted. Used by the
 * quadrature / brute-force pins of the Metropolis step. */
int64_t oracle_run_chain(float *phi, const uint8_t *mask, const float *beta, int Lx, int Ly,
                         float q, float J, uint32_t s_begin, uint32_t s_end, int64_t m, uint64_t seed,
                         double *sum_phi)
{
    int64_t acc = 0, n = (int64_t)Lx * Ly;
    for (uint32_t s = s_begin; s < s_end; ++s) {
        acc += oracle_sweep(phi, mask, beta, Lx, Ly, q, J, s, m, seed, 0);
        if (sum_phi)
            for (int64_t i = 0; i < n; ++i) sum_phi[i] += (double)phi[i];
    }
    return acc;
}

/* ------------------------------------------------------------ full pipeline */
typedef struct {
    float q, J;
    int lb, rs, ns, init_mode, n_avg;
    int order;  /* 0 = single checkerboard (SC), 1 = double checkerboard (DC, row f3) */
} oracle_cfg;

/* Parameter stage (a1-a5): transform, block stats, block T, median, expand, smooth,
 * beta. Outputs: phi0 (known angles), T (per site), beta, zmin/zmax. Returns
 * 0 ok, 1 degenerate range, -1 no samples, -2 no sample bonds. */
int oracle_parameters(const float *z, const uint8_t *mask, int Lx, int Ly, const oracle_cfg *cfg,
                      const float *Tk, const float *ek, int K,
                      float *phi0, float *T, float *beta, float *zmin, float *zmax,
                      int64_t *SP, int64_t *NK, float *Tb_out)
{
    int64_t n = (int64_t)Lx * Ly;
    int st = oracle_transform(z, mask, n, zmin, zmax, phi0);
    if (st < 0) return -1;
    int nbx = (Lx + cfg->lb - 1) / cfg->lb, nby = (Ly + cfg->lb - 1) / cfg->lb;
    int64_t nblocks = (int64_t)nbx * nby;
    int64_t *SB = (int64_t *)malloc(sizeof(int64_t) * (size_t)nblocks);
    int64_t *NB = (int64_t *)malloc(sizeof(int64_t) * (size_t)nblocks);
    float *Tb = (float *)malloc(sizeof(float) * (size_t)nblocks);
    oracle_block_stats(phi0, mask, Lx, Ly, cfg->lb, cfg->q, SB, NB, SP, NK);
    int64_t na = oracle_block_temperatures(SB, NB, nblocks, Tk, ek, K, Tb);
    int rc = st;
    if (na == 0 && st == 0) rc = -2;
    if (na > 0) {
        oracle_expand(Tb, Lx, Ly, cfg->lb, T);
        oracle_smooth(T, Lx, Ly, cfg->rs, cfg->ns);
        for (int64_t i = 0; i < n; ++i) beta[i] = 1.0f / T[i];
        if (Tb_out) memcpy(Tb_out, Tb, sizeof(float) * (size_t)nblocks);
    }
    free(SB); free(NB); free(Tb);
    return rc;
}

int64_t oracle_grid_energy_fx(const float *phi, int Lx, int Ly, float q);
double oracle_energy_from_fx(int64_t E_fx, int Lx, int Ly);

/* Realizations m in [m_begin, m_end): init, S sweeps, accumulate the last n_avg
 * (P:95 conditional mean). acc (fp64, length Lx*Ly) is added to; energy
 * (nullable, (m_end-m_begin)*S) receives the whole-grid specific energy after each
 * sweep; phi_out (nullable, (m_end-m_begin)*Lx*Ly) receives the final states. */
void oracle_simulate(const float *phi0, const uint8_t *mask, const float *beta, int Lx, int Ly,
                     const oracle_cfg *cfg, const int64_t *SP, const int64_t *NK,
                     int64_t m_begin, int64_t m_end, int S, uint64_t seed,
                     double *acc, double *energy, float *phi_out, int64_t *accepted)
{
    int64_t n = (int64_t)Lx * Ly;
    float *phi = (float *)malloc(sizeof(float) * (size_t)n);
    int64_t nacc = 0;
    for (int64_t m = m_begin; m < m_end; ++m) {
        memcpy(phi, phi0, sizeof(float) * (size_t)n);
        oracle_init(phi, mask, Lx, Ly, cfg->lb, SP, NK, cfg->init_mode, m, seed);
        for (int s = 1; s <= S; ++s) {
            nacc += cfg->order == 1
                        ? oracle_sweep_dc(phi, mask, beta, Lx, Ly, cfg->q, cfg->J, (uint32_t)s, m, seed, cfg->lb)
                        : oracle_sweep(phi, mask, beta, Lx, Ly, cfg->q, cfg->J, (uint32_t)s, m, seed, 0);
            if (s > S - cfg->n_avg)
                for (int64_t i = 0; i < n; ++i)
                    if (!mask[i]) acc[i] += (double)phi[i];
            if (energy)  /* ARITH §J fixed-point definition (pinned against the fp64 one) */
                energy[(m - m_begin) * S + (s - 1)] =
                    oracle_energy_from_fx(oracle_grid_energy_fx(phi, Lx, Ly, cfg->q), Lx, Ly);
        }
        if (phi_out) memcpy(phi_out + (m - m_begin) * n, phi, sizeof(float) * (size_t)n);
    }
    if (accepted) *accepted = nacc;
    free(phi);
}

/* Whole-grid bond sum in fixed point (ARITH §J): sum over all bonds of
 * llrint(cos_spec(q(phi_i - phi_j)) * 2^32), every unordered bond once. */
int64_t oracle_grid_energy_fx(const float *phi, int Lx, int Ly, float q)
{
    int64_t sum = 0;
    for (int r = 0; r < Ly; ++r)
        for (int c = 0; c < Lx; ++c) {
            int64_t i = (int64_t)r * Lx + c;
            if (c + 1 < Lx) sum += llrintf(oracle_cos_spec(q * (phi[i] - phi[i + 1])) * 0x1p32f);
            if (r + 1 < Ly) sum += llrintf(oracle_cos_spec(q * (phi[i] - phi[i + Lx])) * 0x1p32f);
        }
    return sum;
}

/* e = (-(double)E_fx * 2^-32) / N_bonds (ARITH §J). */
double oracle_energy_from_fx(int64_t E_fx, int Lx, int Ly)
{
    double nb = (double)(2 * (int64_t)Lx * Ly - Lx - Ly);
    return (-(double)E_fx * 0x1p-32) / nb;
}

/* Equilibrium test of ARITH §K on y[0 .. n_fit-1] (the last n_fit energies): least-squares
 * slope b against t = 0..n_fit-1, residual scale, tau = 2 sigma / n_fit; 1 iff b >= -tau. */
int oracle_equilibrium_test(const double *y, int n_fit, double slope_tol)
{
    double xbar = (double)(n_fit - 1) / 2.0;
    double sy = 0.0;
    for (int t = 0; t < n_fit; ++t) sy = sy + y[t];
    double ybar = sy / (double)n_fit;
    double sxx = 0.0, sxy = 0.0;
    for (int t = 0; t < n_fit; ++t) {
        double dx = (double)t - xbar;
        sxx = sxx + dx * dx;
        sxy = sxy + dx * (y[t] - ybar);
    }
    double b = sxy / sxx;
    double a = ybar - b * xbar;
    double sse = 0.0;
    for (int t = 0; t < n_fit; ++t) {
        double res = y[t] - a - b * (double)t;
        sse = sse + res * res;
    }
    double tau = 2.0 * sqrt(sse / (double)(n_fit - 2)) / (double)n_fit;
    if (slope_tol > tau) tau = slope_tol;  /* tau = max(2 sigma / n_fit, slope_tol) */
    return b >= -tau;
}

/* Reading R22: the slope tolerance derived from the data, tau = SE(e_s) / n_fit,
 * the standard error of the sample specific energy of Eq.(2) spread over the fit
 * window: SE^2 = var(b) / N_SP over the sample bonds' cosines b = cos_spec(q (phi_i - phi_j)),
 * each unordered pair once; the sums are exact fixed point (S1 = sum llrint(b 2^32),
 * S2 = sum llrint(fp32(b b) 2^32)), then fp64 in this order. Pinned against the fp64/libm
 * sample standard deviation and hand lattices (test_derived_slope_tolerance_*). */
double oracle_derived_slope_tol(const float *phi, const uint8_t *mask, int Lx, int Ly, float q, int n_fit)
{
    int64_t S1 = 0, S2 = 0, N = 0;
    for (int r = 0; r < Ly; ++r)
        for (int c = 0; c < Lx; ++c) {
            int64_t i = (int64_t)r * Lx + c;
            if (!mask[i]) continue;
            if (c + 1 < Lx && mask[i + 1]) {
                float b = oracle_cos_spec(q * (phi[i] - phi[i + 1]));
                S1 += llrintf(b * 0x1p32f); S2 += llrintf((b * b) * 0x1p32f); ++N;
            }
            if (r + 1 < Ly && mask[i + Lx]) {
                float b = oracle_cos_spec(q * (phi[i] - phi[i + Lx]));
                S1 += llrintf(b * 0x1p32f); S2 += llrintf((b * b) * 0x1p32f); ++N;
            }
        }
    if (N < 1) return 0.0;
    double n = (double)N;
    double mean = ((double)S1 * 0x1p-32) / n;
    double m2 = ((double)S2 * 0x1p-32) / n;
    double var = m2 - mean * mean;
    if (var < 0.0) var = 0.0;
    return sqrt(var / n) / (double)n_fit;
}

/* Adaptive protocol (row f1; ARITH §K): realization m sweeps until the energy
 * trace passes the equilibrium test at a check sweep (s = n_fit + k n_f), then runs
 * n_avg more sweeps accumulating each; capped at S_max. acc (fp64, Lx*Ly) is added to;
 * s_eq[m - m_begin] receives the equilibrium sweep (negated if forced by the cap);
 * energy (nullable, (m_end-m_begin)*S_max) the per-sweep energies (0 after the stop). */
void oracle_simulate_adaptive(const float *phi0, const uint8_t *mask, const float *beta, int Lx, int Ly,
                              const oracle_cfg *cfg, const int64_t *SP, const int64_t *NK,
                              int64_t m_begin, int64_t m_end, int n_fit, int n_f, int S_max, double slope_tol,
                              uint64_t seed,
                              double *acc, int32_t *s_eq, double *energy, float *phi_out)
{
    int64_t n = (int64_t)Lx * Ly;
    /* slope_tol < 0: the tolerance derived from the samples (R22) */
    if (slope_tol < 0.0) slope_tol = oracle_derived_slope_tol(phi0, mask, Lx, Ly, cfg->q, n_fit);
    float *phi = (float *)malloc(sizeof(float) * (size_t)n);
    double *e = (double *)malloc(sizeof(double) * (size_t)(S_max + 1));
    for (int64_t m = m_begin; m < m_end; ++m) {
        memcpy(phi, phi0, sizeof(float) * (size_t)n);
        oracle_init(phi, mask, Lx, Ly, cfg->lb, SP, NK, cfg->init_mode, m, seed);
        int eq = 0, stop = S_max;
        for (int s = 1; s <= stop; ++s) {
            if (cfg->order == 1)
                oracle_sweep_dc(phi, mask, beta, Lx, Ly, cfg->q, cfg->J, (uint32_t)s, m, seed, cfg->lb);
            else
                oracle_sweep(phi, mask, beta, Lx, Ly, cfg->q, cfg->J, (uint32_t)s, m, seed, 0);
            e[s] = oracle_energy_from_fx(oracle_grid_energy_fx(phi, Lx, Ly, cfg->q), Lx, Ly);
            if (energy) energy[(m - m_begin) * S_max + (s - 1)] = e[s];
            if (eq) {
                for (int64_t i = 0; i < n; ++i)
                    if (!mask[i]) acc[i] += (double)phi[i];
                continue;
            }
            int check = s >= n_fit + n_f && (s - n_fit) % n_f == 0 && s + cfg->n_avg <= S_max;
            if (check && oracle_equilibrium_test(&e[s - n_fit + 1], n_fit, slope_tol)) {
                eq = s;
                stop = s + cfg->n_avg;
            } else if (s == S_max - cfg->n_avg) {
                eq = -s;  /* forced by the cap */
                stop = S_max;
            }
        }
        s_eq[m - m_begin] = eq;
        if (phi_out) memcpy(phi_out + (m - m_begin) * n, phi, sizeof(float) * (size_t)n);
    }
    free(phi);
    free(e);
}

/* Back-transform of the conditional mean, P:95 (ARITH §I). */
void oracle_predict(const float *z, const uint8_t *mask, int64_t n, const double *acc,
                    int64_t M, int n_avg, float zmin, float zmax, int degenerate, float *out)
{
    for (int64_t i = 0; i < n; ++i) {
        if (mask[i]) { out[i] = z[i]; continue; }
        if (degenerate) { out[i] = zmin; continue; }
        double mean = acc[i] / (double)(M * (int64_t)n_avg);
        out[i] = (float)((double)zmin + ((double)zmax - (double)zmin) * (mean / (double)TWO_PI_F));
    }
}

/* One local-move Metropolis sweep (calibration only): phi' = phi + step*(2u-1),
 * rejected outside [0, 2pi_f] (symmetric proposal, so the stationary law is the same
 * Gibbs measure as the uniform proposal's; it equilibrates far faster at low T). */
static void local_sweep(float *phi, int L, float beta, float q, float step, uint32_t sweep,
                        int64_t m, uint64_t seed)
{
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    for (int colour = 0; colour < 2; ++colour)
        for (int r = 0; r < L; ++r)
            for (int c = 0; c < L; ++c) {
                if (((r + c) & 1) != colour) continue;
                int64_t i = (int64_t)r * L + c;
                uint32_t ctr[4] = {(uint32_t)i, sweep, (uint32_t)m, 3u};
                uint32_t w[4];
                oracle_philox4x32_10(ctr, key, w);
                float prop = phi[i] + step * (2.0f * oracle_uniform(w[0]) - 1.0f);
                if (prop < 0.0f || prop > TWO_PI_F) continue;
                float dE = oracle_delta_energy_direct(phi, L, L, r, c, prop, q, 1.0f);
                if (dE <= 0.0f || oracle_uniform(w[1]) < oracle_exp_spec(-(dE * beta))) phi[i] = prop;
            }
}

/* Unconditional simulation at uniform T (all sites free) for the e(T) calibration
 * curve (reading R2: the T<->e relation the matching of P:90 inverts). init_mode
 * 1 = RANDOM, 2 = ORDERED (all phi = pi). step <= 0: the uniform proposal of the
 * conditional simulation; step > 0: local moves of half-width step. Returns the mean
 * whole-grid specific energy over sweeps n_eq+1 .. n_eq+n_meas (per-sweep values in
 * trace, nullable). */
double oracle_unconditional_energy(int L, float T, float q, int init_mode, int n_eq, int n_meas,
                                   uint64_t seed, int64_t m, double *trace, float step)
{
    int64_t n = (int64_t)L * L;
    float *phi = (float *)malloc(sizeof(float) * (size_t)n);
    float *beta = (float *)malloc(sizeof(float) * (size_t)n);
    uint8_t *mask = (uint8_t *)calloc((size_t)n, 1);
    int64_t SP = 0, NK = 0;
    for (int64_t i = 0; i < n; ++i) { phi[i] = 0x1.921fb6p+1f; beta[i] = 1.0f / T; }
    if (init_mode == 1) oracle_init(phi, mask, L, L, L, &SP, &NK, 1, m, seed);
    double sum = 0.0;
    for (int s = 1; s <= n_eq + n_meas; ++s) {
        if (step > 0.0f) local_sweep(phi, L, 1.0f / T, q, step, (uint32_t)s, m, seed);
        else oracle_sweep(phi, mask, beta, L, L, q, 1.0f, (uint32_t)s, m, seed, 0);
        double e = oracle_energy_from_fx(oracle_grid_energy_fx(phi, L, L, q), L, L);  /* ARITH §J */
        if (trace) trace[s - 1] = e;
        if (s > n_eq) sum += e;
    }
    free(phi); free(beta); free(mask);
    return sum / (double)n_meas;
}

/* Prediction errors of Eq.(3), P:184-192 (AAE, RASE) and MARE (reading R16). */
void oracle_score(const float *pred, const float *truth, const uint8_t *mask, int64_t n,
                  double *mae, double *rmse, double *mare, int64_t *n_excl)
{
    double sa = 0.0, s2 = 0.0, sr = 0.0;
    int64_t P = 0, Pr = 0, ex = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (mask[i]) continue;
        double e = (double)truth[i] - (double)pred[i];
        sa += fabs(e); s2 += e * e; ++P;
        if (truth[i] != 0.0f) { sr += fabs(e) / fabs((double)truth[i]); ++Pr; } else ++ex;
    }
    *mae = P ? sa / (double)P : 0.0;
    *rmse = P ? sqrt(s2 / (double)P) : 0.0;
    *mare = Pr ? sr / (double)Pr : 0.0;
    *n_excl = ex;
}
