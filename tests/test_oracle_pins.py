"""Pins of the CPU oracle against things other than itself (`-m "not gpu"`).

Each test names the pin type (KAT, libm, closed form, hand lattice, quadrature,
brute force, invariant) and the passage it pins (P:<line> = PAPER.md). A plausible
mistake in the oracle — a dropped term, a wrong sign or index, a transposed operand —
fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TWO_PI_F = np.float32(2 * np.pi)
S2 = math.sqrt(0.5)


# ------------------------------------------------------------------ Philox (KAT)
@pytest.mark.parametrize("ctr,key,expect", [
    ([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
    ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
    ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
     [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
])
def test_philox_known_answers(ctr, key, expect):
    """Random123 Philox4x32-10 KAT vectors (library routine / KAT)."""
    assert [int(x) for x in O.philox4x32_10(ctr, key)] == expect


def test_uniform_is_24bit_exact():
    assert O.uniform(0) == 0.0
    assert O.uniform(0xffffffff) == 1.0 - 2.0 ** -24
    assert O.uniform(0x80000000) == 0.5


# ------------------------------------------------------------- cos / exp vs libm
def test_cos_spec_against_libm():
    """|cos_spec - cos| <= 3.5e-7 on [-pi_f, pi_f] (libm, fp64)."""
    xs = np.linspace(-np.pi, np.pi, 200001).astype(np.float32)
    err = max(abs(O.cos_spec(x) - math.cos(float(x))) for x in xs[::7])
    assert err < 3.5e-7
    assert O.cos_spec(0.0) == 1.0
    assert O.cos_spec(float(np.float32(np.pi))) == -1.0


def test_exp_spec_against_libm():
    """exp_spec within 2 ulp relative of exp on [-80, 0]; 0 below -80 (libm)."""
    xs = np.linspace(-80, 0, 40001).astype(np.float32)
    worst = max(abs(O.exp_spec(x) - math.exp(float(x))) / math.exp(float(x)) for x in xs)
    assert worst < 2 * 2 ** -23
    assert O.exp_spec(0.0) == 1.0
    assert O.exp_spec(-80.5) == 0.0


# --------------------------------------------------- bond energy (hand values, Eq.(1))
@pytest.mark.parametrize("a,b,expect", [(1.3, 1.3, -1.0), (0.0, np.pi, 0.0), (0.0, 2 * np.pi, 1.0)])
def test_bond_energy_hand_values(a, b, expect):
    """-J cos[q(phi_i - phi_j)] at q = 1/2 (SPEC bond_energy examples)."""
    assert abs(O.bond_energy(a, b) - expect) < 4e-7
    assert O.bond_energy(a, b) == O.bond_energy(b, a)


def test_bond_energy_scales_with_J_and_q():
    assert abs(O.bond_energy(0.0, 2.0, q=0.25, J=3.0) + 3.0 * math.cos(0.5)) < 2e-6


# ------------------------------------------------------------ transform (closed form)
def test_transform_endpoints_and_midpoint():
    """phi(z_min) = 0, phi(z_max) = 2pi_f, phi(mid) = pi."""
    z = np.array([[3.0, 7.0], [5.0, np.nan]], np.float32)
    mask = np.array([[1, 1], [1, 0]], np.uint8)
    phi, lo, hi, st = O.to_angles(np.nan_to_num(z), mask)
    assert st == 0 and lo == 3.0 and hi == 7.0
    assert phi[0, 0] == 0.0 and phi[0, 1] == TWO_PI_F
    assert abs(phi[1, 0] - np.pi) <= 4e-7
    assert phi[1, 1] == 0.0  # gap


def test_transform_degenerate_and_roundtrip():
    """Constant samples flag a degenerate range; to_angles -> predict is the identity within fp32 ulp."""
    z = np.full((3, 3), 2.5, np.float32)
    mask = np.ones((3, 3), np.uint8)
    assert O.to_angles(z, mask)[3] == 1
    rng = np.random.default_rng(0)
    z = (rng.standard_normal((16, 16)) * 40 + 100).astype(np.float32)
    phi, lo, hi, st = O.to_angles(z, np.ones_like(z, np.uint8))
    back = O.predict(z, np.zeros_like(z, np.uint8), phi.astype(np.float64), 1, 1, lo, hi, 0)
    assert np.max(np.abs(back - z)) <= 4 * np.spacing(np.float32(hi - lo))


def test_too_few_samples_rejected(calib):
    """SPEC S:31 / SURVEY 8(b): fewer than 2 known sites is an error (status < 0), not a
    degenerate range; exactly 2 equal samples is the degenerate (accepted) case."""
    z = np.full((3, 4), 1.5, np.float32)
    for known in (0, 1):
        mask = np.zeros((3, 4), np.uint8)
        mask.flat[:known] = 1
        assert O.to_angles(z, mask)[3] < 0
        assert O.parameters(z, mask, O.OracleConfig(lb=2), *calib).status < 0
    mask = np.zeros((3, 4), np.uint8)
    mask.flat[:2] = 1
    assert O.to_angles(z, mask)[3] == 1


def test_transform_negative_zero_canonical():
    """ARITH §D: a -0 extremum is returned as +0."""
    z = np.array([[-0.0, 1.0]], np.float32)
    _, lo, _, _ = O.to_angles(z, np.ones((1, 2), np.uint8))
    assert lo == 0.0 and math.copysign(1, lo) == 1.0


# ------------------------------------------------- sample specific energy (Eq.(2))
def test_sample_energy_constant_field():
    """Fully sampled constant field: e_s = -1 with N_SP = 2LxLy - Lx - Ly (SPEC mpr-model)."""
    phi = np.full((5, 7), 1.234, np.float32)
    e, n = O.sample_specific_energy(phi, np.ones((5, 7), np.uint8))
    assert n == 2 * 35 - 7 - 5 and abs(e + 1) < 1e-12


def test_sample_energy_checker_2x2():
    """[[0, pi], [pi, 0]]: every bond has |dphi| = pi, cos(pi/2) = 0 -> e_s = 0, N_SP = 4."""
    phi = np.array([[0, np.pi], [np.pi, 0]], np.float32)
    e, n = O.sample_specific_energy(phi, np.ones((2, 2), np.uint8))
    assert n == 4 and abs(e) < 1e-7


def test_sample_energy_missing_centre_3x3():
    """3x3 with missing centre: the 8 perimeter bonds only."""
    mask = np.ones((3, 3), np.uint8); mask[1, 1] = 0
    rng = np.random.default_rng(1)
    phi = (rng.random((3, 3)) * 2 * np.pi).astype(np.float32)
    e, n = O.sample_specific_energy(phi, mask)
    assert n == 8
    bonds = [((0, 0), (0, 1)), ((0, 1), (0, 2)), ((2, 0), (2, 1)), ((2, 1), (2, 2)),
             ((0, 0), (1, 0)), ((1, 0), (2, 0)), ((0, 2), (1, 2)), ((1, 2), (2, 2))]
    ref = -np.mean([math.cos(0.5 * (float(phi[a]) - float(phi[b]))) for a, b in bonds])
    assert abs(e - ref) < 1e-12


def test_grid_energy_independent_angles():
    """i.i.d. uniform angles: E[cos((x-y)/2)] = (2/pi)^2 -> e = -4/pi^2 (analytic)."""
    rng = np.random.default_rng(2)
    phi = (rng.random((256, 256)) * 2 * np.pi).astype(np.float32)
    assert abs(O.grid_specific_energy(phi) + 4 / np.pi ** 2) < 0.01


def _random_init(L, m, seed=20221202):
    mask = np.zeros((L, L), np.uint8)                      # every site a gap
    zero = np.zeros(1, np.int64)
    return O.init_angles(np.zeros((L, L), np.float32), mask, L, zero, zero, 1, m, seed)


def test_random_init_energy_matches_independent_uniform_angles():
    """RANDOM init (ARITH §G): i.i.d. phi ~ U[0, 2pi) gives the whole-grid energy
    e = -E[cos((x-y)/2)] = -4/pi^2 (closed form, see test_grid_energy_independent_angles).
    3 SE with the bond covariance of shared sites: var ~ 0.336 + 6 * 0.0384 per bond. A
    narrower range (e.g. [0, pi): e = -8/pi^2) or a constant init fails by > 50 SE."""
    L = 128
    nb = 2 * L * (L - 1)
    se = math.sqrt((0.5 - 16 / math.pi ** 4 + 6 * (2 / math.pi ** 2 - 16 / math.pi ** 4)) / nb)
    for m in (0, 1, 7):
        phi = _random_init(L, m)
        assert abs(O.grid_specific_energy(phi) + 4 / math.pi ** 2) < 3 * se, m


def test_random_init_uniform_distribution_ks_and_moments():
    """RANDOM init draws from U[0, 2pi_f): Kolmogorov-Smirnov against the uniform law
    (scipy), the mean pi and variance (2pi)^2/12 within 4 SE, range inside [0, 2pi_f)."""
    from scipy import stats
    L = 128
    n = L * L
    for m in (0, 1):
        phi = _random_init(L, m).ravel().astype(np.float64)
        assert phi.min() >= 0.0 and phi.max() < float(TWO_PI_F)
        assert stats.kstest(phi, stats.uniform(loc=0.0, scale=float(TWO_PI_F)).cdf).pvalue > 1e-3
        sd = 2 * math.pi / math.sqrt(12)
        assert abs(phi.mean() - math.pi) < 4 * sd / math.sqrt(n)
        assert abs(phi.var() - sd ** 2) < 4 * sd ** 2 * math.sqrt(0.8 / n)


def test_random_init_realizations_and_sites_independent():
    """Different realizations (the two words of one Philox call, m = 0/1, and a different
    counter, m = 2) and neighbouring sites are uncorrelated: |corr| < 4/sqrt(n)."""
    L = 128
    n = L * L
    a, b, c = (_random_init(L, m).ravel() for m in (0, 1, 2))
    for x, y in ((a, b), (a, c), (b, c), (a[:-1], a[1:])):
        assert abs(np.corrcoef(x, y)[0, 1]) < 4 / math.sqrt(n)
    assert not np.array_equal(_random_init(16, 0, seed=1), _random_init(16, 0, seed=2))


def test_openmp_build_bit_identical(calib):
    """The OpenMP timing build (liboracle_omp.so: same-colour rows and smoothing rows split
    over threads) computes the same bits as the single-thread parity build."""
    Tk, ek = calib
    rng = np.random.default_rng(5)
    z = rng.standard_normal((37, 45)).astype(np.float32)
    mask = (rng.random(z.shape) > 0.5).astype(np.uint8)
    cfg = O.OracleConfig(lb=8, rs=2, ns=3, init="random")
    try:
        ref = O.fill(z, mask, cfg, Tk, ek, 4, 6, 11, energy=True, states=True)
        assert O.set_threads(4) >= 2
        par = O.fill(z, mask, cfg, Tk, ek, 4, 6, 11, energy=True, states=True)
    finally:
        O.set_threads(1)
    assert np.array_equal(ref["params"].T.view(np.uint32), par["params"].T.view(np.uint32))
    assert np.array_equal(ref["sim"]["phi"].view(np.uint32), par["sim"]["phi"].view(np.uint32))
    assert np.array_equal(ref["pred"].view(np.uint32), par["pred"].view(np.uint32))
    assert np.array_equal(ref["sim"]["energy"], par["sim"]["energy"])


# --------------------------------------------------- the worked 4x4 lattice (golden)
@pytest.fixture(scope="module")
def worked():
    g = json.load(open(os.path.join(GOLD, "worked_4x4.json")))
    z = np.array([[np.nan if v is None else v for v in row] for row in g["z"]], np.float32)
    mask = (~np.isnan(z)).astype(np.uint8)
    return g, np.nan_to_num(z), mask


def test_worked_lattice_transform_and_block_energies(worked):
    """Hand closed forms of SURVEY c.6 from Eq.(2) and P:108 (bond -> block of its left/top end)."""
    g, z, mask = worked
    phi, lo, hi, st = O.to_angles(z, mask)
    assert (lo, hi, int(mask.sum())) == (g["z_min"], g["z_max"], g["N"])
    SB, NB, SP, NK = O.block_stats(phi, mask, 2)
    assert NB.tolist() == g["block_NSP"]
    for (i, j) in [(0, 0), (0, 1), (1, 1)]:
        assert abs(SB[i, j] * 2.0 ** -32 - g["block_sumcos"][i][j]) < 3e-6
        assert abs(O.block_energy(SB[i, j], NB[i, j]) - g["block_e"][i][j]) < 5e-7
    e, n = O.sample_specific_energy(phi, mask)
    assert n == g["global_NSP"] and abs(e - g["global_e_s"]) < 1e-6
    assert NB.tolist() != g["exclusion_variant_NSP"]  # the SPEC exclusion rule is NOT the one implemented


def test_worked_lattice_temperatures_median_sst(worked, toy_table):
    g, z, mask = worked
    Tk, ek = toy_table
    phi, *_ = O.to_angles(z, mask)
    SB, NB, SP, NK = O.block_stats(phi, mask, 2)
    Tb, na = O.block_temperatures(SB, NB, Tk, ek)
    assert na == 3
    for (i, j) in [(0, 0), (0, 1), (1, 1)]:
        assert abs(Tb[i, j] - g["block_T_toy"][i][j]) < 3e-5
    assert Tb[1, 0] == Tb[0, 0]  # lower median of {0.586, 0.837, 1.724}
    assert abs(Tb[1, 0] - g["median_fallback_T"]) < 3e-5
    T = O.smooth(O.expand(Tb, 4, 4, 2), 1, 1)
    assert abs(T[1, 1] - (6 * Tb[0, 0] + 2 * Tb[0, 1] + Tb[1, 1]) / 9) < 1e-6
    assert T[0, 0] == Tb[0, 0]


def test_worked_lattice_block_mean_init(worked):
    g, z, mask = worked
    phi, *_ = O.to_angles(z, mask)
    SB, NB, SP, NK = O.block_stats(phi, mask, 2)
    init = O.init_angles(phi, mask, 2, SP, NK, 0, 0, 1)
    for key, v in g["block_mean_init"].items():
        r, c = map(int, key.strip("()").split(","))
        assert abs(init[r, c] - v) < 1e-6
    assert np.array_equal(init[mask == 1], phi[mask == 1])


def test_worked_lattice_metropolis_energy_change(worked):
    """dE at gap (2,1) with the neighbours of c.6: proposal pi/2 -> 0, 3pi/2 -> 1 (Eq.(1))."""
    g, z, mask = worked
    phi, *_ = O.to_angles(z, mask)
    phi[2, 1] = np.float32(np.pi)
    assert abs(O.delta_energy(phi, 2, 1, np.float32(np.pi / 2))) < 1e-6
    assert abs(O.delta_energy(phi, 2, 1, np.float32(1.5 * np.pi)) - 1.0) < 1e-6


def test_sin_spec_against_libm():
    """|sin_spec - sin| <= 4e-7 on [-pi_f, pi_f] (libm, fp64); exact zero and odd symmetry."""
    xs = np.linspace(-np.pi, np.pi, 200001).astype(np.float32)
    err = max(abs(O.sin_spec(x) - math.sin(float(x))) for x in xs[::7])
    assert err <= 4e-7
    assert O.sin_spec(0.0) == 0.0
    for x in xs[::997]:
        assert np.float32(O.sin_spec(-x)) == -np.float32(O.sin_spec(x))


def _delta_energy_exact(phi, r, c, prop, q, J):
    """Eq.(1) in fp64 with libm: E(phi') - E(phi) over the in-grid neighbours."""
    Ly, Lx = phi.shape
    d = 0.0
    for rr, cc in ((r - 1, c), (r + 1, c), (r, c - 1), (r, c + 1)):
        if 0 <= rr < Ly and 0 <= cc < Lx:
            pj = float(phi[rr, cc])
            d += J * (math.cos(q * (float(phi[r, c]) - pj)) - math.cos(q * (float(prop) - pj)))
    return d


def test_delta_energy_product_form_matches_eq1():
    """The product-identity dE of ARITH §H equals Eq.(1)'s energy difference (fp64 / libm) to
    fp32 accuracy, on interior, edge and corner sites, for several q and J; the direct form
    (calibration) agrees too; a proposal equal to the current angle gives dE = 0 exactly."""
    rng = np.random.default_rng(21)
    phi = (rng.random((5, 6)) * 2 * np.pi).astype(np.float32)
    worst = 0.0
    for q, J in ((0.5, 1.0), (0.35, 1.3), (0.1, 0.7)):
        for r in range(5):
            for c in range(6):
                for prop in (rng.random(6) * 2 * np.pi).astype(np.float32):
                    ex = _delta_energy_exact(phi, r, c, prop, q, J)
                    worst = max(worst, abs(O.delta_energy(phi, r, c, prop, q, J) - ex) / J)
                    assert abs(O.delta_energy_direct(phi, r, c, prop, q, J) - ex) <= 4e-6 * J
                assert O.delta_energy(phi, r, c, phi[r, c], q, J) == 0.0
    assert worst <= 4e-6, worst
    # a sign error in either sine factor would flip dE: check one hand case as well
    two = np.array([[0.0, np.pi]], np.float32)   # site (0,0) with one neighbour at pi
    assert abs(O.delta_energy(two, 0, 0, np.float32(np.pi), 0.5, 1.0) - (-1.0)) < 1e-6  # cos 0 - cos(-pi/2): -1


# ------------------------------------------------------- block stats special cases
def test_single_block_equals_global_energy():
    """l_b >= L: the one block's e_b equals the global e_s of Eq.(2) (reading R4)."""
    rng = np.random.default_rng(3)
    mask = (rng.random((37, 29)) > 0.4).astype(np.uint8)
    phi = (rng.random((37, 29)) * 2 * np.pi).astype(np.float32) * mask
    SB, NB, SP, NK = O.block_stats(phi, mask, 64)
    e, n = O.sample_specific_energy(phi, mask)
    assert NB[0, 0] == n and NK[0, 0] == mask.sum()
    assert abs(O.block_energy(SB[0, 0], NB[0, 0]) - e) < 1e-6


def test_block_stats_brute_force_partition():
    """Per-block bond sums by enumeration on a ragged grid (l_b does not divide L)."""
    rng = np.random.default_rng(4)
    Ly, Lx, lb = 10, 13, 4
    mask = (rng.random((Ly, Lx)) > 0.3).astype(np.uint8)
    phi = (rng.random((Ly, Lx)) * 2 * np.pi).astype(np.float32) * mask
    SB, NB, SP, NK = O.block_stats(phi, mask, lb)
    ref_n = np.zeros_like(NB); ref_s = np.zeros(NB.shape)
    for r in range(Ly):
        for c in range(Lx):
            if not mask[r, c]:
                continue
            for rr, cc in ((r, c + 1), (r + 1, c)):
                if rr < Ly and cc < Lx and mask[rr, cc]:
                    ref_n[r // lb, c // lb] += 1
                    ref_s[r // lb, c // lb] += math.cos(0.5 * (float(phi[r, c]) - float(phi[rr, cc])))
    assert np.array_equal(NB, ref_n)
    assert np.max(np.abs(SB * 2.0 ** -32 - ref_s)) < 1e-5
    assert NB.shape == (3, 4) and NK.sum() == mask.sum()


# ------------------------------------------------------ inversion / median (exact)
def test_inversion_knots_clamps_and_midpoint(calib):
    Tk, ek = calib
    for k in range(len(Tk)):
        assert O.estimate_temperature(ek[k], Tk, ek) == Tk[k]
    assert O.estimate_temperature(-1.0, Tk, ek) == Tk[0]
    assert O.estimate_temperature(0.5, Tk, ek) == Tk[-1]
    for k in (3, 10, 30):
        e_mid = np.float32((np.float64(ek[k]) + ek[k + 1]) / 2)
        w = (np.float64(e_mid) - ek[k]) / (np.float64(ek[k + 1]) - ek[k])
        ref = Tk[k] + w * (np.float64(Tk[k + 1]) - Tk[k])
        assert abs(O.estimate_temperature(e_mid, Tk, ek) - ref) < 1e-6 * Tk[k + 1]


def test_lower_median():
    assert O.lower_median([0.4, 0.1, 0.2]) == np.float32(0.2)
    assert O.lower_median([0.4, 0.1, 0.3, 0.2]) == np.float32(0.2)
    SB = np.array([0, 0, 0, 0], np.int64); NB = np.array([1, 1, 1, 0], np.int64)
    Tk = np.array([0.1, 0.2, 0.4], np.float32); ek = np.array([-0.9, -0.8, -0.7], np.float32)
    SB[:3] = [int(round(0.9 * 2 ** 32)), int(round(0.8 * 2 ** 32)), int(round(0.7 * 2 ** 32))]
    Tb, na = O.block_temperatures(SB, NB, Tk, ek)
    assert na == 3 and abs(Tb[3] - 0.2) < 1e-6


# ----------------------------------------------------------------- SST smoothing
def test_smoothing_invariants():
    """Uniform field invariant, n_s = 0 identity, range contraction (SPEC sv-temperature)."""
    T = np.full((9, 11), 0.0731, np.float32)
    assert np.array_equal(O.smooth(T, 3, 4), T)
    rng = np.random.default_rng(5)
    T = (rng.random((20, 17)) * 0.5 + 0.01).astype(np.float32)
    assert np.array_equal(O.smooth(T, 2, 0), T)
    S = O.smooth(T, 2, 3)
    assert S.min() >= T.min() and S.max() <= T.max()


def test_smoothing_delta_field_hand_convolution():
    """Delta at the centre of 5x5, r_s = 1: the 9 sites of its 3x3 neighbourhood get 1/9;
    delta at the corner: (0,0) -> 1/4, (0,1) -> 1/6, (1,1) -> 1/9 (clipped window counts)."""
    T = np.zeros((5, 5), np.float32); T[2, 2] = 1
    S = O.smooth(T, 1, 1)
    ref = np.zeros((5, 5)); ref[1:4, 1:4] = 1 / 9
    assert np.max(np.abs(S - ref)) < 1e-7
    T = np.zeros((5, 5), np.float32); T[0, 0] = 1
    S = O.smooth(T, 1, 1)
    assert abs(S[0, 0] - 0.25) < 1e-7 and abs(S[0, 1] - 1 / 6) < 1e-7 and abs(S[1, 1] - 1 / 9) < 1e-7
    assert S[2, 2] == 0


# -------------------------------------------------------------- Metropolis pins
def _stationary(neigh, T, q=0.5, n=200001):
    x = np.linspace(0, 2 * np.pi, n)
    logp = sum(np.cos(q * (x - v)) for v in neigh) / T
    p = np.exp(logp - logp.max())
    p /= np.trapezoid(p, x)
    return x, p


def _acceptance_uniform_proposal(p, dx):
    # A = (1/2pi) * integral integral min(p(x), p(y)) dx dy, via the sorted-sum identity
    a = np.sort(p)
    n = len(a)
    k = np.arange(1, n + 1)
    return float(np.sum(a * (2 * (n - k) + 1)) * dx * dx / (2 * np.pi))


@pytest.mark.slow
def test_isolated_gap_site_matches_quadrature():
    """A gap site with 4 frozen neighbours is a 1-D Metropolis chain whose stationary density is
    exp(sum_j cos q(phi - phi_j) / T) on [0, 2pi] (Eq.(1) Gibbs measure); its mean and the
    acceptance rate of the uniform proposal follow by quadrature (brute force)."""
    neigh = [1.0, 1.5, 2.2, 4.0]
    T = 0.3
    x, p = _stationary(neigh, T)
    mean_q = float(np.trapezoid(x * p, x))
    acc_q = _acceptance_uniform_proposal(p, x[1] - x[0])
    phi = np.zeros((3, 3), np.float32)
    phi[0, 1], phi[2, 1], phi[1, 0], phi[1, 2] = neigh  # N, S, W, E
    mask = np.ones((3, 3), np.uint8); mask[1, 1] = 0
    beta = np.full((3, 3), 1 / T, np.float32)
    means, accs = [], []
    for m in range(16):
        ph = phi.copy(); ph[1, 1] = np.float32(np.pi)
        O.run_chain(ph, mask, beta, 1, 101, m=m, seed=11)  # burn-in
        sp, na = O.run_chain(ph, mask, beta, 101, 25101, m=m, seed=11)
        means.append(sp[1, 1] / 25000); accs.append(na / 25000)
    se_m = np.std(means) / np.sqrt(len(means)); se_a = np.std(accs) / np.sqrt(len(accs))
    assert abs(np.mean(means) - mean_q) < 5 * se_m + 1e-3
    assert abs(np.mean(accs) - acc_q) < 5 * se_a + 1e-3
    assert abs(mean_q - 2.12757) < 2e-4 and abs(acc_q - 0.30784) < 2e-4


@pytest.mark.slow
def test_coupled_gaps_4x4_detailed_balance_brute_force():
    """4x4 lattice, uniform T, two ADJACENT gap sites (1,1) [colour A] and (1,2) [colour B]: the
    checkerboard chain must sample the joint Gibbs density pi(x, y) (detailed balance of each
    colour update). <x>, <y> and each site's acceptance rate by 2-D quadrature (brute force)."""
    rng = np.random.default_rng(7)
    phi = (rng.random((4, 4)) * 2 * np.pi).astype(np.float32)
    mask = np.ones((4, 4), np.uint8); mask[1, 1] = 0; mask[1, 2] = 0
    T = 0.4
    q = 0.5
    n = 721
    g = np.linspace(0, 2 * np.pi, n)
    f1 = [phi[0, 1], phi[2, 1], phi[1, 0]]  # fixed neighbours of (1,1): N, S, W
    f2 = [phi[0, 2], phi[2, 2], phi[1, 3]]  # fixed neighbours of (1,2): N, S, E
    a = sum(np.cos(q * (g - v)) for v in f1)
    b = sum(np.cos(q * (g - v)) for v in f2)
    logp = (a[:, None] + b[None, :] + np.cos(q * (g[:, None] - g[None, :]))) / T
    P = np.exp(logp - logp.max()); dx = g[1] - g[0]
    P /= P.sum() * dx * dx
    ex = float((g[:, None] * P).sum() * dx * dx); ey = float((g[None, :] * P).sum() * dx * dx)
    # acceptance of site 1 given y: independence sampler on p(x|y); average over the y-marginal
    py = P.sum(0) * dx
    acc1 = sum(py[j] * dx * _acceptance_uniform_proposal(P[:, j] / (P[:, j].sum() * dx), dx) for j in range(0, n, 4)) * 4
    px = P.sum(1) * dx
    acc2 = sum(px[i] * dx * _acceptance_uniform_proposal(P[i, :] / (P[i, :].sum() * dx), dx) for i in range(0, n, 4)) * 4
    beta = np.full((4, 4), 1 / T, np.float32)
    mx, my, na_all = [], [], []
    for m in range(12):
        ph = phi.copy(); ph[1, 1] = 1.0; ph[1, 2] = 5.0
        O.run_chain(ph, mask, beta, 1, 101, m=m, seed=5)
        sp, na = O.run_chain(ph, mask, beta, 101, 20101, m=m, seed=5)
        mx.append(sp[1, 1] / 20000); my.append(sp[1, 2] / 20000); na_all.append(na / 40000)
    se = lambda v: np.std(v) / np.sqrt(len(v))
    assert abs(np.mean(mx) - ex) < 5 * se(mx) + 2e-3
    assert abs(np.mean(my) - ey) < 5 * se(my) + 2e-3
    assert abs(np.mean(na_all) - (acc1 + acc2) / 2) < 5 * se(na_all) + 2e-3


def test_high_temperature_accepts_everything():
    """T -> infinity: exp(-dE/T) -> 1, acceptance -> 1 (SPEC metropolis_sweep)."""
    rng = np.random.default_rng(8)
    phi = (rng.random((8, 8)) * 2 * np.pi).astype(np.float32)
    mask = (rng.random((8, 8)) > 0.5).astype(np.uint8)
    beta = np.full((8, 8), 1e-6, np.float32)
    _, na = O.run_chain(phi, mask, beta, 1, 201)
    assert na / (200 * (mask == 0).sum()) > 0.999


def test_no_free_sites_is_noop():
    phi = np.full((4, 4), 1.0, np.float32)
    before = phi.copy()
    n = O.sweep(phi, np.ones((4, 4), np.uint8), np.ones((4, 4), np.float32), 1, 0, 1)
    assert n == 0 and np.array_equal(phi, before)


def test_low_temperature_relaxes_to_neighbours():
    """T = 1e-4, 4 neighbours at pi: after 500 sweeps the free site is within 0.05 rad of pi
    (uniform proposal: P(hit the 0.1-rad window in 500 tries) = 0.9997; SURVEY c.4 on S:249)."""
    phi = np.full((3, 3), np.float32(np.pi)); phi[1, 1] = 0.3
    mask = np.ones((3, 3), np.uint8); mask[1, 1] = 0
    O.run_chain(phi, mask, np.full((3, 3), 1e4, np.float32), 1, 501, seed=3)
    assert abs(phi[1, 1] - np.pi) < 0.05


# ---------------------------------------------------------------- invariants
def _problem(L=24, p=0.5, seed=0):
    from inputs.synth import make_problem
    truth, z, mask = make_problem(L, p, seed_field=seed + 1, seed_mask=seed + 2, corr_len=6.0)
    return truth, z, mask


def test_pipeline_invariants(calib):
    """Frozen samples bitwise unchanged, phi in [0, 2pi_f], predictions in [z_min, z_max],
    samples returned bitwise (SPEC invariants)."""
    Tk, ek = calib
    truth, z, mask = _problem()
    cfg = O.OracleConfig(lb=8, rs=1, ns=2)
    res = O.fill(z, mask, cfg, Tk, ek, M=4, S=10, seed=9, states=True)
    p = res["params"]
    phis = res["sim"]["phi"]
    for r in range(4):
        assert np.array_equal(phis[r][mask == 1].view(np.uint32), p.phi0[mask == 1].view(np.uint32))
        assert phis[r].min() >= 0 and phis[r].max() <= TWO_PI_F
    pred = res["pred"]
    assert np.array_equal(pred[mask == 1].view(np.uint32), z[mask == 1].view(np.uint32))
    assert pred[mask == 0].min() >= p.zmin and pred[mask == 0].max() <= p.zmax


def test_parity_safety_order_independence(calib):
    """Same-colour sites never read each other's new value: visiting them in reverse order gives
    a bit-identical sweep (SPEC parity safety)."""
    truth, z, mask = _problem(L=20)
    phi, lo, hi, _ = O.to_angles(np.nan_to_num(z), mask)
    rng = np.random.default_rng(1)
    phi[mask == 0] = (rng.random(int((mask == 0).sum())) * 2 * np.pi).astype(np.float32)
    beta = (rng.random(phi.shape) * 20 + 1).astype(np.float32)
    a, b = phi.copy(), phi.copy()
    for s in range(1, 6):
        O.sweep(a, mask, beta, s, 3, 77, reverse=False)
        O.sweep(b, mask, beta, s, 3, 77, reverse=True)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_determinism_and_realization_sharding(calib):
    """Counter-based RNG: same inputs -> identical chains; realizations [0,M) == [0,k) + [k,M)."""
    Tk, ek = calib
    truth, z, mask = _problem(L=16)
    cfg = O.OracleConfig(lb=8, rs=1, ns=1)
    p = O.parameters(z, mask, cfg, Tk, ek)
    full = O.simulate(p, mask, cfg, 6, 8, 123, states=True)
    again = O.simulate(p, mask, cfg, 6, 8, 123, states=True)
    assert np.array_equal(full["phi"], again["phi"])
    a = O.simulate(p, mask, cfg, 6, 8, 123, m_begin=0, m_end=3, states=True)
    b = O.simulate(p, mask, cfg, 6, 8, 123, m_begin=3, m_end=6, states=True)
    assert np.array_equal(np.concatenate([a["phi"], b["phi"]]), full["phi"])
    assert np.allclose(a["acc"] + b["acc"], full["acc"], rtol=1e-13, atol=0)
    other = O.simulate(p, mask, cfg, 6, 8, 124, states=True)
    assert not np.array_equal(other["phi"], full["phi"])


def test_uniform_T_limit_mpr(calib):
    """l_b >= L reproduces the uniform-T MPR method: a single temperature everywhere, equal to the
    inversion of the global e_s (SPEC BST degeneracy)."""
    Tk, ek = calib
    truth, z, mask = _problem(L=20)
    cfg = O.OracleConfig(lb=64, rs=2, ns=3)
    p = O.parameters(z, mask, cfg, Tk, ek)
    assert np.unique(p.T).size == 1
    phi, *_ = O.to_angles(np.nan_to_num(z), mask)
    e, _ = O.sample_specific_energy(phi, mask)
    assert abs(p.T[0, 0] - O.estimate_temperature(np.float32(e), Tk, ek)) < 1e-5 * p.T[0, 0]


# ------------------------------------------------------------------ metrics
def test_score_hand_values():
    """AAE / RASE of Eq.(3): errors {+3, -4} -> 3.5, sqrt(12.5)."""
    truth = np.array([[10, 20, 5]], np.float32)
    pred = np.array([[7, 24, 5]], np.float32)
    mask = np.array([[0, 0, 1]], np.uint8)
    s = O.score(pred, truth, mask)
    assert s["mae"] == 3.5 and abs(s["rmse"] - math.sqrt(12.5)) < 1e-12
    assert abs(s["mare"] - (3 / 10 + 4 / 20) / 2) < 1e-12
    assert O.score(truth, truth, mask)["rmse"] == 0


def test_window_oracle_equals_full_oracle(calib):
    """The full-size sampling device (oracle.WindowOracle) reproduces the full-grid oracle
    bit for bit inside its window (locality of the smoothing and of the Metropolis chain)."""
    Tk, ek = calib
    from inputs.synth import make_problem
    truth, z, mask = make_problem(70, 0.5, Lx=83, corr_len=6.0)
    for cfg in (O.OracleConfig(lb=8, rs=2, ns=2), O.OracleConfig(lb=16, rs=1, ns=3, init="random")):
        p = O.parameters(z, mask, cfg, Tk, ek)
        full = O.simulate(p, mask, cfg, 3, 5, 77, states=True)["phi"]
        W = O.WindowOracle(z, mask, cfg, Tk, ek)
        for (r0, r1, c0, c1) in [(30, 38, 40, 47), (0, 6, 0, 9), (62, 70, 75, 83)]:
            assert np.array_equal(W.T_window(r0, r1, c0, c1), p.T[r0:r1, c0:c1])
            got = W.states(r0, r1, c0, c1, [0, 2], 5, 77)
            assert np.array_equal(got.view(np.uint32), full[[0, 2], r0:r1, c0:c1].view(np.uint32))


# --------------------------------------------------- ARITH §J/§K (row f1) pins
def test_fixed_point_energy_equals_libm_definition():
    """E_fx (ARITH §J) reproduces the fp64/libm whole-grid energy to cos_spec accuracy."""
    rng = np.random.default_rng(9)
    for L in (17, 64):
        phi = (rng.random((L, L + 3)) * 2 * np.pi).astype(np.float32)
        e_fx = O.energy_from_fx(O.grid_energy_fx(phi), L + 3, L)
        assert abs(e_fx - O.grid_specific_energy(phi)) < 4e-7
    phi = np.full((9, 9), 2.0, np.float32)
    assert O.energy_from_fx(O.grid_energy_fx(phi), 9, 9) == -1.0


def test_equilibrium_test_against_numpy_fit():
    """The ARITH §K slope test decides like an independent numpy least-squares fit
    (np.polyfit) wherever the decision is not within rounding of the threshold."""
    rng = np.random.default_rng(3)
    assert O.equilibrium_test(np.full(20, -0.93))
    assert not O.equilibrium_test(-0.9 - 1e-3 * np.arange(20))
    assert O.equilibrium_test(-0.9 + 1e-3 * np.arange(20))
    agree = 0
    for _ in range(400):
        slope = rng.normal(0, 2e-4)
        y = -0.95 + slope * np.arange(20) + rng.normal(0, 1e-3, 20)
        b, a = np.polyfit(np.arange(20), y, 1)
        tau = 2 * np.sqrt(np.sum((y - a - b * np.arange(20)) ** 2) / 18) / 20
        if abs(b + tau) < 1e-9:
            continue
        assert O.equilibrium_test(y) == (b >= -tau)
        agree += 1
    assert agree > 390


def test_adaptive_protocol_invariants(calib):
    """Equilibrium is declared only at check sweeps n_fit + k n_f (first at 25) or at
    the cap; each realization averages exactly n_avg sweeps (predictions in range); the
    per-block-average start is not slower than the random start on average."""
    Tk, ek = calib
    from inputs.synth import make_problem
    truth, z, mask = make_problem(40, 0.5, corr_len=6.0)
    res = {}
    for init in ("block_mean", "random"):
        cfg = O.OracleConfig(init=init, n_avg=2)
        p = O.parameters(z, mask, cfg, Tk, ek)
        r = O.simulate_adaptive(p, mask, cfg, 6, 21, n_fit=20, n_f=5, S_max=200, energy=True)
        for s in r["s_eq"]:
            assert s > 0 and s >= 25 and (s - 20) % 5 == 0
        pred = O.predict(np.nan_to_num(z), mask, r["acc"], 6, 2, p.zmin, p.zmax, 0)
        assert pred[mask == 0].min() >= p.zmin and pred[mask == 0].max() <= p.zmax
        assert np.all(r["energy"][:, 0] > r["energy"][:, 20])  # relaxation toward equilibrium
        res[init] = r["s_eq"].mean()
    assert res["block_mean"] <= res["random"]
    cfg = O.OracleConfig(n_avg=3)
    p = O.parameters(z, mask, cfg, Tk, ek)
    r = O.simulate_adaptive(p, mask, cfg, 2, 21, n_fit=20, n_f=5, S_max=15)
    assert r["s_eq"].tolist() == [-12, -12]


# ------------------------------------------------------ row f3: double checkerboard
def test_dc_with_one_tile_is_sc():
    """With a single tile (l_b >= L) the DC sweep is the SC sweep, bit for bit."""
    rng = np.random.default_rng(12)
    phi = (rng.random((14, 11)) * 2 * np.pi).astype(np.float32)
    mask = (rng.random((14, 11)) > 0.5).astype(np.uint8)
    beta = (rng.random((14, 11)) * 30 + 1).astype(np.float32)
    a, b = phi.copy(), phi.copy()
    for s in range(1, 6):
        O.sweep(a, mask, beta, s, 4, 9)
        O.sweep_dc(b, mask, beta, s, 4, 9, lb=64)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    c = phi.copy()
    for s in range(1, 6):
        O.sweep_dc(c, mask, beta, s, 4, 9, lb=2)
    assert not np.array_equal(a, c)  # with several tiles the order (and chain) differs


@pytest.mark.slow
def test_dc_coupled_gaps_detailed_balance():
    """The DC order samples the same Gibbs density: two adjacent gaps in different tiles
    (l_b = 2) of a 4x4 lattice, means vs 2-D quadrature (brute force)."""
    rng = np.random.default_rng(7)
    phi = (rng.random((4, 4)) * 2 * np.pi).astype(np.float32)
    mask = np.ones((4, 4), np.uint8); mask[1, 1] = 0; mask[1, 2] = 0
    T, q, n = 0.4, 0.5, 721
    g = np.linspace(0, 2 * np.pi, n)
    a = sum(np.cos(q * (g - v)) for v in [phi[0, 1], phi[2, 1], phi[1, 0]])
    b = sum(np.cos(q * (g - v)) for v in [phi[0, 2], phi[2, 2], phi[1, 3]])
    logp = (a[:, None] + b[None, :] + np.cos(q * (g[:, None] - g[None, :]))) / T
    Pd = np.exp(logp - logp.max()); dx = g[1] - g[0]
    Pd /= Pd.sum() * dx * dx
    ex = float((g[:, None] * Pd).sum() * dx * dx); ey = float((g[None, :] * Pd).sum() * dx * dx)
    beta = np.full((4, 4), 1 / T, np.float32)
    mx, my = [], []
    for m in range(8):
        ph = phi.copy(); ph[1, 1] = 1.0; ph[1, 2] = 5.0
        sx = sy = 0.0
        for s in range(1, 6001):
            O.sweep_dc(ph, mask, beta, s, m, 5, lb=2)
            if s > 100:
                sx += ph[1, 1]; sy += ph[1, 2]
        mx.append(sx / 5900); my.append(sy / 5900)
    se = lambda v: np.std(v) / np.sqrt(len(v))  # noqa: E731
    assert abs(np.mean(mx) - ex) < 5 * se(mx) + 3e-3
    assert abs(np.mean(my) - ey) < 5 * se(my) + 3e-3


def test_equilibrium_slope_tolerance():
    """slope_tol (SPEC's configurable tolerance) relaxes the rule to b >= -max(tau, slope_tol)."""
    y = -0.95 - 1e-4 * np.arange(20)
    assert not O.equilibrium_test(y)
    assert not O.equilibrium_test(y, slope_tol=5e-5)
    assert O.equilibrium_test(y, slope_tol=2e-4)


# ------------------------------------------------ R22: the derived slope tolerance
def test_derived_slope_tolerance_hand_values():
    """A row [0, 0, 2pi] (q = 1/2): bond cosines 1 and cos(-pi) = -1, mean 0, variance 1,
    N_SP = 2 -> SE = 1/sqrt(2), tau = SE / n_fit; a constant field (variance 0) -> 0 exactly;
    no sample bond -> 0."""
    phi = np.array([[0.0, 0.0, float(TWO_PI_F)]], np.float32)
    mask = np.ones((1, 3), np.uint8)
    assert abs(O.derived_slope_tol(phi, mask, 0.5, 20) - math.sqrt(0.5) / 20) < 1e-7
    assert O.derived_slope_tol(np.full((5, 6), 1.3, np.float32), np.ones((5, 6), np.uint8), 0.5, 20) == 0.0
    iso = np.zeros((4, 4), np.uint8)
    iso[0, 0] = iso[2, 2] = 1
    assert O.derived_slope_tol(np.ones((4, 4), np.float32), iso, 0.5, 20) == 0.0


def test_derived_slope_tolerance_matches_libm_sample_sd():
    """The fixed-point definition equals the fp64/libm one, sd(cos q(phi_i - phi_j)) /
    sqrt(N_SP) / n_fit over every unordered sample pair once, to 1e-6 relative."""
    rng = np.random.default_rng(11)
    for p_gap, q, n_fit in ((0.3, 0.5, 20), (0.7, 0.37, 8)):
        phi = (rng.random((40, 33)) * 2 * np.pi).astype(np.float32)
        mask = (rng.random(phi.shape) > p_gap).astype(np.uint8)
        b = []
        for r in range(40):
            for c in range(33):
                if not mask[r, c]:
                    continue
                if c + 1 < 33 and mask[r, c + 1]:
                    b.append(math.cos(q * (float(phi[r, c]) - float(phi[r, c + 1]))))
                if r + 1 < 40 and mask[r + 1, c]:
                    b.append(math.cos(q * (float(phi[r, c]) - float(phi[r + 1, c]))))
        b = np.array(b)
        ref = b.std() / math.sqrt(b.size) / n_fit
        got = O.derived_slope_tol(phi, mask, q, n_fit)
        assert abs(got - ref) <= 1e-6 * ref, (got, ref)


def test_adaptive_with_derived_tolerance_uses_it(calib):
    """slope_tol = "derived" in the oracle's adaptive protocol equals passing the derived
    value explicitly."""
    from inputs.synth import make_problem
    truth, z, mask = make_problem(40, 0.4, corr_len=6.0)
    cfg = O.OracleConfig(lb=8)
    p = O.parameters(z, mask, cfg, *calib)
    tol = O.derived_slope_tol(p.phi0, mask, cfg.q, 10)
    assert tol > 0
    a = O.simulate_adaptive(p, mask, cfg, 4, 5, n_fit=10, n_f=3, S_max=80, slope_tol="derived")
    b = O.simulate_adaptive(p, mask, cfg, 4, 5, n_fit=10, n_f=3, S_max=80, slope_tol=tol)
    assert a["s_eq"].tolist() == b["s_eq"].tolist()
    assert np.array_equal(a["acc"], b["acc"])


def test_sst_division_with_hoisted_reciprocal_is_ieee(tmp_path):
    """The GPU's SST pass divides unclipped window sums by their count as q0 = a RN(1/b),
    q = fma(a - b q0, RN(1/b), q0) (Markstein): equal to the IEEE quotient the oracle uses
    (ARITH §F) for every window count of r_s <= 8 and 3M random sums per count."""
    import subprocess
    src = os.path.join(os.path.dirname(__file__), "native", "markstein_div.c")
    exe = str(tmp_path / "markstein_div")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-o", exe, src, "-lm"])
    out = subprocess.run([exe, "3000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.strip().startswith("0 mismatches")


@pytest.mark.slow
def test_checkerboard_chain_matches_sequential_random_order_metropolis(tmp_path):
    """SPEC acceptance criterion 6 (oracle equivalence): on an 8x8 lattice at a fixed T the
    oracle's checkerboard chain (independence proposal, ARITH §H, colour A then B) and an
    independent random-order single-site Metropolis sampler (fp64/libm, its own RNG,
    tests/native/sequential_metropolis.c) have the same stationary mean specific energy:
    within 4 combined standard errors over independent chains, with 12 frozen samples and
    at two temperatures (the tolerance resolves a ~3 % temperature error)."""
    import subprocess
    exe = str(tmp_path / "seqmc")
    src = os.path.join(os.path.dirname(__file__), "native", "sequential_metropolis.c")
    subprocess.check_call(["gcc", "-O2", "-o", exe, src, "-lm"])
    rng = np.random.default_rng(2212)
    L = 8
    mask = np.zeros((L, L), np.uint8)
    mask.ravel()[rng.choice(L * L, 12, replace=False)] = 1
    phi_known = (rng.random((L, L)) * 2 * np.pi).astype(np.float32)
    phi_init = np.where(mask != 0, phi_known, np.float32(0)).astype(np.float32)
    chains, burn, sweeps = 8, 300, 6000
    for T in (0.35, 1.2):
        # oracle checkerboard chains
        beta = np.full((L, L), np.float32(1.0) / np.float32(T), np.float32)
        means = []
        for m in range(chains):
            ph = phi_init.copy()
            es = 0.0
            for s in range(1, burn + sweeps + 1):
                O.sweep(ph, mask, beta, s, m, 77)
                if s > burn:
                    es += O.grid_specific_energy(ph)
            means.append(es / sweeps)
        cb, cb_se = float(np.mean(means)), float(np.std(means, ddof=1) / np.sqrt(chains))
        # independent sequential sampler
        lines = [f"{L} {L} {T!r} 0.5 1.0 {chains} {burn} {sweeps} 5"]
        lines += [f"{int(mask.ravel()[i])} {float(phi_init.ravel()[i])!r}" for i in range(L * L)]
        out = subprocess.run([exe], input="\n".join(lines) + "\n", capture_output=True, text=True, check=True).stdout
        seq = np.array([float(x) for x in out.split()])
        sq, sq_se = float(seq.mean()), float(seq.std(ddof=1) / np.sqrt(len(seq)))
        tol = 4.0 * math.hypot(cb_se, sq_se)
        assert abs(cb - sq) < tol, f"T={T}: checkerboard {cb:.5f} +- {cb_se:.1e} vs sequential {sq:.5f} +- {sq_se:.1e}"
    # sensitivity (measured when the test was written): the sequential sampler at T = 0.36
    # instead of 0.35 lands 1.7 tolerances away, at 1.25 instead of 1.2 3.2 tolerances


@pytest.mark.slow
def test_sin_and_exp_spec_exhaustive_error_bounds(tmp_path):
    """ARITH §B2 / §C accuracy statements over EVERY fp32 argument (not a sample): the
    degree-11 sin_spec stays within 3.9e-7 of libm on [0, pi_f] (3.84e-7 when the contract
    was frozen) and exp_spec within 1.1 ulp on [-80, 0] (1.05 ulp)."""
    import subprocess
    exe = str(tmp_path / "spec_exhaustive")
    src = os.path.join(os.path.dirname(__file__), "native", "spec_exhaustive.c")
    libdir = os.path.dirname(O.build())
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-o", exe, src, "-L", libdir, "-l:liboracle.so",
                           f"-Wl,-rpath,{libdir}", "-lm"])
    es, ee = map(float, subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split())
    assert es <= 3.9e-7, es
    assert ee <= 1.1, ee
