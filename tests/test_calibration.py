"""Pins of the e(T) calibration curve (reading R2: the T <-> e relation that the energy
matching of PAPER.md:90 inverts) against closed forms, and of the oracle's unconditional
simulation that produced it (scripts/make_calibration.py)."""
import math

import numpy as np
import pytest

import oracle as O

E_INF = -4 / math.pi ** 2                       # independent angles, q = 1/2
C_HIGH = 0.5 + 12 / math.pi ** 2 - 112 / math.pi ** 4  # first-order 1/T coefficient


def harmonic(T, L):
    """Low-T equipartition on an open L x L lattice: (L^2 - 1) modes x T/2 over 2L(L-1) bonds."""
    return -1 + T * (L + 1) / (4 * L)


def test_table_shape_and_monotonicity(calib):
    T, e = calib
    assert len(T) == 48 and T[0] == np.float32(1e-4) and abs(T[-1] - 10) < 1e-5
    assert np.all(np.diff(T) > 0) and np.all(np.diff(e) > 0)
    assert e[0] > -1 and e[-1] < E_INF


def test_table_low_temperature_closed_form(calib):
    """e(T) = -1 + T(L+1)/(4L) + O(T^2) for T << 1 (L = 128, the table's lattice)."""
    T, e = calib
    for t, v in zip(T, e):
        if t <= 0.01:
            assert abs(v - harmonic(float(t), 128)) < 0.02 * float(t) + 3e-7


def test_table_high_temperature_trend(calib):
    """At T = 10 the first-order expansion -4/pi^2 - c/T is within 0.01 (SURVEY c.4)."""
    T, e = calib
    assert abs(e[-1] - (E_INF - C_HIGH / float(T[-1]))) < 0.01


@pytest.mark.parametrize("L,T", [(16, 0.01), (16, 0.05)])
def test_unconditional_low_T_harmonic(L, T):
    es = [O.unconditional_energy(L, T, init="ordered", n_eq=300, n_meas=3000, seed=7, m=m) for m in range(4)]
    se = np.std(es) / 2 + 2e-6
    assert abs(np.mean(es) - harmonic(T, L)) < 5 * se


def test_unconditional_high_T_expansion():
    es = [O.unconditional_energy(24, 100.0, init="random", n_eq=50, n_meas=1500, seed=7, m=m) for m in range(4)]
    ref = E_INF - C_HIGH / 100.0
    assert abs(np.mean(es) - ref) < 5 * np.std(es) / 2 + 3e-4


def test_random_and_ordered_init_agree():
    """The equilibrium energy does not depend on the initial state (no hysteresis at T = 0.3)."""
    a = O.unconditional_energy(24, 0.3, init="ordered", n_eq=400, n_meas=1500, seed=3)
    b = O.unconditional_energy(24, 0.3, init="random", n_eq=400, n_meas=1500, seed=3)
    assert abs(a - b) < 5e-3
