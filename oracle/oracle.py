"""ctypes + numpy wrapper of oracle/mpr_oracle.c (TEST INFRASTRUCTURE ONLY).

Each wrapper names the SPEC-style operation it realises and the paper passage it
follows (P:<line> = /root/reference/PAPER.md). The arithmetic lives in the C file;
this module only marshals arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]

TWO_PI_F = float(np.float32(2.0 * np.pi))


def _build_one(path, extra):
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC):
        tmp = path + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, *extra, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, path)
    return path


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no FMA contraction): liboracle.so (single
    thread, parity) and liboracle_omp.so (the same source with -fopenmp, timing only)."""
    if force:
        for p in (_LIB, _LIB_OMP):
            if os.path.exists(p):
                os.remove(p)
    _build_one(_LIB_OMP, ["-fopenmp"])
    return _build_one(_LIB, [])


_lib = None
_libs = {}


def _load(path):
    if path not in _libs:
        L = C.CDLL(path)
        _declare(L)
        _libs[path] = L
    return _libs[path]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = _load(_LIB)
    return _lib


def set_threads(n: int | None) -> int:
    """Select the build the wrappers below call: n None or 1 -> the single-thread library
    (parity runs); n > 1 (or 0 = all cores) -> the OpenMP build with n threads (timing the
    oracle on the host cores). Returns the thread count in use."""
    global _lib
    build()
    if n is None or n == 1:
        _lib = _load(_LIB)
        return 1
    _lib = _load(_LIB_OMP)
    return int(_lib.oracle_set_threads(int(n) if n > 0 else (os.cpu_count() or 1)))


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


class _Cfg(C.Structure):
    _fields_ = [("q", C.c_float), ("J", C.c_float), ("lb", C.c_int), ("rs", C.c_int),
                ("ns", C.c_int), ("init_mode", C.c_int), ("n_avg", C.c_int), ("order", C.c_int)]


def _declare(L):
    L.oracle_set_threads.argtypes = [C.c_int]; L.oracle_set_threads.restype = C.c_int
    L.oracle_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
    L.oracle_uniform.argtypes = [C.c_uint32]; L.oracle_uniform.restype = C.c_float
    L.oracle_cos_spec.argtypes = [C.c_float]; L.oracle_cos_spec.restype = C.c_float
    L.oracle_sin_spec.argtypes = [C.c_float]; L.oracle_sin_spec.restype = C.c_float
    L.oracle_exp_spec.argtypes = [C.c_float]; L.oracle_exp_spec.restype = C.c_float
    L.oracle_bond_energy.argtypes = [C.c_float] * 4; L.oracle_bond_energy.restype = C.c_float
    L.oracle_transform.argtypes = [_f32p, _u8p, C.c_int64, C.POINTER(C.c_float),
                                   C.POINTER(C.c_float), _f32p]
    L.oracle_transform.restype = C.c_int
    L.oracle_sample_specific_energy.argtypes = [_f32p, _u8p, C.c_int, C.c_int, C.c_float,
                                                C.POINTER(C.c_int64)]
    L.oracle_sample_specific_energy.restype = C.c_double
    L.oracle_grid_specific_energy.argtypes = [_f32p, C.c_int, C.c_int, C.c_float]
    L.oracle_grid_specific_energy.restype = C.c_double
    L.oracle_block_stats.argtypes = [_f32p, _u8p, C.c_int, C.c_int, C.c_int, C.c_float,
                                     _i64p, _i64p, _i64p, _i64p]
    L.oracle_block_energy.argtypes = [C.c_int64, C.c_int64]; L.oracle_block_energy.restype = C.c_float
    L.oracle_estimate_temperature.argtypes = [C.c_float, _f32p, _f32p, C.c_int]
    L.oracle_estimate_temperature.restype = C.c_float
    L.oracle_lower_median.argtypes = [_f32p, C.c_int64]; L.oracle_lower_median.restype = C.c_float
    L.oracle_block_temperatures.argtypes = [_i64p, _i64p, C.c_int64, _f32p, _f32p, C.c_int, _f32p]
    L.oracle_block_temperatures.restype = C.c_int64
    L.oracle_expand.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p]
    L.oracle_smooth.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int]
    L.oracle_init.argtypes = [_f32p, _u8p, C.c_int, C.c_int, C.c_int, _i64p, _i64p, C.c_int,
                              C.c_int64, C.c_uint64]
    L.oracle_sweep.argtypes = [_f32p, _u8p, _f32p, C.c_int, C.c_int, C.c_float, C.c_float,
                               C.c_uint32, C.c_int64, C.c_uint64, C.c_int]
    L.oracle_sweep.restype = C.c_int64
    L.oracle_delta_energy.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float,
                                      C.c_float]
    L.oracle_delta_energy.restype = C.c_float
    L.oracle_delta_energy_direct.argtypes = L.oracle_delta_energy.argtypes
    L.oracle_delta_energy_direct.restype = C.c_float
    L.oracle_run_chain.argtypes = [_f32p, _u8p, _f32p, C.c_int, C.c_int, C.c_float, C.c_float, C.c_uint32,
                                   C.c_uint32, C.c_int64, C.c_uint64, C.c_void_p]
    L.oracle_run_chain.restype = C.c_int64
    L.oracle_half_sweep_rows.argtypes = [_f32p, _u8p, _f32p, C.c_int, C.c_int, C.c_float, C.c_float, C.c_uint32,
                                         C.c_int64, C.c_uint64, C.c_int, C.c_int, C.c_int]
    L.oracle_half_sweep_rows.restype = C.c_int64
    L.oracle_sweep_dc.argtypes = [_f32p, _u8p, _f32p, C.c_int, C.c_int, C.c_float, C.c_float, C.c_uint32,
                                  C.c_int64, C.c_uint64, C.c_int]
    L.oracle_sweep_dc.restype = C.c_int64
    L.oracle_simulate_window.argtypes = [_f32p, _u8p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, _i64p, _i64p, C.c_int, C.c_float, C.c_float, C.c_int64,
                                         C.c_int, C.c_uint64, _f32p]
    L.oracle_parameters.argtypes = [_f32p, _u8p, C.c_int, C.c_int, C.POINTER(_Cfg), _f32p, _f32p,
                                    C.c_int, _f32p, _f32p, _f32p, C.POINTER(C.c_float),
                                    C.POINTER(C.c_float), _i64p, _i64p, C.c_void_p]
    L.oracle_parameters.restype = C.c_int
    L.oracle_simulate.argtypes = [_f32p, _u8p, _f32p, C.c_int, C.c_int, C.POINTER(_Cfg), _i64p,
                                  _i64p, C.c_int64, C.c_int64, C.c_int, C.c_uint64, _f64p,
                                  C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
    L.oracle_predict.argtypes = [_f32p, _u8p, C.c_int64, _f64p, C.c_int64, C.c_int, C.c_float,
                                 C.c_float, C.c_int, _f32p]
    L.oracle_unconditional_energy.argtypes = [C.c_int, C.c_float, C.c_float, C.c_int, C.c_int,
                                              C.c_int, C.c_uint64, C.c_int64, C.c_void_p, C.c_float]
    L.oracle_unconditional_energy.restype = C.c_double
    L.oracle_score.argtypes = [_f32p, _f32p, _u8p, C.c_int64, C.POINTER(C.c_double),
                               C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.oracle_grid_energy_fx.argtypes = [_f32p, C.c_int, C.c_int, C.c_float]
    L.oracle_grid_energy_fx.restype = C.c_int64
    L.oracle_energy_from_fx.argtypes = [C.c_int64, C.c_int, C.c_int]
    L.oracle_energy_from_fx.restype = C.c_double
    L.oracle_derived_slope_tol.argtypes = [_f32p, _u8p, C.c_int, C.c_int, C.c_float, C.c_int]
    L.oracle_derived_slope_tol.restype = C.c_double
    L.oracle_equilibrium_test.argtypes = [_f64p, C.c_int, C.c_double]
    L.oracle_equilibrium_test.restype = C.c_int
    L.oracle_simulate_adaptive.argtypes = [_f32p, _u8p, _f32p, C.c_int, C.c_int, C.POINTER(_Cfg), _i64p, _i64p,
                                           C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                           _f64p,
                                           np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"), C.c_void_p,
                                           C.c_void_p]


# ------------------------------------------------------------------ primitives
def philox4x32_10(ctr, key) -> np.ndarray:
    """Philox4x32-10 (ARITH §A)."""
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def uniform(w: int) -> float:
    return lib().oracle_uniform(int(w))


def cos_spec(x: float) -> float:
    return lib().oracle_cos_spec(float(x))


def sin_spec(x: float) -> float:
    return lib().oracle_sin_spec(float(x))


def exp_spec(x: float) -> float:
    return lib().oracle_exp_spec(float(x))


def bond_energy(phi_i, phi_j, q=0.5, J=1.0) -> float:
    """-J cos[q(phi_i - phi_j)], Eq.(1) P:86-90."""
    return lib().oracle_bond_energy(float(phi_i), float(phi_j), float(q), float(J))


def to_angles(z: np.ndarray, mask: np.ndarray):
    """Data -> spin transform. Returns (phi, zmin, zmax, status)."""
    z = np.ascontiguousarray(z, np.float32)
    mask = np.ascontiguousarray(mask, np.uint8)
    phi = np.zeros(z.shape, np.float32)
    lo, hi = C.c_float(), C.c_float()
    st = lib().oracle_transform(z.ravel(), mask.ravel(), z.size, C.byref(lo), C.byref(hi), phi.ravel())
    return phi, lo.value, hi.value, st


def sample_specific_energy(phi, mask, q=0.5):
    """Eq.(2), fp64 definition. Returns (e_s, N_SP)."""
    phi = np.ascontiguousarray(phi, np.float32); mask = np.ascontiguousarray(mask, np.uint8)
    n = C.c_int64()
    e = lib().oracle_sample_specific_energy(phi.ravel(), mask.ravel(), phi.shape[1], phi.shape[0],
                                            float(q), C.byref(n))
    return e, n.value


def grid_specific_energy(phi, q=0.5) -> float:
    phi = np.ascontiguousarray(phi, np.float32)
    return lib().oracle_grid_specific_energy(phi.ravel(), phi.shape[1], phi.shape[0], float(q))


def block_stats(phi, mask, lb, q=0.5):
    """Block bond sums, fixed point (ARITH §E). Returns SB, NB, SP, NK (nby, nbx)."""
    phi = np.ascontiguousarray(phi, np.float32); mask = np.ascontiguousarray(mask, np.uint8)
    Ly, Lx = phi.shape
    nby, nbx = -(-Ly // lb), -(-Lx // lb)
    arrs = [np.zeros(nby * nbx, np.int64) for _ in range(4)]
    lib().oracle_block_stats(phi.ravel(), mask.ravel(), Lx, Ly, lb, float(q), *arrs)
    return tuple(a.reshape(nby, nbx) for a in arrs)


def block_energy(SB: int, NB: int) -> float:
    return lib().oracle_block_energy(int(SB), int(NB))


def estimate_temperature(e, Tk, ek) -> float:
    """Energy matching by table inversion, P:90 (ARITH §F)."""
    Tk = np.ascontiguousarray(Tk, np.float32); ek = np.ascontiguousarray(ek, np.float32)
    return lib().oracle_estimate_temperature(float(e), Tk, ek, len(Tk))


def lower_median(v) -> float:
    v = np.ascontiguousarray(v, np.float32)
    return lib().oracle_lower_median(v, v.size)


def block_temperatures(SB, NB, Tk, ek):
    """Per-block T with the median fallback of P:108. Returns (Tb, n_available)."""
    SB = np.ascontiguousarray(SB, np.int64); NB = np.ascontiguousarray(NB, np.int64)
    Tk = np.ascontiguousarray(Tk, np.float32); ek = np.ascontiguousarray(ek, np.float32)
    Tb = np.zeros(SB.shape, np.float32)
    na = lib().oracle_block_temperatures(SB.ravel(), NB.ravel(), SB.size, Tk, ek, len(Tk), Tb.ravel())
    return Tb, na


def expand(Tb, Lx, Ly, lb) -> np.ndarray:
    Tb = np.ascontiguousarray(Tb, np.float32)
    T = np.zeros((Ly, Lx), np.float32)
    lib().oracle_expand(Tb.ravel(), Lx, Ly, lb, T.ravel())
    return T


def smooth(T, rs, ns) -> np.ndarray:
    """SST smoothing, P:124 (ARITH §F)."""
    T = np.array(T, np.float32, copy=True, order="C")
    lib().oracle_smooth(T.ravel(), T.shape[1], T.shape[0], int(rs), int(ns))
    return T


def init_angles(phi_known, mask, lb, SP, NK, init_mode, m, seed):
    """BLOCK_MEAN (0) or RANDOM (1) initialisation, P:249 (ARITH §G)."""
    phi = np.array(phi_known, np.float32, copy=True, order="C")
    mask = np.ascontiguousarray(mask, np.uint8)
    lib().oracle_init(phi.ravel(), mask.ravel(), phi.shape[1], phi.shape[0], lb,
                      np.ascontiguousarray(SP, np.int64).ravel(),
                      np.ascontiguousarray(NK, np.int64).ravel(), int(init_mode), int(m), int(seed))
    return phi


def sweep(phi, mask, beta, sweep_index, m, seed, q=0.5, J=1.0, reverse=False) -> int:
    """One checkerboard Metropolis sweep in place (ARITH §H). Returns #accepted."""
    assert phi.dtype == np.float32 and phi.flags.c_contiguous
    mask = np.ascontiguousarray(mask, np.uint8)
    beta = np.ascontiguousarray(beta, np.float32)
    return lib().oracle_sweep(phi.ravel(), mask.ravel(), beta.ravel(), phi.shape[1], phi.shape[0],
                              float(q), float(J), int(sweep_index), int(m), int(seed), int(reverse))


def delta_energy(phi, r, c, prop, q=0.5, J=1.0) -> float:
    """dE of moving site (r, c) to `prop` (Eq.(1); ARITH §H product form)."""
    phi = np.ascontiguousarray(phi, np.float32)
    return lib().oracle_delta_energy(phi.ravel(), phi.shape[1], phi.shape[0], int(r), int(c), float(prop),
                                     float(q), float(J))


def delta_energy_direct(phi, r, c, prop, q=0.5, J=1.0) -> float:
    """dE as the sum of bond-cosine differences (the calibration recipe's form, ARITH §H)."""
    phi = np.ascontiguousarray(phi, np.float32)
    return lib().oracle_delta_energy_direct(phi.ravel(), phi.shape[1], phi.shape[0], int(r), int(c),
                                            float(prop), float(q), float(J))


def run_chain(phi, mask, beta, s_begin, s_end, m=0, seed=1, q=0.5, J=1.0):
    """Sweeps [s_begin, s_end) in place; returns (sum over sweeps of phi per site, #accepted)."""
    assert phi.dtype == np.float32 and phi.flags.c_contiguous
    mask = np.ascontiguousarray(mask, np.uint8); beta = np.ascontiguousarray(beta, np.float32)
    sp = np.zeros(phi.shape, np.float64)
    n = lib().oracle_run_chain(phi.ravel(), mask.ravel(), beta.ravel(), phi.shape[1], phi.shape[0], float(q),
                               float(J), int(s_begin), int(s_end), int(m), int(seed), sp.ctypes.data)
    return sp, n


def sweep_dc(phi, mask, beta, sweep_index, m, seed, lb, q=0.5, J=1.0) -> int:
    """One double-checkerboard sweep in place (row f3, ARITH §H). Returns #accepted."""
    assert phi.dtype == np.float32 and phi.flags.c_contiguous
    mask = np.ascontiguousarray(mask, np.uint8); beta = np.ascontiguousarray(beta, np.float32)
    return lib().oracle_sweep_dc(phi.ravel(), mask.ravel(), beta.ravel(), phi.shape[1], phi.shape[0], float(q),
                                 float(J), int(sweep_index), int(m), int(seed), int(lb))


def half_sweep_rows(phi, mask, beta, sweep, m, seed, colour, r0, r1, q=0.5, J=1.0) -> int:
    """Colour half of one checkerboard sweep over rows [r0, r1) only (row slab), in place."""
    assert phi.dtype == np.float32 and phi.flags.c_contiguous
    mask = np.ascontiguousarray(mask, np.uint8); beta = np.ascontiguousarray(beta, np.float32)
    return lib().oracle_half_sweep_rows(phi.ravel(), mask.ravel(), beta.ravel(), phi.shape[1], phi.shape[0],
                                        float(q), float(J), int(sweep), int(m), int(seed), int(colour), int(r0),
                                        int(r1))


def unconditional_energy(L, T, q=0.5, init="ordered", n_eq=200, n_meas=200, seed=1, m=0,
                         trace=False, step=0.0):
    """Mean specific energy of an unconditional uniform-T run (calibration curve)."""
    tr = np.zeros(n_eq + n_meas, np.float64) if trace else None
    e = lib().oracle_unconditional_energy(int(L), float(T), float(q), 2 if init == "ordered" else 1,
                                          int(n_eq), int(n_meas), int(seed), int(m),
                                          tr.ctypes.data if trace else None, float(step))
    return (e, tr) if trace else e


def score(pred, truth, mask):
    """AAE / RASE of Eq.(3) and MARE; returns dict."""
    pred = np.ascontiguousarray(pred, np.float32); truth = np.ascontiguousarray(truth, np.float32)
    mask = np.ascontiguousarray(mask, np.uint8)
    a, b, c, n = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
    lib().oracle_score(pred.ravel(), truth.ravel(), mask.ravel(), pred.size, C.byref(a), C.byref(b),
                       C.byref(c), C.byref(n))
    return dict(mae=a.value, rmse=b.value, mare=c.value, mare_excluded=n.value)


def grid_energy_fx(phi, q=0.5) -> int:
    """Fixed-point whole-grid bond sum E_fx (ARITH §J)."""
    phi = np.ascontiguousarray(phi, np.float32)
    return lib().oracle_grid_energy_fx(phi.ravel(), phi.shape[1], phi.shape[0], float(q))


def energy_from_fx(E_fx, Lx, Ly) -> float:
    return lib().oracle_energy_from_fx(int(E_fx), int(Lx), int(Ly))


def equilibrium_test(y, slope_tol=0.0) -> bool:
    """ARITH §K slope test on the last n_fit energies."""
    y = np.ascontiguousarray(y, np.float64)
    return bool(lib().oracle_equilibrium_test(y, len(y), float(slope_tol)))


def derived_slope_tol(phi, mask, q=0.5, n_fit=20) -> float:
    """Reading R22: SE(e_s) / n_fit over the sample bonds (exact fixed-point sums, fp64)."""
    phi = np.ascontiguousarray(phi, np.float32); mask = np.ascontiguousarray(mask, np.uint8)
    return lib().oracle_derived_slope_tol(phi.ravel(), mask.ravel(), phi.shape[1], phi.shape[0], float(q), int(n_fit))


def simulate_adaptive(params, mask, cfg, M, seed, n_fit=20, n_f=5, S_max=500, m_begin=0, m_end=None,
                      energy=False, states=False, slope_tol=0.0):
    """Row f1 protocol (ARITH §K) for realizations [m_begin, m_end): returns
    dict(acc, s_eq (negative = forced by the cap), energy, phi). slope_tol="derived" (or < 0):
    the R22 tolerance SE(e_s) / n_fit."""
    if slope_tol == "derived":
        slope_tol = -1.0
    m_end = M if m_end is None else m_end
    mask = np.ascontiguousarray(mask, np.uint8)
    Ly, Lx = mask.shape
    R = m_end - m_begin
    acc = np.zeros(Lx * Ly, np.float64)
    s_eq = np.zeros(R, np.int32)
    en = np.zeros(R * S_max, np.float64) if energy else None
    ph = np.zeros(R * Lx * Ly, np.float32) if states else None
    c = _Cfg(cfg.q, cfg.J, cfg.lb, cfg.rs, cfg.ns, 0 if cfg.init == "block_mean" else 1, cfg.n_avg,
             1 if cfg.order == "dc" else 0)
    lib().oracle_simulate_adaptive(params.phi0.ravel(), mask.ravel(), params.beta.ravel(), Lx, Ly, C.byref(c),
                                   params.SP.ravel(), params.NK.ravel(), int(m_begin), int(m_end), int(n_fit),
                                   int(n_f), int(S_max), float(slope_tol), int(seed), acc, s_eq,
                                   en.ctypes.data if energy else None, ph.ctypes.data if states else None)
    return dict(acc=acc.reshape(Ly, Lx), s_eq=s_eq, energy=None if en is None else en.reshape(R, S_max),
                phi=None if ph is None else ph.reshape(R, Ly, Lx))


# ------------------------------------------------------------------ pipeline
@dataclass
class OracleConfig:
    q: float = 0.5
    J: float = 1.0
    lb: int = 32
    rs: int = 2
    ns: int = 5
    init: str = "block_mean"   # or "random"
    n_avg: int = 1
    order: str = "sc"          # "sc" single checkerboard, "dc" double checkerboard (row f3)


@dataclass
class OracleParams:
    phi0: np.ndarray
    T: np.ndarray
    beta: np.ndarray
    Tb: np.ndarray
    SP: np.ndarray
    NK: np.ndarray
    zmin: float
    zmax: float
    status: int


def parameters(z, mask, cfg: OracleConfig, Tk, ek) -> OracleParams:
    """a1-a5: transform, block energies, block T + median, expand, smooth."""
    z = np.ascontiguousarray(z, np.float32); mask = np.ascontiguousarray(mask, np.uint8)
    Ly, Lx = z.shape
    nby, nbx = -(-Ly // cfg.lb), -(-Lx // cfg.lb)
    phi0 = np.zeros((Ly, Lx), np.float32)
    T = np.zeros((Ly, Lx), np.float32)
    beta = np.zeros((Ly, Lx), np.float32)
    SP = np.zeros(nby * nbx, np.int64); NK = np.zeros(nby * nbx, np.int64)
    Tb = np.zeros(nby * nbx, np.float32)
    lo, hi = C.c_float(), C.c_float()
    c = _Cfg(cfg.q, cfg.J, cfg.lb, cfg.rs, cfg.ns, 0 if cfg.init == "block_mean" else 1, cfg.n_avg,
             1 if cfg.order == "dc" else 0)
    st = lib().oracle_parameters(np.where(mask != 0, z, np.float32(0)).astype(np.float32).ravel(),
                                 mask.ravel(), Lx, Ly, C.byref(c),
                                 np.ascontiguousarray(Tk, np.float32), np.ascontiguousarray(ek, np.float32),
                                 len(Tk), phi0.ravel(), T.ravel(), beta.ravel(), C.byref(lo), C.byref(hi),
                                 SP, NK, Tb.ctypes.data)
    return OracleParams(phi0, T, beta, Tb.reshape(nby, nbx), SP.reshape(nby, nbx), NK.reshape(nby, nbx),
                        lo.value, hi.value, st)


def simulate(params: OracleParams, mask, cfg: OracleConfig, M, S, seed, m_begin=0, m_end=None,
             energy=False, states=False):
    """a6-a9 for realizations [m_begin, m_end): returns dict(acc, energy, phi, accepted)."""
    m_end = M if m_end is None else m_end
    mask = np.ascontiguousarray(mask, np.uint8)
    Ly, Lx = mask.shape
    R = m_end - m_begin
    acc = np.zeros(Lx * Ly, np.float64)
    en = np.zeros(R * S, np.float64) if energy else None
    ph = np.zeros(R * Lx * Ly, np.float32) if states else None
    nacc = C.c_int64()
    c = _Cfg(cfg.q, cfg.J, cfg.lb, cfg.rs, cfg.ns, 0 if cfg.init == "block_mean" else 1, cfg.n_avg,
             1 if cfg.order == "dc" else 0)
    lib().oracle_simulate(params.phi0.ravel(), mask.ravel(), params.beta.ravel(), Lx, Ly, C.byref(c),
                          params.SP.ravel(), params.NK.ravel(), int(m_begin), int(m_end), int(S),
                          int(seed), acc, en.ctypes.data if energy else None,
                          ph.ctypes.data if states else None, C.byref(nacc))
    return dict(acc=acc.reshape(Ly, Lx), energy=None if en is None else en.reshape(R, S),
                phi=None if ph is None else ph.reshape(R, Ly, Lx), accepted=nacc.value)


def predict(z, mask, acc, M, n_avg, zmin, zmax, degenerate) -> np.ndarray:
    """Back-transformed conditional mean, P:95 (ARITH §I)."""
    z = np.ascontiguousarray(np.where(mask != 0, z, np.float32(0)), np.float32)
    mask = np.ascontiguousarray(mask, np.uint8)
    out = np.zeros(z.shape, np.float32)
    lib().oracle_predict(z.ravel(), mask.ravel(), z.size, np.ascontiguousarray(acc, np.float64).ravel(),
                         int(M), int(n_avg), float(zmin), float(zmax), int(degenerate), out.ravel())
    return out


def fill(z, mask, cfg: OracleConfig, Tk, ek, M, S, seed, energy=False, states=False):
    """Full LE-MPR gap fill (a1-a11) on the CPU. Returns dict(pred, params, sim)."""
    p = parameters(z, mask, cfg, Tk, ek)
    if p.status < 0:
        raise ValueError(f"oracle parameter stage failed: status {p.status}")
    degenerate = p.status == 1
    if degenerate:
        sim = dict(acc=np.zeros(mask.shape), energy=None, phi=None, accepted=0)
    else:
        sim = simulate(p, mask, cfg, M, S, seed, energy=energy, states=states)
    zin = np.where(mask != 0, z, np.float32(0)).astype(np.float32)
    pred = predict(zin, mask, sim["acc"], M, cfg.n_avg, p.zmin, p.zmax, degenerate)
    return dict(pred=pred, params=p, sim=sim)


class WindowOracle:
    """Exact oracle states of a small window of a LARGE grid (full-size sampled parity).

    Global quantities are computed on the whole grid with the oracle's own functions:
    z_min/z_max and the spin transform (a1-a2), block sums, block temperatures and the global
    lower median (a3-a4). The rest of the method is local, so it runs on a crop:
    - SST smoothing (a5) on a crop with margin r_s*n_s around the simulation crop: a clipped
      window at an inner crop edge differs from the global one, and the difference moves
      r_s sites per pass;
    - the simulation (a6-a7) on a crop with margin 2S+2 around the target window: an inner
      crop edge acts as an open boundary, and information moves one site per half-sweep.
    Inside the target window the result is therefore exactly the full-grid oracle's."""

    def __init__(self, z, mask, cfg: OracleConfig, Tk, ek):
        self.z = np.ascontiguousarray(np.where(mask != 0, z, np.float32(0)), np.float32)
        self.mask = np.ascontiguousarray(mask, np.uint8)
        self.cfg, self.Tk, self.ek = cfg, Tk, ek
        self.phi, self.zmin, self.zmax, st = to_angles(self.z, self.mask)
        SB, NB, self.SP, self.NK = block_stats(self.phi, self.mask, cfg.lb, cfg.q)
        self.Tb, self.n_avail = block_temperatures(SB, NB, Tk, ek)

    def T_window(self, r0, r1, c0, c1):
        """Exact SST field on [r0,r1)x[c0,c1) (crop with margin r_s*n_s, expand, smooth)."""
        Ly, Lx = self.mask.shape
        mt = self.cfg.rs * self.cfg.ns
        R0, R1, C0, C1 = max(r0 - mt, 0), min(r1 + mt, Ly), max(c0 - mt, 0), min(c1 + mt, Lx)
        lb = self.cfg.lb
        rows = np.arange(R0, R1) // lb
        cols = np.arange(C0, C1) // lb
        T = np.ascontiguousarray(self.Tb[rows[:, None], cols[None, :]], np.float32)
        T = smooth(T, self.cfg.rs, self.cfg.ns)
        return T[r0 - R0:r1 - R0, c0 - C0:c1 - C0]

    def states(self, r0, r1, c0, c1, realizations, S, seed):
        """Final states (after S sweeps) of realizations on the window [r0,r1)x[c0,c1)."""
        Ly, Lx = self.mask.shape
        ms = 2 * S + 2
        R0, R1, C0, C1 = max(r0 - ms, 0), min(r1 + ms, Ly), max(c0 - ms, 0), min(c1 + ms, Lx)
        T = self.T_window(R0, R1, C0, C1)
        beta = np.ascontiguousarray(np.float32(1.0) / T, np.float32)
        phi0 = np.ascontiguousarray(self.phi[R0:R1, C0:C1])
        mk = np.ascontiguousarray(self.mask[R0:R1, C0:C1])
        out = []
        for m in realizations:
            st = np.zeros_like(phi0)
            lib().oracle_simulate_window(phi0, mk, beta, C1 - C0, R1 - R0, R0, C0, Lx, Ly, self.cfg.lb,
                                         np.ascontiguousarray(self.SP, np.int64).ravel(),
                                         np.ascontiguousarray(self.NK, np.int64).ravel(),
                                         0 if self.cfg.init == "block_mean" else 1, float(self.cfg.q),
                                         float(self.cfg.J), int(m), int(S), int(seed), st)
            out.append(st[r0 - R0:r1 - R0, c0 - C0:c1 - C0].copy())
        return np.stack(out)
