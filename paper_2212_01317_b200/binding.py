"""Thin ctypes binding of libmpr.so (include/mpr.h) — argument marshalling only.

Every function below has the name of the C entry point it calls; all computation
happens in the sm_100a kernels behind the C-ABI. There is no CPU fallback: if the
shared library is missing or no GPU is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# MPR_LIB: load another build of the library (A/B timing of kernel changes)
LIB_PATH = os.environ.get("MPR_LIB", os.path.join(_PKG, "libmpr.so"))

MPR_OK, MPR_ERR_INVALID_ARG, MPR_ERR_STATE, MPR_ERR_TOO_FEW_SAMPLES, MPR_ERR_NO_SAMPLE_BONDS, \
    MPR_ERR_CUDA, MPR_ERR_OOM, MPR_ERR_NCCL = range(8)
STATUS_NAMES = {0: "MPR_OK", 1: "MPR_ERR_INVALID_ARG", 2: "MPR_ERR_STATE", 3: "MPR_ERR_TOO_FEW_SAMPLES",
                4: "MPR_ERR_NO_SAMPLE_BONDS", 5: "MPR_ERR_CUDA", 6: "MPR_ERR_OOM", 7: "MPR_ERR_NCCL"}
MPR_INIT_BLOCK_MEAN, MPR_INIT_RANDOM = 0, 1
MPR_SHARD_REALIZATIONS, MPR_SHARD_ROWS = 0, 1
MPR_NCCL_UNIQUE_ID_BYTES = 128
(MPR_BUF_PHI_KNOWN, MPR_BUF_T, MPR_BUF_BLOCK_T, MPR_BUF_BLOCK_STATS, MPR_BUF_STATE, MPR_BUF_ACC,
 MPR_BUF_ENERGY) = range(7)

# every symbol include/mpr.h declares (checked by tests/test_abi.py)
EXPORTED = ["mpr_config_default", "mpr_init", "mpr_destroy", "mpr_last_error", "mpr_set_data",
            "mpr_set_data_device", "mpr_estimate_local_params", "mpr_simulate", "mpr_reset_accumulator",
            "mpr_simulate_range", "mpr_accumulator_device", "mpr_predict", "mpr_predict_device",
            "mpr_get_info", "mpr_debug_get", "mpr_set_energy_trace", "mpr_set_kernel_timing", "mpr_version",
            "mpr_sync", "mpr_predict_rows", "mpr_set_deferred_reduce", "mpr_accumulate_states",
            "mpr_simulate_adaptive", "mpr_build_calibration", "mpr_nccl_unique_id", "mpr_nccl_comm_init",
            "mpr_nccl_comm_destroy", "mpr_group_create", "mpr_group_destroy", "mpr_filter_check"]


class MprError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class mpr_config(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("J", C.c_float), ("q", C.c_float),
                ("l_b", C.c_int), ("r_s", C.c_int), ("n_s", C.c_int), ("init", C.c_int),
                ("n_avg", C.c_int), ("calib_T", C.POINTER(C.c_float)), ("calib_e", C.POINTER(C.c_float)),
                ("calib_n", C.c_int), ("max_batch", C.c_int64), ("order", C.c_int),
                ("nccl_comm", C.c_void_p), ("group", C.c_void_p), ("group_rank", C.c_int), ("shard", C.c_int),
                ("ordered_reduce", C.c_int)]


class mpr_info(C.Structure):
    _fields_ = [("Lx", C.c_int64), ("Ly", C.c_int64), ("n_samples", C.c_int64), ("n_gaps", C.c_int64),
                ("n_gaps_a", C.c_int64), ("z_min", C.c_float), ("z_max", C.c_float),
                ("degenerate_range", C.c_int), ("n_blocks", C.c_int64), ("n_blocks_fallback", C.c_int64),
                ("median_T", C.c_float), ("M", C.c_int64), ("sweeps", C.c_int64), ("batch", C.c_int64),
                ("kernel_launches", C.c_int64), ("total_launches", C.c_int64), ("sweep_launches", C.c_int64),
                ("sweep_ms", C.c_double), ("last_m_base", C.c_int64), ("last_batch", C.c_int64),
                ("sweep_variant", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("shard", C.c_int32),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("m_begin", C.c_int64), ("m_end", C.c_int64),
                ("n_gaps_local", C.c_int64), ("comm_calls", C.c_int64), ("slope_tol", C.c_double),
                ("sample_bonds", C.c_int64), ("filter_exact_pairs", C.c_int64), ("filter_pairs", C.c_int64)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libmpr.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    vp, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
    L.mpr_config_default.argtypes = [C.POINTER(mpr_config)]; L.mpr_config_default.restype = None
    L.mpr_init.argtypes = [C.POINTER(mpr_config), C.POINTER(vp)]; L.mpr_init.restype = C.c_int
    L.mpr_destroy.argtypes = [vp]; L.mpr_destroy.restype = None
    L.mpr_last_error.argtypes = [vp]; L.mpr_last_error.restype = C.c_char_p
    L.mpr_set_data.argtypes = [vp, vp, vp, i64, i64]; L.mpr_set_data.restype = C.c_int
    L.mpr_set_data_device.argtypes = [vp, vp, vp, i64, i64]; L.mpr_set_data_device.restype = C.c_int
    L.mpr_estimate_local_params.argtypes = [vp, vp]; L.mpr_estimate_local_params.restype = C.c_int
    L.mpr_simulate.argtypes = [vp, i64, i32, u64]; L.mpr_simulate.restype = C.c_int
    L.mpr_reset_accumulator.argtypes = [vp]; L.mpr_reset_accumulator.restype = C.c_int
    L.mpr_simulate_range.argtypes = [vp, i64, i32, u64, i64, i64]; L.mpr_simulate_range.restype = C.c_int
    L.mpr_accumulator_device.argtypes = [vp, C.POINTER(vp), C.POINTER(i64)]
    L.mpr_accumulator_device.restype = C.c_int
    L.mpr_predict.argtypes = [vp, vp]; L.mpr_predict.restype = C.c_int
    L.mpr_predict_device.argtypes = [vp, vp]; L.mpr_predict_device.restype = C.c_int
    L.mpr_get_info.argtypes = [vp, C.POINTER(mpr_info)]; L.mpr_get_info.restype = C.c_int
    L.mpr_debug_get.argtypes = [vp, C.c_int, i64, vp]; L.mpr_debug_get.restype = C.c_int
    L.mpr_set_energy_trace.argtypes = [vp, C.c_int]; L.mpr_set_energy_trace.restype = C.c_int
    L.mpr_set_kernel_timing.argtypes = [vp, C.c_int]; L.mpr_set_kernel_timing.restype = C.c_int
    L.mpr_set_deferred_reduce.argtypes = [vp, C.c_int]; L.mpr_set_deferred_reduce.restype = C.c_int
    L.mpr_accumulate_states.argtypes = [vp]; L.mpr_accumulate_states.restype = C.c_int
    L.mpr_sync.argtypes = [vp]; L.mpr_sync.restype = C.c_int
    L.mpr_predict_rows.argtypes = [vp, vp]; L.mpr_predict_rows.restype = C.c_int
    L.mpr_nccl_unique_id.argtypes = [vp]; L.mpr_nccl_unique_id.restype = C.c_int
    L.mpr_nccl_comm_init.argtypes = [C.c_int, C.c_int, vp, C.c_int, C.POINTER(vp)]
    L.mpr_nccl_comm_init.restype = C.c_int
    L.mpr_nccl_comm_destroy.argtypes = [vp]; L.mpr_nccl_comm_destroy.restype = C.c_int
    L.mpr_group_create.argtypes = [C.c_int, C.POINTER(vp)]; L.mpr_group_create.restype = C.c_int
    L.mpr_group_destroy.argtypes = [vp]; L.mpr_group_destroy.restype = None
    L.mpr_simulate_adaptive.argtypes = [vp, i64, u64, i32, i32, i32, C.c_double, vp]
    L.mpr_simulate_adaptive.restype = C.c_int
    L.mpr_build_calibration.argtypes = [vp, vp, i32, i32, C.c_float, i32, i32, i32, u64, vp, vp]
    L.mpr_build_calibration.restype = C.c_int
    L.mpr_version.argtypes = []; L.mpr_version.restype = C.c_char_p
    L.mpr_filter_check.argtypes = [C.c_int, vp]; L.mpr_filter_check.restype = C.c_int
    _lib = L
    return L


def _check(ctx, status):
    if status != MPR_OK:
        msg = load_library().mpr_last_error(ctx).decode() if ctx else ""
        raise MprError(status, msg)


# ----------------------------------------------------------- same-name wrappers
def mpr_config_default() -> mpr_config:
    cfg = mpr_config()
    load_library().mpr_config_default(C.byref(cfg))
    return cfg


def mpr_init(cfg: mpr_config):
    ctx = C.c_void_p()
    st = load_library().mpr_init(C.byref(cfg), C.byref(ctx))
    if st != MPR_OK:
        raise MprError(st, "mpr_init failed (see stderr)")
    return ctx


def mpr_destroy(ctx) -> None:
    load_library().mpr_destroy(ctx)


def mpr_set_data(ctx, grid: np.ndarray, mask: np.ndarray) -> None:
    """Host arrays (Ly, Lx): float32 grid (gaps may be NaN), uint8 mask (1 = sample)."""
    g = np.ascontiguousarray(grid, np.float32)
    m = np.ascontiguousarray(mask, np.uint8)
    assert g.shape == m.shape and g.ndim == 2
    Ly, Lx = g.shape
    _check(ctx, load_library().mpr_set_data(ctx, g.ctypes.data, m.ctypes.data, Lx, Ly))


def mpr_set_data_device(ctx, grid_ptr: int, mask_ptr: int, Lx: int, Ly: int) -> None:
    _check(ctx, load_library().mpr_set_data_device(ctx, grid_ptr, mask_ptr, Lx, Ly))


def mpr_estimate_local_params(ctx, want_T: bool = False, shape=None):
    if want_T:  # row slabs write their own rows only: the rest stays NaN
        T = np.full(shape, np.nan, np.float32)
        _check(ctx, load_library().mpr_estimate_local_params(ctx, T.ctypes.data))
        return T
    _check(ctx, load_library().mpr_estimate_local_params(ctx, None))
    return None


def mpr_simulate(ctx, M: int, sweeps: int, seed: int) -> None:
    _check(ctx, load_library().mpr_simulate(ctx, M, sweeps, seed))


def mpr_reset_accumulator(ctx) -> None:
    _check(ctx, load_library().mpr_reset_accumulator(ctx))


def mpr_simulate_range(ctx, M: int, sweeps: int, seed: int, m_begin: int, m_end: int) -> None:
    _check(ctx, load_library().mpr_simulate_range(ctx, M, sweeps, seed, m_begin, m_end))


def mpr_accumulator_device(ctx):
    p, n = C.c_void_p(), C.c_int64()
    _check(ctx, load_library().mpr_accumulator_device(ctx, C.byref(p), C.byref(n)))
    return p.value, n.value


def mpr_predict(ctx, shape) -> np.ndarray:
    out = np.empty(shape, np.float32)
    _check(ctx, load_library().mpr_predict(ctx, out.ctypes.data))
    return out


def mpr_predict_device(ctx, out_ptr: int) -> None:
    _check(ctx, load_library().mpr_predict_device(ctx, out_ptr))


def mpr_get_info(ctx) -> dict:
    info = mpr_info()
    _check(ctx, load_library().mpr_get_info(ctx, C.byref(info)))
    return {k: getattr(info, k) for k, _ in mpr_info._fields_}


def mpr_debug_get(ctx, which: int, index: int, out: np.ndarray) -> np.ndarray:
    _check(ctx, load_library().mpr_debug_get(ctx, which, index, out.ctypes.data))
    return out


def mpr_set_energy_trace(ctx, enable: bool) -> None:
    _check(ctx, load_library().mpr_set_energy_trace(ctx, 1 if enable else 0))


def mpr_set_kernel_timing(ctx, enable: bool) -> None:
    _check(ctx, load_library().mpr_set_kernel_timing(ctx, 1 if enable else 0))


def mpr_set_deferred_reduce(ctx, enable: bool) -> None:
    _check(ctx, load_library().mpr_set_deferred_reduce(ctx, 1 if enable else 0))


def mpr_accumulate_states(ctx) -> None:
    _check(ctx, load_library().mpr_accumulate_states(ctx))


def mpr_sync(ctx) -> None:
    _check(ctx, load_library().mpr_sync(ctx))


def mpr_predict_rows(ctx, rows: int, Lx: int) -> np.ndarray:
    """The rank's own rows of the prediction ((row_end - row_begin) x Lx)."""
    out = np.empty((rows, Lx), np.float32)
    _check(ctx, load_library().mpr_predict_rows(ctx, out.ctypes.data))
    return out


def mpr_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(MPR_NCCL_UNIQUE_ID_BYTES)
    _check(None, load_library().mpr_nccl_unique_id(buf))
    return buf.raw


def mpr_nccl_comm_init(world: int, rank: int, uid: bytes, device: int) -> int:
    comm = C.c_void_p()
    buf = C.create_string_buffer(uid, MPR_NCCL_UNIQUE_ID_BYTES)
    _check(None, load_library().mpr_nccl_comm_init(world, rank, buf, device, C.byref(comm)))
    return comm.value


def mpr_nccl_comm_destroy(comm: int) -> None:
    _check(None, load_library().mpr_nccl_comm_destroy(comm))


def mpr_group_create(world: int) -> int:
    g = C.c_void_p()
    _check(None, load_library().mpr_group_create(world, C.byref(g)))
    return g.value


def mpr_group_destroy(group: int) -> None:
    load_library().mpr_group_destroy(group)


def mpr_build_calibration(ctx, T, L=128, q=0.5, n_eq=400, n_meas=800, reps=2, seed=20221202):
    """Row f2: e(T) table on the GPU (defaults = scripts/make_calibration.py). Returns (e, e_raw)."""
    T = np.ascontiguousarray(T, np.float32)
    e = np.zeros(len(T), np.float32)
    raw = np.zeros(len(T), np.float64)
    _check(ctx, load_library().mpr_build_calibration(ctx, T.ctypes.data, len(T), L, q, n_eq, n_meas, reps, seed,
                                                     e.ctypes.data, raw.ctypes.data))
    return e, raw


def mpr_simulate_adaptive(ctx, M, seed, n_fit=20, n_f=5, max_sweeps=500, slope_tol=0.0) -> np.ndarray:
    """Adaptive equilibration (ARITH §K); returns s_eq per realization
    (negative = forced by max_sweeps). slope_tol="derived" (or < 0): SE(e_s) / n_fit (R22)."""
    if slope_tol == "derived":
        slope_tol = -1.0
    s_eq = np.zeros(M, np.int32)
    _check(ctx, load_library().mpr_simulate_adaptive(ctx, M, seed, n_fit, n_f, max_sweeps, float(slope_tol),
                                                     s_eq.ctypes.data))
    return s_eq


def mpr_version() -> str:
    return load_library().mpr_version().decode()


def mpr_filter_check(device: int = 0):
    """(passed, sfu_sine_err, max_exp_x24) of the default kernel's rejection filter."""
    err = np.zeros(2, np.float64)
    ok = load_library().mpr_filter_check(int(device), err.ctypes.data)
    return bool(ok), float(err[0]), float(err[1])


# ----------------------------------------------------------- convenience layer
def load_calibration(path: str | None = None):
    """(T_k, e_k) float32 arrays of the shipped e(T) table (data/calib_q0.5.txt)."""
    path = path or os.path.join(_PKG, "data", "calib_q0.5.txt")
    T, e = [], []
    with open(path) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            a, b = line.split()[:2]
            T.append(float.fromhex(a)); e.append(float.fromhex(b))
    return np.array(T, np.float32), np.array(e, np.float32)


@dataclass
class Config:
    """Method parameters (defaults: PAPER.md:260 l_b = 32, n_s = 5; DESIGN.md readings)."""
    J: float = 1.0
    q: float = 0.5
    l_b: int = 32
    r_s: int = 2
    n_s: int = 5
    init: str = "block_mean"
    n_avg: int = 1
    device: int = 0
    max_batch: int = 0
    order: str = "sc"   # "sc" single checkerboard, "dc" double checkerboard (row f3)
    # multi-rank (include/mpr.h mpr_shard): a communicator (NCCL comm handle from
    # mpr_nccl_comm_init, or an in-process group from mpr_group_create + this rank) and
    # the decomposition "realizations" or "rows"
    nccl_comm: int | None = None
    group: int | None = None
    group_rank: int = 0
    shard: str = "realizations"
    ordered_reduce: bool = False


class LeMpr:
    """One device context: set_data -> estimate_local_params -> simulate -> predict."""

    def __init__(self, cfg: Config | None = None, calib=None, stream: int | None = None):
        cfg = cfg or Config()
        self.cfg = cfg
        T, e = calib if calib is not None else load_calibration()
        self._T = np.ascontiguousarray(T, np.float32)
        self._e = np.ascontiguousarray(e, np.float32)
        c = mpr_config_default()
        c.device, c.J, c.q, c.l_b, c.r_s, c.n_s = cfg.device, cfg.J, cfg.q, cfg.l_b, cfg.r_s, cfg.n_s
        c.init = MPR_INIT_BLOCK_MEAN if cfg.init == "block_mean" else MPR_INIT_RANDOM
        c.n_avg, c.max_batch = cfg.n_avg, cfg.max_batch
        c.order = 1 if cfg.order == "dc" else 0
        c.nccl_comm, c.group, c.group_rank = cfg.nccl_comm, cfg.group, cfg.group_rank
        if cfg.shard not in ("realizations", "rows"):
            raise ValueError("shard must be 'realizations' or 'rows'")
        c.shard = MPR_SHARD_ROWS if cfg.shard == "rows" else MPR_SHARD_REALIZATIONS
        c.ordered_reduce = 1 if cfg.ordered_reduce else 0
        c.stream = stream
        c.calib_T = self._T.ctypes.data_as(C.POINTER(C.c_float))
        c.calib_e = self._e.ctypes.data_as(C.POINTER(C.c_float))
        c.calib_n = len(self._T)
        self.ctx = mpr_init(c)
        self.shape = None

    def close(self):
        if getattr(self, "ctx", None):
            mpr_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_data(self, grid, mask):
        self.shape = tuple(np.shape(grid))
        mpr_set_data(self.ctx, grid, mask)

    def set_data_device(self, grid_ptr, mask_ptr, Lx, Ly):
        self.shape = (Ly, Lx)
        mpr_set_data_device(self.ctx, grid_ptr, mask_ptr, Lx, Ly)

    def estimate_local_params(self, want_T=False):
        return mpr_estimate_local_params(self.ctx, want_T, self.shape)

    def simulate(self, M, sweeps, seed):
        mpr_simulate(self.ctx, M, sweeps, seed)

    def simulate_range(self, M, sweeps, seed, m_begin, m_end):
        mpr_simulate_range(self.ctx, M, sweeps, seed, m_begin, m_end)

    def simulate_adaptive(self, M, seed, n_fit=20, n_f=5, max_sweeps=500, slope_tol=0.0):
        return mpr_simulate_adaptive(self.ctx, M, seed, n_fit, n_f, max_sweeps, slope_tol)

    def reset_accumulator(self):
        mpr_reset_accumulator(self.ctx)

    def predict(self):
        return mpr_predict(self.ctx, self.shape)

    def info(self):
        return mpr_get_info(self.ctx)

    def debug(self, which, index=0):
        Ly, Lx = self.shape
        inf = self.info()
        # Lx*Ly buffers: row slabs fill their own rows only, the rest stays NaN
        if which in (MPR_BUF_PHI_KNOWN, MPR_BUF_T, MPR_BUF_STATE):
            out = np.full((Ly, Lx), np.nan, np.float32)
        elif which == MPR_BUF_ACC:
            out = np.full((Ly, Lx), np.nan, np.float64)
        elif which == MPR_BUF_BLOCK_T:
            out = np.empty(inf["n_blocks"], np.float32)
        elif which == MPR_BUF_BLOCK_STATS:
            out = np.empty((4, inf["n_blocks"]), np.int64)
        elif which == MPR_BUF_ENERGY:
            out = np.empty((inf["M"], inf["sweeps"]), np.float64)
        else:
            raise ValueError(which)
        return mpr_debug_get(self.ctx, which, index, out)

    def set_energy_trace(self, enable=True):
        mpr_set_energy_trace(self.ctx, enable)

    def set_kernel_timing(self, enable=True):
        mpr_set_kernel_timing(self.ctx, enable)

    def simulate_device_acc(self):
        """(device pointer, count) of the fp64 per-gap accumulator, for an external all-reduce."""
        return mpr_accumulator_device(self.ctx)

    def _device_view(self, ptr, n, typestr):
        import torch

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                        "version": 3, "stream": None}
        return torch.as_tensor(_View(), device=torch.device("cuda", self.cfg.device))

    def accumulator_tensor(self):
        """Zero-copy torch view (cuda, float64) of the per-gap accumulator owned by the
        context, via __cuda_array_interface__ (valid until the next set_data/close)."""
        ptr, n = mpr_accumulator_device(self.ctx)
        return self._device_view(ptr, max(n, 1), "<f8")

    def predict_device(self, out_ptr):
        mpr_predict_device(self.ctx, out_ptr)

    def predict_rows(self):
        """The own rows of the prediction (row slabs; the whole grid otherwise)."""
        inf = self.info()
        return mpr_predict_rows(self.ctx, inf["row_end"] - inf["row_begin"], self.shape[1])

    def set_deferred_reduce(self, enable=True):
        """simulate_range keeps its states; accumulate_states adds them later (ordered
        multi-rank reduction, bit-identical to one GPU)."""
        mpr_set_deferred_reduce(self.ctx, enable)

    def accumulate_states(self):
        mpr_accumulate_states(self.ctx)

    def sync(self):
        mpr_sync(self.ctx)


def fill(grid, mask, M=100, sweeps=30, seed=20221202, cfg: Config | None = None, calib=None):
    """Gap-fill one grid on the GPU: returns the float32 predictions (samples unchanged)."""
    m = LeMpr(cfg, calib)
    try:
        m.set_data(grid, mask)
        m.estimate_local_params()
        m.simulate(M, sweeps, seed)
        return m.predict()
    finally:
        m.close()
