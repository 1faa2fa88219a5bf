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
    MPR_ERR_CUDA, MPR_ERR_OOM = range(7)
STATUS_NAMES = {0: "MPR_OK", 1: "MPR_ERR_INVALID_ARG", 2: "MPR_ERR_STATE", 3: "MPR_ERR_TOO_FEW_SAMPLES",
                4: "MPR_ERR_NO_SAMPLE_BONDS", 5: "MPR_ERR_CUDA", 6: "MPR_ERR_OOM"}
MPR_INIT_BLOCK_MEAN, MPR_INIT_RANDOM = 0, 1
(MPR_BUF_PHI_KNOWN, MPR_BUF_T, MPR_BUF_BLOCK_T, MPR_BUF_BLOCK_STATS, MPR_BUF_STATE, MPR_BUF_ACC,
 MPR_BUF_ENERGY) = range(7)

# every symbol include/mpr.h declares (checked by tests/test_abi.py)
EXPORTED = ["mpr_config_default", "mpr_init", "mpr_destroy", "mpr_last_error", "mpr_set_data",
            "mpr_set_data_device", "mpr_estimate_local_params", "mpr_simulate", "mpr_reset_accumulator",
            "mpr_simulate_range", "mpr_accumulator_device", "mpr_predict", "mpr_predict_device",
            "mpr_get_info", "mpr_debug_get", "mpr_set_energy_trace", "mpr_set_kernel_timing", "mpr_version",
            "mpr_slab_begin", "mpr_slab_half_sweep", "mpr_slab_row_states", "mpr_slab_end", "mpr_sync",
            "mpr_slab_state_ipc_handle", "mpr_slab_state_device", "mpr_slab_set_peer",
            "mpr_set_deferred_reduce", "mpr_accumulate_states",
            "mpr_simulate_adaptive", "mpr_build_calibration"]


class MprError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class mpr_config(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("J", C.c_float), ("q", C.c_float),
                ("l_b", C.c_int), ("r_s", C.c_int), ("n_s", C.c_int), ("init", C.c_int),
                ("n_avg", C.c_int), ("calib_T", C.POINTER(C.c_float)), ("calib_e", C.POINTER(C.c_float)),
                ("calib_n", C.c_int), ("max_batch", C.c_int64), ("order", C.c_int)]


class mpr_info(C.Structure):
    _fields_ = [("Lx", C.c_int64), ("Ly", C.c_int64), ("n_samples", C.c_int64), ("n_gaps", C.c_int64),
                ("n_gaps_a", C.c_int64), ("z_min", C.c_float), ("z_max", C.c_float),
                ("degenerate_range", C.c_int), ("n_blocks", C.c_int64), ("n_blocks_fallback", C.c_int64),
                ("median_T", C.c_float), ("M", C.c_int64), ("sweeps", C.c_int64), ("batch", C.c_int64),
                ("kernel_launches", C.c_int64), ("total_launches", C.c_int64), ("sweep_launches", C.c_int64),
                ("sweep_ms", C.c_double), ("last_m_base", C.c_int64), ("last_batch", C.c_int64),
                ("sweep_variant", C.c_int32)]


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
    L.mpr_slab_begin.argtypes = [vp, i64, i32, u64, i64, i64, i64, i64]; L.mpr_slab_begin.restype = C.c_int
    L.mpr_slab_half_sweep.argtypes = [vp, i32, C.c_int]; L.mpr_slab_half_sweep.restype = C.c_int
    L.mpr_slab_row_states.argtypes = [vp, i64, C.c_int, C.POINTER(vp), C.POINTER(i64)]
    L.mpr_slab_row_states.restype = C.c_int
    L.mpr_slab_state_ipc_handle.argtypes = [vp, vp]; L.mpr_slab_state_ipc_handle.restype = C.c_int
    L.mpr_slab_state_device.argtypes = [vp, C.POINTER(vp)]; L.mpr_slab_state_device.restype = C.c_int
    L.mpr_slab_set_peer.argtypes = [vp, C.c_int, vp, vp]; L.mpr_slab_set_peer.restype = C.c_int
    L.mpr_set_deferred_reduce.argtypes = [vp, C.c_int]; L.mpr_set_deferred_reduce.restype = C.c_int
    L.mpr_accumulate_states.argtypes = [vp]; L.mpr_accumulate_states.restype = C.c_int
    L.mpr_slab_end.argtypes = [vp]; L.mpr_slab_end.restype = C.c_int
    L.mpr_sync.argtypes = [vp]; L.mpr_sync.restype = C.c_int
    L.mpr_simulate_adaptive.argtypes = [vp, i64, u64, i32, i32, i32, C.c_double, vp]
    L.mpr_simulate_adaptive.restype = C.c_int
    L.mpr_build_calibration.argtypes = [vp, vp, i32, i32, C.c_float, i32, i32, i32, u64, vp, vp]
    L.mpr_build_calibration.restype = C.c_int
    L.mpr_version.argtypes = []; L.mpr_version.restype = C.c_char_p
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
    if want_T:
        T = np.empty(shape, np.float32)
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


def mpr_slab_begin(ctx, M, sweeps, seed, m_begin, m_end, row_begin, row_end) -> None:
    _check(ctx, load_library().mpr_slab_begin(ctx, M, sweeps, seed, m_begin, m_end, row_begin, row_end))


def mpr_slab_half_sweep(ctx, sweep, colour) -> None:
    _check(ctx, load_library().mpr_slab_half_sweep(ctx, sweep, colour))


def mpr_slab_row_states(ctx, row, colour):
    p, n = C.c_void_p(), C.c_int64()
    _check(ctx, load_library().mpr_slab_row_states(ctx, row, colour, C.byref(p), C.byref(n)))
    return p.value, n.value


def mpr_set_deferred_reduce(ctx, enable: bool) -> None:
    _check(ctx, load_library().mpr_set_deferred_reduce(ctx, 1 if enable else 0))


def mpr_accumulate_states(ctx) -> None:
    _check(ctx, load_library().mpr_accumulate_states(ctx))


MPR_IPC_HANDLE_BYTES = 64


def mpr_slab_state_ipc_handle(ctx) -> bytes:
    buf = C.create_string_buffer(MPR_IPC_HANDLE_BYTES)
    _check(ctx, load_library().mpr_slab_state_ipc_handle(ctx, buf))
    return buf.raw


def mpr_slab_state_device(ctx) -> int:
    p = C.c_void_p()
    _check(ctx, load_library().mpr_slab_state_device(ctx, C.byref(p)))
    return p.value


def mpr_slab_set_peer(ctx, side, ipc_handle: bytes | None = None, dev_ptr: int | None = None) -> None:
    h = C.create_string_buffer(ipc_handle, MPR_IPC_HANDLE_BYTES) if ipc_handle is not None else None
    _check(ctx, load_library().mpr_slab_set_peer(ctx, side, h, dev_ptr))


def mpr_slab_end(ctx) -> None:
    _check(ctx, load_library().mpr_slab_end(ctx))


def mpr_sync(ctx) -> None:
    _check(ctx, load_library().mpr_sync(ctx))


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
    (negative = forced by max_sweeps)."""
    s_eq = np.zeros(M, np.int32)
    _check(ctx, load_library().mpr_simulate_adaptive(ctx, M, seed, n_fit, n_f, max_sweeps, float(slope_tol),
                                                     s_eq.ctypes.data))
    return s_eq


def mpr_version() -> str:
    return load_library().mpr_version().decode()


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
        if which in (MPR_BUF_PHI_KNOWN, MPR_BUF_T, MPR_BUF_STATE):
            out = np.empty((Ly, Lx), np.float32)
        elif which == MPR_BUF_ACC:
            out = np.empty((Ly, Lx), np.float64)
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

    # ---- row-slab mode (include/mpr.h mpr_slab_*) ----
    def slab_begin(self, M, sweeps, seed, m_begin, m_end, row_begin, row_end):
        mpr_slab_begin(self.ctx, M, sweeps, seed, m_begin, m_end, row_begin, row_end)

    def slab_half_sweep(self, sweep, colour):
        mpr_slab_half_sweep(self.ctx, sweep, colour)

    def row_view(self, row, colour):
        """Zero-copy (cuda, float32) view of the colour-`colour` gap states of `row`; the
        halo exchange sends from / receives into it in place."""
        ptr, n = mpr_slab_row_states(self.ctx, row, colour)
        if n == 0:
            import torch
            return torch.empty(0, dtype=torch.float32, device=torch.device("cuda", self.cfg.device))
        return self._device_view(ptr, n, "<f4")

    def commit_row(self, row, colour, tensor):
        """Received halo rows land in place (row_view is zero-copy): nothing to do."""

    def set_deferred_reduce(self, enable=True):
        """simulate_range keeps its states; accumulate_states adds them later (ordered
        multi-rank reduction, bit-identical to one GPU)."""
        mpr_set_deferred_reduce(self.ctx, enable)

    def accumulate_states(self):
        mpr_accumulate_states(self.ctx)

    def state_ipc_handle(self) -> bytes:
        """cudaIpcMemHandle_t of this slab's state buffer (for a neighbour process)."""
        return mpr_slab_state_ipc_handle(self.ctx)

    def state_device(self) -> int:
        """Device pointer of this slab's state buffer (for a neighbour in this process)."""
        return mpr_slab_state_device(self.ctx)

    def set_peer(self, side, ipc_handle=None, dev_ptr=None):
        """Register the upper (side 0) / lower (side 1) neighbour's state buffer: the
        half-sweep kernel then writes the boundary rows into it (fused halo exchange)."""
        mpr_slab_set_peer(self.ctx, side, ipc_handle, dev_ptr)

    def slab_end(self):
        mpr_slab_end(self.ctx)

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
