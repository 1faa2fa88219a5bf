"""B200-native LE-MPR (SV-MPR) gap filling — arXiv 2212.01317 hot path.

The computation lives in libmpr.so (hand-written sm_100a CUDA behind the C-ABI of
include/mpr.h); this package is the thin Python binding plus the multi-GPU
realization-sharding driver. Importing it never falls back to a CPU path.
"""
from .binding import (  # noqa: F401
    Config, LeMpr, MprError, fill, load_calibration, load_library, mpr_accumulator_device,
    mpr_config_default, mpr_debug_get, mpr_destroy, mpr_estimate_local_params, mpr_get_info, mpr_init,
    mpr_predict, mpr_predict_device, mpr_reset_accumulator, mpr_set_data, mpr_set_data_device,
    mpr_set_energy_trace, mpr_set_kernel_timing, mpr_simulate, mpr_simulate_range, mpr_slab_begin,
    mpr_build_calibration, mpr_simulate_adaptive, mpr_slab_end, mpr_slab_half_sweep, mpr_slab_row_states, mpr_sync, mpr_version,
)

__all__ = [n for n in dir() if n.startswith("mpr_")] + ["Config", "LeMpr", "MprError", "fill",
                                                       "load_calibration", "load_library"]
