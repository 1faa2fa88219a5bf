"""B200-native LE-MPR (SV-MPR) gap filling — arXiv 2212.01317 hot path.

The computation lives in libmpr.so (hand-written sm_100a CUDA behind the C-ABI of
include/mpr.h), including the multi-GPU decompositions (realization shards, row slabs);
this package is the thin Python binding plus communicator set-up (sharding.py).
Importing it never falls back to a CPU path.
"""
from .binding import (  # noqa: F401
    Config, LeMpr, MprError, fill, load_calibration, load_library, mpr_accumulator_device,
    mpr_build_calibration, mpr_config_default, mpr_debug_get, mpr_destroy, mpr_estimate_local_params,
    mpr_get_info, mpr_group_create, mpr_group_destroy, mpr_init, mpr_nccl_comm_destroy, mpr_nccl_comm_init,
    mpr_nccl_unique_id, mpr_predict, mpr_predict_device, mpr_predict_rows, mpr_reset_accumulator, mpr_set_data,
    mpr_set_data_device, mpr_set_energy_trace, mpr_set_kernel_timing, mpr_simulate, mpr_simulate_adaptive,
    mpr_simulate_range, mpr_sync, mpr_version,
)

__all__ = [n for n in dir() if n.startswith("mpr_")] + ["Config", "LeMpr", "MprError", "fill",
                                                       "load_calibration", "load_library"]
