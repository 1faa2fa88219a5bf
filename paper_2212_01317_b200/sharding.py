"""Multi-GPU plumbing around libmpr's in-library decompositions (
include/mpr.h ``mpr_shard``).

The decompositions themselves run inside libmpr.so (api.cu): every rank makes the same
C-ABI calls with a communicator in its config, and the library shards the realizations
(one NCCL all-reduce of the fp64 accumulators, or the rank-ordered chain) or splits the
grid into row slabs (distributed parameter stage, one-row halo exchange per colour
half-sweep, all-gathered predictions). This module only creates communicators:

* ``make_nccl_comm``: one process per GPU (torchrun) — rank 0 draws an NCCL unique id
  through libmpr, the id travels over the torch process group, every rank initialises its
  communicator through libmpr (so the library and the communicator share one libnccl).
* ``run_group``: W contexts in ONE process (one host thread each; one or several devices):
  libmpr's in-process transport, whose collectives are host-synchronous copies between the
  contexts' device buffers. It runs the multi-rank code path where one process owns all the
  devices, and on a single GPU for tests (no kernel ever waits on another).

It never computes any part of the method itself.
"""
from __future__ import annotations

import threading

from . import binding as B


def shard_range(M: int, world: int, rank: int) -> tuple[int, int]:
    """Global realization ids [m_begin, m_end) of `rank` — the same rule as api.cu's
    shard_range (tests compare both): contiguous, aligned to realization pairs (one Philox
    call serves ids 2k and 2k+1, ARITH §A), covering [0, M) once, sizes within one pair."""
    if M < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    npairs = (M + 1) // 2
    p0 = rank * npairs // world
    p1 = (rank + 1) * npairs // world
    return min(2 * p0, M), min(2 * p1, M)


def row_range(Ly: int, world: int, rank: int) -> tuple[int, int]:
    """Own rows [r0, r1) of row slab `rank` — api.cu's row_range; sizes within one row."""
    if Ly < world or world < 1 or not 0 <= rank < world:
        raise ValueError("need at least one row per rank")
    return rank * Ly // world, (rank + 1) * Ly // world


def make_nccl_comm(device: int, group=None) -> int:
    """NCCL communicator (handle for ``Config.nccl_comm``) over the ranks of the torch
    process group `group`: the unique id is drawn by rank 0 and broadcast over torch."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = [B.mpr_nccl_unique_id() if rank == 0 else None]
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast_object_list(obj, src=src, group=group)
    return B.mpr_nccl_comm_init(world, rank, obj[0], device)


def destroy_nccl_comm(comm: int) -> None:
    B.mpr_nccl_comm_destroy(comm)


def run_group(world: int, fn, timeout: float | None = None):
    """Run fn(rank, group_handle) on `world` host threads sharing one in-process libmpr
    communicator (``Config(group=handle, group_rank=rank)``); returns the per-rank results.
    ctypes releases the GIL inside the C calls, so the ranks meet in the library's
    collectives. An exception on any rank is re-raised after every thread has ended (the
    library's group barrier times out, MPR_GROUP_TIMEOUT_S, if a rank never arrives)."""
    g = B.mpr_group_create(world)
    results, errors = [None] * world, [None] * world

    def body(r):
        try:
            results[r] = fn(r, g)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errors[r] = e

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    try:
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout)
    finally:
        if all(not t.is_alive() for t in threads):
            B.mpr_group_destroy(g)
    for e in errors:
        if e is not None:
            raise e
    return results


def distributed_fill(grid, mask, M: int, sweeps: int, seed: int, cfg: B.Config | None = None, calib=None,
                     stream: int | None = None):
    """SPMD gap fill: every rank calls this with the same arguments and a config carrying
    its communicator and decomposition; returns the whole prediction on every rank."""
    eng = B.LeMpr(cfg, calib, stream=stream)
    try:
        eng.set_data(grid, mask)
        eng.estimate_local_params()
        eng.simulate(M, sweeps, seed)
        return eng.predict()
    finally:
        eng.close()
