"""Multi-GPU realization sharding (BASELINE.json north star: "sharding
independent realizations, with an NCCL allreduce of the per-site accumulators over NVLink").

The M realizations of a fill are independent Markov chains whose random numbers are
keyed by their GLOBAL realization id (docs/ARITH.md §A), so any partition of the ids
over ranks reproduces the single-GPU chains bit for bit. Every rank recomputes the
(deterministic, bit-exact) parameter stage itself — cheaper than broadcasting a T field —
simulates its contiguous, pair-aligned range of ids, and one all-reduce (NCCL over
NVLink on GPUs; gloo in the CPU tests) sums the per-gap fp64 accumulators. Every rank
then back-transforms the same sums.

This module is plumbing only: it never computes any part of the method itself.
"""
from __future__ import annotations

from typing import Protocol

import torch
import torch.distributed as dist


def shard_range(M: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous range [m_begin, m_end) of global realization ids for `rank`.

    Ranges are aligned to realization pairs (one Philox call serves ids 2k and 2k+1,
    ARITH §A), cover [0, M) exactly once, and differ in size by at most one pair."""
    if M < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    npairs = (M + 1) // 2
    p0 = rank * npairs // world
    p1 = (rank + 1) * npairs // world
    return min(2 * p0, M), min(2 * p1, M)


def slab_realization_chunks(M: int) -> list[tuple[int, int]]:
    """Realization ranges a row-slab fill runs one after the other (each is one state batch
    of mpr_slab_begin). The default sweep kernel moves two realization pairs per thread and
    needs a multiple of 4 realizations, so M = 4k + r runs as [0, 4k) then [4k, M). The
    chains do not depend on the split (global Philox ids, ARITH §A)."""
    if M < 1:
        raise ValueError("M must be >= 1")
    k = (M // 4) * 4
    if k == 0 or k == M:
        return [(0, M)]
    return [(0, k), (k, M)]


class Engine(Protocol):
    def set_data(self, grid, mask): ...
    def estimate_local_params(self, want_T: bool = False): ...
    def reset_accumulator(self): ...
    def simulate_range(self, M, sweeps, seed, m_begin, m_end): ...
    def accumulator_tensor(self) -> torch.Tensor: ...
    def predict(self): ...


def allreduce_accumulator(acc: torch.Tensor, group=None) -> None:
    """Sum the per-gap accumulators of all ranks in place (a10 of SURVEY §8(a))."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)


def row_range(Ly: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous rows [r0, r1) of a row slab; sizes differ by at most one row."""
    if Ly < world or world < 1 or not 0 <= rank < world:
        raise ValueError("need at least one row per rank")
    return rank * Ly // world, (rank + 1) * Ly // world


def exchange_halo(engine, colour: int, r0: int, r1: int, rank: int, world: int, group=None) -> None:
    """After the colour-`colour` half-sweep: send the colour's gap states of the first and
    last own rows to the neighbouring slabs, receive theirs into the ghost rows (one row
    per side). Row sizes are global facts, so both ends agree on them."""
    ops, recvs = [], []
    peer = lambda r: r if group is None else dist.get_global_rank(group, r)  # noqa: E731
    if rank > 0:
        snd, rcv = engine.row_view(r0, colour), engine.row_view(r0 - 1, colour)
        if snd.numel():
            ops.append(dist.P2POp(dist.isend, snd, peer(rank - 1), group))
        if rcv.numel():
            ops.append(dist.P2POp(dist.irecv, rcv, peer(rank - 1), group))
            recvs.append((r0 - 1, rcv))
    if rank < world - 1:
        snd, rcv = engine.row_view(r1 - 1, colour), engine.row_view(r1, colour)
        if snd.numel():
            ops.append(dist.P2POp(dist.isend, snd, peer(rank + 1), group))
        if rcv.numel():
            ops.append(dist.P2POp(dist.irecv, rcv, peer(rank + 1), group))
            recvs.append((r1, rcv))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for row, t in recvs:
        engine.commit_row(row, colour, t)


def connect_peer_halo(engine, rank: int, world: int, group=None) -> None:
    """Fused halo exchange set-up (after every slab_begin): all-gather the ranks' state
    buffer IPC handles and register the neighbours' buffers, so each half-sweep kernel
    writes its boundary rows straight into the neighbours' ghost rows over NVLink."""
    handles = [None] * world
    dist.all_gather_object(handles, engine.state_ipc_handle(), group=group)
    if rank > 0:
        engine.set_peer(0, ipc_handle=handles[rank - 1])
    if rank < world - 1:
        engine.set_peer(1, ipc_handle=handles[rank + 1])
    dist.barrier(group=group)  # every mapping is in place before any kernel writes through it


def distributed_fill_slabs(engine, grid, mask, M: int, sweeps: int, seed: int, group=None, halo: str = "peer"):
    """SPMD gap fill with the grid split into row slabs (one per rank) and a one-row halo
    exchange per colour half-sweep; every rank runs all M realizations on its rows. The
    chains are bit-identical to the single-GPU run (global Philox counters).

    halo="peer": the half-sweep kernel writes the boundary rows into the neighbours'
    state buffers (IPC-mapped peer memory); the host only orders half-sweeps (sync +
    barrier). halo="nccl": the boundary rows are sent with NCCL point-to-point calls."""
    if halo not in ("peer", "nccl"):
        raise ValueError("halo must be 'peer' or 'nccl'")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    Ly = grid.shape[0]
    r0, r1 = row_range(Ly, world, rank)
    engine.set_data(grid, mask)
    engine.estimate_local_params()
    engine.reset_accumulator()
    peer = halo == "peer" and world > 1
    for m0, m1 in slab_realization_chunks(M):
        engine.slab_begin(M, sweeps, seed, m0, m1, r0, r1)
        if peer:
            connect_peer_halo(engine, rank, world, group)
        for s in range(1, sweeps + 1):
            for colour in (0, 1):
                engine.slab_half_sweep(s, colour)
                if peer:  # the kernels wrote the halos; finish the half-sweep everywhere
                    engine.sync()
                    dist.barrier(group=group)
                elif world > 1:
                    exchange_halo(engine, colour, r0, r1, rank, world, group)
        engine.slab_end()
    allreduce_accumulator(engine.accumulator_tensor(), group)
    return engine.predict()


def ordered_reduce_accumulator(engine, rank: int, world: int, group=None) -> None:
    """Deterministic reduction across ranks, bit-identical to one GPU: the accumulator
    travels rank 0 -> 1 -> ... -> W-1, each rank adding its realizations (ascending ids,
    mpr_accumulate_states) on top of the sum of the ranks before it; the last rank
    broadcasts the total. Needs simulate_range under set_deferred_reduce(True)."""
    acc = engine.accumulator_tensor()
    peer = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))
    if rank > 0:
        dist.recv(acc, peer(rank - 1), group=group)
    engine.accumulate_states()
    if rank < world - 1:
        dist.send(acc, peer(rank + 1), group=group)
    if world > 1:
        dist.broadcast(acc, peer(world - 1), group=group)


def distributed_fill(engine: Engine, grid, mask, M: int, sweeps: int, seed: int, group=None,
                     reduce: str = "allreduce"):
    """SPMD gap fill: every rank calls this with the same arguments; returns the
    predictions (identical on every rank). reduce="allreduce": one all-reduce of the
    accumulators (equal to one GPU up to fp64 summation order); reduce="ordered": the
    chained reduction, bit-identical to one GPU."""
    if reduce not in ("allreduce", "ordered"):
        raise ValueError("reduce must be 'allreduce' or 'ordered'")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m0, m1 = shard_range(M, world, rank)
    engine.set_data(grid, mask)
    engine.estimate_local_params()
    engine.reset_accumulator()
    if reduce == "ordered":
        engine.set_deferred_reduce(True)
        engine.simulate_range(M, sweeps, seed, m0, m1)
        ordered_reduce_accumulator(engine, rank, world, group)
        engine.set_deferred_reduce(False)
    else:
        engine.simulate_range(M, sweeps, seed, m0, m1)
        allreduce_accumulator(engine.accumulator_tensor(), group)
    return engine.predict()
