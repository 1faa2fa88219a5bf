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


def distributed_fill(engine: Engine, grid, mask, M: int, sweeps: int, seed: int, group=None):
    """SPMD gap fill: every rank calls this with the same arguments; returns the
    predictions (identical on every rank)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m0, m1 = shard_range(M, world, rank)
    engine.set_data(grid, mask)
    engine.estimate_local_params()
    engine.reset_accumulator()
    engine.simulate_range(M, sweeps, seed, m0, m1)
    allreduce_accumulator(engine.accumulator_tensor(), group)
    return engine.predict()
