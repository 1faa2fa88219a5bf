"""Multi-rank host logic on CPU (world_size 2-3, gloo): the decompositions libmpr runs with
a communicator (api.cu), modelled step for step with oracle primitives in
tests/dist_model.py, must reproduce the single-process oracle bit for bit:

* row slabs (MPR_SHARD_ROWS): the distributed parameter stage (min/max all-reduce, z/mask
  ghost-row exchange for the cross-slab bonds, all-reduced exact block sums, the lower
  median on every rank, the smoothing halo of r_s * n_s rows) and the per-half-sweep
  boundary-row exchange;
* realization shards (MPR_SHARD_REALIZATIONS): pair-aligned id ranges, all-reduce (equal up
  to fp64 summation order) or the rank-ordered chain (bit-identical).
Every rank holds NaN outside its rows, so a step that reads outside them shows up.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_01317_b200.sharding import row_range, shard_range


@pytest.mark.parametrize("M,world", [(10, 2), (7, 2), (1, 2), (100, 8), (3, 4), (0, 3)])
def test_shard_range_covers_exactly_once(M, world):
    ranges = [shard_range(M, world, r) for r in range(world)]
    ids = [m for a, b in ranges for m in range(a, b)]
    assert ids == list(range(M))
    for a, b in ranges:
        assert a % 2 == 0  # pair-aligned starts (Philox pairs, ARITH §A)
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 2


def test_row_range():
    rr = [row_range(10, 3, r) for r in range(3)]
    assert rr == [(0, 3), (3, 6), (6, 10)]
    for Ly, W in ((16384, 8), (21, 5), (7, 7)):
        parts = [row_range(Ly, W, r) for r in range(W)]
        assert parts[0][0] == 0 and parts[-1][1] == Ly
        assert all(parts[i][1] == parts[i + 1][0] for i in range(W - 1))
        assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1
    with pytest.raises(ValueError):
        row_range(3, 4, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = {
    # name: (L, Lx, p, gaps, corr, cfg kwargs, M, S, seed)
    "sst": (21, 18, 0.6, "random", 5.0, dict(lb=8, rs=1, ns=2), 4, 5, 41),
    "wide_halo": (26, 13, 0.5, "random", 4.0, dict(lb=4, rs=2, ns=3, init="random"), 3, 4, 7),
    "mpr_one_block": (17, 20, 0.4, "cloud", 6.0, dict(lb=64, rs=1, ns=1), 2, 4, 3),
}


def _problem(name):
    from inputs.synth import make_problem
    L, Lx, p, gaps, corr, kw, M, S, seed = CASES[name]
    truth, z, mask = make_problem(L, p, Lx=Lx, gaps=gaps, corr_len=corr)
    return z, mask, kw, M, S, seed


def _slab_worker(rank, world, port, out, name):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from tests.conftest import read_calibration
    from tests.dist_model import slab_fill
    z, mask, kw, M, S, seed = _problem(name)
    Tk, ek = read_calibration()
    pred, p = slab_fill(z, mask, O.OracleConfig(**kw), Tk, ek, M, S, seed, rank, world)
    out[rank] = (pred, p["T"], p["SB"], p["NB"], p["SP"], p["NK"], p["Tb"])
    dist.destroy_process_group()


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_row_slabs_bit_exact(calib, world, name):
    """The row-slab decomposition: all-reduced block sums equal the global ones, each rank's
    SST rows equal the global field's (halo r_s n_s wide enough), and the predictions
    all-gathered from the slabs equal the single-process oracle bit for bit."""
    import oracle as O
    z, mask, kw, M, S, seed = _problem(name)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_slab_worker, args=(world, _free_port(), out, name), nprocs=world, join=True)
    cfg = O.OracleConfig(**kw)
    ref = O.fill(z, mask, cfg, *calib, M=M, S=S, seed=seed)
    SB, NB, SP, NK = O.block_stats(ref["params"].phi0, mask, cfg.lb, cfg.q)
    for r in range(world):
        pred, T, sb, nb, sp, nk, Tb = out[r]
        for a, b in ((sb, SB), (nb, NB), (sp, SP), (nk, NK)):
            assert np.array_equal(a, b)
        assert np.array_equal(Tb.view(np.uint32), ref["params"].Tb.view(np.uint32))
        r0, r1 = row_range(z.shape[0], world, r)
        assert np.array_equal(T[r0:r1].view(np.uint32), ref["params"].T[r0:r1].view(np.uint32))
        assert np.array_equal(pred.view(np.uint32), ref["pred"].view(np.uint32))


def _shard_worker(rank, world, port, out, ordered):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from inputs.synth import make_problem
    from tests.conftest import read_calibration
    from tests.dist_model import shard_fill
    truth, z, mask = make_problem(24, 0.5, corr_len=5.0)
    out[rank] = shard_fill(z, mask, O.OracleConfig(lb=8, rs=1, ns=2), *read_calibration(), M=7, S=6, seed=31,
                           rank=rank, world=world, ordered=ordered)
    dist.destroy_process_group()


@pytest.mark.parametrize("ordered", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_realization_shards(calib, world, ordered):
    """ordered: bit-identical to one process; all-reduce: equal up to fp64 reassociation."""
    import oracle as O
    from inputs.synth import make_problem
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(world, _free_port(), out, ordered), nprocs=world, join=True)
    truth, z, mask = make_problem(24, 0.5, corr_len=5.0)
    ref = O.fill(z, mask, O.OracleConfig(lb=8, rs=1, ns=2), *calib, M=7, S=6, seed=31)["pred"]
    for r in range(world):
        if ordered:
            assert np.array_equal(out[r].view(np.uint32), ref.view(np.uint32))
        else:
            assert np.max(np.abs(out[r] - ref)) <= 1e-6 * (np.nanmax(z) - np.nanmin(z))
        assert np.array_equal(out[r], out[0])
