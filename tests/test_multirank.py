"""Multi-rank (realization sharding) host logic on CPU: world_size-2 gloo process group.

The product's sharding driver (paper_2212_01317_b200/sharding.py) is run with an
oracle-backed engine injected by the test (the product never imports oracle/): each rank
simulates its shard of global realization ids, the accumulators are all-reduced over
gloo, and the predictions must equal the single-process fill up to fp64 reassociation.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_01317_b200.sharding import distributed_fill, shard_range


@pytest.mark.parametrize("M,world", [(10, 2), (7, 2), (1, 2), (100, 8), (3, 4), (0, 3)])
def test_shard_range_covers_exactly_once(M, world):
    ranges = [shard_range(M, world, r) for r in range(world)]
    ids = [m for a, b in ranges for m in range(a, b)]
    assert ids == list(range(M))
    for a, b in ranges:
        assert a % 2 == 0  # pair-aligned starts (Philox pairs, ARITH §A)
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 2


class OracleEngine:
    """CPU stand-in with the Engine interface, backed by oracle/ (test-only)."""

    def __init__(self, calib, cfg):
        import oracle as O
        self.O, self.calib, self.cfg = O, calib, cfg

    def set_data(self, grid, mask):
        self.z, self.mask = grid, mask

    def estimate_local_params(self, want_T=False):
        self.p = self.O.parameters(self.z, self.mask, self.cfg, *self.calib)

    def reset_accumulator(self):
        self.acc = torch.zeros(self.z.size, dtype=torch.float64)
        self.M = 0

    deferred = False
    pending = None

    def set_deferred_reduce(self, enable=True):
        self.deferred = enable

    def simulate_range(self, M, sweeps, seed, m0, m1):
        self.M = M
        if m1 > m0:
            r = self.O.simulate(self.p, self.mask, self.cfg, M, sweeps, seed, m_begin=m0, m_end=m1,
                                states=self.deferred)
            if self.deferred:  # keep the final states (n_avg = 1), add them in accumulate_states
                self.pending = r["phi"]
            else:
                self.acc += torch.from_numpy(r["acc"].ravel())

    def accumulate_states(self):
        acc = self.acc.numpy().reshape(self.mask.shape)  # a view: the adds land in self.acc
        gaps = self.mask == 0
        for phi in (self.pending if self.pending is not None else []):  # ascending realization ids
            acc[gaps] += phi[gaps].astype(np.float64)
        self.pending = None

    def accumulator_tensor(self):
        return self.acc

    def predict(self):
        acc = self.acc.numpy().reshape(self.z.shape)
        return self.O.predict(np.nan_to_num(self.z), self.mask, acc, self.M, self.cfg.n_avg,
                              self.p.zmin, self.p.zmax, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ordered_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from inputs.synth import make_problem
    from tests.conftest import read_calibration
    truth, z, mask = make_problem(24, 0.5, corr_len=5.0)
    eng = OracleEngine(read_calibration(), O.OracleConfig(lb=8, rs=1, ns=2))
    out[rank] = distributed_fill(eng, z, mask, M=7, sweeps=6, seed=31, reduce="ordered")
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ordered_reduce_bit_identical_to_single_process(calib, world):
    """reduce="ordered": the accumulator travels rank 0 -> W-1, each rank adding its
    realizations in ascending order, so the predictions equal the single-process oracle
    bit for bit (the all-reduce is only equal up to fp64 summation order)."""
    import oracle as O
    from inputs.synth import make_problem
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ordered_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    truth, z, mask = make_problem(24, 0.5, corr_len=5.0)
    ref = O.fill(z, mask, O.OracleConfig(lb=8, rs=1, ns=2), *calib, M=7, S=6, seed=31)["pred"]
    for r in range(world):
        assert np.array_equal(out[r].view(np.uint32), ref.view(np.uint32))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from inputs.synth import make_problem
    from tests.conftest import read_calibration
    truth, z, mask = make_problem(24, 0.5, corr_len=5.0)
    eng = OracleEngine(read_calibration(), O.OracleConfig(lb=8, rs=1, ns=2))
    pred = distributed_fill(eng, z, mask, M=7, sweeps=6, seed=31)
    out[rank] = pred
    dist.destroy_process_group()


def test_gloo_world2_equals_single_process(calib):
    import oracle as O
    from inputs.synth import make_problem
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    truth, z, mask = make_problem(24, 0.5, corr_len=5.0)
    ref = O.fill(z, mask, O.OracleConfig(lb=8, rs=1, ns=2), *calib, M=7, S=6, seed=31)["pred"]
    for r in range(2):
        assert np.max(np.abs(out[r] - ref)) <= 1e-6 * (np.nanmax(z) - np.nanmin(z))
    assert np.array_equal(out[0], out[1])


# ------------------------------------------------------------------ row slabs
class OracleSlabEngine(OracleEngine):
    """Row-slab interface on top of the oracle: dense per-realization states, own rows
    updated by oracle.half_sweep_rows, halo rows exchanged through row_view/commit_row."""

    def slab_begin(self, M, sweeps, seed, m0, m1, r0, r1):
        from multiprocessing import shared_memory
        self.M, self.S, self.seed, self.m0, self.m1, self.r0, self.r1 = M, sweeps, seed, m0, m1, r0, r1
        init = np.stack([self.O.init_angles(self.p.phi0, self.mask, self.cfg.lb, self.p.SP, self.p.NK,
                                            0 if self.cfg.init == "block_mean" else 1, m, seed)
                         for m in range(m0, m1)])
        # the state lives in a shared-memory segment so neighbour processes can write into it,
        # as the GPU kernel writes into IPC-mapped neighbour buffers (halo="peer")
        self.shm = shared_memory.SharedMemory(create=True, size=init.nbytes)
        self.phi = np.ndarray(init.shape, init.dtype, buffer=self.shm.buf)
        self.phi[...] = init
        self.peers = [None, None]

    def state_ipc_handle(self):
        return self.shm.name.encode()

    def set_peer(self, side, ipc_handle=None, dev_ptr=None):
        from multiprocessing import shared_memory
        seg = shared_memory.SharedMemory(name=ipc_handle.decode())
        self.peers[side] = (seg, np.ndarray(self.phi.shape, self.phi.dtype, buffer=seg.buf))

    def sync(self):
        pass

    def slab_half_sweep(self, s, colour):
        for k, m in enumerate(range(self.m0, self.m1)):
            ph = np.ascontiguousarray(self.phi[k])
            self.O.half_sweep_rows(ph, self.mask, self.p.beta, s, m, self.seed, colour, self.r0, self.r1,
                                   q=self.cfg.q, J=self.cfg.J)
            self.phi[k] = ph
        # fused halo: the boundary rows' colour-c gap states land in the neighbours' buffers
        for side, row in ((0, self.r0), (1, self.r1 - 1)):
            if self.peers[side] is not None:
                cols = self._cols(row, colour)
                self.peers[side][1][:, row, cols] = self.phi[:, row, cols]

    def _cols(self, row, colour):
        Lx = self.mask.shape[1]
        return [c for c in range(Lx) if ((row + c) & 1) == colour and not self.mask[row, c]]

    def row_view(self, row, colour):
        cols = self._cols(row, colour)
        return torch.from_numpy(np.ascontiguousarray(self.phi[:, row, cols].T.ravel()))

    def commit_row(self, row, colour, t):
        cols = self._cols(row, colour)
        self.phi[:, row, cols] = t.numpy().reshape(len(cols), -1).T

    def slab_end(self):
        rows = slice(self.r0, self.r1)
        gaps = np.zeros(self.mask.shape, bool)
        gaps[rows] = self.mask[rows] == 0
        acc = self.acc.numpy().reshape(self.mask.shape)  # a view: adds land in self.acc
        for k in range(self.phi.shape[0]):  # realization order, as the oracle accumulates
            acc[gaps] += self.phi[k][gaps].astype(np.float64)
        for side in (0, 1):
            if self.peers[side] is not None:
                self.peers[side][0].close()
        self.peers = [None, None]
        dist.barrier()  # no neighbour still writes into this segment
        self.phi = self.phi.copy()
        self.shm.close()
        self.shm.unlink()


def _slab_worker(rank, world, port, out, halo):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from inputs.synth import make_problem
    from paper_2212_01317_b200.sharding import distributed_fill_slabs
    from tests.conftest import read_calibration
    truth, z, mask = make_problem(21, 0.6, Lx=18, corr_len=5.0)
    eng = OracleSlabEngine(read_calibration(), O.OracleConfig(lb=8, rs=1, ns=2))
    out[rank] = distributed_fill_slabs(eng, z, mask, M=6, sweeps=5, seed=41, halo=halo)  # chunks [0,4), [4,6)
    dist.destroy_process_group()


@pytest.mark.parametrize("halo", ["peer", "nccl"])
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_row_slabs_bit_exact(calib, world, halo):
    """Row-slab decomposition with one-row halos per colour half-sweep reproduces the
    single-process chains bit for bit (global Philox counters). halo="peer"
    runs the fused-exchange protocol (handle all-gather, neighbour registration, boundary
    rows written into the neighbours' shared buffers, sync + barrier per half-sweep);
    halo="nccl" the point-to-point exchange."""
    import oracle as O
    from inputs.synth import make_problem
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_slab_worker, args=(world, _free_port(), out, halo), nprocs=world, join=True)
    truth, z, mask = make_problem(21, 0.6, Lx=18, corr_len=5.0)
    ref = O.fill(z, mask, O.OracleConfig(lb=8, rs=1, ns=2), *calib, M=6, S=5, seed=41)["pred"]
    for r in range(world):
        assert np.array_equal(out[r].view(np.uint32), ref.view(np.uint32))


def test_row_range():
    from paper_2212_01317_b200.sharding import row_range
    rr = [row_range(10, 3, r) for r in range(3)]
    assert rr == [(0, 3), (3, 6), (6, 10)]


@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 6, 7, 8, 10, 64, 100, 101])
def test_slab_realization_chunks(M):
    """Row-slab realization split: covers [0, M) once, in order, the first chunk a multiple of
    4 whenever M >= 4 (the two-pair sweep kernel's batch), at most two chunks."""
    from paper_2212_01317_b200.sharding import slab_realization_chunks
    ch = slab_realization_chunks(M)
    assert ch[0][0] == 0 and ch[-1][1] == M and len(ch) <= 2
    assert all(a < b for a, b in ch) and all(ch[i][1] == ch[i + 1][0] for i in range(len(ch) - 1))
    if M >= 4:
        assert ch[0][1] % 4 == 0
    if len(ch) == 2:
        assert ch[1][1] - ch[1][0] < 4
