"""CPU model of libmpr's multi-rank decompositions (test infrastructure).

Each rank of a torch.distributed (gloo) group runs the same steps, in the same order and
with the same collectives, as api.cu does with a communicator — but every computation is
an oracle/ primitive (or, for the one-line data transform, ARITH §D in numpy float32) on
WHOLE-GRID arrays in which everything outside the rank's local rows is NaN (values) or 0
(mask). A step that read outside the rows a rank is meant to hold would therefore poison
its result, and the tests compare the end result with the single-process oracle bit for bit.

Row slabs (MPR_SHARD_ROWS), rank w of W, own rows [r0, r1) = [w Ly / W, (w+1) Ly / W):
  1. own rows of z / mask; ghost rows r0-1 and r1 by neighbour exchange;
  2. (z_min, z_max) over own samples, all-reduce MIN / MAX; transform of the local rows;
  3. block sums of the own rows (bonds to the ghost row below included, the ghost row's
     own terms excluded), all-reduce SUM -> every rank holds every block's sums;
  4. block temperatures + lower median (identical on every rank);
  5. expand on rows [r0 - H, r1 + H), H = max(r_s n_s, 1), n_s smoothing passes;
  6. per realization: init, then per colour half-sweep the own rows, then the colour's
     boundary-row states to the neighbours' ghost rows;
  7. accumulate own gap sites, predict own rows, all-gather the rows.
Realization shards (MPR_SHARD_REALIZATIONS): every rank holds the whole problem and runs
shard_range(M, W, w); the fp64 accumulators are summed by all-reduce, or by the ordered
chain (rank 0 -> W-1, then a broadcast) which is bit-identical to one process.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

import oracle as O
from paper_2212_01317_b200.sharding import row_range, shard_range

TWO_PI_F = np.float32(2 * np.pi)


def _exchange_rows(arr, r0, r1, rank, world, fill):
    """Ghost rows r0-1 / r1 of `arr` from the neighbours (their first / last own row)."""
    Ly = arr.shape[0]
    ops = []
    bufs = {}
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(arr[r0])), rank - 1))
        bufs["up"] = torch.from_numpy(np.full(arr.shape[1], fill, arr.dtype))
        ops.append(dist.P2POp(dist.irecv, bufs["up"], rank - 1))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(arr[r1 - 1])), rank + 1))
        bufs["dn"] = torch.from_numpy(np.full(arr.shape[1], fill, arr.dtype))
        ops.append(dist.P2POp(dist.irecv, bufs["dn"], rank + 1))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if "up" in bufs:
        arr[r0 - 1] = bufs["up"].numpy()
    if "dn" in bufs and r1 < Ly:
        arr[r1] = bufs["dn"].numpy()


def slab_parameters(z_full, mask_full, cfg: O.OracleConfig, Tk, ek, rank, world):
    """Steps 1-5: the local arrays of rank `rank` (NaN / 0 outside its rows)."""
    Ly, Lx = z_full.shape
    r0, r1 = row_range(Ly, world, rank)
    lr0, lr1 = max(r0 - 1, 0), min(r1 + 1, Ly)
    z = np.full(z_full.shape, np.nan, np.float32)
    mask = np.zeros(mask_full.shape, np.uint8)
    z[r0:r1] = z_full[r0:r1]
    mask[r0:r1] = mask_full[r0:r1]
    _exchange_rows(z, r0, r1, rank, world, np.nan)
    _exchange_rows(mask, r0, r1, rank, world, 0)
    # 2. extrema over own samples, all-reduced (min / max are exact)
    own = mask[r0:r1] != 0
    vals = z[r0:r1][own]
    lo = torch.tensor([vals.min() if vals.size else np.inf], dtype=torch.float32)
    hi = torch.tensor([vals.max() if vals.size else -np.inf], dtype=torch.float32)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    zmin, zmax = np.float32(lo.item()) + np.float32(0), np.float32(hi.item()) + np.float32(0)
    s = TWO_PI_F / np.float32(zmax - zmin)  # ARITH §D, fp32
    phi = np.zeros(z.shape, np.float32)
    loc = np.zeros(z.shape, bool)
    loc[lr0:lr1] = True
    known = loc & (mask != 0)
    phi[known] = np.minimum((z[known] - zmin) * s, TWO_PI_F)
    phi[~loc] = np.nan
    # 3. block sums of the own rows: all terms of rows [r0, r1] minus the ghost row's own terms
    lb = cfg.lb
    m_own = np.zeros_like(mask)
    m_own[r0:min(r1 + 1, Ly)] = mask[r0:min(r1 + 1, Ly)]
    ph0 = np.nan_to_num(phi, nan=0.0).astype(np.float32)
    stats = [a.astype(np.int64) for a in O.block_stats(ph0, m_own, lb, cfg.q)]
    if r1 < Ly:
        m_gh = np.zeros_like(mask)
        m_gh[r1] = mask[r1]
        for a, b in zip(stats, O.block_stats(ph0, m_gh, lb, cfg.q)):
            a -= b
    t = torch.from_numpy(np.stack([a.ravel() for a in stats]))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    SB, NB, SP, NK = (x.reshape(stats[0].shape) for x in t.numpy())
    # 4. block temperatures and the lower median: the same on every rank
    Tb, n_avail = O.block_temperatures(SB, NB, Tk, ek)
    # 5. expansion and smoothing on the halo-extended rows only
    H = max(cfg.rs * cfg.ns, 1)
    t0, t1 = max(r0 - H, 0), min(r1 + H, Ly)
    T_ext = O.expand(Tb, Lx, Ly, lb)[t0:t1]
    T_loc = O.smooth(T_ext, cfg.rs, cfg.ns)
    T = np.full(z.shape, np.nan, np.float32)
    T[r0:r1] = T_loc[r0 - t0:r1 - t0]
    beta = np.full(z.shape, np.nan, np.float32)
    beta[r0:r1] = np.float32(1.0) / T[r0:r1]
    return dict(r0=r0, r1=r1, lr0=lr0, lr1=lr1, z=z, mask=mask, phi=phi, beta=beta, T=T, Tb=Tb, SB=SB, NB=NB,
                SP=SP, NK=NK, zmin=zmin, zmax=zmax, n_avail=n_avail)


def _halo(phi, mask, r0, r1, colour, rank, world):
    """Colour-`colour` gap states of the boundary rows to the neighbours' ghost rows."""
    Ly, Lx = phi.shape
    cols = lambda r: [c for c in range(Lx) if ((r + c) & 1) == colour and not mask[r, c]]  # noqa: E731
    ops, recv = [], []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(phi[r0, cols(r0)].copy()), rank - 1))
        buf = torch.zeros(len(cols(r0 - 1)), dtype=torch.float32)
        ops.append(dist.P2POp(dist.irecv, buf, rank - 1))
        recv.append((r0 - 1, buf))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(phi[r1 - 1, cols(r1 - 1)].copy()), rank + 1))
        buf = torch.zeros(len(cols(r1)), dtype=torch.float32)
        ops.append(dist.P2POp(dist.irecv, buf, rank + 1))
        recv.append((r1, buf))
    ops = [op for op in ops if op.tensor.numel()]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for r, buf in recv:
        phi[r, cols(r)] = buf.numpy()


def slab_fill(z_full, mask_full, cfg: O.OracleConfig, Tk, ek, M, S, seed, rank, world):
    """Steps 1-7; returns (prediction on every rank, local params dict)."""
    p = slab_parameters(z_full, mask_full, cfg, Tk, ek, rank, world)
    Ly, Lx = z_full.shape
    r0, r1, lr0, lr1 = p["r0"], p["r1"], p["lr0"], p["lr1"]
    mask = p["mask"]
    acc = np.zeros(z_full.shape, np.float64)
    gaps_own = np.zeros(z_full.shape, bool)
    gaps_own[r0:r1] = mask[r0:r1] == 0
    init_mode = 0 if cfg.init == "block_mean" else 1
    phi0 = np.nan_to_num(p["phi"], nan=0.0).astype(np.float32)
    for m in range(M):
        phi = O.init_angles(phi0, mask, cfg.lb, p["SP"], p["NK"], init_mode, m, seed)
        phi[:lr0] = np.nan
        phi[lr1:] = np.nan
        beta = np.nan_to_num(p["beta"], nan=0.0).astype(np.float32)  # read at own sites only
        for s in range(1, S + 1):
            for colour in (0, 1):
                O.half_sweep_rows(phi, mask, beta, s, m, seed, colour, r0, r1, q=cfg.q, J=cfg.J)
                _halo(phi, mask, r0, r1, colour, rank, world)
        if cfg.n_avg != 1:
            raise NotImplementedError("the model accumulates the final sweep only")
        acc[gaps_own] += phi[gaps_own].astype(np.float64)
    zin = np.where(mask != 0, np.nan_to_num(p["z"]), np.float32(0)).astype(np.float32)
    pred_own = O.predict(zin, mask, acc, M, cfg.n_avg, p["zmin"], p["zmax"], 0)[r0:r1]
    parts = [None] * world
    dist.all_gather_object(parts, (r0, r1, pred_own))
    pred = np.full(z_full.shape, np.nan, np.float32)
    for a, b, rows in parts:
        pred[a:b] = rows
    return pred, p


def shard_fill(z, mask, cfg: O.OracleConfig, Tk, ek, M, S, seed, rank, world, ordered=False):
    """Realization shards: the rank's range of ids, then all-reduce or the ordered chain."""
    p = O.parameters(z, mask, cfg, Tk, ek)
    m0, m1 = shard_range(M, world, rank)
    gaps = mask == 0
    acc = torch.zeros(z.size, dtype=torch.float64)
    if ordered:
        if rank > 0:
            dist.recv(acc, rank - 1)
        if m1 > m0:
            st = O.simulate(p, mask, cfg, M, S, seed, m_begin=m0, m_end=m1, states=True)["phi"]
            a = acc.numpy().reshape(mask.shape)
            for phi in st:  # ascending ids, as the single process adds them
                a[gaps] += phi[gaps].astype(np.float64)
        if rank < world - 1:
            dist.send(acc, rank + 1)
        dist.broadcast(acc, world - 1)
    else:
        if m1 > m0:
            acc += torch.from_numpy(O.simulate(p, mask, cfg, M, S, seed, m_begin=m0, m_end=m1)["acc"].ravel())
        dist.all_reduce(acc, op=dist.ReduceOp.SUM)
    zin = np.where(mask != 0, z, np.float32(0)).astype(np.float32)
    return O.predict(zin, mask, acc.numpy().reshape(mask.shape), M, cfg.n_avg, p.zmin, p.zmax, 0)
