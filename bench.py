#!/usr/bin/env python3
"""LE-MPR gap-filling benchmark (BASELINE.json metric: gap-site spin updates/s and fill time).

One "step" = one pass of the whole hot path over one synthetic
problem: set_data (device-resident input) -> estimate_local_params -> simulate
(M realizations x S sweeps, with the reduction over ranks inside libmpr) -> predict.

Headline line (N=1: BASELINE config 2): 1024^2 Matern nu=0.5 heterogeneous field, 33%
random gaps, M = 100 per rank, S = 30, SST l_b=32 r_s=2 n_s=5. At N > 1 the realizations
are sharded inside libmpr (MPR_SHARD_REALIZATIONS over an NCCL communicator: weak
scaling, M per rank fixed, one NCCL all-reduce of the fp64 accumulators).
Sub-record "c4_rows" (every N): BASELINE config 4 — 16384^2, 50% random gaps, M = 10,
S = 30 — split into row slabs over the N ranks (MPR_SHARD_ROWS: strong scaling; the
north star's < 1 s target), device-resident and end-to-end fill time, the half-sweep
kernel's roofline, and each rank's H2D (its own rows only) and D2H (its own rows).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C2]

Rank 0 prints ONE JSON line. `--impl reference` times the CPU oracle (the reference arm
of this tier) on all host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from inputs.synth import CONFIGS, SEED_SIM, make_problem  # noqa: E402

METRIC = "gap-site spin updates/sec (LE-MPR conditional simulation, whole fill)"
# FP32 lane-ops the arithmetic contract fixes per gap-site update (ARITH §H
# product form with the degree-11 sine of §B2: sin of the half difference 8, four
# neighbour sine terms of 8, the sum phi' + phi 1, dE / beta 3, exp_spec 12, 4 conversions
# = 60) + half a Philox4x32-10 call (10 rounds x 2 IMAD.WIDE + 2 LOP3 = 40 per pair) = 80.
ALG_OPS_PER_UPDATE = 80
UNIT = "updates/s"
# how each config scales over ranks: weak (M per rank) or strong (M in total)
SCALING = {"C1": "weak", "C2": "weak", "C3": "strong", "C4": "strong"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mpr", choices=["mpr", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--M", type=int, default=None, help="realizations (per rank for weak-scaling configs)")
    ap.add_argument("--sweeps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-realizations", type=int, default=100)
    ap.add_argument("--ref-sample-realizations", type=int, default=20)
    ap.add_argument("--cpu-threads", type=int, default=0, help="oracle threads (0 = all host cores)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 row-slab sub-record")
    ap.add_argument("--c4-steps", type=int, default=3)
    ap.add_argument("--reduce", default="allreduce", choices=["allreduce", "ordered"],
                    help="realization shards at N > 1: one NCCL all-reduce of the accumulators, or the "
                         "ordered chain (bit-identical to one GPU)")
    ap.add_argument("--decomp", default=None, choices=["realizations", "rows"],
                    help="multi-GPU split of the headline line (default: rows for C4, realizations otherwise)")
    ap.add_argument("--emulate", type=int, default=0,
                    help="W > 1: run the multi-rank path with W contexts on this ONE GPU (libmpr's in-process "
                         "transport, one host thread each) and check it against one context; a functional "
                         "line, not a scaling measurement")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_problem(cfg_name):
    """The config's synthetic problem; C3/C4 are cached as .npy under /tmp (generation of
    the 16384^2 field takes ~1 min on the host)."""
    c = dict(CONFIGS[cfg_name])
    cache = os.path.join("/tmp", "mpr_inputs")
    path = os.path.join(cache, f"{cfg_name}_{c['L']}_{c['p']}_{c['gaps']}_{c['nu']}.npz")
    if c["L"] >= 4096 and os.path.exists(path):
        d = np.load(path)
        return c, d["truth"], d["z"], d["mask"]
    truth, z, mask = make_problem(c["L"], c["p"], gaps=c["gaps"], nu=c["nu"])
    if c["L"] >= 4096:
        try:
            os.makedirs(cache, exist_ok=True)
            tmp = path + f".tmp{os.getpid()}.npz"
            np.savez(tmp, truth=truth, z=z, mask=mask)
            os.replace(tmp, path)
        except OSError:
            pass
    return c, truth, z, mask


def describe(name, c, M, S, per_rank):
    return (f"{name}: {c['L']}x{c['L']} Whittle-Matern nu={c['nu']} heterogeneous field, "
            f"{int(round(c['p'] * 100))}% {c['gaps']} gaps, M={M}{' per rank' if per_rank else ' in total'}, "
            f"S={S} sweeps, SST l_b=32 r_s=2 n_s=5, BLOCK_MEAN init, n_avg=1")


def algorithmic_bytes_per_update(p, n_avg=1, S=30, b_T=4):
    """B_alg = 4/p + 8 + b_T bytes per gap-site update (+ 8 n_avg/S when the
    accumulation is a separate buffer, i.e. n_avg > 1)."""
    return 4.0 / p + 8.0 + b_T + (8.0 * n_avg / S if n_avg > 1 else 0.0)


def cpu_info():
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed regions."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = f"/tmp/mpr_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


def cpu_baseline_sample(z, mask, M_sample, S, c, threads=0):
    """Time the CPU oracle, as it stands, on a bounded sample of the same workload: the
    full parameter stage + M_sample realizations x S sweeps, on `threads` host cores (the
    OpenMP build of the same source: same-colour rows split over threads, bit-identical
    to the single-thread oracle; 0 = all cores)."""
    import oracle as O
    from paper_2212_01317_b200.binding import load_calibration
    Tk, ek = load_calibration()
    cfg = O.OracleConfig()
    used = O.set_threads(threads)
    try:
        t0 = time.perf_counter()
        p = O.parameters(z, mask, cfg, Tk, ek)
        sim = O.simulate(p, mask, cfg, M_sample, S, SEED_SIM)
        zin = np.where(mask != 0, z, np.float32(0)).astype(np.float32)
        O.predict(zin, mask, sim["acc"], M_sample, 1, p.zmin, p.zmax, 0)
        dt = time.perf_counter() - t0
    finally:
        O.set_threads(1)
    P = int((mask == 0).sum())
    upd = P * S * M_sample
    nproc, model = cpu_info()
    return {"value": upd / dt, "unit": UNIT, "cores": used, "kind": "oracle", "nproc": nproc, "cpu_model": model,
            "sample": f"{c['L']}x{c['L']} grid, p={c['p']}: full parameter stage + realizations 0..{M_sample - 1} "
                      f"x {S} sweeps = {upd:.3e} gap-site updates in {dt:.2f} s ({used} threads, oracle/ as is)",
            "seconds": dt}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    c, truth, z, mask = load_problem(args.config)
    M = args.M or c["M"]
    S = args.sweeps or c["sweeps"]
    P = int((mask == 0).sum())
    Ms = max(1, args.ref_sample_realizations)
    for _ in range(args.warmup):
        cpu_baseline_sample(z, mask, Ms, S, c, args.cpu_threads)
    times, last = [], None
    for _ in range(args.steps):
        last = cpu_baseline_sample(z, mask, Ms, S, c, args.cpu_threads)
        times.append(last["seconds"])
    total = sum(times)
    value = P * S * Ms * args.steps / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
            "higher_is_better": True, "scaling": SCALING[args.config], "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": describe(args.config, c, M, S, SCALING[args.config] == "weak"),
                       "sample_realizations_per_step": Ms},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                             "nproc": last["nproc"], "cpu_model": last["cpu_model"],
                             "sample": f"per step: parameter stage + {Ms} realizations x {S} sweeps "
                                       f"({P * S * Ms:.3e} updates), {last['cores']} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


class Workload:
    """One config run through libmpr with this rank's communicator: device-resident and
    end-to-end (pinned host buffers) timings, and the half-sweep kernel's device time."""

    def __init__(self, name, decomp, M, S, comm, ws, rank, local, dev, stream):
        import torch

        import paper_2212_01317_b200 as Pk
        self.name, self.decomp, self.S, self.ws, self.rank = name, decomp, S, ws, rank
        self.c, self.truth, self.z, self.mask = load_problem(name)
        self.P = int((self.mask == 0).sum())
        Ly, Lx = self.z.shape
        self.Ly, self.Lx = Ly, Lx
        self.M = M
        self.rows = decomp == "rows"
        cfg = Pk.Config(device=local, nccl_comm=comm, shard="rows" if self.rows else "realizations",
                        ordered_reduce=False)
        self.eng = Pk.LeMpr(cfg, Pk.load_calibration(), stream=stream.cuda_stream)
        self.Pk, self.torch, self.dev, self.stream = Pk, torch, dev, stream
        from paper_2212_01317_b200.sharding import row_range
        self.r0, self.r1 = row_range(Ly, ws, rank) if self.rows else (0, Ly)
        zs = np.ascontiguousarray(np.nan_to_num(self.z[self.r0:self.r1], nan=0.0))
        ms = np.ascontiguousarray(self.mask[self.r0:self.r1])
        # device-resident inputs: the own rows only (row slabs) or the whole grid
        self.z_dev = torch.from_numpy(zs).to(dev)
        self.m_dev = torch.from_numpy(ms).to(dev)
        self.out_dev = torch.empty((Ly, Lx), dtype=torch.float32, device=dev)
        # pinned host buffers of the e2e leg: the whole grid (the C-ABI copies the own rows)
        self.z_pin = torch.from_numpy(np.nan_to_num(self.z, nan=0.0)).pin_memory()
        self.m_pin = torch.from_numpy(self.mask).pin_memory()
        self.out_pin = torch.empty((self.r1 - self.r0, Lx), dtype=torch.float32).pin_memory()
        self.lib = Pk.load_library()

    def step_device(self):
        e = self.eng
        e.set_data_device(self.z_dev.data_ptr(), self.m_dev.data_ptr(), self.Lx, self.Ly)
        e.estimate_local_params()
        e.simulate(self.M, self.S, SEED_SIM)
        e.predict_device(self.out_dev.data_ptr())

    def step_host(self):
        e, L, ck = self.eng, self.lib, self.Pk.binding._check
        ck(e.ctx, L.mpr_set_data(e.ctx, self.z_pin.data_ptr(), self.m_pin.data_ptr(), self.Lx, self.Ly))
        e.shape = (self.Ly, self.Lx)
        e.estimate_local_params()
        e.simulate(self.M, self.S, SEED_SIM)
        ck(e.ctx, L.mpr_predict_rows(e.ctx, self.out_pin.data_ptr()))  # the own rows

    def updates_per_step(self):
        return self.P * self.S * self.M

    def h2d_bytes(self):
        return (self.r1 - self.r0) * self.Lx * 5

    def d2h_bytes(self):
        return (self.r1 - self.r0) * self.Lx * 4


def barrier(dev, ws):
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)


def max_over_ranks(x, dev, ws):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_workload(w: Workload, steps, warmup, dev, ws, e2e=True, flush=None):
    """Device-timed steps (CUDA events on the library's stream, max over ranks), the
    half-sweep kernel's device time, and the e2e wall time through the C-ABI."""
    import torch
    for _ in range(max(warmup, 0)):
        w.step_device()
    barrier(dev, ws)
    w.eng.set_kernel_timing(True)
    launches0 = w.eng.info()["total_launches"]
    barrier(dev, ws)
    total_ms = 0.0
    for _ in range(steps):
        if flush is not None:
            flush.fill_(1.0)  # L2 flush between timed steps (256 MiB > 126 MB L2), outside the events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(w.stream)
        w.step_device()
        e1.record(w.stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    barrier(dev, ws)
    info = w.eng.info()
    w.eng.set_kernel_timing(False)
    total_ms = max_over_ranks(total_ms, dev, ws)
    res = {"ms_per_step": total_ms / steps, "launches": info["total_launches"] - launches0,
           "sweep_ms": info["sweep_ms"], "sweep_launches": info["sweep_launches"], "info": info,
           "value": w.updates_per_step() * steps / (total_ms / 1000.0)}
    if e2e:
        for _ in range(max(warmup, 1)):  # first use of the host-buffer path, untimed
            w.step_host()
        barrier(dev, ws)
        t0 = time.perf_counter()
        for _ in range(steps):
            w.step_host()
        barrier(dev, ws)
        wall = max_over_ranks(time.perf_counter() - t0, dev, ws)
        res["e2e"] = {"value": w.updates_per_step() * steps / wall, "unit": UNIT,
                      "h2d_bytes_per_step": int(w.h2d_bytes()), "d2h_bytes_per_step": int(w.d2h_bytes()),
                      "fill_time_ms": 1000 * wall / steps}
    return res


def e2e_pipelined(w: Workload, steps, warmup, n_ctx=2):
    """Serving-style end-to-end throughput (one GPU): n_ctx contexts, each on its own CUDA
    stream and driven by its own host thread, fill the steps round-robin. Every fill still
    makes the public C-ABI calls with the H2D of its inputs from pinned host memory and the
    D2H of its prediction inside the timed region; one context's copies and host work
    overlap another's kernels (a stream of grids to fill, e.g. a time series)."""
    import threading
    import torch
    Pk, L, ck = w.Pk, w.lib, w.Pk.binding._check
    engs, outs = [w.eng], [w.out_pin]
    for _ in range(n_ctx - 1):
        st = torch.cuda.Stream(w.dev)
        engs.append(Pk.LeMpr(Pk.Config(device=w.dev.index or 0), Pk.load_calibration(), stream=st.cuda_stream))
        outs.append(torch.empty_like(w.out_pin).pin_memory())

    def fill(e, out):
        ck(e.ctx, L.mpr_set_data(e.ctx, w.z_pin.data_ptr(), w.m_pin.data_ptr(), w.Lx, w.Ly))
        e.shape = (w.Ly, w.Lx)
        e.estimate_local_params()
        e.simulate(w.M, w.S, SEED_SIM)
        ck(e.ctx, L.mpr_predict_rows(e.ctx, out.data_ptr()))

    for e, o in zip(engs, outs):
        for _ in range(max(warmup, 1)):
            fill(e, o)
    torch.cuda.synchronize(w.dev)
    errs = []

    def worker(k):
        try:
            for _ in range(k, steps, n_ctx):
                fill(engs[k], outs[k])
        except Exception as ex:  # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(n_ctx)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize(w.dev)
    wall = time.perf_counter() - t0
    for e in engs[1:]:
        e.close()
    if errs:
        raise errs[0]
    return {"value": w.updates_per_step() * steps / wall, "unit": UNIT, "contexts": n_ctx,
            "fill_time_ms": 1000 * wall / steps, "h2d_bytes_per_step": int(w.h2d_bytes()),
            "d2h_bytes_per_step": int(w.d2h_bytes()),
            "how": "fills issued round-robin by one host thread per context (own CUDA stream); each fill "
                   "copies its inputs from pinned host memory and its prediction back"}


def sweep_roofline(w: Workload, r, steps, peaks):
    """The half-sweep kernel (CUDA events on the library's stream around its launches)
    against the FP32-lane ALU peak, and the SURVEY §8(d) algorithmic-byte view beside it."""
    info = r["info"]
    sweep_s = r["sweep_ms"] / 1000.0
    own_gaps = info["n_gaps"] if not w.rows else int((w.mask[w.r0:w.r1] == 0).sum())
    m_own = info["m_end"] - info["m_begin"]
    upd = own_gaps * w.S * m_own * steps
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    b_upd = algorithmic_bytes_per_update(w.c["p"])
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    alu_peak = 148 * 128 * sm_mhz * 1e6 / 1e9  # Gop/s: SMs x FP32 lanes x max SM clock
    alu = ALG_OPS_PER_UPDATE * upd / sweep_s / 1e9 if sweep_s > 0 else None
    hbm = b_upd * upd / sweep_s / 1e9 if sweep_s > 0 else None
    traffic = None
    pipe = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "sweep_traffic.json")))
        if prof.get("config") == w.name:
            traffic = prof.get("dram_bytes_per_launch")
            if "fmaheavy_busy_frac_of_elapsed" in prof:
                # the bound pipe as ncu measures it on this config's launch (FFMA2 and Philox's
                # IMAD.WIDE share it): how busy it is, not a lane-op count
                pipe = {"pipe": "fma_heavy", "busy_frac": prof["fmaheavy_busy_frac_of_elapsed"],
                        "issue_active_frac": prof.get("issue_active_frac"), "source": prof.get("pipe_source")}
    except Exception:
        pass
    batch = info.get("batch", 0)
    variant = info.get("sweep_variant", 0)
    kernel = (f"k_sweep_quad (variant {variant}: two realization pairs per thread)"
              if variant in (22, 28, 33) and batch % 4 == 0 else f"k_sweep_half (variant {13 if variant in (22, 28, 33) else variant})")
    return {"bound": "alu", "kernel": kernel, "achieved": alu, "peak": alu_peak, "unit": "Gop/s",
            "frac": (alu / alu_peak) if alu else None, "traffic": traffic,
            "algorithmic_ops_per_update": ALG_OPS_PER_UPDATE,
            "peak_derivation": f"148 SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (max SM clock)",
            "sweep_launches_timed": r["sweep_launches"],
            "sweep_ms_per_launch": r["sweep_ms"] / max(r["sweep_launches"], 1),
            "sweep_share_of_step": r["sweep_ms"] / max(r["ms_per_step"] * steps, 1e-9),
            "sweep_updates_per_s": upd / sweep_s if sweep_s > 0 else None,
            "pipe_view": pipe,
            "hbm_view": {"achieved": hbm, "peak": hbm_peak, "unit": "GB/s",
                         "frac": (hbm / hbm_peak) if hbm else None,
                         "frac_of_8TBps": (hbm / 8000.0) if hbm else None,
                         "algorithmic_bytes_per_update": b_upd,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"
                         if "hbm_gbs" in peaks else "fallback 6650 GB/s (B200_PROFILING.md)"}}


def c4_subrecord(args, comm, ws, rank, local, dev, stream, peaks):
    """BASELINE C4 as row slabs over the N ranks (strong scaling): device and e2e timings and
    the sweep roofline, as a sub-record of the headline line."""
    w4 = Workload("C4", "rows", CONFIGS["C4"]["M"], CONFIGS["C4"]["sweeps"], comm, ws, rank, local, dev, stream)
    try:
        r4 = time_workload(w4, args.c4_steps, args.warmup, dev, ws, e2e=not args.no_e2e)
        c4 = {"config": {"workload": describe("C4", w4.c, w4.M, w4.S, False), "parallelism": f"row slabs x{ws}",
                         "rows_per_rank": w4.r1 - w4.r0, "gap_sites": w4.P, "updates_per_step": w4.updates_per_step(),
                         "input_per_rank": "own rows only (H2D of the slab; device memory holds own rows + 1 ghost "
                                           "row per side + the r_s n_s temperature halo)"},
              "steps": args.c4_steps, "warmup": args.warmup, "value": r4["value"], "unit": UNIT,
              "fill_time_ms": r4["ms_per_step"], "gpu_launches": int(r4["launches"]),
              "roofline": sweep_roofline(w4, r4, args.c4_steps, peaks), "target": "< 1000 ms end to end on 8 B200"}
        if "e2e" in r4:
            c4["e2e"] = r4["e2e"]
        return c4
    finally:
        w4.eng.close()


def run_mpr(args):
    import torch
    import torch.distributed as dist

    import paper_2212_01317_b200 as Pk
    from paper_2212_01317_b200.sharding import destroy_nccl_comm, make_nccl_comm

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    comm = make_nccl_comm(local) if ws > 1 else None
    if ws > 1:  # one rank generates (and caches) the large inputs, the others then read them
        if rank == 0:
            load_problem(args.config)
            if not args.no_c4:
                load_problem("C4")
        dist.barrier()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass

    name = args.config
    c0 = CONFIGS[name]
    scaling = SCALING[name]
    decomp = args.decomp or ("rows" if name == "C4" else "realizations")
    if decomp == "rows":
        scaling = "strong"
    M_arg = args.M or c0["M"]
    M_glob = M_arg * ws if scaling == "weak" else M_arg
    S = args.sweeps or c0["sweeps"]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    w = Workload(name, decomp, M_glob, S, comm, ws, rank, local, dev, stream)

    clocks = ClockSampler(local) if not args.no_clocks else None
    if clocks:
        clocks.start()
    r = time_workload(w, args.steps, args.warmup, dev, ws, e2e=not args.no_e2e, flush=flush)
    roof = sweep_roofline(w, r, args.steps, peaks)
    if ws == 1 and not args.no_e2e and name != "C4":
        try:
            r["e2e_pipelined"] = e2e_pipelined(w, args.steps, args.warmup)
        except Exception as ex:
            r["e2e_pipelined"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    c4 = None
    if not args.no_c4 and name != "C4":
        del flush
        w.eng.close()
        torch.cuda.empty_cache()
        try:
            c4 = c4_subrecord(args, comm, ws, rank, local, dev, stream, peaks)
        except Exception as ex:  # the optional sub-record must not cost the headline line
            c4 = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    else:
        w.eng.close()
    ck = clocks.stop() if clocks else None

    if rank == 0:
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": describe(name, w.c, M_arg, S, scaling == "weak"), "L": w.c["L"], "p": w.c["p"],
                           "gaps": w.c["gaps"], "gap_sites": w.P, "M_per_rank": M_arg if scaling == "weak" else None,
                           "M_total": M_glob, "sweeps": S, "updates_per_step": w.updates_per_step(),
                           "parallelism": (f"row slabs x{ws}" if decomp == "rows" else f"realizations x{ws}")
                           + (" (libmpr + NCCL)" if ws > 1 else ""),
                           "l2": "flushed between timed steps (256 MiB write, outside the events)"},
                "fill_time_ms": r["ms_per_step"],
                "gpu_launches": int(r["launches"]),
                "roofline": roof,
                "clocks": ck}
        if "e2e" in r:
            line["e2e"] = r["e2e"]
        if "e2e_pipelined" in r:
            line["e2e_pipelined"] = r["e2e_pipelined"]
        if c4 is not None:
            line["c4_rows"] = c4
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = {k: v for k, v in cpu_baseline_sample(w.z, w.mask, args.cpu_sample_realizations, S,
                                                                          w.c, args.cpu_threads).items()
                                    if k != "seconds"}
        print(json.dumps(line), flush=True)
    if comm:
        destroy_nccl_comm(comm)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_emulated(args):
    """W ranks as W contexts in this process on one GPU (in-process transport): the same SPMD
    calls as the NCCL path, timed per rank by wall clock around each whole fill (all ranks
    share the GPU, so this is not a scaling number); the all-gathered predictions are
    compared bit for bit with one context's."""
    import torch

    import paper_2212_01317_b200 as Pk
    from paper_2212_01317_b200.sharding import run_group
    W = args.emulate
    name = args.config
    decomp = args.decomp or ("rows" if name == "C4" else "realizations")
    c, truth, z, mask = load_problem(name)
    M = args.M or c["M"]
    S = args.sweeps or c["sweeps"]
    P_sites = int((mask == 0).sum())
    calib = Pk.load_calibration()
    ref = Pk.fill(z, mask, M, S, SEED_SIM, Pk.Config(), calib)

    def fn(rank, g):
        m = Pk.LeMpr(Pk.Config(group=g, group_rank=rank, shard=decomp), calib)
        times = []
        for k in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m.set_data(z, mask)
            m.estimate_local_params()
            m.simulate(M, S, SEED_SIM)
            m.predict_rows()
            torch.cuda.synchronize()
            if k >= args.warmup:
                times.append(time.perf_counter() - t0)
        full = m.predict()
        inf = m.info()
        m.close()
        return times, inf, full

    res = run_group(W, fn)
    per_step = max(sum(t) for t, _, _ in res) / args.steps
    same = all(np.array_equal(f.view(np.uint32), ref.view(np.uint32)) for _, _, f in res)
    line = {"metric": METRIC, "value": P_sites * S * M / per_step, "unit": UNIT, "n_gpus": 1, "emulated": True,
            "n_contexts": W, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * per_step,
            "higher_is_better": True, "scaling": "strong" if decomp == "rows" else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": describe(name, c, M, S, False), "parallelism": f"{decomp} x{W} on one GPU "
                       "(in-process transport)"},
            "bit_identical_to_one_context": bool(same),
            "per_rank": [{"rank": inf["rank"], "rows": [inf["row_begin"], inf["row_end"]],
                          "realizations": [inf["m_begin"], inf["m_end"]], "gap_sites_local": inf["n_gaps_local"],
                          "collectives": inf["comm_calls"]} for _, inf, _ in res],
            "note": "W contexts share ONE GPU: wall time of the SPMD fill, not a multi-GPU scaling measurement"}
    print(json.dumps(line), flush=True)
    return 0 if same else 1


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.emulate > 1:
        return run_emulated(args)
    return run_mpr(args)


if __name__ == "__main__":
    sys.exit(main())
