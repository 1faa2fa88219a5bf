#!/usr/bin/env python3
"""LE-MPR gap-filling benchmark (BASELINE.json metric: gap-site spin updates/s and fill time).

One "step" = one pass of the whole hot path over one synthetic
problem: set_data (device-resident input) -> estimate_local_params -> simulate
(M realizations x S sweeps) -> [all-reduce of the accumulator over ranks] -> predict.
The N=1 workload is BASELINE config 2 (1024^2 Matern nu=0.5 heterogeneous field, 33%
random gaps, M = 100, S = 30, SST l_b=32 r_s=2 n_s=5). Multi-GPU: realizations are
sharded over ranks (weak scaling: M per rank fixed), then one NCCL all-reduce of the
per-gap accumulator.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C2]

Rank 0 prints ONE JSON line. `--impl reference` times the CPU oracle (the reference arm
of this tier) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
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
# product form: sin of the half difference 9, four neighbour sine terms of 9, the sum
# phi' + phi 1, dE / beta 3, exp_spec 12, 4 conversions = 65) + half a Philox4x32-10 call
# (10 rounds x 2 IMAD.WIDE + 2 LOP3 = 40 per pair) = 85.
ALG_OPS_PER_UPDATE = 85
UNIT = "updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mpr", choices=["mpr", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--M", type=int, default=None, help="realizations per rank (default: config)")
    ap.add_argument("--sweeps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-realizations", type=int, default=4)
    ap.add_argument("--ref-sample-realizations", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--reduce", default="allreduce", choices=["allreduce", "ordered"],
                    help="realization sharding at N > 1: one NCCL all-reduce of the accumulators, or the "
                         "ordered chain (bit-identical to one GPU)")
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"],
                    help="row slabs at N > 1: the sweep kernel writes the boundary rows into the "
                         "neighbours' IPC-mapped state buffers (peer), or NCCL send/recv (nccl)")
    ap.add_argument("--decomp", default="realizations", choices=["realizations", "rows"],
                    help="multi-GPU split: realization shards (weak scaling, default) or row slabs "
                         "with one-row halos (strong scaling)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(cfg_name, args):
    c = dict(CONFIGS[cfg_name])
    M = args.M or c["M"]
    S = args.sweeps or c["sweeps"]
    truth, z, mask = make_problem(c["L"], c["p"], gaps=c["gaps"], nu=c["nu"])
    P = int((mask == 0).sum())
    desc = (f"{cfg_name}: {c['L']}x{c['L']} Whittle-Matern nu={c['nu']} heterogeneous field, "
            f"{int(round(c['p'] * 100))}% {c['gaps']} gaps, M={M} per rank, S={S} sweeps, "
            f"SST l_b=32 r_s=2 n_s=5, BLOCK_MEAN init, n_avg=1")
    return c, M, S, truth, z, mask, P, desc


def algorithmic_bytes_per_update(p, n_avg=1, S=30, b_T=4):
    """B_alg = 4/p + 8 + b_T bytes per gap-site update (+ 8 n_avg/S when the
    accumulation is a separate buffer, i.e. n_avg > 1)."""
    return 4.0 / p + 8.0 + b_T + (8.0 * n_avg / S if n_avg > 1 else 0.0)


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


def cpu_baseline_sample(z, mask, M_sample, S, c):
    """Time the CPU oracle, as it stands (single thread), on a bounded sample of the same
    workload: the full parameter stage + M_sample realizations x S sweeps."""
    import oracle as O
    from paper_2212_01317_b200.binding import load_calibration
    Tk, ek = load_calibration()
    cfg = O.OracleConfig()
    t0 = time.perf_counter()
    p = O.parameters(z, mask, cfg, Tk, ek)
    sim = O.simulate(p, mask, cfg, M_sample, S, SEED_SIM)
    zin = np.where(mask != 0, z, np.float32(0)).astype(np.float32)
    O.predict(zin, mask, sim["acc"], M_sample, 1, p.zmin, p.zmax, 0)
    dt = time.perf_counter() - t0
    P = int((mask == 0).sum())
    upd = P * S * M_sample
    return {"value": upd / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{c['L']}x{c['L']} grid, p={c['p']}: full parameter stage + realizations 0..{M_sample - 1} "
                      f"x {S} sweeps = {upd:.3e} gap-site updates in {dt:.2f} s (single thread, oracle/ as is)",
            "seconds": dt}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    c, M, S, truth, z, mask, P, desc = workload(args.config, args)
    Ms = max(1, args.ref_sample_realizations)
    for _ in range(args.warmup):
        cpu_baseline_sample(z, mask, Ms, S, c)
    times = []
    for _ in range(args.steps):
        r = cpu_baseline_sample(z, mask, Ms, S, c)
        times.append(r["seconds"])
    total = sum(times)
    value = P * S * Ms * args.steps / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": desc, "sample_realizations_per_step": Ms},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"per step: parameter stage + {Ms} realizations x {S} sweeps "
                                       f"({P * S * Ms:.3e} updates), single thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_mpr(args):
    import torch
    import torch.distributed as dist

    import paper_2212_01317_b200 as Pk

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    c, M, S, truth, z, mask, P, desc = workload(args.config, args)
    n = z.size
    Ly, Lx = z.shape
    stream = torch.cuda.current_stream(dev)
    calib = Pk.load_calibration()
    cfg = Pk.Config(device=local)
    eng = Pk.LeMpr(cfg, calib, stream=stream.cuda_stream)
    from paper_2212_01317_b200.sharding import (allreduce_accumulator, connect_peer_halo, exchange_halo,
                                                ordered_reduce_accumulator, row_range, shard_range,
                                                slab_realization_chunks)
    ordered = ws > 1 and args.decomp == "realizations" and args.reduce == "ordered"
    eng.set_deferred_reduce(ordered)
    rows = args.decomp == "rows"
    if rows:  # strong scaling: the whole M on every rank, the grid split into row slabs
        M_glob = M
        m0, m1 = 0, M
        r0, r1 = row_range(Ly, ws, rank)
    else:     # weak scaling: M realizations per rank
        M_glob = M * ws
        m0, m1 = shard_range(M_glob, ws, rank)

    # device-resident inputs (the "value" leg) and pinned host buffers (the e2e leg)
    z_dev = torch.from_numpy(np.nan_to_num(z, nan=0.0)).to(dev)
    m_dev = torch.from_numpy(mask).to(dev)
    out_dev = torch.empty((Ly, Lx), dtype=torch.float32, device=dev)
    z_pin = torch.from_numpy(np.nan_to_num(z, nan=0.0)).pin_memory()
    m_pin = torch.from_numpy(mask).pin_memory()
    out_pin = torch.empty((Ly, Lx), dtype=torch.float32).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def allreduce_acc():
        if ordered:
            ordered_reduce_accumulator(eng, rank, ws)
        elif ws > 1:
            allreduce_accumulator(eng.accumulator_tensor())

    def simulate():
        if not rows:
            eng.simulate_range(M_glob, S, SEED_SIM, m0, m1)
            return
        peer = ws > 1 and args.halo == "peer"
        for c0, c1 in slab_realization_chunks(M_glob):
            eng.slab_begin(M_glob, S, SEED_SIM, c0, c1, r0, r1)
            if peer:
                connect_peer_halo(eng, rank, ws)
            for s in range(1, S + 1):
                for colour in (0, 1):
                    eng.slab_half_sweep(s, colour)
                    if peer:  # the kernels wrote the halos into the neighbours' buffers
                        eng.sync()
                        dist.barrier()
                    elif ws > 1:
                        exchange_halo(eng, colour, r0, r1, rank, ws)
            eng.slab_end()

    def step_device():
        eng.set_data_device(z_dev.data_ptr(), m_dev.data_ptr(), Lx, Ly)
        eng.estimate_local_params()
        eng.reset_accumulator()
        simulate()
        allreduce_acc()
        eng.predict_device(out_dev.data_ptr())

    def step_host():
        Pk.binding._check(eng.ctx, Pk.load_library().mpr_set_data(eng.ctx, z_pin.data_ptr(), m_pin.data_ptr(), Lx, Ly))
        eng.shape = (Ly, Lx)
        eng.estimate_local_params()
        eng.reset_accumulator()
        simulate()
        allreduce_acc()
        Pk.binding._check(eng.ctx, Pk.load_library().mpr_predict(eng.ctx, out_pin.data_ptr()))

    def barrier():
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(args.warmup, 0)):
        step_device()
    barrier()
    eng.set_kernel_timing(True)
    launches0 = eng.info()["total_launches"]
    clocks = ClockSampler(local) if not args.no_clocks else None
    if clocks:
        clocks.start()
    barrier()
    total_ms = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (256 MiB > 126 MB L2), outside the events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step_device()
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    barrier()
    info = eng.info()
    launches = info["total_launches"] - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    updates_per_step = P * S * M_glob
    value = updates_per_step * args.steps / (total_ms / 1000.0)

    # dominant kernel: the half-sweep (CUDA events on the library's stream around the sweep loops)
    sweep_ms, sweep_n = info["sweep_ms"], info["sweep_launches"]
    P_loc = int((mask[r0:r1] == 0).sum()) if rows else P
    sweep_updates = P_loc * S * (m1 - m0) * args.steps
    sweep_s = sweep_ms / 1000.0
    b_upd = algorithmic_bytes_per_update(c["p"])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_achieved = b_upd * sweep_updates / sweep_s / 1e9 if sweep_s > 0 else None
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    alu_peak = 148 * 128 * sm_mhz * 1e6 / 1e9  # Gop/s: SMs x FP32 lanes x max SM clock
    alu_achieved = ALG_OPS_PER_UPDATE * sweep_updates / sweep_s / 1e9 if sweep_s > 0 else None
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "sweep_traffic.json")))
        if prof.get("config") == args.config:
            traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass

    # e2e through the public API with pinned host buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        for _ in range(max(args.warmup, 1)):  # first use of the host-buffer path, untimed
            step_host()
        barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            step_host()
        barrier()
        wall = time.perf_counter() - w0
        tw = torch.tensor([wall], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        wall = float(tw.item())
        e2e = {"value": updates_per_step * args.steps / wall, "unit": UNIT,
               "h2d_bytes_per_step": int(n * 4 + n * 1), "d2h_bytes_per_step": int(n * 4),
               "fill_time_ms": 1000 * wall / args.steps}
    ck = clocks.stop() if clocks else None

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if rows else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": desc, "L": c["L"], "p": c["p"], "gaps": c["gaps"], "gap_sites": P,
                           "M_per_rank": M, "M_total": M_glob, "sweeps": S,
                           "updates_per_step": updates_per_step, "parallelism": (f"row slabs x{ws}" + (f", {args.halo} halo" if ws > 1 else "")) if rows
                           else f"realizations x{ws}" + (f", {args.reduce} reduce" if ws > 1 else ""),
                           "l2": "flushed between timed steps (256 MiB write, outside the events)"},
                "fill_time_ms": total_ms / args.steps,
                "gpu_launches": int(launches),
                "roofline": {"bound": "alu", "kernel": sweep_kernel_name(info.get("sweep_variant", 0),
                                                               (lambda c: c[1] - c[0])(slab_realization_chunks(M_glob)[0])
                                                               if rows else info.get("batch", 0)),
                             "achieved": alu_achieved,
                             "peak": alu_peak, "unit": "Gop/s",
                             "frac": (alu_achieved / alu_peak) if alu_achieved else None,
                             "traffic": traffic,
                             "algorithmic_ops_per_update": ALG_OPS_PER_UPDATE,
                             "peak_derivation": f"148 SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (max SM clock)",
                             "sweep_launches_timed": sweep_n, "sweep_ms_per_launch": sweep_ms / max(sweep_n, 1),
                             "sweep_share_of_step": sweep_ms / max(total_ms, 1e-9),
                             "sweep_updates_per_s": sweep_updates / sweep_s if sweep_s > 0 else None,
                             "hbm_view": {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                                          "frac": (hbm_achieved / hbm_peak) if hbm_achieved else None,
                                          "frac_of_8TBps": (hbm_achieved / 8000.0) if hbm_achieved else None,
                                          "algorithmic_bytes_per_update": b_upd,
                                          "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"
                                          if "hbm_gbs" in peaks else "fallback 6650 GB/s (B200_PROFILING.md)"}},
                "clocks": ck}
        if e2e:
            line["e2e"] = e2e
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = {k: v for k, v in cpu_baseline_sample(z, mask, args.cpu_sample_realizations, S,
                                                                          c).items() if k != "seconds"}
        print(json.dumps(line), flush=True)
    eng.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def sweep_kernel_name(variant, batch):
    """Name of the half-sweep kernel the library launched (mpr_info.sweep_variant and the
    realization batch: the quad kernel needs an even pair count)."""
    if variant in (22, 28) and batch % 4 == 0:
        return f"k_sweep_quad (variant {variant}: two realization pairs per thread)"
    return f"k_sweep_half (variant {13 if variant in (22, 28) else variant})"


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_mpr(args)


if __name__ == "__main__":
    sys.exit(main())
