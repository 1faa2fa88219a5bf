#!/usr/bin/env python3
"""BASELINE config 5 sweep on one B200: fill time and gap-site updates/s versus grid size L,
missing ratio p, smoothing window w = 2 r_s + 1 and realization count M, plus the paper's
(L, p) points (256 / 2048 / 8192 at p = 0.85, Tables 2-3) with the adaptive protocol.

Each point: device-resident fill (set_data -> estimate -> simulate -> predict) timed with CUDA
events (median of `--reps` after one warm-up) and the host-buffer end-to-end fill (wall clock).
Prints one JSON line per point.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2212_01317_b200 as P
    from inputs.synth import heterogeneous_field, random_mask

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--max-L", type=int, default=16384)
    ap.add_argument("--only-paper", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    calib = P.load_calibration()
    fields = {}

    def field(L):
        if L not in fields:
            fields.clear()
            fields[L] = heterogeneous_field(L)
        return fields[L]

    def run(L, p, M, S=30, rs=2, adaptive=False, tag="", slope_tol=0.0):
        truth = field(L)
        mask = random_mask(L, L, p)
        z = np.where(mask != 0, truth, np.float32(0)).astype(np.float32)
        Pg = int((mask == 0).sum())
        eng = P.LeMpr(P.Config(r_s=rs), calib, stream=stream.cuda_stream)
        zd = torch.from_numpy(z).to(dev)
        md = torch.from_numpy(mask).to(dev)
        out = torch.empty((L, L), device=dev)
        sweeps_used = []

        def fill():
            eng.set_data_device(zd.data_ptr(), md.data_ptr(), L, L)
            eng.estimate_local_params()
            if adaptive:
                s = eng.simulate_adaptive(M, 7, n_fit=20, n_f=5, max_sweeps=500, slope_tol=slope_tol)
                sweeps_used.append(float(np.mean(np.abs(s)) + 1))
            else:
                eng.simulate(M, S, 7)
            eng.predict_device(out.data_ptr())

        fill()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fill()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        # end to end through the C-ABI from pinned host buffers (H2D of z + mask and D2H of the
        # predictions inside), after one untimed use of the host path; median of --reps
        zp = torch.from_numpy(z).pin_memory()
        mp = torch.from_numpy(mask).pin_memory()
        op = torch.empty((L, L), dtype=torch.float32).pin_memory()
        L_ = P.load_library()

        def fill_host():
            P.binding._check(eng.ctx, L_.mpr_set_data(eng.ctx, zp.data_ptr(), mp.data_ptr(), L, L))
            eng.shape = (L, L)
            eng.estimate_local_params()
            if adaptive:
                eng.simulate_adaptive(M, 7, n_fit=20, n_f=5, max_sweeps=500, slope_tol=slope_tol)
            else:
                eng.simulate(M, S, 7)
            P.binding._check(eng.ctx, L_.mpr_predict(eng.ctx, op.data_ptr()))

        fill_host()
        es = []
        for _ in range(a.reps):
            w0 = time.perf_counter()
            fill_host()
            es.append(1e3 * (time.perf_counter() - w0))
        e2e = float(np.median(es))
        sw = float(np.mean(sweeps_used)) if adaptive else S
        rec = dict(tag=tag, L=L, p=p, gap_sites=Pg, M=M, window=2 * rs + 1, protocol=f"adaptive tol={slope_tol:g}" if adaptive else f"S={S}",
                   mean_sweeps=sw, fill_ms=t, e2e_fill_ms=e2e, updates_per_s=Pg * sw * M / (t / 1e3))
        print(json.dumps(rec), flush=True)
        eng.close()

    Ls = [] if a.only_paper else [L for L in (256, 1024, 2048, 4096, 8192, 16384) if L <= a.max_L]
    for L in Ls:                       # size sweep (p = 0.5, w = 5, M = 10)
        run(L, 0.5, 10, tag="size")
    for p in (() if a.only_paper else (0.33, 0.5, 0.9)):  # missing-ratio sweep at 4096^2
        run(4096, p, 10, tag="ratio")
    for rs in (() if a.only_paper else (1, 2, 4, 7)):     # smoothing window 3..15 at 4096^2
        run(4096, 0.5, 10, rs=rs, tag="window")
    for M in (() if a.only_paper else (10, 100, 1000)):   # realization count at 1024^2
        run(1024, 0.5, M, tag="realizations")
    for L in (256, 2048, 8192):        # the paper's sizes at p = 0.85 (Tables 2-3), one chain
        if L <= a.max_L:
            for tol in (0.0, 1e-5):
                run(L, 0.85, 1, adaptive=True, tag="paper-point adaptive M=1", slope_tol=tol)
                run(L, 0.85, 100, adaptive=True, tag="paper-point adaptive M=100", slope_tol=tol)


if __name__ == "__main__":
    main()
