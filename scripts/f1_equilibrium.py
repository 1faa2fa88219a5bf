#!/usr/bin/env python3
"""Row f1 on the GPU: for MPR (one global T, RANDOM init), SV-MPR BST
(l_b = 32, n_s = 0) and SST (l_b = 32, n_s = 5, r_s = 2; both BLOCK_MEAN init):
  * the energy trace over S fixed sweeps (mean over the realizations of the last batch):
    e_s (Eq.(2) over all sample bonds), e_eq (mean of the last 10 sweeps), e(1);
  * the adaptive protocol with the DERIVED slope tolerance (reading R22: SE(e_s) / n_fit,
    n_fit = 20, n_f = 5, cap 200): the tolerance, s_eq of every realization, device time.
Fields: "hetero" (smooth variance heterogeneity, inputs.synth.heterogeneous_field) and
"walls" (sharp variance domain walls, inputs.synth.domain_wall_field). One JSON line per
(field, L, p, method)."""
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
    from inputs.synth import domain_wall_field, heterogeneous_field, random_mask
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="256,2048,8192")
    ap.add_argument("--ps", default="0.3,0.85")
    ap.add_argument("--fields", default="hetero,walls")
    ap.add_argument("--M", type=int, default=10)
    ap.add_argument("--S", type=int, default=60)
    ap.add_argument("--corr-len", type=float, default=2.0,
                    help="Matern correlation length in sites (2: rough, sample T of the order of the paper's 0.07)")
    a = ap.parse_args()
    calib = P.load_calibration()
    for field in a.fields.split(","):
        for L in map(int, a.sizes.split(",")):
            truth = (heterogeneous_field(L, corr_len=a.corr_len) if field == "hetero"
                     else domain_wall_field(L, corr_len=a.corr_len))
            for p in map(float, a.ps.split(",")):
                mask = random_mask(L, L, p)
                z = np.where(mask != 0, truth, np.float32(np.nan)).astype(np.float32)
                methods = {"MPR": P.Config(l_b=L, n_s=0, init="random"),
                           "BST": P.Config(l_b=32, n_s=0, init="block_mean"),
                           "SST": P.Config(l_b=32, n_s=5, r_s=2, init="block_mean")}
                for name, cfg in methods.items():
                    m = P.LeMpr(cfg, calib)
                    m.set_data(z, mask)
                    m.set_energy_trace(True)
                    m.estimate_local_params()
                    stats = m.debug(P.binding.MPR_BUF_BLOCK_STATS)
                    e_s = float(-(stats[0].sum() * 2.0 ** -32) / stats[1].sum())
                    m.simulate(a.M, a.S, 2022)
                    inf = m.info()
                    E = m.debug(P.binding.MPR_BUF_ENERGY)
                    lo, hi = inf["last_m_base"], min(inf["last_m_base"] + inf["last_batch"], a.M)
                    curve = E[lo:hi].mean(axis=0)
                    e_eq = float(curve[-10:].mean())
                    m.set_energy_trace(False)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    s_eq = m.simulate_adaptive(a.M, 7, n_fit=20, n_f=5, max_sweeps=200, slope_tol="derived")
                    dt = time.perf_counter() - t0
                    inf = m.info()
                    m.close()
                    print(json.dumps(dict(field=field, corr_len=a.corr_len, L=L, p=p, method=name, M=a.M, S=a.S,
                                          e_s=e_s, e_eq=e_eq, median_T=inf["median_T"],
                                          e_first=float(curve[0]), e_eq_minus_e_s=e_eq - e_s,
                                          slope_tol_derived=inf["slope_tol"], s_eq=[int(x) for x in s_eq],
                                          s_eq_median=float(np.median(np.abs(s_eq))),
                                          forced=int((s_eq < 0).sum()), adaptive_wall_s=dt,
                                          curve=[float(x) for x in curve])), flush=True)


if __name__ == "__main__":
    main()
