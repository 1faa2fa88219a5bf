#!/usr/bin/env python3
"""SPEC acceptance criteria 3 and 4 on the GPU (row f1), on SPEC's
validation generator (the two-regime field, scripts/validate_methods.make_truth) at 512^2,
p = 0.3, over 20 paired runs (run k: mask seed 1000 + k, simulation seed k):
  3. equilibration speed: the adaptive protocol (n_fit = 20, n_f = 5, derived tolerance,
     reading R22, cap 200) with RANDOM init reaches equilibrium in <= 50 sweeps, and with
     BLOCK_MEAN init in strictly fewer sweeps than RANDOM on >= 80 % of the runs (SST);
  4. equilibrium-energy ordering: the post-equilibrium mean specific energy (sweeps 51-60 of a
     60-sweep run, BLOCK_MEAN init) satisfies e(BST) > e(SST) on >= 80 % of the runs.
Prints one JSON line per run and a summary line."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def main():
    import paper_2212_01317_b200 as P
    from inputs.synth import random_mask
    from validate_methods import make_truth
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--corr-len", type=float, default=0.0,
                    help="field correlation length in sites (0: the validation default L/32; 2: rough, sample "
                         "temperatures of the order of the paper's T = 0.067)")
    a = ap.parse_args()
    L, p, runs = 512, 0.3, 20
    if a.corr_len > 0:
        from inputs.synth import domain_wall_field
        truth = domain_wall_field(L, tile=L // 2, low=0.1, high=10.0, corr_len=a.corr_len, seed=2212)
    else:
        truth = make_truth(L, "two-regime")
    calib = P.load_calibration()
    res = []
    for k in range(runs):
        mask = random_mask(L, L, p, seed=1000 + k)
        z = np.where(mask != 0, truth, np.float32(np.nan)).astype(np.float32)
        rec = {"run": k}
        for init in ("random", "block_mean"):
            m = P.LeMpr(P.Config(l_b=32, n_s=5, r_s=2, init=init), calib)
            m.set_data(z, mask)
            m.estimate_local_params()
            s = m.simulate_adaptive(1, k, n_fit=20, n_f=5, max_sweeps=200, slope_tol="derived")
            rec[f"s_eq_SST_{init}"] = int(s[0])
            m.close()
        for name, cfg in (("BST", P.Config(l_b=32, n_s=0)), ("SST", P.Config(l_b=32, n_s=5, r_s=2))):
            m = P.LeMpr(cfg, calib)
            m.set_data(z, mask)
            m.set_energy_trace(True)
            m.estimate_local_params()
            m.simulate(1, 60, k)
            E = m.debug(P.binding.MPR_BUF_ENERGY)
            rec[f"e_eq_{name}"] = float(E[0, -10:].mean())
            m.close()
        if k == 0:
            m = P.LeMpr(P.Config(l_b=32, n_s=5, r_s=2), calib)
            m.set_data(z, mask)
            m.estimate_local_params()
            rec["median_T"] = m.info()["median_T"]
            m.close()
        res.append(rec)
        print(json.dumps(rec), flush=True)
    sr = np.array([abs(r["s_eq_SST_random"]) for r in res])
    sb = np.array([abs(r["s_eq_SST_block_mean"]) for r in res])
    forced_r = sum(r["s_eq_SST_random"] < 0 for r in res)
    ebst = np.array([r["e_eq_BST"] for r in res])
    esst = np.array([r["e_eq_SST"] for r in res])
    print(json.dumps({"summary": True, "L": L, "p": p, "runs": runs, "corr_len": a.corr_len or L / 32,
                      "crit3_random_max_sweeps": int(sr.max()), "crit3_random_forced": int(forced_r),
                      "crit3_random_le_50": bool(sr.max() <= 50 and forced_r == 0),
                      "crit3_block_mean_faster_frac": float(np.mean(sb < sr)),
                      "s_eq_random_median": float(np.median(sr)), "s_eq_block_mean_median": float(np.median(sb)),
                      "crit4_bst_above_sst_frac": float(np.mean(ebst > esst)),
                      "e_eq_BST_mean": float(ebst.mean()), "e_eq_SST_mean": float(esst.mean())}), flush=True)


if __name__ == "__main__":
    main()
