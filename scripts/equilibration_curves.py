#!/usr/bin/env python3
"""Analogue of the paper's Fig. `fig:Equi_energies_wasatch_p03` on a
synthetic heterogeneous field: the whole-grid specific energy e(s) after each sweep,
averaged over M realizations, for MPR (one global T, RANDOM init), SV-MPR BST (l_b = 32,
n_s = 0) and SST (l_b = 32, n_s = 5), both BLOCK_MEAN init, next to the sample energy e_s
of Eq.(2). Everything runs on the GPU through the C-ABI (fused fixed-point energy trace,
ARITH §J); one JSON line per method with the curve and summary numbers:
  e_s, e_eq (mean of the last 10 sweeps), e(1), and s_rel: the first sweep whose mean
  energy is within 0.1 % of e_eq.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2212_01317_b200 as P
    from inputs.synth import heterogeneous_field, random_mask

    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=4096)
    ap.add_argument("--p", type=float, default=0.3)
    ap.add_argument("--M", type=int, default=100)
    ap.add_argument("--S", type=int, default=60)
    ap.add_argument("--nu", type=float, default=0.5)
    ap.add_argument("--corr-len", type=float, default=2.0)
    ap.add_argument("--spread", type=float, default=1.0, help="variance heterogeneity (1 = homogeneous)")
    a = ap.parse_args()
    truth = heterogeneous_field(a.L, nu=a.nu, corr_len=a.corr_len, spread=a.spread)
    mask = random_mask(a.L, a.L, a.p)
    z = np.where(mask != 0, truth, np.float32(np.nan)).astype(np.float32)
    calib = P.load_calibration()
    methods = {
        "MPR": P.Config(l_b=a.L, n_s=0, init="random"),
        "BST": P.Config(l_b=32, n_s=0, init="block_mean"),
        "SST": P.Config(l_b=32, n_s=5, r_s=2, init="block_mean"),
    }
    for name, cfg in methods.items():
        m = P.LeMpr(cfg, calib)
        m.set_data(z, mask)
        m.set_energy_trace(True)
        m.estimate_local_params()
        stats = m.debug(P.binding.MPR_BUF_BLOCK_STATS)
        e_s = float(-(stats[0].sum() * 2.0 ** -32) / stats[1].sum())  # Eq.(2) over all sample bonds
        # the energy trace covers the realizations of the last launch batch
        m.simulate(a.M, a.S, 2022)
        inf = m.info()
        E = m.debug(P.binding.MPR_BUF_ENERGY)
        lo, hi = inf["last_m_base"], min(inf["last_m_base"] + inf["last_batch"], a.M)
        curve = E[lo:hi].mean(axis=0)
        e_eq = float(curve[-10:].mean())
        s_rel = int(np.argmax(np.abs(curve - e_eq) <= 1e-3 * abs(e_eq)) + 1)
        print(json.dumps(dict(method=name, L=a.L, p=a.p, nu=a.nu, corr_len=a.corr_len, spread=a.spread, M=a.M, realizations_in_curve=hi - lo, S=a.S, e_s=e_s,
                              e_eq=e_eq, e_first=float(curve[0]), s_rel=s_rel, curve=[float(x) for x in curve])),
              flush=True)
        m.close()


if __name__ == "__main__":
    main()
