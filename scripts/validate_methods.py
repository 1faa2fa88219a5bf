#!/usr/bin/env python3
"""Row f4 validation harness (§3.2, Table 2, fig:err-p): MPR (one global T,
l_b >= L) vs SV-MPR BST (l_b = 32, n_s = 0) vs SV-MPR SST (l_b = 32, n_s = 5) on synthetic
heterogeneous fields. For each missing ratio p, K random thinnings of the same field are
filled on the GPU; AAE and RASE (Eq.(3)) are averaged over the thinnings (MAAE, MRASE) and
reported with the paired error ratios err_SV-MPR / err_MPR of fig:err-p.

  python scripts/validate_methods.py [--L 256] [--K 20] [--M 20] [--ps 0.3,0.5,0.7,0.85]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def errors(pred, truth, mask):
    gaps = mask == 0
    e = truth[gaps].astype(np.float64) - pred[gaps].astype(np.float64)
    return float(np.mean(np.abs(e))), float(np.sqrt(np.mean(e * e)))


def run(L=256, K=20, M=20, S=30, ps=(0.3, 0.5, 0.7, 0.85), skew=True, seed_field=2212):
    import paper_2212_01317_b200 as P
    from inputs.synth import heterogeneous_field, random_mask
    truth = heterogeneous_field(L, corr_len=max(L / 32, 4.0), skew=skew, seed=seed_field)
    calib = P.load_calibration()
    methods = {"MPR": P.Config(l_b=max(L, 2), n_s=0), "BST": P.Config(l_b=32, n_s=0),
               "SST": P.Config(l_b=32, n_s=5, r_s=2)}
    engines = {k: P.LeMpr(c, calib) for k, c in methods.items()}
    rows = []
    for p in ps:
        errs = {k: [] for k in methods}
        for k in range(K):
            mask = random_mask(L, L, p, seed=1000 + k)
            z = np.where(mask != 0, truth, np.nan).astype(np.float32)
            for name, eng in engines.items():
                eng.set_data(z, mask)
                eng.estimate_local_params()
                eng.simulate(M, S, 20221202 + k)
                errs[name].append(errors(eng.predict(), truth, mask))
        rec = {"L": L, "p": p, "K": K, "M": M, "S": S}
        for name in methods:
            a = np.array(errs[name])
            rec[f"MAAE_{name}"] = float(a[:, 0].mean())
            rec[f"MRASE_{name}"] = float(a[:, 1].mean())
        for name in ("BST", "SST"):
            ra = np.array(errs[name]) / np.array(errs["MPR"])
            rec[f"ratio_AAE_{name}"] = float(ra[:, 0].mean())
            rec[f"ratio_RASE_{name}"] = float(ra[:, 1].mean())
            rec[f"win_rate_RASE_{name}"] = float(np.mean(ra[:, 1] < 1))
        rows.append(rec)
        print(json.dumps(rec), flush=True)
    for eng in engines.values():
        eng.close()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=256)
    ap.add_argument("--K", type=int, default=20)
    ap.add_argument("--M", type=int, default=20)
    ap.add_argument("--S", type=int, default=30)
    ap.add_argument("--ps", default="0.3,0.5,0.7,0.85")
    ap.add_argument("--no-skew", action="store_true")
    a = ap.parse_args()
    run(a.L, a.K, a.M, a.S, tuple(float(x) for x in a.ps.split(",")), skew=not a.no_skew)


if __name__ == "__main__":
    main()
