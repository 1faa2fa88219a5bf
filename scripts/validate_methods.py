#!/usr/bin/env python3
"""Row f4 validation harness (§3.2, Table 2, fig:err-p): MPR (one global T,
l_b >= L) vs SV-MPR BST (l_b = 32, n_s = 0) vs SV-MPR SST (l_b = 32, n_s = 5) on synthetic
heterogeneous fields. For each missing ratio p, K random thinnings of the same field are
filled on the GPU; AAE and RASE (Eq.(3)) are averaged over the thinnings (MAAE, MRASE) and
reported with the paired error ratios err_SV-MPR / err_MPR of fig:err-p.

  python scripts/validate_methods.py [--L 256] [--K 20] [--M 20] [--ps 0.3,0.5,0.7,0.85]
  python scripts/validate_methods.py --sweep lb|ns --L 512 --K 10   (SST vs l_b / n_s at p = 0.7)
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


def make_truth(L, field="heterogeneous", skew=True, seed_field=2212):
    """The synthetic field: 'heterogeneous' (smooth variance variation, inputs.synth) or
    'two-regime' (SPEC's validation generator: a low-variance (sigma 0.1) and a high-variance
    (sigma 10) domain, here the 2x2 quadrant checkerboard of inputs.synth.domain_wall_field)."""
    from inputs.synth import domain_wall_field, heterogeneous_field
    if field == "two-regime":
        return domain_wall_field(L, tile=L // 2, low=0.1, high=10.0, corr_len=max(L / 32, 4.0), seed=seed_field)
    return heterogeneous_field(L, corr_len=max(L / 32, 4.0), skew=skew, seed=seed_field)


def run(L=256, K=20, M=20, S=30, ps=(0.3, 0.5, 0.7, 0.85), skew=True, seed_field=2212, field="heterogeneous"):
    import paper_2212_01317_b200 as P
    from inputs.synth import random_mask
    truth = make_truth(L, field, skew, seed_field)
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
        rec = {"field": field, "L": L, "p": p, "K": K, "M": M, "S": S}
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


def run_param_sweep(param, values, L=512, K=10, M=20, S=30, p=0.7, skew=True, seed_field=2212):
    """SV-MPR SST error ratios to MPR versus one parameter: the block side l_b (BST and SST)
    or the number of smoothing passes n_s (SST; n_s = 0 is BST). Same fields and thinnings
    as run(); one JSON line per value."""
    import paper_2212_01317_b200 as P
    from inputs.synth import heterogeneous_field, random_mask
    truth = heterogeneous_field(L, corr_len=max(L / 32, 4.0), skew=skew, seed=seed_field)
    calib = P.load_calibration()
    mpr = P.LeMpr(P.Config(l_b=max(L, 2), n_s=0), calib)
    masks = [random_mask(L, L, p, seed=1000 + k) for k in range(K)]
    base = []
    for k, mask in enumerate(masks):
        z = np.where(mask != 0, truth, np.nan).astype(np.float32)
        mpr.set_data(z, mask)
        mpr.estimate_local_params()
        mpr.simulate(M, S, 20221202 + k)
        base.append(errors(mpr.predict(), truth, mask))
    mpr.close()
    base = np.array(base)
    rows = []
    for v in values:
        cfg = P.Config(l_b=v, n_s=5, r_s=2) if param == "lb" else P.Config(l_b=32, n_s=v, r_s=2)
        eng = P.LeMpr(cfg, calib)
        errs = []
        for k, mask in enumerate(masks):
            z = np.where(mask != 0, truth, np.nan).astype(np.float32)
            eng.set_data(z, mask)
            eng.estimate_local_params()
            eng.simulate(M, S, 20221202 + k)
            errs.append(errors(eng.predict(), truth, mask))
        eng.close()
        ra = np.array(errs) / base
        rec = {"sweep": param, param: v, "L": L, "p": p, "K": K, "M": M, "S": S,
               "MAAE_MPR": float(base[:, 0].mean()), "MRASE_MPR": float(base[:, 1].mean()),
               "MAAE": float(np.array(errs)[:, 0].mean()), "MRASE": float(np.array(errs)[:, 1].mean()),
               "ratio_AAE": float(ra[:, 0].mean()), "ratio_RASE": float(ra[:, 1].mean())}
        rows.append(rec)
        print(json.dumps(rec), flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=256)
    ap.add_argument("--K", type=int, default=20)
    ap.add_argument("--M", type=int, default=20)
    ap.add_argument("--S", type=int, default=30)
    ap.add_argument("--ps", default="0.3,0.5,0.7,0.85")
    ap.add_argument("--no-skew", action="store_true")
    ap.add_argument("--field", default="heterogeneous", choices=["heterogeneous", "two-regime"])
    ap.add_argument("--sweep", default="p", choices=["p", "lb", "ns"],
                    help="p: MPR/BST/SST vs missing ratio; lb: SST vs block side; ns: vs smoothing passes")
    ap.add_argument("--values", default=None, help="comma list for --sweep lb / ns")
    a = ap.parse_args()
    if a.sweep == "p":
        run(a.L, a.K, a.M, a.S, tuple(float(x) for x in a.ps.split(",")), skew=not a.no_skew, field=a.field)
    else:
        vals = a.values or ("8,16,32,64,128" if a.sweep == "lb" else "0,1,2,5,10")
        run_param_sweep(a.sweep, [int(x) for x in vals.split(",")], L=a.L, K=a.K, M=a.M, S=a.S,
                        skew=not a.no_skew)


if __name__ == "__main__":
    main()
