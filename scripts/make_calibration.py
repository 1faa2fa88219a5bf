#!/usr/bin/env python3
"""Build the e(T) calibration table that the energy matching of PAPER.md:90 inverts.

The paper defers the T <-> e relation to its reference [mz-dth18]; we
realise it as in SPEC.md:170-178 (reading R2 in DESIGN.md): for each T of a
log-spaced grid, an UNCONDITIONAL simulation (all sites free) of the MPR model on an
open L x L lattice, run with the oracle's own checkerboard Metropolis (oracle/, never
the CUDA path), records the mean whole-grid specific energy after equilibration.
Pool-adjacent-violators makes e non-decreasing, then ties are split by one fp32 ulp
so that e is strictly increasing (ARITH §F needs a strictly increasing table).

The table is pinned in tests/test_calibration.py by the closed forms
e(T) = -1 + T(L+1)/(4L) (harmonic, low T) and e(T) = -4/pi^2 - c/T (high T).

Output: paper_2212_01317_b200/data/calib_q0.5.txt (hex floats, exact round trip).
"""
from __future__ import annotations

import argparse
import os
import sys
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args):
    import oracle as O
    L, T, q, n_eq, n_meas, seed, m = args
    step = float(min(2 * np.pi, 3.0 * np.sqrt(T)))  # local moves: ~40% acceptance at any T
    return O.unconditional_energy(L, T, q=q, init="ordered", n_eq=n_eq, n_meas=n_meas, seed=seed, m=m,
                                  step=step)


def pava(y: np.ndarray) -> np.ndarray:
    """Isotonic (non-decreasing) least-squares fit, pool adjacent violators."""
    vals, wts, lens = [], [], []
    for v in y:
        vals.append(float(v)); wts.append(1.0); lens.append(1)
        while len(vals) > 1 and vals[-2] > vals[-1]:
            v2, w2, l2 = vals.pop(), wts.pop(), lens.pop()
            v1, w1, l1 = vals.pop(), wts.pop(), lens.pop()
            vals.append((v1 * w1 + v2 * w2) / (w1 + w2)); wts.append(w1 + w2); lens.append(l1 + l2)
    out = []
    for v, l in zip(vals, lens):
        out.extend([v] * l)
    return np.array(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=128)
    ap.add_argument("--K", type=int, default=48)
    ap.add_argument("--tmin", type=float, default=1e-4)
    ap.add_argument("--tmax", type=float, default=10.0)
    ap.add_argument("--q", type=float, default=0.5)
    ap.add_argument("--n-eq", type=int, default=400)
    ap.add_argument("--n-meas", type=int, default=800)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--seed", type=int, default=20221202)
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2212_01317_b200", "data", "calib_q0.5.txt"))
    a = ap.parse_args()
    Ts = np.float32(np.logspace(np.log10(a.tmin), np.log10(a.tmax), a.K))
    jobs = [(a.L, float(T), a.q, a.n_eq, a.n_meas, a.seed, m) for T in Ts for m in range(a.reps)]
    with Pool(os.cpu_count()) as pool:
        res = pool.map(_run, jobs)
    e_raw = np.array(res).reshape(a.K, a.reps).mean(1)
    e_iso = pava(e_raw).astype(np.float32)
    for k in range(1, a.K):  # strictly increasing in fp32
        if e_iso[k] <= e_iso[k - 1]:
            e_iso[k] = np.nextafter(e_iso[k - 1], np.float32(1))
    with open(a.out, "w") as f:
        f.write(f"# MPR calibration curve e(T): q={a.q} L={a.L} open boundary, unconditional "
                f"checkerboard Metropolis (oracle, local moves of half-width min(2pi, 3 sqrt T)), ordered init, n_eq={a.n_eq} n_meas={a.n_meas} "
                f"reps={a.reps} seed={a.seed}; PAVA + strict-increase fix\n")
        f.write("# columns: T (fp32 hex)  e (fp32 hex)  e_raw (fp64)\n")
        for T, e, er in zip(Ts, e_iso, e_raw):
            f.write(f"{float(T).hex()} {float(e).hex()} {er:.9f}\n")
    print(f"wrote {a.out}")
    for T, e, er in zip(Ts, e_iso, e_raw):
        print(f"T={T:.6g} e={e:.7f} raw={er:.7f}")


if __name__ == "__main__":
    main()
