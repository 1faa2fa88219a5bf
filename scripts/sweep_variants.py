#!/usr/bin/env python3
"""Time the half-sweep kernel variants (MPR_SWEEP_VARIANT) on one config; check they agree bitwise."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs.synth import CONFIGS, make_problem  # noqa: E402


def sm_clock():
    """Current SM clock (MHz) right after a measurement, or None without nvidia-smi."""
    import subprocess
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                             capture_output=True, text=True, timeout=10).stdout
        return int(out.strip().splitlines()[0])
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--variants", default="5,13,22,28")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--M", type=int, default=None)
    ap.add_argument("--max-batch", default="0", help="comma list of max_batch values to try")
    ap.add_argument("--rounds", type=int, default=1, help="repeat the whole variant list (interleaved)")
    a = ap.parse_args()
    import paper_2212_01317_b200 as P
    c = CONFIGS[a.config]
    M = a.M or c["M"]
    truth, z, mask = make_problem(c["L"], c["p"], gaps=c["gaps"], nu=c["nu"])
    Pg = int((mask == 0).sum())
    calib = P.load_calibration()
    ref = None
    runs = [(int(v), int(b)) for v in a.variants.split(",") for b in a.max_batch.split(",")] * a.rounds
    for v, mb in runs:
        os.environ["MPR_SWEEP_VARIANT"] = str(v)
        m = P.LeMpr(P.Config(max_batch=mb), calib)
        m.set_data(z, mask)
        m.estimate_local_params()
        m.simulate(M, c["sweeps"], 1)  # warm-up
        m.set_kernel_timing(True)
        for _ in range(a.reps):
            m.simulate(M, c["sweeps"], 1)
        inf = m.info()
        pred = m.predict()
        if ref is None:
            ref = pred
        same = bool(np.array_equal(pred.view(np.uint32), ref.view(np.uint32)))
        per = inf["sweep_ms"] / inf["sweep_launches"]
        ups = Pg * M / 2 / (per / 1e3)
        per = inf["sweep_ms"] / a.reps / (2 * c["sweeps"])  # per half-sweep of the whole M
        ups = Pg * M / 2 / (per / 1e3)
        print(json.dumps({"variant": v, "max_batch": mb, "batch": inf["batch"], "config": a.config, "M": M,
                          "ms_per_halfsweep_allM": per,
                          "updates_per_s": ups, "bitwise_equal_to_first": same, "sm_mhz": sm_clock()}), flush=True)
        m.close()


if __name__ == "__main__":
    main()
