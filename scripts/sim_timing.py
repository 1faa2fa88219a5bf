#!/usr/bin/env python3
"""Wall time of mpr_simulate for a config, with and without CUDA graphs (MPR_NO_GRAPHS)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import paper_2212_01317_b200 as P
    from inputs.synth import CONFIGS, make_problem
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    c = CONFIGS[name]
    L = int(sys.argv[2]) if len(sys.argv) > 2 else c["L"]
    p = float(sys.argv[3]) if len(sys.argv) > 3 else c["p"]
    M = int(sys.argv[4]) if len(sys.argv) > 4 else c["M"]
    truth, z, mask = make_problem(L, p, gaps=c["gaps"], nu=c["nu"])
    Pg = int((mask == 0).sum())
    ref = None
    for ng in ("0", "1"):
        os.environ["MPR_NO_GRAPHS"] = ng
        m = P.LeMpr(P.Config(), P.load_calibration())
        m.set_data(z, mask)
        m.estimate_local_params()
        for _ in range(3):
            m.simulate(M, c["sweeps"], 7)
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            m.simulate(M, c["sweeps"], 7)
            ts.append(time.perf_counter() - t0)
        pred = m.predict()
        same = ref is None or bool(np.array_equal(pred.view(np.uint32), ref.view(np.uint32)))
        ref = pred if ref is None else ref
        t = float(np.median(ts))
        print(f"L={L} p={p} M={M} graphs={'off' if ng == '1' else 'on'}: simulate {1e3 * t:.3f} ms, "
              f"{Pg * c['sweeps'] * M / t:.3e} updates/s, bitwise_same={same}")
        m.close()


if __name__ == "__main__":
    main()
