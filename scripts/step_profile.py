#!/usr/bin/env python3
"""Host-side breakdown of one bench step (C2): wall time of each C-ABI call, synchronised."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2212_01317_b200 as P
    from inputs.synth import CONFIGS, make_problem
    c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
    truth, z, mask = make_problem(c["L"], c["p"], gaps=c["gaps"], nu=c["nu"])
    Ly, Lx = z.shape
    dev = torch.device("cuda", 0)
    zd = torch.from_numpy(np.nan_to_num(z)).to(dev)
    md = torch.from_numpy(mask).to(dev)
    out = torch.empty((Ly, Lx), device=dev)
    eng = P.LeMpr(P.Config(), P.load_calibration(), stream=torch.cuda.current_stream(dev).cuda_stream)
    stages = {}
    for it in range(8):
        t = {}
        t0 = time.perf_counter()
        eng.set_data_device(zd.data_ptr(), md.data_ptr(), Lx, Ly); torch.cuda.synchronize(); t["set_data"] = time.perf_counter()
        eng.estimate_local_params(); torch.cuda.synchronize(); t["estimate"] = time.perf_counter()
        eng.reset_accumulator(); torch.cuda.synchronize(); t["reset_acc"] = time.perf_counter()
        eng.simulate_range(c["M"], c["sweeps"], 1, 0, c["M"]); torch.cuda.synchronize(); t["simulate"] = time.perf_counter()
        eng.predict_device(out.data_ptr()); torch.cuda.synchronize(); t["predict"] = time.perf_counter()
        prev = t0
        if it >= 3:
            for k, v in t.items():
                stages.setdefault(k, []).append(1e3 * (v - prev))
                prev = v
    for k, v in stages.items():
        print(f"{k:12s} {np.median(v):8.3f} ms")
    print(f"{'total':12s} {sum(np.median(v) for v in stages.values()):8.3f} ms")


if __name__ == "__main__":
    main()
