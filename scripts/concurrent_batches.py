#!/usr/bin/env python3
"""Would the 2-realization tail batch of a 4k + 2 split overlap with the 4k batch? Two
independent contexts on two CUDA streams of one GPU, one simulating M = 8 and the other
M = 2 (same grid), timed alone and concurrently from two host threads."""
import sys, os, time, threading, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_01317_b200 as P
from inputs.synth import heterogeneous_field, random_mask

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
truth = heterogeneous_field(L); mask = random_mask(L, L, 0.5)
z = np.where(mask != 0, truth, np.float32(0)).astype(np.float32)
calib = P.load_calibration()
dev = torch.device('cuda', 0)
zd = torch.from_numpy(z).to(dev); md = torch.from_numpy(mask).to(dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
engs = []
for s in (s1, s2):
    e = P.LeMpr(P.Config(), calib, stream=s.cuda_stream)
    e.set_data_device(zd.data_ptr(), md.data_ptr(), L, L); e.estimate_local_params()
    engs.append(e)
def run(e, M):
    e.simulate(M, 30, 7)
for e, M in ((engs[0], 8), (engs[1], 2)):
    run(e, M)
torch.cuda.synchronize()
res = {}
for name, jobs in (("M8 alone", [(0, 8)]), ("M2 alone", [(1, 2)]), ("M8 + M2 sequential", [(0, 8), (1, 2)])):
    t0 = time.perf_counter()
    for i, M in jobs:
        run(engs[i], M)
    torch.cuda.synchronize()
    res[name] = 1e3 * (time.perf_counter() - t0)
ts = [threading.Thread(target=run, args=(engs[0], 8)), threading.Thread(target=run, args=(engs[1], 2))]
t0 = time.perf_counter()
for t in ts: t.start()
for t in ts: t.join()
torch.cuda.synchronize()
res["M8 || M2 concurrent"] = 1e3 * (time.perf_counter() - t0)
print(json.dumps({"L": L, **{k: round(v, 2) for k, v in res.items()}}))
