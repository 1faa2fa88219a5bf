import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2212_01317_b200 as P
from inputs.synth import heterogeneous_field, random_mask
import os
L = 8192
truth = heterogeneous_field(L); mask = random_mask(L, L, 0.85)
z = np.where(mask != 0, truth, np.float32(0)).astype(np.float32)
dev = torch.device('cuda', 0); st = torch.cuda.current_stream(dev)
zd = torch.from_numpy(z).to(dev); md = torch.from_numpy(mask).to(dev)
for v in sys.argv[1].split(','):
    os.environ['MPR_SWEEP_VARIANT'] = v
    eng = P.LeMpr(P.Config(), P.load_calibration(), stream=st.cuda_stream)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        eng.set_data_device(zd.data_ptr(), md.data_ptr(), L, L); eng.estimate_local_params()
        s = eng.simulate_adaptive(1, 7, n_fit=20, n_f=5, max_sweeps=500, slope_tol=0.0)
        torch.cuda.synchronize(); print(v, rep, round(1e3 * (time.perf_counter() - t0), 1), flush=True)
    eng.close()
