import os, sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2212_01317_b200 as P
from inputs.synth import heterogeneous_field, random_mask
L = 2048
truth = heterogeneous_field(L); mask = random_mask(L, L, 0.85)
z = np.where(mask != 0, truth, np.float32(0)).astype(np.float32)
calib = P.load_calibration()
dev = torch.device('cuda', 0); st = torch.cuda.current_stream(dev)
zd = torch.from_numpy(z).to(dev); md = torch.from_numpy(mask).to(dev)
for v in sys.argv[1].split(','):
    os.environ['MPR_SWEEP_VARIANT'] = v
    eng = P.LeMpr(P.Config(), calib, stream=st.cuda_stream)
    eng.set_data_device(zd.data_ptr(), md.data_ptr(), L, L); eng.estimate_local_params()
    for M, tol in ((100, 1e-5), (100, 0.0)):
        eng.simulate_adaptive(M, 7, n_fit=20, n_f=5, max_sweeps=200, slope_tol=tol)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s = eng.simulate_adaptive(M, 7, n_fit=20, n_f=5, max_sweeps=200, slope_tol=tol)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
        print(json.dumps(dict(variant=int(v), M=M, tol=tol, ms=1e3 * t, mean_sweeps=float(np.mean(np.abs(s)) + 1), s_sum=int(np.sum(s)))), flush=True)
    eng.close()
