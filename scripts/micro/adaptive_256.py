import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2212_01317_b200 as P
from inputs.synth import heterogeneous_field, random_mask
L = 256
truth = heterogeneous_field(L); mask = random_mask(L, L, 0.85)
z = np.where(mask != 0, truth, np.float32(0)).astype(np.float32)
eng = P.LeMpr(P.Config(), P.load_calibration())
for _ in range(2):
    eng.set_data(z, mask); eng.estimate_local_params()
    s = eng.simulate_adaptive(1, 7, n_fit=20, n_f=5, max_sweeps=500, slope_tol=1e-5)
    eng.predict()
print("ok", s)
