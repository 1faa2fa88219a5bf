"""A/B timing of the energy-trace half-sweep kernels: simulate(M, S) with the energy trace
on, L^2 grid, p = 0.85; prints ms per half-sweep (library kernel timing)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2212_01317_b200 as P
from inputs.synth import heterogeneous_field, random_mask
L, M = int(sys.argv[1]), int(sys.argv[2])
truth = heterogeneous_field(L); mask = random_mask(L, L, 0.85)
z = np.where(mask != 0, truth, np.float32(0)).astype(np.float32)
for energy in (False, True):
    eng = P.LeMpr(P.Config(), P.load_calibration())
    eng.set_data(z, mask); eng.estimate_local_params(); eng.set_energy_trace(energy)
    eng.simulate(M, 10, 1)
    eng.set_kernel_timing(True)
    eng.simulate(M, 30, 1)
    inf = eng.info()
    print(f"L={L} M={M} energy={energy}: {inf['sweep_ms'] / (2 * 30):.4f} ms per half-sweep", flush=True)
    eng.close()
