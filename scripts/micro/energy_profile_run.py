"""A short energy-trace fill (C2-size, M = 100) for ncu captures of the energy kernels."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2212_01317_b200 as P
from inputs.synth import make_problem
truth, z, mask = make_problem(1024, 0.33, nu=0.5)
eng = P.LeMpr(P.Config(), P.load_calibration())
eng.set_data(z, mask); eng.estimate_local_params(); eng.set_energy_trace(True)
eng.simulate(100, 6, 1)
print("ok")
