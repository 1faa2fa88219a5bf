"""Device time of small fixed-S fills (latency-bound regime): whole fill vs the sweep part."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2212_01317_b200 as P
from inputs.synth import make_problem
dev = torch.device('cuda', 0); st = torch.cuda.current_stream(dev)
for L, M in ((64, 12), (256, 12), (512, 12), (1024, 12)):
    truth, z, mask = make_problem(L, 0.5)
    zd = torch.from_numpy(np.nan_to_num(z)).to(dev); md = torch.from_numpy(mask).to(dev)
    eng = P.LeMpr(P.Config(), P.load_calibration(), stream=st.cuda_stream)
    out = torch.empty((L, L), device=dev)
    def fill():
        eng.set_data_device(zd.data_ptr(), md.data_ptr(), L, L); eng.estimate_local_params()
        eng.simulate(M, 30, 1); eng.predict_device(out.data_ptr())
    for _ in range(3): fill()
    eng.set_kernel_timing(True)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); fill(); e1.record(st); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    inf = eng.info()
    print(f"L={L} M={M}: fill {np.median(ts):.3f} ms, sweeps {inf['sweep_ms']/10:.3f} ms "
          f"({inf['sweep_launches']//10} launches)", flush=True)
    eng.close()
