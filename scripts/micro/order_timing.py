"""SC vs DC update order (row f3): device time of a C2 fill and of its sweeps; DC on the
paper's shared-memory tiles (MPR_DC_TILED=1) and on phase lists (0)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2212_01317_b200 as P
from inputs.synth import make_problem
dev = torch.device('cuda', 0); st = torch.cuda.current_stream(dev)
truth, z, mask = make_problem(1024, 0.33, nu=0.5)
zd = torch.from_numpy(np.nan_to_num(z)).to(dev); md = torch.from_numpy(mask).to(dev)
for order, tiled in (("sc", "1"), ("dc", "1"), ("dc", "0")):
    os.environ["MPR_DC_TILED"] = tiled
    for M in (100, 10):
        eng = P.LeMpr(P.Config(order=order), P.load_calibration(), stream=st.cuda_stream)
        out = torch.empty((1024, 1024), device=dev)
        def fill():
            eng.set_data_device(zd.data_ptr(), md.data_ptr(), 1024, 1024); eng.estimate_local_params()
            eng.simulate(M, 30, 1); eng.predict_device(out.data_ptr())
        for _ in range(2): fill()
        eng.set_kernel_timing(True)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); fill(); e1.record(st); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        inf = eng.info()
        print(f"order={order} tiled={tiled} M={M}: fill {np.median(ts):.3f} ms, sweeps {inf['sweep_ms']/5:.3f} ms, "
              f"{inf['sweep_launches']//5} sweep launches", flush=True)
        eng.close()
