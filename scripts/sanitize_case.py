#!/usr/bin/env python3
"""Small end-to-end cases for compute-sanitizer: SC and DC orders, energy trace, n_avg > 1,
adaptive protocol, row slabs (emulated), and the calibration builder."""
import os
import sys


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2212_01317_b200 as P
    from inputs.synth import make_problem
    calib = P.load_calibration()
    truth, z, mask = make_problem(45, 0.5, Lx=38, corr_len=5.0)
    for cfg, energy in ((P.Config(l_b=8, n_s=2, r_s=1), True), (P.Config(l_b=8, order="dc"), False),
                        (P.Config(n_avg=3, init="random"), True)):
        m = P.LeMpr(cfg, calib)
        m.set_data(z, mask)
        m.set_energy_trace(energy)
        m.estimate_local_params()
        m.simulate(5, 6, 3)      # odd pair count: the one-pair fallback kernel
        m.simulate(8, 4, 5)      # two pairs per thread: the quad kernel
        m.predict()
        if cfg.order == "sc":
            m.set_energy_trace(False)
            m.simulate_adaptive(3, 4, n_fit=5, n_f=2, max_sweeps=20)
            m.predict()
        m.close()
    # row slabs: three contexts joined by the in-process communicator
    from paper_2212_01317_b200.sharding import run_group

    def slab(rank, g):
        m = P.LeMpr(P.Config(l_b=8, n_s=2, r_s=1, group=g, group_rank=rank, shard="rows"), calib)
        m.set_data(z, mask)
        m.estimate_local_params()
        m.simulate(4, 3, 1)
        out = m.predict()
        m.close()
        return out
    run_group(3, slab)
    m = P.LeMpr(P.Config(), calib)
    P.mpr_build_calibration(m.ctx, calib[0][:6], L=16, n_eq=5, n_meas=5, reps=2)
    m.close()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
