"""GPU (libmpr.so, sm_100a) vs CPU oracle parity, through the C-ABI.

Bars (BASELINE.json north star):
- spin transform, masks, block statistics, temperature field: bit-exact;
- Markov-chain states after k sweeps: bit-exact (shared Philox stream, docs/ARITH.md);
- predictions: within 1e-3 of the data range (bit-exact when n_avg = 1 on one GPU);
- MAE / RMSE / MARE: within 1e-4 relative; energy trace: within 1e-5 relative.
"""
import numpy as np
import pytest

import oracle as O
from inputs.synth import make_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_01317_b200 import _build
    _build.build()
    import paper_2212_01317_b200 as P
    P.load_library()
    return P


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32 if a.dtype == np.float32 else np.uint64)


def assert_bitwise(a, b, what):
    a = np.ascontiguousarray(a); b = np.ascontiguousarray(b)
    assert a.shape == b.shape, what
    diff = np.flatnonzero(bits(a).ravel() != bits(b).ravel())
    assert diff.size == 0, f"{what}: {diff.size} mismatches, first at {np.unravel_index(diff[0], a.shape)}: " \
                           f"gpu={a.ravel()[diff[0]]!r} oracle={b.ravel()[diff[0]]!r}"


def gpu_run(P, z, mask, cfg, calib, M, S, seed, energy=False):
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    m.set_energy_trace(energy)
    T = m.estimate_local_params(want_T=True)
    m.simulate(M, S, seed)
    out = dict(T=T, pred=m.predict(), info=m.info(), phiK=m.debug(P.binding.MPR_BUF_PHI_KNOWN),
               Tb=m.debug(P.binding.MPR_BUF_BLOCK_T), stats=m.debug(P.binding.MPR_BUF_BLOCK_STATS),
               acc=m.debug(P.binding.MPR_BUF_ACC))
    inf = out["info"]
    lo, hi = inf["last_m_base"], min(inf["last_m_base"] + inf["last_batch"], M)
    out["states"] = {r: m.debug(P.binding.MPR_BUF_STATE, r) for r in range(lo, hi)}
    if energy:
        out["energy"] = m.debug(P.binding.MPR_BUF_ENERGY)
    m.close()
    return out


def ocfg(cfg):
    return O.OracleConfig(q=cfg.q, J=cfg.J, lb=cfg.l_b, rs=cfg.r_s, ns=cfg.n_s, init=cfg.init, n_avg=cfg.n_avg,
                          order=cfg.order)


def compare(P, z, mask, truth, cfg, calib, M, S, seed, energy=False, exact_pred=True):
    g = gpu_run(P, z, mask, cfg, calib, M, S, seed, energy=energy)
    Tk, ek = calib
    o = O.fill(z, mask, ocfg(cfg), Tk, ek, M, S, seed, energy=energy, states=True)
    p = o["params"]
    assert_bitwise(g["phiK"], p.phi0, "phi at samples")
    assert g["info"]["z_min"] == p.zmin and g["info"]["z_max"] == p.zmax
    # block statistics element by element (ARITH §E exact int64): SB, NB, SP, NK
    SB, NB, SP, NK = O.block_stats(p.phi0, mask, cfg.l_b, cfg.q)
    for k, (name, ref) in enumerate((("SB", SB), ("NB", NB), ("SP", SP), ("NK", NK))):
        assert np.array_equal(g["stats"][k], ref.ravel()), f"block statistic {name} differs"
    assert np.array_equal(SP.ravel(), p.SP.ravel()) and np.array_equal(NK.ravel(), p.NK.ravel())
    assert_bitwise(g["Tb"], p.Tb.ravel(), "block temperatures")
    assert_bitwise(g["T"], p.T, "temperature field")
    for r, st in g["states"].items():
        assert_bitwise(st, o["sim"]["phi"][r], f"state of realization {r}")
    rng = p.zmax - p.zmin
    gaps = mask == 0
    if exact_pred:
        assert_bitwise(g["acc"][gaps], o["sim"]["acc"][gaps], "accumulator")
        assert_bitwise(g["pred"], o["pred"], "predictions")
    else:
        assert np.max(np.abs(g["pred"][gaps] - o["pred"][gaps])) <= 1e-3 * rng
        assert_bitwise(g["pred"][~gaps], z[~gaps], "samples returned bitwise")
    sg, so = O.score(g["pred"], truth, mask), O.score(o["pred"], truth, mask)
    for k in ("mae", "rmse", "mare"):
        assert abs(sg[k] - so[k]) <= 1e-4 * abs(so[k]) + 1e-12, k
    if energy:
        assert_bitwise(g["energy"], o["sim"]["energy"], "energy trace (ARITH §J fixed point)")
    return g, o


def test_c1_config_bit_exact(P, calib):
    """BASELINE config 1: 64x64 Matern, 50% random gaps, M = 10, S = 30, SST defaults."""
    truth, z, mask = make_problem(64, 0.5)
    compare(P, z, mask, truth, P.Config(), calib, 10, 30, 20221202, energy=True)


def test_ragged_odd_m_random_init(P, calib):
    """Sizes that divide nothing (67 x 45), l_b = 8, r_s = 3, n_s = 2, odd M, RANDOM init."""
    truth, z, mask = make_problem(45, 0.4, Lx=67, corr_len=8.0)
    cfg = P.Config(l_b=8, r_s=3, n_s=2, init="random")
    compare(P, z, mask, truth, cfg, calib, 7, 12, 99)


def test_generic_q_and_J(P, calib):
    """q != 1/2 and J != 1 take the generic (non-specialised) cos path; still bit-exact."""
    truth, z, mask = make_problem(40, 0.6, Lx=36, corr_len=5.0)
    compare(P, z, mask, truth, P.Config(q=0.3, J=2.0, l_b=16, n_s=1, r_s=1), calib, 4, 10, 5)


def test_n_avg_tolerance(P, calib):
    """Averaging the last 5 sweeps: states bit-exact, predictions within 1e-3 of the range."""
    truth, z, mask = make_problem(48, 0.5, corr_len=6.0)
    compare(P, z, mask, truth, P.Config(n_avg=5), calib, 6, 15, 3, exact_pred=False)


def test_batched_realizations(P, calib):
    """max_batch = 4 forces 3 launch batches for M = 10 (pairs of the Philox stream split)."""
    truth, z, mask = make_problem(32, 0.5, corr_len=5.0)
    compare(P, z, mask, truth, P.Config(max_batch=4, l_b=8), calib, 10, 8, 17)


def test_cloud_gaps_bst_and_mpr_modes(P, calib):
    """Clustered gaps (70%), BST (n_s = 0) and uniform MPR (l_b >= L) special cases."""
    truth, z, mask = make_problem(96, 0.7, gaps="cloud", corr_len=10.0)
    compare(P, z, mask, truth, P.Config(n_s=0), calib, 4, 10, 1)
    compare(P, z, mask, truth, P.Config(l_b=128, n_s=0), calib, 4, 10, 2)


def test_small_blocks_many_fallbacks(P, calib):
    """l_b = 2 at 90% missing: most blocks have no sample bond and take the lower median."""
    truth, z, mask = make_problem(50, 0.9, corr_len=4.0)
    g, o = compare(P, z, mask, truth, P.Config(l_b=2, n_s=1, r_s=1), calib, 2, 6, 8)
    assert g["info"]["n_blocks_fallback"] > 0


@pytest.mark.parametrize("rs,ns", [(0, 2), (1, 3), (3, 5), (7, 2), (16, 1)])
def test_sst_field_bit_exact_window_sizes(P, calib, rs, ns):
    """a5 at window widths 1..33 (r_s <= 16, the C-ABI limit) on a ragged grid large enough
    for interior (no bounds check) and edge tiles of k_smooth: T is bit-exact vs the oracle."""
    Tk, ek = calib
    truth, z, mask = make_problem(161, 0.4, Lx=198, corr_len=8.0)
    cfg = P.Config(r_s=rs, n_s=ns, l_b=16)
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    T = m.estimate_local_params(want_T=True)
    m.close()
    p = O.parameters(z, mask, ocfg(cfg), Tk, ek)
    assert_bitwise(T, p.T, f"T field r_s={rs} n_s={ns}")


@pytest.mark.parametrize("scale,rs,ns", [(1.0, 2, 5), (100.0, 2, 3), (300.0, 3, 2), (1e-2, 1, 2), (1e-3, 2, 2)])
def test_sst_fixed_point_paths_bit_exact(P, calib, scale, rs, ns):
    """The specialised SST pass forms the exact window sums in fp64 when every term is an
    integer-valued float below the 2^53 bound ((2 r_s + 1)^2 T_max < 2^13, T_min >= 2^-17),
    else in int64 (tables scaled by 100 and 300: the int64 path; by 1e-3: T_min < 2^-17, the
    int64 path with llrint rounding). Both give the oracle's T field bit for bit, from the
    first (T_b-reading) pass on, on a grid with interior and edge tiles."""
    Tk, ek = calib
    Ts = (Tk.astype(np.float64) * scale).astype(np.float32)
    truth, z, mask = make_problem(150, 0.45, Lx=203, corr_len=7.0)
    cfg = P.Config(r_s=rs, n_s=ns, l_b=16)
    m = P.LeMpr(cfg, (Ts, ek))
    m.set_data(z, mask)
    T = m.estimate_local_params(want_T=True)
    m.close()
    p = O.parameters(z, mask, ocfg(cfg), Ts, ek)
    assert_bitwise(T, p.T, f"T field (table x{scale}, r_s={rs}, n_s={ns})")


@pytest.mark.parametrize("narrow", ["", "1"])
@pytest.mark.parametrize("rs,scale,Lx", [(1, 1.0, 200), (2, 1.0, 1024), (3, 100.0, 132), (4, 1.0, 260), (4, 300.0, 128)])
def test_sst_wide_tile_bit_exact(P, calib, monkeypatch, narrow, rs, scale, Lx):
    """The 4-columns-per-thread SST pass (r_s <= 4, Lx % 4 == 0: float4 loads, halo by lane
    shuffles, register-sliding horizontal sums; fp64 or int64 sums by the table's range) and,
    with MPR_SST_NARROW, the one-column pass: T equals the oracle's bit for bit on grids with
    partial edge tiles in both directions."""
    if narrow:
        monkeypatch.setenv("MPR_SST_NARROW", narrow)
    Tk, ek = calib
    Ts = (Tk.astype(np.float64) * scale).astype(np.float32)
    truth, z, mask = make_problem(77, 0.5, Lx=Lx, corr_len=5.0)
    cfg = P.Config(r_s=rs, n_s=3, l_b=16)
    m = P.LeMpr(cfg, (Ts, ek))
    m.set_data(z, mask)
    T = m.estimate_local_params(want_T=True)
    m.close()
    p = O.parameters(z, mask, ocfg(cfg), Ts, ek)
    assert_bitwise(T, p.T, f"T field (r_s={rs}, table x{scale}, Lx={Lx}, narrow={bool(narrow)})")


def test_sharded_ranges_equal_single_call(P, calib):
    """simulate_range over [0,4) then [4,10) == simulate(10) bit for bit (global realization ids)."""
    truth, z, mask = make_problem(40, 0.5, corr_len=6.0)
    cfg = P.Config(l_b=8)
    ref = gpu_run(P, z, mask, cfg, calib, 10, 8, 77)
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask); m.estimate_local_params(); m.reset_accumulator()
    m.simulate_range(10, 8, 77, 0, 4)
    m.simulate_range(10, 8, 77, 4, 10)
    assert_bitwise(m.predict(), ref["pred"], "predictions of the sharded run")
    m.close()


def test_degenerate_no_gap_and_errors(P, calib):
    Tk, ek = calib
    z = np.full((8, 8), 3.25, np.float32); mask = np.ones((8, 8), np.uint8); mask[2, 3] = 0; z[2, 3] = np.nan
    m = P.LeMpr(P.Config(), calib)
    m.set_data(z, mask); m.estimate_local_params(); m.simulate(4, 5, 1)
    out = m.predict()
    assert out[2, 3] == np.float32(3.25) and m.info()["degenerate_range"] == 1
    # no gaps: predictions are the input, bitwise
    truth, _, _ = make_problem(16, 0.5)
    m.set_data(truth, np.ones((16, 16), np.uint8)); m.estimate_local_params(); m.simulate(2, 3, 1)
    assert_bitwise(m.predict(), truth, "P = 0 returns the input")
    # too few samples
    mask = np.zeros((8, 8), np.uint8); mask[0, 0] = 1
    with pytest.raises(P.MprError) as e:
        m.set_data(np.zeros((8, 8), np.float32), mask)
    assert e.value.status == P.binding.MPR_ERR_TOO_FEW_SAMPLES
    # no sample bonds: samples only on colour A
    mask = (np.add.outer(np.arange(8), np.arange(8)) % 2 == 0).astype(np.uint8)
    m.set_data(np.arange(64, dtype=np.float32).reshape(8, 8), mask)
    with pytest.raises(P.MprError) as e:
        m.estimate_local_params()
    assert e.value.status == P.binding.MPR_ERR_NO_SAMPLE_BONDS
    # out of order
    m2 = P.LeMpr(P.Config(), calib)
    with pytest.raises(P.MprError) as e:
        m2.simulate(1, 1, 1)
    assert e.value.status == P.binding.MPR_ERR_STATE
    # non-finite sample
    bad = np.ones((4, 4), np.float32); bad[1, 1] = np.inf
    with pytest.raises(P.MprError) as e:
        m2.set_data(bad, np.ones((4, 4), np.uint8))
    assert e.value.status == P.binding.MPR_ERR_INVALID_ARG
    m.close(); m2.close()


@pytest.mark.slow
def test_c2_full_size_sampled(P, calib):
    """BASELINE config 2 at full size (1024^2, p = 0.33, M = 100, S = 30) in the launch
    configuration bench.py times: the whole parameter stage bit-exact, and realizations
    0, 57, 99 (sampled; each one is a 1e7-update oracle run) bit-exact."""
    Tk, ek = calib
    truth, z, mask = make_problem(1024, 0.33, nu=0.5)
    cfg = P.Config()
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    T = m.estimate_local_params(want_T=True)
    m.simulate(100, 30, 20221202)
    pred = m.predict()
    p = O.parameters(z, mask, ocfg(cfg), Tk, ek)
    assert_bitwise(T, p.T, "temperature field (1024^2)")
    for r in (0, 57, 99):
        st = m.debug(P.binding.MPR_BUF_STATE, r)
        o = O.simulate(p, mask, ocfg(cfg), 100, 30, 20221202, m_begin=r, m_end=r + 1, states=True)
        assert_bitwise(st, o["phi"][0], f"realization {r} at 1024^2")
    gaps = mask == 0
    assert_bitwise(pred[~gaps], z[~gaps], "samples")
    assert pred[gaps].min() >= p.zmin and pred[gaps].max() <= p.zmax
    m.close()


@pytest.mark.slow
def test_c2_full_predictions_bit_exact(P, calib):
    """BASELINE config 2 exactly as bench.py runs it (1024^2, p = 0.33, M = 100, S = 30, the
    default kernels and launch configuration): the accumulator over all 100 realizations and
    the whole prediction grid equal the oracle's bit for bit. The oracle runs its OpenMP
    build on the host cores (~1e9 updates; the same C source, pinned bit-identical to the
    single-thread parity build by test_openmp_build_bit_identical)."""
    Tk, ek = calib
    truth, z, mask = make_problem(1024, 0.33, nu=0.5)
    cfg = P.Config()
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    m.estimate_local_params()
    m.simulate(100, 30, 20221202)
    pred = m.predict()
    acc = m.debug(P.binding.MPR_BUF_ACC)
    m.close()
    oc = ocfg(cfg)
    try:
        O.set_threads(0)
        p = O.parameters(z, mask, oc, Tk, ek)
        sim = O.simulate(p, mask, oc, 100, 30, 20221202)
        opred = O.predict(np.nan_to_num(z), mask, sim["acc"], 100, 1, p.zmin, p.zmax, 0)
    finally:
        O.set_threads(1)
    gaps = mask == 0
    assert_bitwise(acc[gaps], sim["acc"][gaps], "accumulator over 100 realizations (1024^2)")
    assert_bitwise(pred, opred, "predictions (1024^2, M = 100)")


def group_run(P, z, mask, cfg_kw, calib, M, S, seed, world, shard="rows", ordered=False, energy=False,
              device_input=False, states=True):
    """`world` contexts on this GPU joined by libmpr's in-process communicator (one host
    thread each), every one running the SPMD call sequence with shard="rows" or
    "realizations"; returns each rank's results (own rows of the Lx*Ly debug buffers)."""
    import torch
    from paper_2212_01317_b200.sharding import row_range, run_group
    Ly, Lx = z.shape

    def fn(rank, g):
        cfg = P.Config(**cfg_kw, group=g, group_rank=rank, shard=shard, ordered_reduce=ordered)
        m = P.LeMpr(cfg, calib)
        try:
            if device_input:  # row slabs: the device buffers hold the own rows only
                r0, r1 = row_range(Ly, world, rank) if shard == "rows" else (0, Ly)
                zd = torch.from_numpy(np.ascontiguousarray(np.nan_to_num(z[r0:r1]))).cuda()
                md = torch.from_numpy(np.ascontiguousarray(mask[r0:r1])).cuda()
                m.set_data_device(zd.data_ptr(), md.data_ptr(), Lx, Ly)
            else:
                m.set_data(z, mask)
            m.set_energy_trace(energy)
            T = m.estimate_local_params(want_T=True)
            m.simulate(M, S, seed)
            out = dict(T=T, pred=m.predict(), rows=m.predict_rows(), info=m.info(),
                       stats=m.debug(P.binding.MPR_BUF_BLOCK_STATS), Tb=m.debug(P.binding.MPR_BUF_BLOCK_T),
                       phiK=m.debug(P.binding.MPR_BUF_PHI_KNOWN))
            inf = out["info"]
            if states:
                lo, hi = inf["last_m_base"], min(inf["last_m_base"] + inf["last_batch"], M)
                out["states"] = {r: m.debug(P.binding.MPR_BUF_STATE, r) for r in range(lo, hi)}
            if energy:
                out["energy"] = m.debug(P.binding.MPR_BUF_ENERGY)
            return out
        finally:
            m.close()

    return run_group(world, fn)


def check_row_slabs(P, z, mask, cfg_kw, calib, M, S, seed, world, energy=True, device_input=False):
    """Every rank of a row-slab run against the oracle: block sums (global on every rank),
    z_min / z_max, the own rows of phi, T and the last batch's states bitwise, the energy
    trace bitwise, the all-gathered predictions bitwise (n_avg = 1), and slab-local memory
    (a rank holds its own rows' gap sites plus one ghost row per side)."""
    from paper_2212_01317_b200.sharding import row_range
    cfg = P.Config(**cfg_kw)
    Tk, ek = calib
    o = O.fill(z, mask, ocfg(cfg), Tk, ek, M, S, seed, energy=energy, states=True)
    p = o["params"]
    SB, NB, SP, NK = O.block_stats(p.phi0, mask, cfg.l_b, cfg.q)
    res = group_run(P, z, mask, cfg_kw, calib, M, S, seed, world, energy=energy, device_input=device_input)
    Ly, Lx = z.shape
    gaps = mask == 0
    for rank, g in enumerate(res):
        r0, r1 = row_range(Ly, world, rank)
        inf = g["info"]
        assert (inf["rank"], inf["world"], inf["row_begin"], inf["row_end"]) == (rank, world, r0, r1)
        assert inf["n_gaps"] == int(gaps.sum()) and inf["z_min"] == p.zmin and inf["z_max"] == p.zmax
        assert inf["sample_bonds"] == int(NB.sum())
        local = int(gaps[max(r0 - 1, 0):min(r1 + 1, Ly)].sum())
        assert inf["n_gaps_local"] == local, "slab-local gap sites: own rows + ghost rows"
        for k, ref in enumerate((SB, NB, SP, NK)):
            assert np.array_equal(g["stats"][k], ref.ravel()), f"rank {rank}: block statistic {k}"
        assert_bitwise(g["Tb"], p.Tb.ravel(), f"rank {rank}: block temperatures")
        assert_bitwise(g["phiK"][r0:r1], p.phi0[r0:r1], f"rank {rank}: phi at samples")
        assert_bitwise(g["T"][r0:r1], p.T[r0:r1], f"rank {rank}: temperature rows")
        for r, st in g["states"].items():
            assert_bitwise(st[r0:r1], o["sim"]["phi"][r][r0:r1], f"rank {rank}: state rows of realization {r}")
        if cfg.n_avg == 1:
            assert_bitwise(g["pred"], o["pred"], f"rank {rank}: predictions")
            assert_bitwise(g["rows"], o["pred"][r0:r1], f"rank {rank}: own prediction rows")
        else:
            assert np.max(np.abs(g["pred"][gaps] - o["pred"][gaps])) <= 1e-3 * (p.zmax - p.zmin)
        if energy:
            assert_bitwise(g["energy"], o["sim"]["energy"], f"rank {rank}: energy trace")
    return res


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_row_slabs_distributed_bit_exact(P, calib, monkeypatch, world, overlap):
    """Row slabs inside libmpr (MPR_SHARD_ROWS) on `world` contexts: the
    distributed parameter stage, the halo exchange after every colour half-sweep (overlapped
    with the interior rows on the comm stream, or in line: MPR_HALO_OVERLAP) and the
    all-gathered predictions reproduce the oracle bit for bit on every rank."""
    monkeypatch.setenv("MPR_HALO_OVERLAP", overlap)
    truth, z, mask = make_problem(61, 0.5, Lx=52, corr_len=6.0)
    check_row_slabs(P, z, mask, dict(l_b=8, n_s=2, r_s=1), calib, 6, 10, 123, world)


def test_row_slabs_device_input_wide_halo_random_init(P, calib):
    """Device-resident own-row inputs (mpr_set_data_device with the slab's rows only), an SST
    halo r_s n_s = 6 wider than a slab, RANDOM init, cloud gaps, M = 4k + 2 realizations."""
    truth, z, mask = make_problem(40, 0.6, Lx=33, gaps="cloud", corr_len=5.0)
    check_row_slabs(P, z, mask, dict(l_b=4, n_s=3, r_s=2, init="random"), calib, 10, 7, 77, 4, device_input=True)


def test_row_slabs_mpr_one_block_and_n_avg(P, calib):
    """Uniform MPR (one block spanning every slab: its sums come from all ranks) and n_avg > 1."""
    truth, z, mask = make_problem(37, 0.5, Lx=29, corr_len=6.0)
    check_row_slabs(P, z, mask, dict(l_b=64, n_s=0), calib, 4, 8, 5, 3)
    check_row_slabs(P, z, mask, dict(l_b=8, n_s=1, r_s=1, n_avg=3), calib, 4, 8, 6, 2, energy=False)


@pytest.mark.parametrize("ordered", [False, True])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_realization_shards_distributed(P, calib, world, ordered):
    """Realization shards inside libmpr (MPR_SHARD_REALIZATIONS): the rank's pair-aligned id
    range (= sharding.shard_range), then the all-reduce (equal up to fp64 reassociation) or
    the rank-ordered chain (bit-identical); the energy trace summed over the ranks."""
    from paper_2212_01317_b200.sharding import shard_range
    truth, z, mask = make_problem(48, 0.45, Lx=41, corr_len=6.0)
    M, S, seed = 11, 9, 4242
    Tk, ek = calib
    cfg = P.Config()
    o = O.fill(z, mask, ocfg(cfg), Tk, ek, M, S, seed, energy=True)
    res = group_run(P, z, mask, {}, calib, M, S, seed, world, shard="realizations", ordered=ordered, energy=True,
                    states=False)
    rng = o["params"].zmax - o["params"].zmin
    for rank, g in enumerate(res):
        assert (g["info"]["m_begin"], g["info"]["m_end"]) == shard_range(M, world, rank)
        if ordered:
            assert_bitwise(g["pred"], o["pred"], f"rank {rank}: ordered-reduce predictions")
        else:
            assert np.max(np.abs(g["pred"] - o["pred"])) <= 1e-6 * rng
        assert_bitwise(g["energy"], o["sim"]["energy"], f"rank {rank}: energy trace")
        assert_bitwise(g["pred"], res[0]["pred"], "every rank holds the same predictions")


def test_adaptive_realization_shards_distributed(P, calib):
    """The adaptive protocol (row f1) with realization shards: each rank decides its own
    realizations on the device; s_eq and the accumulators are summed over the ranks."""
    from paper_2212_01317_b200.sharding import run_group
    truth, z, mask = make_problem(40, 0.5, corr_len=6.0)
    M, seed = 7, 13
    Tk, ek = calib
    cfg = P.Config(n_avg=2)
    oc = ocfg(cfg)
    p = O.parameters(z, mask, oc, Tk, ek)
    r = O.simulate_adaptive(p, mask, oc, M, seed, n_fit=8, n_f=3, S_max=60, slope_tol=1e-4)
    ref = O.predict(np.nan_to_num(z), mask, r["acc"], M, 2, p.zmin, p.zmax, 0)

    def fn(rank, g):
        m = P.LeMpr(P.Config(n_avg=2, group=g, group_rank=rank), calib)
        m.set_data(z, mask); m.estimate_local_params()
        s_eq = m.simulate_adaptive(M, seed, n_fit=8, n_f=3, max_sweeps=60, slope_tol=1e-4)
        pred = m.predict()
        m.close()
        return s_eq, pred
    for s_eq, pred in run_group(3, fn):
        assert s_eq.tolist() == r["s_eq"].tolist()
        assert np.max(np.abs(pred - ref)) <= 1e-3 * (p.zmax - p.zmin)


@pytest.mark.parametrize("overlap", ["1", "0"])
def test_adaptive_row_slabs_distributed(P, calib, monkeypatch, overlap):
    """The adaptive protocol on row slabs (3 contexts): each rank sweeps its rows for every
    realization, the partial whole-grid energies are summed over the ranks before each
    device check, so every rank takes the oracle's decisions (s_eq) and predicts the
    oracle's values (derived tolerance, n_avg = 2 within the tolerance)."""
    from paper_2212_01317_b200.sharding import run_group
    monkeypatch.setenv("MPR_HALO_OVERLAP", overlap)
    truth, z, mask = make_problem(45, 0.5, Lx=38, corr_len=6.0)
    M, seed = 6, 19
    Tk, ek = calib
    for n_avg in (1, 2):
        cfg = P.Config(n_avg=n_avg, l_b=8, n_s=2, r_s=1)
        oc = ocfg(cfg)
        p = O.parameters(z, mask, oc, Tk, ek)
        r = O.simulate_adaptive(p, mask, oc, M, seed, n_fit=8, n_f=3, S_max=70, slope_tol="derived")
        ref = O.predict(np.nan_to_num(z), mask, r["acc"], M, n_avg, p.zmin, p.zmax, 0)

        def fn(rank, g):
            m = P.LeMpr(P.Config(n_avg=n_avg, l_b=8, n_s=2, r_s=1, group=g, group_rank=rank, shard="rows"), calib)
            m.set_data(z, mask)
            m.estimate_local_params()
            s_eq = m.simulate_adaptive(M, seed, n_fit=8, n_f=3, max_sweeps=70, slope_tol="derived")
            pred = m.predict()
            m.close()
            return s_eq, pred
        for s_eq, pred in run_group(3, fn):
            assert s_eq.tolist() == r["s_eq"].tolist()
            if n_avg == 1:
                assert_bitwise(pred, ref, "adaptive row-slab predictions")
            else:
                assert np.max(np.abs(pred - ref)) <= 1e-3 * (p.zmax - p.zmin)


def test_nccl_transport_world1(P, calib, monkeypatch):
    """The NCCL transport on the device: a communicator made through libmpr
    (mpr_nccl_unique_id / mpr_nccl_comm_init, libnccl resolved at run time) and, with
    MPR_FORCE_COMM=1, the multi-rank code paths at world size 1 — every all-reduce,
    broadcast and the predictions' all-gather run as real NCCL operations on the stream
    (neighbour exchanges have no peers at world 1). Results equal the single context."""
    monkeypatch.setenv("MPR_FORCE_COMM", "1")
    truth, z, mask = make_problem(40, 0.5, corr_len=6.0)
    ref = gpu_run(P, z, mask, P.Config(l_b=8), calib, 6, 8, 3)
    uid = P.mpr_nccl_unique_id()
    comm = P.mpr_nccl_comm_init(1, 0, uid, 0)
    try:
        for shard, ordered in (("rows", False), ("realizations", False), ("realizations", True)):
            m = P.LeMpr(P.Config(l_b=8, nccl_comm=comm, shard=shard, ordered_reduce=ordered), calib)
            m.set_data(z, mask)
            T = m.estimate_local_params(want_T=True)
            m.simulate(6, 8, 3)
            pred = m.predict()
            inf = m.info()
            m.close()
            assert inf["world"] == 1 and inf["comm_calls"] > 0, (shard, inf["comm_calls"])
            assert_bitwise(T, ref["T"], f"T ({shard})")
            assert_bitwise(pred, ref["pred"], f"predictions ({shard}, ordered={ordered})")
    finally:
        P.mpr_nccl_comm_destroy(comm)


def _full_size_sampled(P, calib, L, p, gaps, nu, M, S, windows):
    """Full-size run in bench's launch configuration; oracle.WindowOracle gives the exact
    oracle states and predictions of sampled windows (bit-exact comparison). States are
    read for the first and last realization of the last launch batch (the ones still
    resident); the predictions check every realization of every batch."""
    Tk, ek = calib
    truth, z, mask = make_problem(L, p, gaps=gaps, nu=nu)
    cfg = P.Config()
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    T = m.estimate_local_params(want_T=True)
    m.simulate(M, S, 20221202)
    pred = m.predict()
    info = m.info()
    lo = info["last_m_base"]
    realizations = sorted({lo, min(lo + info["last_batch"], M) - 1})
    W = O.WindowOracle(z, mask, ocfg(cfg), Tk, ek)
    assert info["z_min"] == W.zmin and info["z_max"] == W.zmax
    assert np.array_equal(m.debug(P.binding.MPR_BUF_BLOCK_T).reshape(W.Tb.shape).view(np.uint32),
                          W.Tb.view(np.uint32))
    states = {r: m.debug(P.binding.MPR_BUF_STATE, r) for r in realizations}
    m.close()
    for (r0, r1, c0, c1) in windows:
        assert_bitwise(T[r0:r1, c0:c1], W.T_window(r0, r1, c0, c1), f"T window {(r0, c0)}")
        ref = W.states(r0, r1, c0, c1, range(M), S, 20221202)
        for r in realizations:
            assert_bitwise(states[r][r0:r1, c0:c1], ref[r], f"state of realization {r} at {(r0, c0)}")
        acc = np.zeros(ref.shape[1:])
        for k in range(M):
            acc += ref[k].astype(np.float64)
        zw = np.ascontiguousarray(np.nan_to_num(z[r0:r1, c0:c1]))
        mw = np.ascontiguousarray(mask[r0:r1, c0:c1])
        pw = O.predict(zw, mw, np.where(mw == 0, acc, 0.0), M, 1, W.zmin, W.zmax, 0)
        assert_bitwise(pred[r0:r1, c0:c1], pw, f"predictions at {(r0, c0)}")
    gapm = mask == 0
    assert_bitwise(pred[~gapm], z[~gapm], "samples returned bitwise")
    assert pred[gapm].min() >= W.zmin and pred[gapm].max() <= W.zmax


@pytest.mark.slow
def test_fixed_point_bound_32768_mpr_energy_trace(P, calib):
    """The API's largest grid, Lx*Ly = 2^30 (32768^2), in uniform-MPR mode (one block: its
    SB sums all 2^31 - 2^16 sample bonds) with the energy trace on: a field so smooth that
    every bond cosine rounds to 1.0f puts SB and the grid energy's fixed-point sum at
    (2^31 - 2^16) * 2^32 = 2^63 - 2^48, the int64 limit ARITH §E/§J guarantees. SB, e_s and
    the traced energies must be exact / finite (an overflow would wrap them negative)."""
    L = 32768
    r = np.arange(L, dtype=np.float32)
    z = (r[:, None] + r[None, :]) * np.float32(1e-6)
    mask = np.ones((L, L), np.uint8)
    gaps = [(0, 0), (1, 5), (L // 2, L // 2), (L - 1, L - 1), (L - 1, 17), (12345, 23456)]
    for (a, b) in gaps:
        mask[a, b] = 0
        z[a, b] = np.nan
    cfg = P.Config(l_b=L, n_s=0)
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    m.set_energy_trace(True)
    m.estimate_local_params()
    stats = m.debug(P.binding.MPR_BUF_BLOCK_STATS)
    del z
    n_bonds_all = 2 * L * L - 2 * L
    # bonds touching a gap are not sample bonds
    missing = sum((a > 0) + (a < L - 1) + (b > 0) + (b < L - 1) for (a, b) in gaps)
    nsp = n_bonds_all - missing
    assert int(stats[1][0]) == nsp
    assert int(stats[0][0]) == nsp * (1 << 32), "SB must be exactly N_SP * 2^32 (no wrap-around)"
    m.simulate(2, 3, 5)
    E = m.debug(P.binding.MPR_BUF_ENERGY)
    inf = m.info()
    m.close()
    assert np.all(np.isfinite(E)) and np.all(E <= -0.999999) and np.all(E >= -1.0), E
    assert inf["n_gaps"] == len(gaps)


@pytest.mark.slow
def test_c4_row_slabs_windows_vs_oracle(P, calib):
    """C4 (16384^2, 50% random gaps, M = 10, S = 30) split into 4 row slabs (contexts on this
    GPU, in-process transport): windows straddling every slab boundary and the grid edges
    are bit-exact against the oracle (oracle.WindowOracle), on every rank that owns rows of
    them; each rank holds ~1/4 of the gap sites."""
    from paper_2212_01317_b200.sharding import row_range, run_group
    L, M, S, seed, W = 16384, 10, 30, 20221202, 4
    Tk, ek = calib
    truth, z, mask = make_problem(L, 0.5)
    bounds = [row_range(L, W, w)[0] for w in range(1, W)]
    wins = [(b - 6, b + 6, 8000, 8012) for b in bounds] + [(0, 8, 16376, 16384), (16376, 16384, 0, 8)]

    def fn(rank, g):
        m = P.LeMpr(P.Config(group=g, group_rank=rank, shard="rows"), calib)
        m.set_data(z, mask)
        T = m.estimate_local_params(want_T=True)
        m.simulate(M, S, seed)
        pred = m.predict_rows()
        inf = m.info()
        lo = inf["last_m_base"]
        st = {rr: m.debug(P.binding.MPR_BUF_STATE, rr) for rr in (lo, min(lo + inf["last_batch"], M) - 1)}
        r0, r1 = inf["row_begin"], inf["row_end"]
        out = []
        for (a, b, c0, c1) in wins:
            ra, rb = max(a, r0), min(b, r1)
            if ra < rb:
                out.append(((a, b, c0, c1), ra, rb, T[ra:rb, c0:c1].copy(), pred[ra - r0:rb - r0, c0:c1].copy(),
                            {k: v[ra:rb, c0:c1].copy() for k, v in st.items()}))
        m.close()
        return inf, out

    res = run_group(W, fn)
    Wo = O.WindowOracle(z, mask, ocfg(P.Config()), Tk, ek)
    P_total = int((mask == 0).sum())
    for rank, (inf, out) in enumerate(res):
        assert inf["n_gaps_local"] < P_total / W * 1.01 + 2 * L
        for (a, b, c0, c1), ra, rb, T, pred, st in out:
            assert_bitwise(T, Wo.T_window(ra, rb, c0, c1), f"rank {rank} T window {(ra, c0)}")
            ref = Wo.states(ra, rb, c0, c1, range(M), S, seed)
            for rr, v in st.items():
                assert_bitwise(v, ref[rr], f"rank {rank} state {rr} window {(ra, c0)}")
            acc = np.zeros(ref.shape[1:])
            for k in range(M):  # realization order, as the oracle accumulates
                acc += ref[k].astype(np.float64)
            zw = np.ascontiguousarray(np.nan_to_num(z[ra:rb, c0:c1]))
            mw = np.ascontiguousarray(mask[ra:rb, c0:c1])
            pw = O.predict(zw, mw, np.where(mw == 0, acc, 0.0), M, 1, Wo.zmin, Wo.zmax, 0)
            assert_bitwise(pred, pw, f"rank {rank} predictions window {(ra, c0)}")


@pytest.mark.slow
def test_c3_full_size_sampled(P, calib):
    """BASELINE config 3 at full size: 4096^2, 70% cloud gaps, M = 8 (one GPU's shard of 64)."""
    L = 4096
    wins = [(2040, 2056, 2040, 2056), (0, 12, 0, 12), (4084, 4096, 1000, 1016), (777, 793, 4080, 4096)]
    _full_size_sampled(P, calib, L, 0.7, "cloud", 1.5, 8, 30, wins)


@pytest.mark.slow
def test_c4_full_size_sampled(P, calib):
    """BASELINE config 4 at full size: 16384^2, 50% random gaps, M = 10, S = 30 (the north
    star's < 1 s target workload), sampled windows bit-exact vs the oracle."""
    L = 16384
    wins = [(8190, 8202, 8190, 8202), (0, 10, 16374, 16384), (12000, 12010, 3, 13)]
    _full_size_sampled(P, calib, L, 0.5, "random", 1.5, 10, 30, wins)


@pytest.mark.parametrize("init,n_avg", [("block_mean", 1), ("random", 1), ("block_mean", 3)])
def test_adaptive_equilibration_matches_oracle(P, calib, init, n_avg):
    """Row f1 (ARITH §K): the per-realization equilibrium sweeps agree exactly
    with the oracle (exact fixed-point energies + the same fp64 slope test), and so do the
    predictions (bit-exact for n_avg = 1, within 1e-3 of the range otherwise)."""
    Tk, ek = calib
    truth, z, mask = make_problem(48, 0.5, corr_len=6.0)
    cfg = P.Config(init=init, n_avg=n_avg)
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    m.estimate_local_params()
    s_eq = m.simulate_adaptive(6, 11, n_fit=20, n_f=5, max_sweeps=120)
    pred = m.predict()
    m.close()
    oc = ocfg(cfg)
    p = O.parameters(z, mask, oc, Tk, ek)
    r = O.simulate_adaptive(p, mask, oc, 6, 11, n_fit=20, n_f=5, S_max=120)
    assert s_eq.tolist() == r["s_eq"].tolist()
    ref = O.predict(np.nan_to_num(z), mask, r["acc"], 6, n_avg, p.zmin, p.zmax, 0)
    if n_avg == 1:
        assert_bitwise(pred, ref, "adaptive predictions")
    else:
        assert np.max(np.abs(pred - ref)) <= 1e-3 * (p.zmax - p.zmin)


def test_adaptive_forced_cap(P, calib):
    """A cap too short for any check sweep forces s_eq = max_sweeps - n_avg (negated)."""
    truth, z, mask = make_problem(32, 0.5, corr_len=5.0)
    m = P.LeMpr(P.Config(), calib)
    m.set_data(z, mask)
    m.estimate_local_params()
    s_eq = m.simulate_adaptive(3, 5, n_fit=20, n_f=5, max_sweeps=12)
    assert s_eq.tolist() == [-11, -11, -11]
    m.close()


@pytest.mark.slow
def test_sv_mpr_beats_mpr_on_heterogeneous_field(P):
    """Row f4 (fig:err-p; SPEC acceptance #1): on a field with domains of
    very different variability, block/site-specific temperatures (BST, SST) predict better
    than one global temperature (MPR) — paired over random thinnings."""
    import sys
    sys.path.insert(0, "scripts")
    from validate_methods import run
    rows = run(L=256, K=4, M=10, S=30, ps=(0.85,))
    r = rows[0]
    for name in ("BST", "SST"):
        assert r[f"ratio_AAE_{name}"] < 0.9 and r[f"ratio_RASE_{name}"] < 1.0
        assert r[f"win_rate_RASE_{name}"] == 1.0


@pytest.mark.slow
def test_sv_mpr_beats_mpr_two_regime_spec1(P):
    """SPEC acceptance #1 on its two-regime field (sigma 0.1 and 10 domains, 256^2): for
    p = 0.5 and 0.8, MRASE(BST)/MRASE(MPR) < 1 and MRASE(SST)/MRASE(MPR) < 1 on paired
    thinnings (the full run, K = 20, M = 20, p = 0.5/0.7/0.8: ratios 0.70-0.85, every
    thinning won; profiles/r02_validation_spec1_two_regime.jsonl)."""
    import sys
    sys.path.insert(0, "scripts")
    from validate_methods import run
    for r in run(L=256, K=4, M=10, S=30, ps=(0.5, 0.8), field="two-regime"):
        for name in ("BST", "SST"):
            assert r[f"ratio_RASE_{name}"] < 1.0 and r[f"win_rate_RASE_{name}"] == 1.0


@pytest.mark.slow
def test_gpu_calibration_table_equals_shipped(P, calib):
    """Row f2: the e(T) table built on the GPU with the recipe of scripts/make_calibration.py
    is bit-identical to the shipped table the oracle wrote (same chains, exact fixed-point
    energies, same averaging and monotone fit)."""
    Tk, ek = calib
    m = P.LeMpr(P.Config(), calib)
    e, raw = P.mpr_build_calibration(m.ctx, Tk, L=128, q=0.5, n_eq=400, n_meas=800, reps=2, seed=20221202)
    m.close()
    assert_bitwise(e, ek, "GPU calibration table")
    # and it is a valid table: strictly increasing, harmonic at low T
    assert np.all(np.diff(e) > 0)
    assert abs(e[0] - (-1 + Tk[0] * 129 / 512)) < 3e-6


@pytest.mark.parametrize("lb", [8, 2])
def test_dc_order_bit_exact(P, calib, lb):
    """Row f3: double-checkerboard update order (even tiles A, B; odd tiles A, B), states and
    predictions bit-exact vs the oracle."""
    truth, z, mask = make_problem(52, 0.5, Lx=47, corr_len=6.0)
    compare(P, z, mask, truth, P.Config(l_b=lb, order="dc", n_s=1, r_s=1), calib, 6, 12, 31)


@pytest.mark.parametrize("tiled", ["1", "0"])
@pytest.mark.parametrize("lb,M,kw", [(32, 40, {}), (13, 10, dict(n_avg=3)), (64, 6, dict(q=0.3, J=1.5)),
                                      (5, 34, dict(init="random")), (96, 4, {})])
def test_dc_tiles_and_lists_bit_exact(P, calib, monkeypatch, tiled, lb, M, kw):
    """Row f3 both ways (MPR_DC_TILED): the paper's shared-memory tiles (one CTA per tile of a
    parity and realization chunk, both colours inside the tile; several chunks when M > 16)
    and the phase-list launches: states and predictions equal the oracle's DC order, on
    ragged grids whose edge tiles are partial, with n_avg > 1, generic q and RANDOM init."""
    monkeypatch.setenv("MPR_DC_TILED", tiled)
    truth, z, mask = make_problem(99, 0.55, Lx=131, corr_len=7.0)
    cfg = P.Config(l_b=lb, order="dc", n_s=1, r_s=1, **kw)
    compare(P, z, mask, truth, cfg, calib, M, 7, 41, exact_pred=cfg.n_avg == 1)


def test_context_reuse_across_masks_with_equal_counts(P, calib):
    """One context, two problems with the SAME numbers of gap sites of each colour but other
    gap positions (so other DC phase segments, records and neighbour ids), in SC and DC order:
    the cached CUDA graph of the first problem must not be replayed for the second (its key
    holds every pointer, size and segment the launches bake in). Both fills equal fresh
    single-use contexts bit for bit."""
    truth, z, mask = make_problem(48, 0.5, Lx=40, corr_len=6.0)
    # the same multiset of colour-A / colour-B gaps, shifted by two columns (colour kept)
    mask2 = np.roll(mask, 2, axis=1)
    z2 = np.roll(z, 2, axis=1)
    assert ((mask == 0) & ((np.indices(mask.shape).sum(0) & 1) == 0)).sum() == \
           ((mask2 == 0) & ((np.indices(mask.shape).sum(0) & 1) == 0)).sum()
    for order in ("sc", "dc"):
        cfg = P.Config(order=order, l_b=8, n_s=1, r_s=1)
        refs = [P.fill(zz, mm, 6, 5, 9, cfg, calib) for zz, mm in ((z, mask), (z2, mask2))]
        m = P.LeMpr(cfg, calib)
        for zz, mm, ref in ((z, mask, refs[0]), (z2, mask2, refs[1]), (z, mask, refs[0])):
            m.set_data(zz, mm)
            m.estimate_local_params()
            m.simulate(6, 5, 9)
            assert_bitwise(m.predict(), ref, f"reused context ({order})")
        m.close()


def test_dc_rejects_sc_only_features(P, calib):
    truth, z, mask = make_problem(32, 0.5, corr_len=5.0)
    m = P.LeMpr(P.Config(order="dc", l_b=8), calib)
    m.set_data(z, mask)
    m.estimate_local_params()
    with pytest.raises(P.MprError):
        m.simulate_adaptive(2, 1, max_sweeps=40)
    m.set_energy_trace(True)
    with pytest.raises(P.MprError):
        m.simulate(2, 3, 1)
    m.close()


@pytest.mark.parametrize("n_avg,init", [(1, "block_mean"), (2, "random")])
def test_adaptive_with_derived_tolerance(P, calib, n_avg, init):
    """slope_tol = "derived" (reading R22: SE(e_s) / n_fit from the exact sums of the sample
    bonds' cosines and squared cosines): the library's tolerance equals the oracle's bit for
    bit, and so do s_eq and the predictions."""
    Tk, ek = calib
    truth, z, mask = make_problem(56, 0.45, Lx=49, corr_len=6.0)
    cfg = P.Config(n_avg=n_avg, init=init)
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    m.estimate_local_params()
    s_eq = m.simulate_adaptive(6, 21, n_fit=10, n_f=4, max_sweeps=90, slope_tol="derived")
    pred, inf = m.predict(), m.info()
    m.close()
    oc = ocfg(cfg)
    p = O.parameters(z, mask, oc, Tk, ek)
    tol = O.derived_slope_tol(p.phi0, mask, oc.q, 10)
    assert inf["slope_tol"] == tol and tol > 0
    SB, NB, SP, NK = O.block_stats(p.phi0, mask, oc.lb, oc.q)
    assert inf["sample_bonds"] == int(NB.sum())
    r = O.simulate_adaptive(p, mask, oc, 6, 21, n_fit=10, n_f=4, S_max=90, slope_tol="derived")
    assert s_eq.tolist() == r["s_eq"].tolist()
    ref = O.predict(np.nan_to_num(z), mask, r["acc"], 6, n_avg, p.zmin, p.zmax, 0)
    if n_avg == 1:
        assert_bitwise(pred, ref, "adaptive (derived tolerance) predictions")
    else:
        assert np.max(np.abs(pred - ref)) <= 1e-3 * (p.zmax - p.zmin)


def test_adaptive_with_slope_tolerance(P, calib):
    """The relaxed test (slope_tol > 0) stops earlier and still agrees with the oracle."""
    Tk, ek = calib
    truth, z, mask = make_problem(48, 0.5, corr_len=6.0)
    cfg = P.Config()
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    m.estimate_local_params()
    s_eq = m.simulate_adaptive(4, 12, n_fit=20, n_f=5, max_sweeps=200, slope_tol=2e-5)
    pred = m.predict()
    m.close()
    oc = ocfg(cfg)
    p = O.parameters(z, mask, oc, Tk, ek)
    r = O.simulate_adaptive(p, mask, oc, 4, 12, n_fit=20, n_f=5, S_max=200, slope_tol=2e-5)
    assert s_eq.tolist() == r["s_eq"].tolist() and all(25 <= s < 200 for s in s_eq)
    assert_bitwise(pred, O.predict(np.nan_to_num(z), mask, r["acc"], 4, 1, p.zmin, p.zmax, 0), "predictions")


@pytest.mark.parametrize("variant", [5, 13, 14, 22, 28, 33, 40, 41])
def test_every_sweep_variant_bit_exact(P, calib, variant, monkeypatch):
    """Each half-sweep kernel variant (scalar / packed f32x2 arithmetic, one or two pairs per
    thread, early Philox; MPR_SWEEP_VARIANT) reproduces the oracle bit for bit: q = 1/2 with the energy trace, generic q, the DC
    order (glist path), and even pair counts without energy (the quad kernels' domain)."""
    monkeypatch.setenv("MPR_SWEEP_VARIANT", str(variant))
    truth, z, mask = make_problem(48, 0.45, Lx=53, corr_len=6.0)
    compare(P, z, mask, truth, P.Config(), calib, 7, 9, 1234 + variant, energy=True)
    compare(P, z, mask, truth, P.Config(q=0.35, J=1.3, r_s=1), calib, 4, 6, 99)
    compare(P, z, mask, truth, P.Config(order="dc", l_b=8, r_s=1), calib, 5, 6, 7)
    # even pair counts without the energy trace (the quad-pair kernels run, no fallback)
    compare(P, z, mask, truth, P.Config(), calib, 8, 7, 55)
    compare(P, z, mask, truth, P.Config(order="dc", l_b=8, max_batch=4), calib, 12, 5, 56)
    compare(P, z, mask, truth, P.Config(), calib, 16, 5, 57, energy=True)  # 8k realizations


def test_split_tail_batch_bit_exact(P, calib, monkeypatch):
    """The 4k + 2 batch split of large problems (MPR_SPLIT_MIN_P = 0 applies it at any size):
    the two-pair kernel on the 4k batch, the one-pair kernel on the 2-realization tail. States
    of the tail batch, accumulator, predictions and the energy trace of every realization
    equal the oracle's, for a full tail (M = 10), a half tail (M = 9, one valid realization),
    n_avg > 1 with random init, and generic q."""
    monkeypatch.setenv("MPR_SPLIT_MIN_P", "0")
    truth, z, mask = make_problem(45, 0.55, Lx=61, corr_len=6.0)
    g, _ = compare(P, z, mask, truth, P.Config(), calib, 10, 7, 31, energy=True)
    assert g["info"]["last_batch"] == 2 and g["info"]["last_m_base"] == 8
    compare(P, z, mask, truth, P.Config(), calib, 9, 6, 32, energy=True)
    compare(P, z, mask, truth, P.Config(n_avg=3, init="random"), calib, 14, 6, 33, exact_pred=False)
    compare(P, z, mask, truth, P.Config(q=0.3, J=0.8, r_s=1), calib, 6, 5, 34)


def _fuzz_case(k):
    """Seeded random small problem + configuration (case k)."""
    rng = np.random.default_rng(9000 + k)
    Ly, Lx = int(rng.integers(2, 41)), int(rng.integers(2, 41))
    p = float(rng.uniform(0.05, 0.95))
    gaps = "cloud" if (rng.random() < 0.3 and min(Ly, Lx) >= 8) else "random"
    truth, z, mask = make_problem(Ly, p, Lx=Lx, gaps=gaps, corr_len=float(rng.uniform(2, 12)),
                                  seed_field=int(rng.integers(1 << 30)), seed_mask=int(rng.integers(1 << 30)))
    order = "dc" if rng.random() < 0.25 else "sc"
    cfg_kw = dict(l_b=int(rng.integers(2, 48)), r_s=int(rng.integers(0, 5)), n_s=int(rng.integers(0, 4)),
                  q=0.5 if rng.random() < 0.5 else float(rng.uniform(0.1, 0.5)), J=float(rng.uniform(0.5, 2.0)),
                  init="random" if rng.random() < 0.5 else "block_mean", order=order,
                  max_batch=int(rng.choice([0, 2, 4])))
    M, S = int(rng.integers(1, 8)), int(rng.integers(1, 9))
    cfg_kw["n_avg"] = 1 if rng.random() < 0.7 else int(rng.integers(1, S + 1))
    return truth, z, mask, cfg_kw, M, S, int(rng.integers(1 << 40)), order == "sc"


FUZZ_CASES = int(__import__("os").environ.get("MPR_FUZZ_CASES", "150"))


@pytest.mark.parametrize("k", range(FUZZ_CASES))
def test_fuzz_small_problems_bit_exact(P, calib, k):
    """Randomised small problems (2..40 sites per side, any missing ratio, random or cloud
    gaps) under random configurations (l_b, r_s, n_s, q, J, init, SC/DC order, batch
    splits, M, S, n_avg): states bit-exact vs the oracle (predictions too when n_avg = 1,
    else within the n_avg tolerance), or the same rejection on both sides."""
    truth, z, mask, cfg_kw, M, S, seed, energy = _fuzz_case(k)
    cfg = P.Config(**cfg_kw)
    Tk, ek = calib
    if O.parameters(z, mask, ocfg(cfg), Tk, ek).status < 0:
        # the oracle rejects the problem (too few samples / no sample bond): so must the library
        m = P.LeMpr(cfg, calib)
        with pytest.raises(P.MprError):
            m.set_data(z, mask)
            m.estimate_local_params()
        m.close()
        return
    compare(P, z, mask, truth, cfg, calib, M, S, seed, energy=energy, exact_pred=cfg.n_avg == 1)


def test_context_lifecycle_releases_device_memory(P, calib):
    """20 full init -> fill -> destroy cycles (graphs, batches, energy buffers, row slabs)
    leave the device's free memory where it was: the context frees what it allocates."""
    import torch
    truth, z, mask = make_problem(96, 0.5, corr_len=8.0)

    def cycle(k):
        m = P.LeMpr(P.Config(max_batch=4 if k % 2 else 0), calib)
        m.set_data(z, mask)
        m.set_energy_trace(k % 3 == 0)
        m.estimate_local_params()
        m.simulate(6, 5, k)
        m.predict()
        m.close()
        if k % 4 == 1:  # row slabs: two contexts joined by the in-process communicator
            group_run(P, z, mask, {}, calib, 4, 3, k, 2, energy=True)

    cycle(0)  # first use: lazily created device state (CUDA context, module load)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for k in range(1, 21):
        cycle(k)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 <= 4 << 20, f"device memory not released: {(free0 - free1) / 2**20:.1f} MiB"


def test_concurrent_contexts_on_separate_streams(P, calib):
    """The header's thread-safety rule: distinct contexts may run concurrently. Two host
    threads drive two contexts on two CUDA streams (ctypes drops the GIL in the calls);
    each result equals its sequential run bit for bit."""
    import threading
    import torch
    probs = [make_problem(80, 0.4, corr_len=7.0), make_problem(72, 0.6, Lx=90, corr_len=5.0, gaps="cloud")]
    cfgs = [P.Config(), P.Config(l_b=16, r_s=1, init="random")]
    ref = [gpu_run(P, z, mask, cfg, calib, 10, 12, 3 + i)["pred"] for i, ((_, z, mask), cfg) in enumerate(zip(probs, cfgs))]
    out, errs = [None, None], []

    def work(i):
        try:
            st = torch.cuda.Stream()
            _, z, mask = probs[i]
            m = P.LeMpr(cfgs[i], calib, stream=st.cuda_stream)
            for _ in range(5):
                m.set_data(z, mask)
                m.estimate_local_params()
                m.simulate(10, 12, 3 + i)
                out[i] = m.predict()
            m.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        assert_bitwise(out[i], ref[i], f"context {i} under concurrency")


@pytest.mark.slow
def test_block_mean_init_equilibrates_faster_than_random(P, calib):
    """Row f1 energy-trace product (fig:Equi_energies): averaged over the
    realizations, the whole-grid energy of MPR with RANDOM init starts far above its plateau
    and needs many sweeps, while BLOCK_MEAN init (BST/SST) starts near the plateau."""
    from inputs.synth import heterogeneous_field, random_mask
    L = 256
    truth = heterogeneous_field(L, nu=0.5, corr_len=2.0, spread=1.0)
    mask = random_mask(L, L, 0.3)
    z = np.where(mask != 0, truth, np.float32(np.nan)).astype(np.float32)
    res = {}
    for name, cfg in (("MPR", P.Config(l_b=L, n_s=0, init="random")), ("BST", P.Config(l_b=32, n_s=0))):
        m = P.LeMpr(cfg, calib)
        m.set_data(z, mask)
        m.set_energy_trace(True)
        m.estimate_local_params()
        m.simulate(20, 50, 7)
        curve = m.debug(P.binding.MPR_BUF_ENERGY).mean(axis=0)
        m.close()
        e_eq = curve[-10:].mean()
        res[name] = (curve[0] - e_eq, int(np.argmax(np.abs(curve - e_eq) <= 1e-3 * abs(e_eq)) + 1))
    assert res["MPR"][0] > 10 * res["BST"][0] > 0
    assert res["MPR"][1] >= 10 and res["BST"][1] < res["MPR"][1]


@pytest.mark.parametrize("k", range(int(__import__("os").environ.get("MPR_FUZZ_ADAPTIVE_CASES", "24"))))
def test_fuzz_adaptive_protocol_matches_oracle(P, calib, k):
    """Row f1 randomised: small problems under random n_fit, n_f, caps, slope tolerances,
    n_avg, init and M. The per-realization equilibrium sweeps (decided on the device)
    equal the oracle's, and so do the predictions (bit-exact for n_avg = 1)."""
    rng = np.random.default_rng(7000 + k)
    Ly, Lx = int(rng.integers(6, 40)), int(rng.integers(6, 40))
    truth, z, mask = make_problem(Ly, float(rng.uniform(0.2, 0.8)), Lx=Lx, corr_len=float(rng.uniform(2, 10)),
                                  seed_field=int(rng.integers(1 << 30)), seed_mask=int(rng.integers(1 << 30)))
    n_avg = int(rng.integers(1, 4))
    cfg = P.Config(l_b=int(rng.integers(4, 33)), n_s=int(rng.integers(0, 3)), r_s=1, n_avg=n_avg,
                   init="random" if rng.random() < 0.5 else "block_mean")
    n_fit, n_f = int(rng.integers(4, 25)), int(rng.integers(1, 8))
    S_max = int(rng.integers(n_avg + 2, 90))
    tol = float(rng.choice([0.0, 1e-6, 1e-5, 1e-4]))
    M, seed = int(rng.integers(1, 9)), int(rng.integers(1 << 40))
    Tk, ek = calib
    oc = ocfg(cfg)
    p = O.parameters(z, mask, oc, Tk, ek)
    if p.status < 0:
        pytest.skip("problem rejected by the oracle (covered by the fixed-S fuzz)")
    m = P.LeMpr(cfg, calib)
    m.set_data(z, mask)
    m.estimate_local_params()
    s_eq = m.simulate_adaptive(M, seed, n_fit=n_fit, n_f=n_f, max_sweeps=S_max, slope_tol=tol)
    pred = m.predict()
    m.close()
    r = O.simulate_adaptive(p, mask, oc, M, seed, n_fit=n_fit, n_f=n_f, S_max=S_max, slope_tol=tol)
    assert s_eq.tolist() == r["s_eq"].tolist()
    ref = O.predict(np.nan_to_num(z), mask, r["acc"], M, n_avg, p.zmin, p.zmax, 0)
    if n_avg == 1:
        assert_bitwise(pred, ref, "adaptive predictions")
    else:
        assert np.max(np.abs(pred - ref)) <= 1e-3 * (p.zmax - p.zmin)


@pytest.mark.parametrize("k", range(int(__import__("os").environ.get("MPR_FUZZ_SLAB_CASES", "12"))))
def test_fuzz_row_slabs_match_oracle(P, calib, k):
    """Row slabs randomised: random grids, world sizes 2..8 (contexts on one GPU joined by the
    in-process communicator), l_b, r_s, n_s, init, n_avg, M, S: every rank bit-exact against
    the oracle (predictions within the n_avg tolerance when n_avg > 1)."""
    rng = np.random.default_rng(8000 + k)
    Ly, Lx = int(rng.integers(12, 70)), int(rng.integers(6, 60))
    truth, z, mask = make_problem(Ly, float(rng.uniform(0.2, 0.8)), Lx=Lx, corr_len=float(rng.uniform(2, 10)),
                                  seed_field=int(rng.integers(1 << 30)), seed_mask=int(rng.integers(1 << 30)))
    n_avg = int(rng.integers(1, 3))
    kw = dict(l_b=int(rng.integers(2, 24)), n_s=int(rng.integers(0, 4)), r_s=int(rng.integers(0, 4)), n_avg=n_avg,
              init="random" if rng.random() < 0.5 else "block_mean")
    M, S = int(rng.integers(1, 11)), int(rng.integers(n_avg, 9))
    world = int(rng.integers(2, min(8, Ly) + 1))
    Tk, ek = calib
    if O.parameters(z, mask, ocfg(P.Config(**kw)), Tk, ek).status < 0:
        pytest.skip("problem rejected by the oracle (covered by the fixed-S fuzz)")
    check_row_slabs(P, z, mask, kw, calib, M, S, 99 + k, world, energy=n_avg == 1,
                    device_input=bool(rng.random() < 0.5))


@pytest.mark.parametrize("world,M", [(2, 12), (3, 10), (4, 7), (2, 100)])
def test_ordered_reduce_bit_identical_to_single_context(P, calib, world, M):
    """Realization sharding with the ordered reduction (mpr_set_deferred_reduce +
    mpr_accumulate_states): contexts on one GPU standing in for ranks simulate their shards
    independently, then the accumulator is passed on in rank order (device copies where
    NCCL would send/recv) and each adds its realizations. The predictions equal the
    single-context run bit for bit."""
    import torch
    from paper_2212_01317_b200.sharding import shard_range
    truth, z, mask = make_problem(72, 0.45, Lx=61, corr_len=6.0)
    cfg = P.Config()
    ref = gpu_run(P, z, mask, cfg, calib, M, 9, 4242)["pred"]
    engs = [P.LeMpr(cfg, calib) for _ in range(world)]
    for w, e in enumerate(engs):
        e.set_data(z, mask); e.estimate_local_params(); e.reset_accumulator()
        e.set_deferred_reduce(True)
        m0, m1 = shard_range(M, world, w)
        e.simulate_range(M, 9, 4242, m0, m1)
    for w, e in enumerate(engs):
        if w > 0:
            e.accumulator_tensor().copy_(engs[w - 1].accumulator_tensor())
            torch.cuda.synchronize()
        e.accumulate_states()
    pred = engs[-1].predict()
    for e in engs:
        e.close()
    assert_bitwise(pred, ref, f"ordered reduction over {world} shards")


def test_deferred_reduce_state_rules(P, calib):
    """A pending deferred batch blocks the next simulate call; accumulating twice is a
    STATE error; a range wider than one batch is rejected."""
    truth, z, mask = make_problem(32, 0.5, corr_len=5.0)
    m = P.LeMpr(P.Config(max_batch=4), calib)
    m.set_data(z, mask); m.estimate_local_params(); m.reset_accumulator()
    m.set_deferred_reduce(True)
    with pytest.raises(P.MprError):
        m.simulate_range(10, 3, 1, 0, 10)  # needs 3 batches of 4
    m.simulate_range(10, 3, 1, 0, 4)
    with pytest.raises(P.MprError):
        m.simulate_range(10, 3, 1, 4, 8)   # previous states not accumulated
    m.accumulate_states()
    with pytest.raises(P.MprError):
        m.accumulate_states()
    m.close()


def test_filter_check_premises(P, monkeypatch):
    """The SFU rejection filter's premises (variant 40) measured on this device
    over every fp32 argument: the SFU sine within 4e-6 of ARITH §B2's sine on |y| <= 3.2, and
    exp_spec(x) * 2^24 < 1 on [-80, -17]; a context asking for variant 40 then runs it."""
    ok, e_sin, e_exp = P.binding.mpr_filter_check(0)
    print(f"SFU sine max error {e_sin:.3e}, max exp_spec*2^24 on [-80,-17] {e_exp:.6f}")
    assert ok and 0.0 < e_sin <= 4e-6 and 0.0 < e_exp < 1.0
    monkeypatch.setenv("MPR_SWEEP_VARIANT", "40")
    m = P.LeMpr(P.Config(), P.load_calibration())
    assert m.info()["sweep_variant"] == 40
    m.close()


@pytest.mark.parametrize("case", ["smooth", "rough", "edges"])
def test_filter_paths_bit_exact(P, calib, case, monkeypatch):
    """Variant 40 / 41 with the filter statistics on: the certified rejections and the queued
    exact pairs (full warps and the partial flush at the end) reproduce the oracle bit for bit,
    with n_avg > 1 (certified rejections accumulate their unchanged state), the DC lists,
    generic q and J, odd pair counts (41) and RANDOM init. 'smooth': low temperatures, most
    pairs certified; 'rough': a white-noise field at high temperatures, most pairs exact;
    'edges': a thin grid where most sites miss a neighbour."""
    monkeypatch.setenv("MPR_FILTER_STATS", "1")
    monkeypatch.setenv("MPR_SWEEP_VARIANT", "40")
    if case == "smooth":
        truth, z, mask = make_problem(96, 0.4, Lx=80, corr_len=12.0)
    elif case == "rough":
        rng = np.random.default_rng(7)
        truth = rng.standard_normal((64, 72)).astype(np.float32)
        mask = (rng.random((64, 72)) > 0.5).astype(np.uint8)
        z = truth.copy(); z[mask == 0] = np.nan
    else:
        truth, z, mask = make_problem(3, 0.5, Lx=203, corr_len=4.0)
    runs = [(P.Config(), 8, 9, 11, True), (P.Config(n_avg=3, init="random"), 12, 8, 12, False),
            (P.Config(order="dc", l_b=8), 8, 6, 13, True), (P.Config(q=0.3, J=1.7, r_s=1), 6, 6, 14, True),
            (P.Config(), 6, 7, 15, True)]
    fracs = []
    for cfg, M, S, seed, exact in runs:
        g, _ = compare(P, z, mask, truth, cfg, calib, M, S, seed, exact_pred=exact)
        inf = g["info"]
        assert inf["sweep_variant"] == 40 and inf["filter_pairs"] > 0
        fracs.append(inf["filter_exact_pairs"] / inf["filter_pairs"])
    print(case, "exact-path fraction per run", [round(f, 3) for f in fracs])
    if case == "smooth":
        assert max(fracs) < 0.5
    if case == "rough":
        assert min(fracs) > 0.2


def test_multiwave_launches_bit_exact(P, calib, monkeypatch):
    """Half-sweep launches spanning several resident waves of CTAs (MPR_SWEEP_WAVES = 8 makes
    every launch here larger than one wave): SC and DC order, n_avg > 1 with RANDOM init,
    the energy-trace kernels (per-CTA atomics from every wave), generic q and an odd pair
    count (the one-pair kernel) against the oracle."""
    monkeypatch.setenv("MPR_SWEEP_WAVES", "8")
    truth, z, mask = make_problem(256, 0.5, corr_len=12.0)
    g, _ = compare(P, z, mask, truth, P.Config(), calib, 48, 4, 501)
    assert g["info"]["kernel_launches"] > 0
    compare(P, z, mask, truth, P.Config(n_avg=2, init="random"), calib, 40, 4, 502, exact_pred=False)
    compare(P, z, mask, truth, P.Config(order="dc", l_b=16), calib, 48, 3, 503)
    compare(P, z, mask, truth, P.Config(), calib, 48, 3, 504, energy=True)
    compare(P, z, mask, truth, P.Config(q=0.4, J=1.2), calib, 48, 3, 505)
    compare(P, z, mask, truth, P.Config(), calib, 46, 3, 506)
