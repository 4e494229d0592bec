"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle on the same inputs."""
import hashlib

import numpy as np
import pytest

import paper_1012_4382_b200 as xf
from oracle import oracle as orc
from paper_1012_4382_b200 import _native as N
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun
from tests.cases import BATH300, DIMER, FMO, RATES, TRAJ_CASES, site_rho

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- tables (A1)

def test_device_tables_bit_exact_small(golden_tables):
    keys = sorted({k.rsplit("_", 1)[0] for k in golden_tables.files})
    for key in keys:
        m, n = (int(x[1:]) for x in key.split("_"))
        g = xf.enumerate_hierarchy(m, n)
        for name in ("indices", "tiers", "plus", "minus"):
            arr = getattr(g, name)
            assert arr.dtype == np.int32
            assert np.array_equal(arr, golden_tables[f"{key}_{name}"]), (key, name)


@pytest.mark.parametrize("key", ["M7_N6", "M7_N8", "M7_N10", "M14_N4", "M14_N6", "M14_N8"])
def test_device_tables_bit_exact_hashed(golden_hashes, key):
    m, n = (int(x[1:]) for x in key.split("_"))
    ref = golden_hashes[key]
    g = xf.enumerate_hierarchy(m, n)
    assert g.n_tot == ref["n_tot"]
    for name in ("indices", "tiers", "plus", "minus"):
        assert _sha(getattr(g, name)) == ref[name], (key, name)


def test_locality_permutation_is_lexicographic():
    g = xf.enumerate_hierarchy(5, 4)
    perm = np.asarray(g.perm)
    assert sorted(perm.tolist()) == list(range(g.n_tot))
    order = np.argsort(perm)
    rows = [tuple(r) for r in g.indices[order]]
    assert rows == sorted(rows)          # device order = pure lexicographic
    assert perm[0] == 0                  # the root stays first


def test_index_of_and_errors():
    g = xf.enumerate_hierarchy(7, 3)
    for k in range(g.n_tot):
        assert xf.index_of(g, g.indices[k]) == k
    with pytest.raises(KeyError):
        xf.index_of(g, (4, 0, 0, 0, 0, 0, 0))
    with pytest.raises(ValueError):
        xf.enumerate_hierarchy(64, 64)
    with pytest.raises(ValueError):
        xf.enumerate_hierarchy(0, 4)


# ------------------------------------------------- Level-2 kernel ABI (A3-A6)

@pytest.mark.parametrize("case", ["fmo_n2", "fmo_n3_77k", "dimer_n4", "dephasing_n5"])
def test_rhs_shim_matches_reference_kernel(golden_rhs, case):
    from paper_1012_4382_b200 import kernels
    g = golden_rhs
    n_sites, n_max = int(g[case + "_n_sites"]), int(g[case + "_n_max"])
    graph = xf.enumerate_hierarchy(n_sites, n_max)
    sig = g[case + "_sig"]
    out = np.empty_like(sig)
    kernels.hierarchy_rhs_kernel(out, sig, g[case + "_h"], g[case + "_site_of"], graph.plus,
                                 graph.minus, graph.indices.astype(np.float64),
                                 graph.tiers * float(g[case + "_gamma"]), float(g[case + "_a"]),
                                 float(g[case + "_b"]), g[case + "_decay"])
    ref = g[case + "_out"]
    assert np.max(np.abs(out - ref)) <= 1e-14 * np.max(np.abs(ref))


@pytest.mark.parametrize("case", ["fmo_n2", "dimer_n4"])
def test_elementwise_shims(golden_rhs, case):
    from paper_1012_4382_b200 import kernels
    g = golden_rhs
    x = g[case + "_sig"].reshape(-1).copy()
    y = g[case + "_out"].reshape(-1).copy()
    tmp = np.empty_like(x)
    kernels.add_scaled(tmp, x, y, 0.37)
    assert np.max(np.abs(tmp - g[case + "_add_scaled"])) <= 1e-15 * np.max(np.abs(tmp))
    s2 = x.copy()
    kernels.rk4_update(s2, x, y, tmp, x[::-1].copy(), 0.125)
    assert np.max(np.abs(s2 - g[case + "_rk4_update"])) <= 1e-15 * np.max(np.abs(s2))
    assert kernels.max_abs2(y) == float(g[case + "_max_abs2"])


# ------------------------------------------------------- propagation (A7-A10)

@pytest.mark.parametrize("name", list(TRAJ_CASES))
def test_trajectory_matches_reference(golden_traj, name):
    arrays, meta = golden_traj
    system, bath, rates, kw, rho0 = TRAJ_CASES[name]
    traj = xf.propagate_from(system, bath, rates, xf.PropagationConfig(**kw), rho0)
    assert traj.stop_reason == meta[name]["stop_reason"]
    assert np.array_equal(traj.times_fs, arrays[name + "_times"])
    assert np.max(np.abs(traj.populations - arrays[name + "_pops"])) < 1e-10
    assert np.max(np.abs(traj.final_rho - arrays[name + "_final_rho"])) < 1e-10
    if name + "_matrices" in arrays.files:
        assert np.max(np.abs(traj.matrices - arrays[name + "_matrices"])) < 1e-10


def test_efficiency_and_trapping_time(golden_traj):
    arrays, meta = golden_traj
    system, bath, rates, kw, rho0 = TRAJ_CASES["fmo_n2_eta"]
    traj = xf.propagate_from(system, bath, rates, xf.PropagationConfig(**kw), rho0)
    assert abs(xf.efficiency(traj) - meta["fmo_n2_eta"]["eta"]) < 1e-10
    assert abs(xf.trapping_time(traj) - meta["fmo_n2_eta"]["trapping_time_ps"]) < 1e-8
    assert abs(xf.efficiency(traj) + traj.ground_population()[-1] - 1.0) < 1e-5


def test_divergence_guard_message(golden_traj):
    _, meta = golden_traj
    cfg = xf.PropagationConfig(dt_fs=150.0, n_max=2, t_end_fs=30000.0, residual=None)
    with pytest.raises(xf.PropagationDiverged) as exc:
        xf.propagate(FMO, BATH300, RATES, cfg, 1)
    assert str(exc.value) == meta["diverge"]["message"]


def test_hard_cap_message(golden_traj):
    _, meta = golden_traj
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=0, residual=1e-5, hard_cap_fs=500.0)
    with pytest.raises(xf.ConvergenceFailure) as exc:
        xf.propagate(FMO, BATH300, xf.MarkovRates.none(), cfg, 1)
    assert str(exc.value) == meta["hardcap"]["message"]


@pytest.mark.parametrize("K", [0, 1])
def test_layouts_orderings_kernels_agree(K):
    base = dict(dt_fs=2.5, n_max=3, t_end_fs=300.0, residual=None, n_matsubara=K,
                record_matrices=True, record_stride=10)
    ref = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(**base), 1)
    for layout in ("hermitian", "general"):
        for ordering in ("lex", "lex-split", "reference"):
            for kernel in ("auto", "generic"):
                cfg = xf.PropagationConfig(**base, layout=layout, ordering=ordering, kernel=kernel)
                t = xf.propagate(FMO, BATH300, RATES, cfg, 1)
                assert np.max(np.abs(t.populations - ref.populations)) < 1e-13, (layout, ordering)
                assert np.max(np.abs(t.matrices - ref.matrices)) < 1e-13, (layout, ordering)


def test_chunking_does_not_change_results():
    base = dict(dt_fs=5.0, n_max=2, residual=1e-5, record_stride=3)
    a = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(**base, chunk_steps=1), 1)
    b = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(**base, chunk_steps=97), 1)
    assert np.array_equal(a.times_fs, b.times_fs)
    assert np.array_equal(a.populations, b.populations)


def test_zero_truncation_equals_markov_only():
    cfg = xf.PropagationConfig(dt_fs=1.0, n_max=0, t_end_fs=200.0, residual=None)
    a = xf.propagate(FMO, BATH300, RATES, cfg, 1).populations
    b = xf.propagate(FMO, xf.BathParams.from_timescale(0.0, 166.0, 300.0), RATES, cfg, 1).populations
    assert np.max(np.abs(a - b)) == 0.0


def test_t_end_zero_and_initial_residual():
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=2, t_end_fs=0.0, residual=None)
    traj = xf.propagate(FMO, BATH300, RATES, cfg, 1)
    assert traj.times_fs.tolist() == [0.0] and traj.stop_reason == "t_end"
    rho0 = np.zeros((9, 9), complex)
    rho0[8, 8] = 1.0  # everything already trapped
    traj = xf.propagate_from(FMO, BATH300, RATES, xf.PropagationConfig(dt_fs=2.5, n_max=2), rho0)
    assert traj.stop_reason == "residual" and len(traj.times_fs) == 1


def test_input_validation():
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=0, t_end_fs=10.0, residual=None)
    bad = site_rho(1)
    bad[0, 1] = bad[1, 0] = 0.1
    with pytest.raises(ValueError):
        xf.propagate_from(FMO, BATH300, RATES, cfg, bad)
    with pytest.raises(ValueError):
        xf.propagate(FMO, BATH300, RATES, cfg, 8)
    with pytest.raises(ValueError):
        xf.propagate_from(FMO, BATH300, RATES, cfg, np.eye(3))


# --------------------------------------------------------- K >= 1 (unpinned)

@pytest.mark.parametrize("n_max", [2, 3])
def test_matsubara_k1_matches_oracle(n_max):
    cfg = xf.PropagationConfig(dt_fs=1.0, n_max=n_max, t_end_fs=150.0, residual=None,
                               n_matsubara=1, record_stride=5)
    traj = xf.propagate(FMO, BATH300, RATES, cfg, 1)
    ref = orc.propagate_from(FMO, BATH300, RATES, cfg, site_rho(1))
    assert np.max(np.abs(traj.populations - ref["populations"])) < 1e-10
    assert np.max(np.abs(traj.final_rho - ref["final_rho"])) < 1e-10


def test_matsubara_zero_coefficient_equals_k0():
    bath = xf.BathParams.from_timescale(20.0, 100.0, 77.0)
    nu, a, b = xf.bath_modes(bath, 0)
    ops0 = BlockOperands(DIMER, bath, xf.MarkovRates.none(), 0)
    ops1 = BlockOperands(DIMER, bath, xf.MarkovRates.none(), 1,
                         modes=(np.array([nu[0], 3.0]), np.array([a[0], 0.0]), np.array([b[0], 0.0])))
    out = []
    for ops in (ops0, ops1):
        with DeviceRun(ops, 3, 0.5, t_end_fs=200.0) as run:
            run.set_rho0(np.diag([1.0, 0.0]).astype(complex), [])
            assert run.run() == N.HB_OK
            out.append(run.records()[1])
    assert np.max(np.abs(out[0] - out[1])) < 1e-15


@pytest.mark.slow
def test_long_eta_twin(golden_long):
    arrays, meta = golden_long
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=6, residual=1e-5, record_stride=100)
    traj = xf.propagate(FMO, BATH300, RATES, cfg, 1)
    m = meta["fmo_n6_eta"]
    assert traj.stop_reason == "residual"
    assert np.array_equal(traj.times_fs, arrays["fmo_n6_eta_times"])
    assert np.max(np.abs(traj.populations - arrays["fmo_n6_eta_pops"])) < 1e-10
    assert abs(xf.efficiency(traj) - m["eta"]) < 1e-10
    # the trapping time <t> (observables.py:85-110) from the same records
    assert abs(xf.trapping_time(traj) - m["trapping_time_ps"]) < 1e-8


def test_large_hierarchy_two_steps_vs_oracle():
    """Config 4 shape (FMO 300 K, N_max=8, K=1, 319,770 ADOs): two RK4 steps."""
    cfg = xf.PropagationConfig(dt_fs=1.0, n_max=8, t_end_fs=2.0, residual=None, n_matsubara=1)
    traj = xf.propagate(FMO, BATH300, RATES, cfg, 1)
    orc.set_threads(8)
    ref = orc.propagate_from(FMO, BATH300, RATES, cfg, site_rho(1))
    orc.set_threads(1)
    assert np.max(np.abs(traj.populations - ref["populations"])) < 1e-12
    assert np.max(np.abs(traj.final_rho - ref["final_rho"])) < 1e-12


# ------------------------------------------------- dense definition (A11)

def test_dense_heom_rhs_matches_reference():
    g = np.load("tests/golden/dense_cases.npz")
    graph = xf.enumerate_hierarchy(7, 2)
    out = xf.heom_rhs(xf.HierarchyState(g["sig"]), graph, FMO, BATH300, RATES)
    ref = g["out"]
    assert np.max(np.abs(out - ref)) <= 1e-14 * np.max(np.abs(ref))


def test_dense_rk4_matches_reference_and_fast_path():
    """test_heom.py:120-130: 40 dense RK4 steps vs the fast propagator."""
    g = np.load("tests/golden/dense_cases.npz")
    graph = xf.enumerate_hierarchy(7, 2)
    state = xf.HierarchyState.initial(graph, FMO, site_rho(1))
    for _ in range(40):
        state = xf.rk4_step(state, graph, FMO, BATH300, RATES, 2.5)
    assert state.time_fs == float(g["rk40_time"])
    assert np.max(np.abs(state.sigma - g["rk40_sigma"])) < 1e-12
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=2, t_end_fs=100.0, residual=None)
    traj = xf.propagate(FMO, BATH300, RATES, cfg, 1)
    assert np.max(np.abs(traj.populations[-1] - np.real(np.diag(state.rho)))) < 1e-13


# ------------------------------------------------- sharding (8(e)), one GPU

@pytest.mark.parametrize("n_shards,n_max,K", [(2, 3, 1), (3, 3, 1), (4, 5, 1), (8, 5, 1), (3, 6, 0)])
def test_sharded_run_is_bit_exact(n_shards, n_max, K):
    """ONE hierarchy split over in-process shards (local numbering, owned + halo
    slots only, four launch groups, cross halos): every ADO of the final state,
    the records and the sinks equal the unsharded run bit for bit."""
    from paper_1012_4382_b200.shard import ShardedRun
    ops = BlockOperands(FMO, BATH300, RATES, K)
    rho0 = np.zeros((7, 7), complex)
    rho0[0, 0] = 1.0
    n_tot = xf.hierarchy_size(7 * (K + 1), n_max)
    with DeviceRun(ops, n_max, 1.0, t_end_fs=30.0, layout="hermitian") as ref:
        ref.set_rho0(rho0, [0.0, 0.0])
        assert ref.run() == N.HB_OK
        steps_ref, pops_ref, _ = ref.records()
        sig_ref, sinks_ref = ref.sigma0()
        state_ref, _ = ref.state(n_tot)
    sr = ShardedRun(ops, n_max, 1.0, 30.0, n_shards)
    try:
        assert all(L.halo_entries() > 0 for L in sr.layouts)
        assert sum(L.n_owned for L in sr.layouts) == n_tot
        sr.set_rho0(rho0, [0.0, 0.0])
        assert sr.run() == 1  # t_end
        steps, pops, _ = sr.records()
        sig, sinks = sr.sigma0()
        state = sr.state(n_tot)
    finally:
        sr.close()
    assert np.array_equal(steps, steps_ref)
    assert np.array_equal(pops, pops_ref)          # bit-exact: same kernels, complete halos
    assert np.array_equal(sig, sig_ref) and np.array_equal(sinks, sinks_ref)
    assert np.array_equal(state, state_ref)


def test_sharded_single_precision_is_bit_exact():
    from paper_1012_4382_b200.shard import ShardedRun
    ops = BlockOperands(FMO, BATH300, RATES, 1)
    rho0 = np.zeros((7, 7), complex)
    rho0[0, 0] = 1.0
    with DeviceRun(ops, 3, 1.0, t_end_fs=30.0, layout="hermitian", precision="single") as ref:
        ref.set_rho0(rho0, [0.0, 0.0])
        assert ref.run() == N.HB_OK
        _, pops_ref, _ = ref.records()
    sr = ShardedRun(ops, 3, 1.0, 30.0, 3, precision="single")
    try:
        sr.set_rho0(rho0, [0.0, 0.0])
        assert sr.run() == 1
        _, pops, _ = sr.records()
    finally:
        sr.close()
    assert np.array_equal(pops, pops_ref)


# ------------------------------------------------- sweeps (8(f) rank 2)

def test_sweep_is_worker_count_invariant():
    """cli.py:279-284 / test_cli.py:182-190: results independent of the worker count."""
    from paper_1012_4382_b200.sweep import SweepPoint, fmo_point_runner, run_points
    cfg = xf.PropagationConfig(dt_fs=5.0, n_max=2, residual=1e-5, record_stride=20)
    pts = [SweepPoint(temperature_k=t, lam_cm1=lam) for t in (77.0, 300.0) for lam in (20.0, 55.0)]
    runner = fmo_point_runner(cfg, RATES)
    seq = run_points(pts, runner, workers=1)
    par = run_points(pts, runner, workers=4)
    assert [r.point for r in par] == pts
    for a, b in zip(seq, par):
        assert a.efficiency == b.efficiency and a.trapping_time_ps == b.trapping_time_ps
        assert a.steps == b.steps and a.stop_reason == "residual"
    ref = orc.propagate_from(FMO, xf.BathParams.from_timescale(55.0, 166.0, 300.0), RATES, cfg,
                             site_rho(1))
    assert abs(seq[3].efficiency - ref["populations"][-1, 8]) < 1e-10


# ------------------------------------------------- other shapes vs the oracle

def _random_system(n, seed, ground=False):
    rng = np.random.default_rng(seed)
    a = rng.normal(0.0, 60.0, (n, n))
    h = (a + a.T) / 2.0
    h[np.diag_indices(n)] = rng.normal(0.0, 120.0, n)
    if ground:
        full = np.zeros((n + 1, n + 1))
        full[1:, 1:] = h
        return xf.ExcitonSystem(h_cm1=full, site_indices=tuple(range(1, n + 1)), ground_index=0)
    return xf.ExcitonSystem(h_cm1=h, site_indices=tuple(range(n)))


@pytest.mark.parametrize("n,K,n_max,ground", [(1, 0, 5, False), (3, 1, 3, True), (5, 1, 3, False),
                                              (8, 0, 2, False), (9, 0, 1, False), (4, 2, 2, False)])
def test_other_shapes_match_oracle(n, K, n_max, ground):
    system = _random_system(n, 100 + n, ground)
    rates = xf.MarkovRates(0.0, 1.0 / 50000.0) if ground else xf.MarkovRates.none()
    bath = xf.BathParams.from_timescale(25.0, 120.0, 250.0)
    cfg = xf.PropagationConfig(dt_fs=1.0, n_max=n_max, t_end_fs=60.0, residual=None,
                               n_matsubara=K, record_stride=7, record_matrices=True)
    d = system.dimension
    rho0 = np.zeros((d, d), complex)
    first = system.site_indices[0]
    rho0[first, first] = 1.0
    traj = xf.propagate_from(system, bath, rates, cfg, rho0)
    ref = orc.propagate_from(system, bath, rates, cfg, rho0)
    assert np.array_equal(traj.times_fs, ref["times_fs"])
    assert np.max(np.abs(traj.populations - ref["populations"])) < 1e-10
    assert np.max(np.abs(traj.matrices - ref["matrices"])) < 1e-10


def test_nccl_shard_path_world_one_is_bit_exact():
    """The NCCL sharded path (hb_nccl_init, hb_shard_steps: launch groups, second
    stream, guard all-reduce) at world size 1 -- the only size one GPU can run --
    equals the unsharded run bit for bit; multi-GPU halos are covered by the
    in-process shards above and the gloo protocol test (tests/test_shard_host.py)."""
    import socket
    import torch.distributed as dist
    from paper_1012_4382_b200.shard import NcclShardedRun
    ops = BlockOperands(FMO, BATH300, RATES, 1)
    rho0 = np.zeros((7, 7), complex)
    rho0[0, 0] = 1.0
    with DeviceRun(ops, 4, 1.0, t_end_fs=60.0, layout="hermitian") as ref:
        ref.set_rho0(rho0, [0.0, 0.0])
        assert ref.run() == N.HB_OK
        _, pops_ref, _ = ref.records()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        sr = NcclShardedRun(ops, 4, 1.0, 60.0, 0, 1, 0, dist, record_stride=1)
        try:
            sr.set_rho0(rho0, [0.0, 0.0])
            assert sr.run(chunk=25) == 1
            _, pops, _ = sr.run_.records()
            assert sr.describe()["halo_ados_max"] == 0
            assert sr.launch_count() > 0
        finally:
            sr.close()
    finally:
        dist.destroy_process_group()
    assert np.array_equal(pops, pops_ref)
