"""Full-hierarchy parity of the production kernel (k_mm4, through the C ABI).

Every ADO of the hierarchy -- not only sigma^0 -- is compared with the oracle's
propagation (oracle/heom_oracle.c ``or_propagate``, a restatement of
heom.py:286-406 and _kernels.py:23-58) after 1 and 10 RK4 steps from a random
Hermitian hierarchy, tier by tier, each tier against its own magnitude.  That
is the reference's own full-state check (test_heom.py:120-130: the fast path
against the dense definition on every ADO) applied to the device.  From
physical initial conditions the deep tiers are ~(dt theta)^tier after a few
steps, so errors in the top-tier paths (the paired-site gather rounds of tiles
without raise links, the skipped raise-link tables of top-tier tiles) would sit
far below any absolute tolerance.  Here tier t is random with magnitude s^t,
s = sqrt(a_0) (the scale at which the raise term +i[V, sigma_{n+e}] and the
lower term n theta sigma_{n-e} of _kernels.py:41-57 are of the same size, so
10 steps neither blow up nor decay), and every tier -- the top tier included --
must agree to 1e-13 of its own size: a perturbed branch shows at 1e-3 or more.

Also: the config-3 K=1 hierarchy (N_max=6, 38,760 ADOs, dt 1.25 fs) for 1,600
steps and config 4 (N_max=8, K=1, 319,770 ADOs) for 50 steps, both from
rho0 = |1><1| against the oracle at 1e-10.
"""
import os

import numpy as np
import pytest

import paper_1012_4382_b200 as xf
from oracle import oracle as orc
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun
from tests.cases import BATH300, FMO, RATES, site_rho

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


def random_hermitian_hierarchy(tiers, d, seed):
    rng = np.random.default_rng(seed)
    n_tot = tiers.shape[0]
    a = rng.standard_normal((n_tot, d, d)) + 1j * rng.standard_normal((n_tot, d, d))
    s = np.sqrt(xf.bath_modes(BATH300, 0)[1][0])  # sqrt(a_0), a_0 = 2 lam kT (fs^-2)
    return 0.5 * (a + np.conj(np.transpose(a, (0, 2, 1)))) * (s ** tiers)[:, None, None]


def _device_state(K, n_max, ordering, precision, steps, sig0):
    ops = BlockOperands(FMO, BATH300, RATES, K)
    with DeviceRun(ops, n_max, 1.0, t_end_fs=float(steps), ordering=ordering,
                   precision=precision, record_stride=1) as run:
        run.set_state(sig0, [0.0, 0.0])
        run.run()
        assert run.result.steps == steps
        sig, sinks = run.state(sig0.shape[0])
        _, pops, _ = run.records()
    return sig, sinks, pops


def _oracle_state(K, n_max, steps, sig0):
    cfg = xf.PropagationConfig(dt_fs=1.0, n_max=n_max, t_end_fs=float(steps), residual=None,
                               n_matsubara=K)
    orc.set_threads(THREADS)
    try:
        ref = orc.propagate_from(FMO, BATH300, RATES, cfg, site_rho(1), init_state=sig0)
    finally:
        orc.set_threads(1)
    return ref


_CACHE = {}


def _case(K, n_max, steps):
    key = (K, n_max, steps)
    if key not in _CACHE:
        tiers = orc.enumerate_hierarchy(7 * (K + 1), n_max)[1]
        sig0 = random_hermitian_hierarchy(tiers, 7, seed=100 * K + 10 * n_max + steps)
        _CACHE.clear()  # the N_max=8, K=1 states are 250 MB each
        _CACHE[key] = (sig0, _oracle_state(K, n_max, steps, sig0), tiers)
    return _CACHE[key]


# kernels by size (hb_api.cu KParams::split): N_max = 3, 4 -> k_mm4ab 2 + 2 warps;
# K = 0, N_max = 8 (202 tiles) and K = 1, N_max = 5 (364 tiles) -> 1 + 1 warps;
# K = 1, N_max = 8 -> k_mm4 (one warp per tile, paired rounds on the top tier)
FULL_CASES = [(K, n, steps, order)
              for K in (0, 1) for n in (3, 4, 8) for steps in (1, 10)
              for order in ("reference", "lex", "lex-split")] + \
             [(1, 5, steps, "reference") for steps in (1, 10)]


def _tier_errors(sig, want, tiers):
    """max |device - oracle| / max |oracle| per tier"""
    out = []
    for t in range(int(tiers.max()) + 1):
        sel = tiers == t
        out.append(float(np.max(np.abs(sig[sel] - want[sel])) / np.max(np.abs(want[sel]))))
    return np.array(out)


@pytest.mark.parametrize("K,n_max,steps,ordering", FULL_CASES)
def test_every_ado_matches_oracle_double(K, n_max, steps, ordering):
    sig0, ref, tiers = _case(K, n_max, steps)
    sig, sinks, pops = _device_state(K, n_max, ordering, "double", steps, sig0)
    err = _tier_errors(sig, ref["final_state"], tiers)
    assert np.all(err <= 1e-13), err
    sink_ref = ref["populations"][-1][[0, 8]]
    assert np.max(np.abs(sinks - sink_ref)) <= 1e-13 * max(1.0, np.max(np.abs(sink_ref)))
    assert np.max(np.abs(pops - ref["populations"])) <= 1e-13 * np.max(np.abs(ref["populations"]))


@pytest.mark.parametrize("K,n_max,ordering", [(0, 4, "reference"), (1, 3, "lex"),
                                              (1, 4, "reference"), (1, 8, "reference"),
                                              (1, 8, "lex-split")])
def test_every_ado_matches_oracle_single(K, n_max, ordering):
    """precision='single' (float32 state and RHS, heom.py:93-94) on the same
    random hierarchies: every ADO within float32 accuracy of the FP64 oracle."""
    steps = 10
    sig0, ref, tiers = _case(K, n_max, steps)
    sig, _, _ = _device_state(K, n_max, ordering, "single", steps, sig0)
    err = _tier_errors(sig, ref["final_state"], tiers)
    assert np.all(err <= 1e-5), err


def test_paired_rounds_are_exercised():
    """The tier-major order puts the top tier in whole tiles past P.top_tile:
    at N_max = 8, K = 1 that is 64 % of the ADOs (6,359 of 9,993 tiles)."""
    n_tot = xf.hierarchy_size(14, 8)
    top = xf.hierarchy_size(13, 8)
    first_top_tile = -(-(n_tot - top) // 32)
    n_tiles = -(-n_tot // 32)
    assert (n_tot, top) == (319770, 203490)
    assert n_tiles - first_top_tile == 6359


@pytest.mark.slow
def test_config3_k1_1600_steps_vs_oracle():
    """Config 3 hierarchy at K = 1 (N_max = 6, 38,760 ADOs, dt 1.25 fs): 1,600
    RK4 steps (2 ps) from |1><1| with trap and sinks, against the oracle."""
    cfg = xf.PropagationConfig(dt_fs=1.25, n_max=6, t_end_fs=2000.0, residual=None,
                               n_matsubara=1, record_stride=40)
    traj = xf.propagate(FMO, BATH300, RATES, cfg, 1)
    orc.set_threads(THREADS)
    try:
        ref = orc.propagate_from(FMO, BATH300, RATES, cfg, site_rho(1))
    finally:
        orc.set_threads(1)
    assert len(traj.times_fs) == len(ref["times_fs"]) == 41
    assert np.max(np.abs(traj.populations - ref["populations"])) < 1e-10
    assert np.max(np.abs(traj.final_rho - ref["final_rho"])) < 1e-10


@pytest.mark.slow
def test_config4_50_steps_vs_oracle():
    """Config 4 (FMO 300 K, N_max = 8, K = 1, 319,770 ADOs, dt 1 fs): 50 steps
    from |1><1|, every ADO of the final state against the oracle."""
    cfg = xf.PropagationConfig(dt_fs=1.0, n_max=8, t_end_fs=50.0, residual=None, n_matsubara=1,
                               record_stride=5)
    ops = BlockOperands(FMO, BATH300, RATES, 1)
    with DeviceRun(ops, 8, 1.0, t_end_fs=50.0, record_stride=5) as run:
        rho0 = np.zeros((7, 7), complex)
        rho0[0, 0] = 1.0  # site 1 (block position 0)
        run.set_rho0(rho0, [0.0, 0.0])
        run.run()
        sig, _ = run.state(319770)
        _, pops, _ = run.records()
    orc.set_threads(THREADS)
    try:
        ref = orc.propagate_from(FMO, BATH300, RATES, cfg, site_rho(1))
    finally:
        orc.set_threads(1)
    assert np.max(np.abs(pops - ref["populations"])) < 1e-10
    assert np.max(np.abs(sig - ref["final_state"])) < 1e-10
    # the deep tiers are ~1e-15 after 50 steps (absolute 1e-10 says nothing about
    # them): every tier against its own size as well
    tiers = orc.enumerate_hierarchy(14, 8)[1]
    err = _tier_errors(sig, ref["final_state"], tiers)
    assert np.all(err <= 1e-10), err
