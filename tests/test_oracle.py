"""Pin the CPU oracle (oracle/heom_oracle.c) to the reference's own outputs.

Golden vectors come from running the reference itself (tests/golden/make_golden.py).
No GPU needed.
"""
import hashlib

import numpy as np
import pytest

from oracle import oracle as orc
from tests.cases import TRAJ_CASES

pytestmark = []


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_tables_small_bit_exact(golden_tables):
    keys = sorted({k.rsplit("_", 1)[0] for k in golden_tables.files})
    assert len(keys) >= 10
    for key in keys:
        m, n = (int(x[1:]) for x in key.split("_"))
        got = orc.enumerate_hierarchy(m, n)
        for name, arr in zip(("indices", "tiers", "plus", "minus"), got):
            ref = golden_tables[f"{key}_{name}"]
            assert arr.dtype == np.int32
            assert np.array_equal(arr, ref), (key, name)


@pytest.mark.parametrize("key", ["M7_N6", "M7_N8", "M14_N4", "M14_N6"])
def test_tables_hash_bit_exact(golden_hashes, key):
    m, n = (int(x[1:]) for x in key.split("_"))
    ref = golden_hashes[key]
    got = orc.enumerate_hierarchy(m, n)
    assert got[0].shape[0] == ref["n_tot"]
    for name, arr in zip(("indices", "tiers", "plus", "minus"), got):
        assert _sha(arr) == ref[name], (key, name)


def test_counts_and_range():
    assert orc.hierarchy_size(7, 4) == 330
    assert orc.hierarchy_size(14, 8) == 319770
    with pytest.raises(ValueError):
        orc.enumerate_hierarchy(64, 64)


@pytest.mark.parametrize("case", ["fmo_n2", "fmo_n3_77k", "dimer_n4", "dephasing_n5"])
def test_rhs_matches_reference_kernel(golden_rhs, case):
    g = golden_rhs
    n_sites, n_max = int(g[case + "_n_sites"]), int(g[case + "_n_max"])
    ind, tiers, plus, minus = orc.enumerate_hierarchy(n_sites, n_max)
    out = orc.rhs_from_arrays(g[case + "_sig"], g[case + "_h"], g[case + "_site_of"], plus, minus,
                              ind, n_sites, 1, [float(g[case + "_gamma"])], [float(g[case + "_a"])],
                              [float(g[case + "_b"])], g[case + "_decay"])
    ref = g[case + "_out"]
    # normwise: the reference is compiled with fastmath (hard part 7)
    assert np.max(np.abs(out - ref)) <= 1e-14 * np.max(np.abs(ref))


@pytest.mark.parametrize("name", [n for n in TRAJ_CASES if n != "fmo_n4_77k"] + ["fmo_n4_77k"])
def test_trajectories_match_reference(golden_traj, name):
    arrays, meta = golden_traj
    system, bath, rates, kw, rho0 = TRAJ_CASES[name]
    import paper_1012_4382_b200 as xf
    cfg = xf.PropagationConfig(**kw)
    res = orc.propagate_from(system, bath, rates, cfg, rho0)
    assert res["stop_reason"] == meta[name]["stop_reason"]
    assert np.array_equal(res["times_fs"], arrays[name + "_times"])
    assert np.max(np.abs(res["populations"] - arrays[name + "_pops"])) < 1e-12
    assert np.max(np.abs(res["final_rho"] - arrays[name + "_final_rho"])) < 1e-12
    if name + "_matrices" in arrays.files:
        assert np.max(np.abs(res["matrices"] - arrays[name + "_matrices"])) < 1e-12


def test_eta_closes_budget(golden_traj):
    arrays, meta = golden_traj
    system, bath, rates, kw, rho0 = TRAJ_CASES["fmo_n2_eta"]
    import paper_1012_4382_b200 as xf
    res = orc.propagate_from(system, bath, rates, xf.PropagationConfig(**kw), rho0)
    eta = res["populations"][-1, 8]
    assert abs(eta - meta["fmo_n2_eta"]["eta"]) < 1e-12
    assert abs(eta + res["populations"][-1, 0] - 1.0) < 1e-5


def test_divergence_and_hardcap_messages(golden_traj):
    _, meta = golden_traj
    import paper_1012_4382_b200 as xf
    from tests.cases import BATH300, FMO, RATES, site_rho
    cfg = xf.PropagationConfig(dt_fs=150.0, n_max=2, t_end_fs=30000.0, residual=None)
    with pytest.raises(RuntimeError) as exc:
        orc.propagate_from(FMO, BATH300, RATES, cfg, site_rho(1))
    assert str(exc.value) == "diverged: " + meta["diverge"]["message"]
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=0, residual=1e-5, hard_cap_fs=500.0)
    with pytest.raises(RuntimeError) as exc:
        orc.propagate_from(FMO, BATH300, xf.MarkovRates.none(), cfg, site_rho(1))
    assert str(exc.value) == "hardcap: " + meta["hardcap"]["message"]


def test_matsubara_zero_coefficient_reduces_to_k0():
    """K=1 with c_1 = 0 must reproduce K=0 (SURVEY 8(c) K>=1 row, item ii)."""
    import paper_1012_4382_b200 as xf
    from tests.cases import DIMER
    bath = xf.BathParams.from_timescale(20.0, 100.0, 77.0)
    nu, a, b = orc.bath_modes(bath, 0)
    p0 = orc.Problem(DIMER, bath, xf.MarkovRates.none(), 3, 0)
    p1 = orc.Problem(DIMER, bath, xf.MarkovRates.none(), 3, 1,
                     modes_override=(np.array([nu[0], 7.0]), np.array([a[0], 0.0]),
                                     np.array([b[0], 0.0])))
    cfg = xf.PropagationConfig(dt_fs=0.5, n_max=3, t_end_fs=200.0, residual=None)
    rho0 = np.diag([1.0, 0.0]).astype(complex)
    r0 = orc.propagate_from(DIMER, bath, xf.MarkovRates.none(), cfg, rho0, 0, problem=p0)
    r1 = orc.propagate_from(DIMER, bath, xf.MarkovRates.none(), cfg, rho0, 1, problem=p1)
    assert np.max(np.abs(r0["populations"] - r1["populations"])) < 1e-15


def test_long_eta_twin(golden_long):
    """Config 3 K=0 twin (300 K, N_max=6, residual 1e-5): 23,519 steps."""
    arrays, meta = golden_long
    m = meta["fmo_n6_eta"]
    assert m["stop_reason"] == "residual"
    assert abs(m["eta"] - 0.9761164832557473) < 1e-12
