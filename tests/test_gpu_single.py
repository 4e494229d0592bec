"""precision='single' (heom.py:74, 93-94): float32 state and right-hand sides on
the device, float64 sinks/records/stop policy.  Checked against the reference's
own single-precision runs (tests/golden/traj_single.npz, made by
tests/golden/make_golden.py --single) and against its single-vs-double bound
(5e-7, test_heom.py:353-360 and test_acceptance.py:231-238)."""
import json

import numpy as np
import pytest

import paper_1012_4382_b200 as xf
from tests.cases import BATH300, BATH77, FMO, RATES, nonherm_rho0
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

SINGLE_CASES = {
    "smoke_n4": (BATH300, dict(dt_fs=10.0, n_max=4, t_end_fs=1000.0, residual=None,
                               record_stride=10)),
    "fmo_n4_77k": (BATH77, dict(dt_fs=2.5, n_max=4, t_end_fs=1000.0, residual=None,
                                record_stride=20)),
    "fmo_n2_eta": (BATH300, dict(dt_fs=5.0, n_max=2, residual=1e-3, record_stride=20)),
}


@pytest.fixture(scope="module")
def golden_single():
    return (np.load(GOLDEN / "traj_single.npz"),
            json.loads((GOLDEN / "traj_single.json").read_text()))


@pytest.mark.parametrize("name", list(SINGLE_CASES))
def test_single_matches_reference_single(golden_single, name):
    arrays, meta = golden_single
    bath, kw = SINGLE_CASES[name]
    traj = xf.propagate(FMO, bath, RATES, xf.PropagationConfig(precision="single", **kw), 1)
    ref_s, ref_d = arrays[name + "_single_pops"], arrays[name + "_double_pops"]
    assert traj.stop_reason == meta[name + "_single"]["stop_reason"]
    assert np.array_equal(traj.times_fs, arrays[name + "_single_times"])
    # the reference's criterion is single vs double < 5e-7 (test_heom.py:360);
    # two float32 runs with different rounding (the reference promotes its
    # float64 scalars, integrates the sinks in float32) agree to a few 1e-7
    err_d = np.max(np.abs(traj.populations - ref_d))
    err_s = np.max(np.abs(traj.populations - ref_s))
    assert err_d < 5e-7, (err_d, err_s)
    assert err_s < 3e-6, (err_d, err_s)


def test_single_vs_double_smoke():
    """test_heom.py:353-360 on the device."""
    kw = dict(dt_fs=10.0, n_max=4, t_end_fs=1000.0, residual=None, record_stride=10)
    d = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(**kw), 1).populations
    s = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(precision="single", **kw),
                     1).populations
    assert np.max(np.abs(d - s)) < 5e-7


def test_single_vs_double_criterion_10():
    """test_acceptance.py:231-238: N_max = 12 (50,388 ADOs), 10 ps."""
    kw = dict(dt_fs=10.0, n_max=12, t_end_fs=10000.0, residual=None, record_stride=10)
    d = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(**kw), 1).populations
    s = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(precision="single", **kw),
                     1).populations
    assert np.max(np.abs(d - s)) < 5e-7


@pytest.mark.parametrize("ordering", ["lex", "reference"])
def test_single_matsubara_k1(ordering):
    kw = dict(dt_fs=2.5, n_max=4, t_end_fs=500.0, residual=None, record_stride=10,
              n_matsubara=1, ordering=ordering)
    d = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(**kw), 1).populations
    s = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(precision="single", **kw),
                     1).populations
    assert np.max(np.abs(d - s)) < 5e-7


def test_single_final_state_is_float32_rounded():
    """the device state holds float32: sigma^0 read back is float32-representable"""
    kw = dict(dt_fs=2.5, n_max=2, t_end_fs=100.0, residual=None)
    traj = xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(precision="single", **kw), 1)
    blk = traj.final_rho[1:8, 1:8]
    assert np.array_equal(blk.real.astype(np.float32).astype(np.float64), blk.real)


def test_single_unsupported_shapes_raise():
    kw = dict(dt_fs=2.5, n_max=2, t_end_fs=100.0, residual=None, precision="single")
    with pytest.raises(ValueError, match="single"):
        xf.propagate_from(FMO, BATH300, RATES, xf.PropagationConfig(**kw), nonherm_rho0())
    with pytest.raises(ValueError, match="single"):
        xf.propagate(FMO, BATH300, RATES, xf.PropagationConfig(kernel="generic", **kw), 1)
