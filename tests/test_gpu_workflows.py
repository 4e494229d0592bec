"""The callers of the propagator: auto_truncate against the
reference's own runs (tests/golden/auto_truncate.*, the cases of
test_heom.py:299-324) and one config-5 sweep point against the oracle."""
import json
import warnings

import numpy as np
import pytest

import paper_1012_4382_b200 as xf
from oracle import oracle as orc
from tests.cases import FMO, RATES, site_rho
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden_at():
    return np.load(GOLDEN / "auto_truncate.npz"), json.loads((GOLDEN / "auto_truncate.json").read_text())


@pytest.mark.parametrize("name", ["pairwise", "zero_coupling", "fmo35_tol"])
@pytest.mark.parametrize("speculate", [True, False])
def test_auto_truncate_matches_reference(golden_at, name, speculate):
    arrays, meta = golden_at
    m = meta[f"at_{name}"]
    lam, gamma_inv, temp = m["bath"]
    bath = xf.BathParams.from_timescale(lam, gamma_inv, temp)
    cfg = xf.PropagationConfig(**m["config"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        n, traj = xf.auto_truncate(FMO, bath, RATES, cfg, 1, speculate=speculate, **m["kwargs"])
        for k, t_ref in m["trapping_times"].items():
            t = xf.trapping_time(xf.propagate(FMO, bath, RATES,
                                              xf.PropagationConfig(**{**m["config"], "n_max": int(k)}), 1))
            assert abs(t - t_ref) < 1e-8, (k, t, t_ref)
    assert n == m["n"]
    assert traj.stop_reason == m["stop_reason"]
    assert np.array_equal(traj.times_fs, arrays[f"at_{name}_times"])
    assert np.max(np.abs(traj.populations - arrays[f"at_{name}_pops"])) < 1e-10


def test_auto_truncate_cap_failure(golden_at):
    _, meta = golden_at
    cfg = xf.PropagationConfig(dt_fs=5.0, n_max=0, t_end_fs=500.0, residual=None)
    with pytest.raises(xf.ConvergenceFailure) as exc:
        xf.auto_truncate(FMO, xf.BathParams.from_timescale(35.0, 166.0, 300.0), RATES, cfg, 1,
                         tol_ps=1e-12, start_n=0, n_cap=2)
    assert str(exc.value) == meta["cap_failure_message"]


@pytest.mark.slow
def test_sweep_point_matches_oracle():
    """One point of the config-5 grid (T = 300 K, lambda = 35 cm^-1, K = 1,
    residual 1e-5) through the sweep worker, against the oracle; N_max = 2 so
    the oracle finishes in seconds (the sweep itself runs N_max = 6)."""
    from paper_1012_4382_b200 import sweep
    cfg = sweep.sweep_config(n_max=2, n_matsubara=1, dt_fs=2.5, residual=1e-5, record_stride=100)
    pt = sweep.SweepPoint(temperature_k=300.0, lam_cm1=35.0)
    res = sweep.fmo_point_runner(cfg, RATES)(pt)
    bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
    ref = orc.propagate_from(FMO, bath, RATES, cfg, site_rho(1))
    assert res.stop_reason == "residual" == ref["stop_reason"]
    assert res.steps == ref["n_steps"]
    assert abs(res.efficiency - ref["populations"][-1, 8]) < 1e-10
