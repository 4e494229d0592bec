"""Host-side logic (no GPU): API types and validation, operand preparation, the
C-ABI library surface, observables.  Mirrors the reference's test_model /
test_observables / the host parts of test_heom."""
import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1012_4382_b200 as xf
from oracle import oracle as orc
from paper_1012_4382_b200 import _native as N
from paper_1012_4382_b200.engine import BlockOperands, bath_coefficients, bath_modes
from paper_1012_4382_b200.hierarchy import GradedLookup
from paper_1012_4382_b200.units import ANGFREQ_RAD_FS
from tests.cases import BATH300, DIMER, FMO, RATES, TWO_LEVEL

ROOT = Path(__file__).resolve().parents[1]


# ------------------------------------------------------------ C-ABI surface

def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "heom_b200.h").read_text()
    declared = set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", header))
    assert declared == set(N.EXPORTS)
    lib = N.lib()
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.hb_hierarchy_size(14, 8) == 319770
    assert lib.hb_hierarchy_size(7, 4) == 330


def test_no_gpu_fails_loudly():
    if N.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(N.NativeError):
        xf.enumerate_hierarchy(7, 2)
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=1, t_end_fs=10.0, residual=None)
    with pytest.raises(N.NativeError):
        xf.propagate(FMO, BATH300, RATES, cfg, 1)


def test_argument_errors_without_device():
    idx = np.zeros(1, np.int32)
    rc = N.lib().hb_graph_build(0, 4, 0, N.ptr(idx), N.ptr(idx), N.ptr(idx), N.ptr(idx), None)
    assert rc == N.HB_ERR_ARG and "at least one site" in N.last_error()
    rc = N.lib().hb_graph_build(64, 64, 0, N.ptr(idx), N.ptr(idx), N.ptr(idx), N.ptr(idx), None)
    assert rc == N.HB_ERR_RANGE and "exceeds the supported index range" in N.last_error()


# ------------------------------------------------------------ API types

def test_config_validation_messages():
    with pytest.raises(ValueError, match="dt must be > 0"):
        xf.PropagationConfig(dt_fs=0.0)
    with pytest.raises(ValueError, match="stop policy"):
        xf.PropagationConfig(t_end_fs=None, residual=None)
    with pytest.raises(ValueError, match="record stride"):
        xf.PropagationConfig(record_stride=0)
    with pytest.raises(ValueError, match="precision"):
        xf.PropagationConfig(precision="half")
    with pytest.raises(ValueError, match="n_matsubara"):
        xf.PropagationConfig(n_matsubara=-1)
    cfg = xf.PropagationConfig()
    assert (cfg.dt_fs, cfg.n_max, cfg.residual, cfg.hard_cap_fs, cfg.blowup_norm) == \
        (2.5, 8, 1e-5, 200_000.0, 1e6)
    assert cfg.n_matsubara == 0 and cfg.dtype == np.complex128


def test_model_types():
    assert FMO.dimension == 9 and FMO.site_count == 7
    assert FMO.h_cm1[1, 2] == -87.7 and FMO.h_cm1[3, 3] == 12210.0
    shifted = xf.build_fmo_system(delta_e_cm1=10.0)
    assert shifted.h_cm1[3, 3] == 12220.0 and shifted.h_cm1[4, 4] == 12330.0
    with pytest.raises(ValueError):
        xf.ExcitonSystem(h_cm1=np.array([[0.0, 1.0], [2.0, 0.0]]), site_indices=(0, 1))
    with pytest.raises(ValueError):
        xf.BathParams(lam_cm1=-1.0, gamma_fs1=0.01, temperature_k=300.0)
    with pytest.raises(ValueError):
        xf.MarkovRates(-1.0, 0.0)
    r = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    assert r.gamma_rc_fs1 == 1.0 / 2500.0 and r.gamma_phot_fs1 == 1.0 / 250000.0
    g = xf.gibbs_state(FMO, 300.0)
    assert abs(np.trace(g) - 1.0) < 1e-12 and np.allclose(g, g.T)
    assert xf.spectral_density(0.0, BATH300) == 0.0


def test_units_match_reference_constants():
    assert ANGFREQ_RAD_FS == 2.0 * math.pi * 2.99792458e-5
    assert xf.units.KB_CM1_PER_K == 0.695035


def test_bath_coefficients_and_modes():
    a, b = bath_coefficients(BATH300)
    assert a == pytest.approx(2.0 * 35.0 * 0.695035 * 300.0 * ANGFREQ_RAD_FS ** 2)
    assert b == pytest.approx(35.0 * ANGFREQ_RAD_FS / 166.0)
    nu, aa, bb = bath_modes(BATH300, 0)
    assert (nu[0], aa[0], bb[0]) == (BATH300.gamma_fs1, a, b)   # K=0 is the reference, bitwise
    nu1, a1, b1 = bath_modes(BATH300, 1)
    onu, oa, ob = orc.bath_modes(BATH300, 1)
    assert np.array_equal(nu1, onu) and np.array_equal(a1, oa) and np.array_equal(b1, ob)
    # Matsubara frequency and the high-temperature limit of a_0
    assert nu1[1] == pytest.approx(2 * math.pi * 0.695035 * 300.0 * ANGFREQ_RAD_FS)
    assert a1[0] == pytest.approx(a, rel=5e-3)


def test_block_operands_match_oracle_restatement():
    for system, rates in ((FMO, RATES), (FMO, xf.MarkovRates.none()), (DIMER, xf.MarkovRates.none()),
                          (TWO_LEVEL, xf.MarkovRates.none())):
        ops = BlockOperands(system, BATH300, rates)
        ref = orc.block_operands(system, rates)
        assert ops.block == ref["block"] and ops.sinks == ref["sinks"]
        assert np.array_equal(ops.h_block, ref["h"])
        assert np.array_equal(ops.site_of, ref["site_of"])
        assert np.array_equal(ops.decay, ref["decay"])
        assert ops.sink_terms == ref["sink_terms"]


def test_sinks_must_be_decoupled():
    h = np.array(FMO.h_cm1)
    h[0, 1] = h[1, 0] = 1.0
    bad = xf.ExcitonSystem(h_cm1=h, site_indices=tuple(range(1, 8)), ground_index=0, rc_index=8,
                           trap_sites=(3, 4))
    with pytest.raises(ValueError, match="decoupled"):
        BlockOperands(bad, BATH300, RATES)


def test_lindblad_and_backaction_values():
    # reference test_heom.py:27-100
    rho = np.zeros((9, 9), complex)
    rho[3, 3] = 1.0
    out = xf.lindblad_markov(rho, FMO, RATES)
    gp, grc = RATES.gamma_phot_fs1, RATES.gamma_rc_fs1
    assert out[3, 3] == pytest.approx(-(gp + grc), rel=1e-14)
    assert out[8, 8] == pytest.approx(grc) and out[0, 0] == pytest.approx(gp)
    rng = np.random.default_rng(3)
    sigma = rng.standard_normal((9, 9)) + 1j * rng.standard_normal((9, 9))
    a, b = bath_coefficients(BATH300)
    for site in (1, 4, 7):
        proj = np.zeros((9, 9))
        proj[site, site] = 1.0
        oracle = 1j * a * (proj @ sigma - sigma @ proj) + b * (proj @ sigma + sigma @ proj)
        assert np.max(np.abs(xf.bath_backaction(FMO, site, sigma, BATH300) - oracle)) < 1e-15


# ------------------------------------------------------------ hierarchy host logic

def test_graded_lookup_matches_reference_tables(golden_tables):
    for key in ("M7_N4", "M4_N5", "M14_N3", "M1_N20"):
        m, n = (int(x[1:]) for x in key.split("_"))
        ind = golden_tables[f"{key}_indices"]
        lk = GradedLookup(m, n, ind)
        assert [lk[tuple(r)] for r in ind] == list(range(len(ind)))
        assert len(lk) == len(ind)
    lk = GradedLookup(7, 2, golden_tables["M7_N2_indices"])
    with pytest.raises(KeyError):
        lk[(3, 0, 0, 0, 0, 0, 0)]
    assert (1, 1, 0, 0, 0, 0, 0) in lk and (3, 0, 0, 0, 0, 0, 0) not in lk


def test_hierarchy_size():
    assert [xf.hierarchy_size(7, n) for n in (4, 6, 8, 10, 12, 16)] == \
        [330, 1716, 6435, 19448, 50388, 245157]
    assert xf.hierarchy_size(14, 8) == 319770


# ------------------------------------------------------------ observables (test_observables.py)

def _traj(t, p):
    pops = np.zeros((len(t), 9))
    pops[:, 8] = p
    pops[:, 0] = 1.0 - p
    return xf.Trajectory(times_fs=np.asarray(t, float), populations=pops,
                         site_indices=tuple(range(1, 8)), ground_index=0, rc_index=8,
                         stop_reason="t_end", final_rho=np.diag(pops[-1]).astype(complex))


def test_trapping_time_analytic():
    tau = 2500.0
    t = np.arange(0.0, 30000.0 + 1e-9, 2.5)
    traj = _traj(t, 1.0 - np.exp(-t / tau))
    expected = (tau - (t[-1] + tau) * np.exp(-t[-1] / tau)) / 1000.0
    assert xf.trapping_time(traj) == pytest.approx(expected, rel=1e-4)
    assert abs(xf.trapping_time(traj, "derivative") - xf.trapping_time(traj, "parts")) < 0.01
    assert xf.efficiency(traj) == pytest.approx(1.0 - np.exp(-t[-1] / tau))
    assert xf.thermal_deviation(np.eye(7) / 7.0, np.diag([1.0] + [0.0] * 6)) == pytest.approx(6 / 7)
