"""Shared problem definitions of the parity suite (mirrors tests/golden/make_golden.py)."""
import numpy as np

import paper_1012_4382_b200 as xf

FMO = xf.build_fmo_system()
RATES = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
BATH300 = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
BATH77 = xf.BathParams.from_timescale(35.0, 166.0, 77.0)
DIMER = xf.ExcitonSystem(h_cm1=np.array([[100.0, 60.0], [60.0, 0.0]]), site_indices=(0, 1))
TWO_LEVEL = xf.ExcitonSystem(h_cm1=np.array([[0.0, 0.0], [0.0, 200.0]]), site_indices=(1,))


def site_rho(i, d=9):
    r = np.zeros((d, d), complex)
    r[i, i] = 1.0
    return r


def nonherm_rho0():
    rho0 = np.zeros((9, 9), dtype=complex)
    rho0[1, 1] = 0.6
    rho0[2, 2] = 0.4
    rho0[1, 2] = 0.3 + 1e-13j
    rho0[2, 1] = 0.3
    return rho0


# name -> (system, bath, rates, config kwargs, rho0)
TRAJ_CASES = {
    "dimer_n4_77k": (DIMER, xf.BathParams.from_timescale(20.0, 100.0, 77.0), xf.MarkovRates.none(),
                     dict(dt_fs=0.5, n_max=4, t_end_fs=1000.0, residual=None, record_stride=20),
                     np.diag([1.0, 0.0]).astype(complex)),
    "fmo_n4_77k": (FMO, BATH77, RATES,
                   dict(dt_fs=2.5, n_max=4, t_end_fs=1000.0, residual=None, record_stride=1),
                   site_rho(1)),
    "fmo_n2_300k": (FMO, BATH300, RATES,
                    dict(dt_fs=2.5, n_max=2, t_end_fs=1000.0, residual=None, record_stride=1),
                    site_rho(1)),
    "fmo_n4_300k_mats": (FMO, BATH300, RATES,
                         dict(dt_fs=2.5, n_max=4, t_end_fs=1000.0, residual=None,
                              record_matrices=True, record_stride=40), site_rho(1)),
    "fmo_n2_eta": (FMO, BATH300, RATES, dict(dt_fs=5.0, n_max=2, residual=1e-5, record_stride=20),
                   site_rho(1)),
    "fmo_n1_eta_site6": (FMO, BATH300, RATES,
                         dict(dt_fs=5.0, n_max=1, residual=1e-5, record_stride=7), site_rho(6)),
    "dephasing_n20": (TWO_LEVEL, xf.BathParams.from_timescale(5.0, 100.0, 300.0),
                      xf.MarkovRates.none(),
                      dict(dt_fs=0.25, n_max=20, t_end_fs=500.0, residual=None, record_stride=20,
                           record_matrices=True), np.full((2, 2), 0.5, complex)),
    "fmo_n0": (FMO, BATH300, RATES, dict(dt_fs=1.0, n_max=0, t_end_fs=200.0, residual=None),
               site_rho(1)),
    "fmo_n2_nonherm": (FMO, BATH300, RATES,
                       dict(dt_fs=2.5, n_max=2, t_end_fs=250.0, residual=None,
                            record_matrices=True, record_stride=10), nonherm_rho0()),
}
