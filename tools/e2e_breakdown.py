"""Where the end-to-end propagate() time of config 4 goes (create, set_rho0,
run, records, close), against the device-timed steps.  Experiment tool."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1012_4382_b200 as xf  # noqa: E402
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun  # noqa: E402

system = xf.build_fmo_system()
bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
steps = 1000
cfg = xf.PropagationConfig(dt_fs=1.0, n_max=8, t_end_fs=float(steps), residual=None,
                           n_matsubara=1, record_stride=1)
xf.propagate(system, bath, rates, cfg, 1)
for _ in range(3):
    t0 = time.perf_counter()
    xf.propagate(system, bath, rates, cfg, 1)
    print("propagate", round(time.perf_counter() - t0, 4))
ops = BlockOperands(system, bath, rates, 1)
rho0 = np.zeros((7, 7), complex)
rho0[0, 0] = 1.0
for _ in range(2):
    t = [time.perf_counter()]
    run = DeviceRun(ops, 8, 1.0, t_end_fs=float(steps), record_stride=1)
    t.append(time.perf_counter())
    run.set_rho0(rho0, [0.0, 0.0])
    t.append(time.perf_counter())
    run.run()
    t.append(time.perf_counter())
    run.records()
    run.sigma0()
    t.append(time.perf_counter())
    run.close()
    t.append(time.perf_counter())
    print("create/set_rho0/run/records/close ms", [round(1e3 * (b - a), 2) for a, b in zip(t, t[1:])])
