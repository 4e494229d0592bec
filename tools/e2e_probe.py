"""Where the host time of one propagate() goes (config 4, 50 steps, a record
every step), phase by phase, after a warm-up call.  Experiment tool."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1012_4382_b200 as xf  # noqa: E402
from paper_1012_4382_b200 import heom  # noqa: E402
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
system = xf.build_fmo_system()
bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
cfg = xf.PropagationConfig(dt_fs=1.0, n_max=8, t_end_fs=steps * 1.0, residual=None, n_matsubara=1,
                           record_stride=1)
xf.propagate(system, bath, rates, cfg, 1)
for rep in range(3):
    t = [time.perf_counter()]
    traj = xf.propagate(system, bath, rates, cfg, 1)
    t.append(time.perf_counter())
    ops = BlockOperands(system, bath, rates, 1)
    t.append(time.perf_counter())
    run = DeviceRun(ops, 8, 1.0, t_end_fs=steps * 1.0, record_stride=1)
    t.append(time.perf_counter())
    rho0 = np.zeros((7, 7), complex)
    rho0[0, 0] = 1
    run.set_rho0(rho0, [0.0, 0.0])
    t.append(time.perf_counter())
    run.run()
    t.append(time.perf_counter())
    recs = run.records()
    t.append(time.perf_counter())
    run.close()
    t.append(time.perf_counter())
    ms = np.diff(t) * 1e3
    print(f"propagate {ms[0]:.2f} ms | ops {ms[1]:.2f} create {ms[2]:.2f} set_rho0 {ms[3]:.2f} "
          f"run {ms[4]:.2f} records {ms[5]:.2f} close {ms[6]:.2f}")
