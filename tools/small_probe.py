"""A few hundred steps of the config-3 eta twin (FMO 300 K, N_max = 6, K = 0,
1,716 ADOs) or its K = 1 hierarchy, for launch lists / timing of small grids.
    python tools/small_probe.py [K] [steps] [chunk]"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1012_4382_b200 as xf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kernel = sys.argv[4] if len(sys.argv) > 4 else "auto"
dt = 2.5 if K == 0 else 1.25
system = xf.build_fmo_system()
bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
n_max = int(os.environ.get("HB_PROBE_NMAX", "6"))
cfg = xf.PropagationConfig(dt_fs=dt, n_max=n_max, t_end_fs=steps * dt, residual=None, n_matsubara=K,
                           record_stride=100, chunk_steps=chunk, kernel=kernel)
xf.propagate(system, bath, rates, cfg, 1)
t0 = time.perf_counter()
xf.propagate(system, bath, rates, cfg, 1)
w = time.perf_counter() - t0
print(f"K={K} N_max={n_max} {steps} steps kernel={kernel}: {1e6 * w / steps:.1f} us/step (end to end)")

# the same steps launched one kernel at a time (hb_time_steps: no CUDA graph), for ncu
import numpy as np  # noqa: E402
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun  # noqa: E402
ops = BlockOperands(system, bath, rates, K)
with DeviceRun(ops, n_max, dt, t_end_fs=1e12, record_stride=10 ** 9, kernel=kernel) as run:
    rho0 = np.zeros((7, 7), complex)
    rho0[0, 0] = 1.0
    run.set_rho0(rho0, [0.0, 0.0])
    run.time_steps(10)
    ms = run.time_steps(steps)
print(f"K={K} N_max={n_max} {steps} steps, stream launches: {1e3 * ms / steps:.1f} us/step (device)")
