"""End-to-end propagate() time against the CUDA-graph body size (chunk_steps):
config 4 for 1,000 steps with a record every step, the config-3 K=0 eta twin,
and the device-timed step of config 4 for comparison.  Experiment tool."""
import sys
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import paper_1012_4382_b200 as xf  # noqa: E402
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun  # noqa: E402

system = xf.build_fmo_system()
bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
ops = BlockOperands(system, bath, rates, 1)
rho0 = np.zeros((7, 7), complex)
rho0[0, 0] = 1.0
with DeviceRun(ops, 8, 1.0, t_end_fs=1e15, record_stride=10 ** 12) as run:
    run.set_rho0(rho0, [0.0, 0.0])
    run.time_steps(10)
    ms = run.time_steps(1000)
print(f"device time_steps(1000): {ms:.1f} ms ({ms:.3f} us/step x1000)")
for chunk in [int(c) for c in (sys.argv[1:] or [1, 2, 4, 8, 16, 64])]:
    for stride, steps in ((1, 1000), (1000, 1000)):
        cfg = xf.PropagationConfig(dt_fs=1.0, n_max=8, t_end_fs=float(steps), residual=None,
                                   n_matsubara=1, record_stride=stride, chunk_steps=chunk)
        xf.propagate(system, bath, rates, cfg, 1)
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            xf.propagate(system, bath, rates, cfg, 1)
            best = min(best, time.perf_counter() - t0)
        print(f"chunk {chunk:3d} config4 {steps} steps stride {stride:4d}: {1e3 * best:.1f} ms "
              f"({best / ms * 1e3:.3f} x device)")
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=6, residual=1e-5, record_stride=100, chunk_steps=chunk)
    xf.propagate(system, bath, rates, replace(cfg, residual=None, t_end_fs=25.0), 1)
    t0 = time.perf_counter()
    tr = xf.propagate(system, bath, rates, cfg, 1)
    w = time.perf_counter() - t0
    print(f"chunk {chunk:3d} eta twin K0 N6: {w:.3f} s, {1e6 * w / 23519:.1f} us/step, eta {xf.efficiency(tr):.15f}")
