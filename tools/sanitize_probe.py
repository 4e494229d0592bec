"""Small runs for compute-sanitizer (memcheck / racecheck / synccheck): FMO with
trap at N_max = 2, K = 0 and 1, through propagate (CUDA-graph WHILE path), the
stream-launched steps (hb_time_steps), the whole-state entry point, the float
path and two in-process shards.  tools/sanitize.sh runs it under each tool."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import paper_1012_4382_b200 as xf  # noqa: E402
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun  # noqa: E402
from paper_1012_4382_b200.shard import ShardedRun  # noqa: E402

system = xf.build_fmo_system()
bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
rho0 = np.zeros((7, 7), complex)
rho0[0, 0] = 1.0
for K in (0, 1):
    cfg = xf.PropagationConfig(dt_fs=1.0, n_max=2, t_end_fs=30.0, residual=None, n_matsubara=K,
                               record_stride=3)
    t = xf.propagate(system, bath, rates, cfg, 1)
    ops = BlockOperands(system, bath, rates, K)
    n_tot = xf.hierarchy_size(ops.modes, 2)
    for prec in ("double", "single"):
        with DeviceRun(ops, 2, 1.0, t_end_fs=1e9, record_stride=10 ** 6, precision=prec) as run:
            run.set_rho0(rho0, [0.0, 0.0])
            run.time_steps(26)
            sig, _ = run.state(n_tot)
        with DeviceRun(ops, 2, 1.0, t_end_fs=10.0, record_stride=1, precision=prec) as run:
            run.set_state(sig, [0.0, 0.0])
            run.run()
    sr = ShardedRun(ops, 2, 1.0, 30.0, 2)
    sr.set_rho0(rho0, [0.0, 0.0])
    sr.run()
    sr.close()
    g = xf.enumerate_hierarchy(ops.modes, 2)
    print(f"K={K}: final p_site1 {t.populations[-1, 1]:.6f}, {n_tot} ADOs, ok")
