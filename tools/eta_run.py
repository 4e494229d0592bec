"""Config 3 (BASELINE.json configs[2]): FMO + trap at 300 K, residual 1e-5
policy, transfer efficiency eta, timed end to end through propagate().

    python tools/eta_run.py [n_max] [K] [dt_fs] [precision]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1012_4382_b200 as xf  # noqa: E402

n_max = int(sys.argv[1]) if len(sys.argv) > 1 else 6
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dt = float(sys.argv[3]) if len(sys.argv) > 3 else 1.25
prec = sys.argv[4] if len(sys.argv) > 4 else "double"
system = xf.build_fmo_system()
bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
cfg = xf.PropagationConfig(dt_fs=dt, n_max=n_max, residual=1e-5, record_stride=100,
                           n_matsubara=K, precision=prec, device=0)
xf.propagate(system, bath, rates, xf.PropagationConfig(dt_fs=dt, n_max=n_max, t_end_fs=10 * dt,
                                                       residual=None, n_matsubara=K,
                                                       precision=prec), 1)  # warm
t0 = time.perf_counter()
traj = xf.propagate(system, bath, rates, cfg, 1)
wall = time.perf_counter() - t0
n_tot = xf.hierarchy_size(7 * (K + 1), n_max)
steps = int(round(traj.times_fs[-1] / dt))
print(json.dumps({"n_max": n_max, "K": K, "dt_fs": dt, "precision": prec, "n_ado": n_tot,
                  "eta": xf.efficiency(traj), "trapping_time_ps": xf.trapping_time(traj),
                  "steps": steps, "t_stop_fs": float(traj.times_fs[-1]), "wall_s": wall,
                  "us_per_step": 1e6 * wall / steps, "ado_steps_per_s": n_tot * steps / wall}))
