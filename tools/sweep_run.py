"""Config 5 on one GPU: one GPU's share (8 points) of the 8 x 8 temperature x
lambda grid, N_max=6, K=1, residual 1e-5, with W concurrent handles.

    python tools/sweep_run.py [workers] [n_points] [precision]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1012_4382_b200 as xf  # noqa: E402
from paper_1012_4382_b200 import sweep  # noqa: E402

workers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prec = sys.argv[3] if len(sys.argv) > 3 else "double"
pts = sweep.temperature_lambda_grid()[::64 // npts][:npts]   # spread over the grid
cfg = sweep.sweep_config(n_max=6, n_matsubara=1, dt_fs=1.0, residual=1e-5, record_stride=100,
                         precision=prec)
rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
runner = sweep.fmo_point_runner(cfg, rates)
sweep.run_points(pts[:1], sweep.fmo_point_runner(
    sweep.sweep_config(n_max=6, n_matsubara=1, dt_fs=1.0, residual=None, t_end_fs=10.0,
                       precision=prec), rates), 1)  # warm
t0 = time.perf_counter()
res = sweep.run_points(pts, runner, workers)
wall = time.perf_counter() - t0
steps = sum(r.steps for r in res)
n_tot = xf.hierarchy_size(14, 6)
print(json.dumps({"workers": workers, "points": npts, "precision": prec, "wall_s": wall,
                  "total_steps": steps, "ado_steps_per_s": n_tot * steps / wall,
                  "eta": [round(r.efficiency, 6) for r in res],
                  "T_lam": [(r.point.temperature_k, r.point.lam_cm1) for r in res]}))
