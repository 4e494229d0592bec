"""Times the config-4 RK4 step (FMO 300 K, N_max=8, K=1) with the kernel knobs
of the environment (HB_FAST_VARIANT, HB_MM4_MINB, HB_BENCH_ORDER, ...) and prints
one JSON line: ms per step and per stage.  Experiment tool, not the bench.

    HB_FAST_VARIANT=7 HB_MM4_MINB=12 python tools/kernel_sweep.py [steps]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1012_4382_b200 as xf  # noqa: E402
from paper_1012_4382_b200.engine import BlockOperands, DeviceRun  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
n_max = int(os.environ.get("HB_SWEEP_NMAX", "8"))
K = int(os.environ.get("HB_SWEEP_K", "1"))
system = xf.build_fmo_system()
bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
ops = BlockOperands(system, bath, rates, K)
run = DeviceRun(ops, n_max, 1.0, t_end_fs=1e15, record_stride=10 ** 12, device=0,
                ordering=os.environ.get("HB_BENCH_ORDER", "reference"),
                precision=os.environ.get("HB_SWEEP_PREC", "double"))
rho0 = np.zeros((7, 7), complex)
rho0[0, 0] = 1.0
run.set_rho0(rho0, [0.0, 0.0])
run.time_steps(20)
ms = min(run.time_steps(steps) for _ in range(3)) / steps
st = np.min([run.time_steps(1, per_stage=True)[1] for _ in range(20)], axis=0)
n_tot = xf.hierarchy_size(ops.modes, n_max)
knobs = {k: v for k, v in os.environ.items() if k.startswith("HB_")}
print(json.dumps({"knobs": knobs, "n_ado": n_tot, "ms_per_step": round(ms, 5),
                  "ado_steps_per_s": n_tot / ms * 1e3,
                  "stage_us": [round(1e3 * x, 1) for x in st]}), flush=True)
run.close()
