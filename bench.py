"""Benchmark: FP64 HEOM RK4 throughput (ADO-RK4-steps/s) on B200.

Workload (BASELINE.json configs[3], the north_star target, one GPU):
7-site FMO (Adolphs-Renger H), 300 K, lambda = 35 cm^-1, gamma^-1 = 166 fs,
Gamma_RC^-1 = 2.5 ps, Gamma_phot^-1 = 250 ps, N_max = 8, K = 1 Matsubara term
(M = 14 modes, 319,770 ADOs), dt = 1 fs, rho0 = |1><1|.  One bench step = one
classical RK4 step of the whole hierarchy (4 fused stage kernels).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints ONE JSON line (rank 0).  Under torchrun (N > 1) every rank propagates its
own full hierarchy (replicas, weak scaling); ranks are timed with CUDA events
and the max over ranks is reported.
``--impl reference`` times the CPU port of the reference path (oracle/, C +
OpenMP over all host cores) on the same workload; the reference itself
(Python + numba) cannot travel to the GPU box.
"""

from __future__ import annotations

import argparse
from dataclasses import replace
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ADO-RK4-steps/sec (FP64)"
UNIT = "ADO-steps/s"
N_MAX, K_MATS, DT = 8, 1, 1.0
D = 7
S_PACKED = 8 * D * D                      # bytes per Hermitian-packed ADO (392 B)
B_ALG_STEP = 12 * S_PACKED                # algorithmic state bytes per ADO-step
B_ALG_STAGE = {1: 2 * S_PACKED, 2: 4 * S_PACKED, 3: 3 * S_PACKED, 4: 3 * S_PACKED}
SURVEY_B_ALG = 16 * 16 * D * D            # SURVEY 8(d) unpacked-scheme figure, 12,544 B
B_ALG_SINGLE = 15 * 4 * D * D             # precision='single': 15 float passes


def workload():
    import paper_1012_4382_b200 as xf
    system = xf.build_fmo_system()
    bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
    rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    return xf, system, bath, rates


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, local, backend):
    if world <= 1:
        return None
    import torch
    import torch.distributed as dist
    if backend == "nccl":
        torch.cuda.set_device(local)
    dist.init_process_group(backend=backend)
    return dist


def barrier(dist, local=0):
    if dist is None:
        return
    import torch
    if dist.get_backend() == "nccl":
        dist.barrier(device_ids=[local])
    else:
        dist.barrier()


def allmax(dist, value, device):
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.file, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=10)
        self.file.flush()
        rows = []
        for line in Path(self.file.name).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.file.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


class CpuBaseline:
    """The C oracle (port of the reference path) on this host's cores, timed on a
    bounded sample of the same workload (whole-hierarchy RK4 steps)."""

    def __init__(self, xf, system, bath, rates, threads=None):
        from oracle import oracle as orc
        self.orc, self.xf = orc, xf
        self.system, self.bath, self.rates = system, bath, rates
        self.threads = threads or os.cpu_count() or 1
        orc.set_threads(self.threads)
        self.pb = orc.Problem(system, bath, rates, N_MAX, K_MATS)
        self.rho0 = np.zeros((9, 9), complex)
        self.rho0[1, 1] = 1.0

    def measure(self, budget_s):
        steps, wall, n = 0, 0.0, 1
        while wall < budget_s and steps < 10_000:
            cfg = self.xf.PropagationConfig(dt_fs=DT, n_max=N_MAX, t_end_fs=n * DT, residual=None,
                                            n_matsubara=K_MATS, record_stride=n)
            t0 = time.perf_counter()
            self.orc.propagate_from(self.system, self.bath, self.rates, cfg, self.rho0,
                                    problem=self.pb)
            dt = time.perf_counter() - t0
            steps += n
            wall += dt
            if dt < budget_s / 8:
                n *= 2
        value = self.pb.n_tot * steps / wall
        return {"value": value, "unit": UNIT, "cores": self.threads, "kind": "port",
                "sample": f"{steps} RK4 steps of the full N_max=8 K=1 hierarchy "
                          f"({self.pb.n_tot} ADOs), {wall:.1f} s wall, oracle/heom_oracle.c "
                          f"OpenMP x{self.threads}"}


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    xf, system, bath, rates = workload()
    budget = float(os.environ.get("HB_REF_BUDGET_S", "20"))
    base = CpuBaseline(xf, system, bath, rates)
    per_step = []
    cb = None
    for _ in range(args.warmup + args.steps):
        cb = base.measure(budget / max(1, args.steps + args.warmup))
        per_step.append(cb["value"])
    value = statistics.median(per_step[args.warmup:]) if args.steps else per_step[-1]
    n_tot = xf.hierarchy_size(14, N_MAX)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n_tot / value,
        "higher_is_better": True, "scaling": "none", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(world),
        "cpu_baseline": {**cb, "value": value},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(world):
    return {"workload": "FMO 300K N_max=8 K=1 (319770 ADOs), RK4 dt=1fs, one step = whole hierarchy",
            "n_max": N_MAX, "n_matsubara": K_MATS, "n_ado": 319770, "dt_fs": DT,
            "layout": "hermitian-packed AoSoA, tier-major ADO order (the reference's)",
            "l2": "inputs larger than L2 (4 x 125 MB state buffers)",
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}


def run_sharded(args, dist, world, rank, local):
    """--shard: config 4 split across the ranks (strong scaling), NCCL halo
    exchange after every stage (paper_1012_4382_b200/shard.py)."""
    import torch
    xf, system, bath, rates = workload()
    from paper_1012_4382_b200.engine import BlockOperands
    from paper_1012_4382_b200.shard import NcclShardedRun
    ops = BlockOperands(system, bath, rates, K_MATS)
    n_tot = xf.hierarchy_size(ops.modes, N_MAX)
    sr = NcclShardedRun(ops, N_MAX, DT, 1e15, rank, world, local, dist)
    rho0 = np.zeros((D, D), complex)
    rho0[0, 0] = 1.0
    sr.set_rho0(rho0, [0.0, 0.0])
    for _ in range(max(3, args.warmup)):
        sr.enqueue_step()
    sr.sync()
    launches0 = N_launch(sr.run_)
    barrier(dist, local)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sr.enqueue_step()
    status, _ = sr.sync()
    wall = time.perf_counter() - t0
    wall = allmax(dist, wall, f"cuda:{local}")
    halo = sr.plan.halo_tiles(rank)
    halo_bytes = sr.cross_plan.bytes_per_stage(rank) if sr.cross_plan is not None else None
    launches = N_launch(sr.run_) - launches0
    sr.close()
    if rank == 0:
        line = {"metric": METRIC, "value": n_tot * args.steps / wall, "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {**config_dict(world),
                           "parallelism": f"sharded x{world} (NCCL compressed cross halos)",
                           "halo_tiles_rank0": halo,
                           "halo_bytes_per_stage_rank0": halo_bytes},
                "gpu_launches": int(launches),
                "status": status}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def N_launch(run):
    return run.launch_count()


def run_b200(args):
    world, rank, local = dist_env()
    import torch
    dist = init_dist(world, local, "nccl" if torch.cuda.is_available() else "gloo")
    if args.shard and world > 1:
        return run_sharded(args, dist, world, rank, local)
    device = local
    xf, system, bath, rates = workload()
    from paper_1012_4382_b200.engine import BlockOperands, DeviceRun
    ops = BlockOperands(system, bath, rates, K_MATS)
    n_tot = xf.hierarchy_size(ops.modes, N_MAX)
    # HB_BENCH_ORDER (experiments): device ADO order of the timed run ('reference' default)
    run = DeviceRun(ops, N_MAX, DT, t_end_fs=1e15, record_stride=10 ** 12, device=device,
                    ordering=os.environ.get("HB_BENCH_ORDER", "reference"))
    rho0 = np.zeros((D, D), complex)
    rho0[0, 0] = 1.0
    run.set_rho0(rho0, [0.0, 0.0])
    torch.cuda.set_device(device)
    run.time_steps(max(3, args.warmup))               # warm-up (untimed)
    launches0 = run.launch_count()
    clocks = ClockSampler(device)
    time.sleep(1.0)                                   # let nvidia-smi start sampling
    barrier(dist, local)
    torch.cuda.synchronize()
    ms = run.time_steps(args.steps)                   # CUDA events on the handle's stream
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier(dist, local)
    launches = run.launch_count() - launches0
    ms_max = allmax(dist, ms, f"cuda:{device}")
    value = n_tot * args.steps * world / (ms_max / 1e3)

    # per-stage kernel durations (events around single launches, same stream)
    _, stage_ms = run.time_steps(1, per_stage=True)
    step_kernel_ms = float(np.sum(stage_ms))
    achieved = n_tot * B_ALG_STEP / (step_kernel_ms / 1e3) / 1e9
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    run.close()

    # same workload with precision='single' (heom.py:74; float32 state, 2,352 B per
    # ADO-step): reported beside the FP64 headline, not instead of it
    single = None
    try:
        run_s = DeviceRun(ops, N_MAX, DT, t_end_fs=1e15, record_stride=10 ** 12, device=device,
                          precision="single")
        run_s.set_rho0(rho0, [0.0, 0.0])
        run_s.time_steps(max(3, args.warmup))
        ms_s = run_s.time_steps(args.steps)
        _, st_s = run_s.time_steps(1, per_stage=True)
        run_s.close()
        single = {"value": n_tot * args.steps / (ms_s / 1e3), "unit": UNIT,
                  "ms_per_step": ms_s / args.steps, "dtype": "f32",
                  "stage_us": [round(1e3 * x, 2) for x in st_s],
                  "bytes_per_ado_step": B_ALG_SINGLE,
                  "achieved_GBps": n_tot * B_ALG_SINGLE / (float(np.sum(st_s)) / 1e3) / 1e9}
    except Exception as exc:  # never let the secondary line kill the headline
        single = {"error": str(exc)}
    # DRAM traffic of the same four stage launches from the committed ncu --set full capture
    traffic = None
    kname = "stage kernels"
    summ = ROOT / "profiles" / "r1_stage_kernels.json"
    if summ.exists():
        try:
            launches_ = json.loads(summ.read_text())["launches"]
            traffic = sum(e["dram_total_MB"] for e in launches_ if "k_" in e["kernel"]) * 1e6
            kname = " | ".join(e["kernel"].split("(")[0].replace("void ", "")
                               for e in launches_ if "k_" in e["kernel"])
        except (KeyError, ValueError, IndexError):
            traffic = None

    # end to end: the public API with host buffers (operands + rho0 in, records out)
    e2e_steps = max(args.steps, 50)
    cfg = xf.PropagationConfig(dt_fs=DT, n_max=N_MAX, t_end_fs=e2e_steps * DT, residual=None,
                               n_matsubara=K_MATS, record_stride=1, device=device)
    xf.propagate(system, bath, rates, cfg, 1)         # warm (module load, graph instantiate)
    best = float("inf")
    for _ in range(3):                                # best of three end-to-end calls
        barrier(dist, local)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        traj = xf.propagate(system, bath, rates, cfg, 1)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    e2e_s = allmax(dist, best, f"cuda:{device}")
    e2e_value = n_tot * e2e_steps * world / e2e_s
    h2d = (D * D * 16 + 16 * 4 * D + 64 * D + 512) / e2e_steps  # rho0 tile, operands, ctl
    d2h = traj.populations.shape[1] * 8 + 8 + 256                  # one record + status per step

    # FMO eta wall-time (BASELINE metric, configs[2]): trap + sinks at 300 K, residual
    # 1e-5 policy, through propagate(); K=1 N_max=6 (38,760 ADOs) and the K=0 twin
    # whose reference run is in tests/golden/traj_long.json
    eta = {}
    if not args.no_eta:
        for tag, (nm, K, dtf) in {"k1_nmax6": (6, 1, 1.25), "k0_nmax6": (6, 0, 2.5)}.items():
            cfg_e = xf.PropagationConfig(dt_fs=dtf, n_max=nm, residual=1e-5, record_stride=100,
                                         n_matsubara=K, device=device)
            xf.propagate(system, bath, rates, replace(cfg_e, residual=None, t_end_fs=10 * dtf), 1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tr = xf.propagate(system, bath, rates, cfg_e, 1)
            w = time.perf_counter() - t0
            eta[tag] = {"eta": float(xf.efficiency(tr)), "wall_s": w,
                        "steps": int(round(tr.times_fs[-1] / dtf)), "dt_fs": dtf,
                        "n_ado": xf.hierarchy_size(7 * (K + 1), nm)}
        eta["reference_k0_nmax6"] = {"eta": 0.9761164832557473, "wall_s": 298.1,
                                     "note": "reference propagate, 1 thread, measured in the "
                                             "build container (SURVEY 8(d).3)"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = CpuBaseline(xf, system, bath, rates).measure(
                float(os.environ.get("HB_CPU_BUDGET_S", "15")))
        except Exception as exc:  # the baseline must never kill the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {exc}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per RK4 step (4 stage launches), ncu",
                         "alg_bytes_per_step": B_ALG_STEP * n_tot,
                         "kernel": f"{kname} (stages 1-4, one launch each per RK4 step; achieved = alg bytes / sum of stage times)",
                         "bytes_per_ado_step": B_ALG_STEP,
                         "stage_us": [round(1e3 * x, 2) for x in stage_ms],
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650"},
            "survey_equivalent": {"b_alg_bytes": SURVEY_B_ALG,
                                  "target_ado_steps_per_s": 0.70 * 6548.2e9 / SURVEY_B_ALG,
                                  "frac_of_survey_roofline": value / world * SURVEY_B_ALG / (peak * 1e9)},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                    "api": "paper_1012_4382_b200.propagate (t_end run, record_stride=1)"},
            "gpu_launches": int(launches),
            "single_precision": single,
            "eta_wall": eta or None,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)   # 1 ps at dt = 1 fs
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-eta", action="store_true", help="skip the config-3 eta wall-time runs")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: split ONE hierarchy across the ranks (NCCL halo exchange) "
                         "instead of independent replicas")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
