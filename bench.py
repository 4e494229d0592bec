"""Benchmark: FP64 HEOM RK4 throughput (ADO-RK4-steps/s) on B200.

Workload (BASELINE.json configs[3], the north_star target):
7-site FMO (Adolphs-Renger H), 300 K, lambda = 35 cm^-1, gamma^-1 = 166 fs,
Gamma_RC^-1 = 2.5 ps, Gamma_phot^-1 = 250 ps, N_max = 8, K = 1 Matsubara term
(M = 14 modes, 319,770 ADOs), dt = 1 fs, rho0 = |1><1|.  One bench step = one
classical RK4 step of the whole hierarchy (4 fused stage kernels + the step
bookkeeping kernel).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Prints ONE JSON line (rank 0).  N = 1: the hierarchy on one GPU.  N > 1
(launched under torchrun, or ``--gpus N`` spawns torchrun itself): ONE
hierarchy sharded across the ranks (strong scaling, NCCL halo exchange of the
stage crosses, paper_1012_4382_b200/shard.py); N independent replicas are timed
as well and reported under "replicas".  Device time = CUDA events, max over
ranks.

``--impl reference`` times the reference itself -- excitonflow.propagate with
its numba kernels, installed unmodified under baseline/_ref -- on this host's
cores (the reference has no Matsubara terms, so on the K = 0 hierarchy of the
same depth: N_max = 8, 7 modes, 6,435 ADOs), with 1 thread and with every core,
and reports the faster.  Without baseline/_ref it falls back to the C port of
the reference path (oracle/).
"""

from __future__ import annotations

import argparse
from dataclasses import replace
import json
import os
import platform
import socket
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
N_ADO = 319770
S_PACKED = 8 * D * D                      # bytes per Hermitian-packed FP64 ADO (392 B)
B_ALG_STEP = 12 * S_PACKED                # algorithmic state bytes per ADO-step
B_ALG_STAGE = {1: 2 * S_PACKED, 2: 4 * S_PACKED, 3: 3 * S_PACKED, 4: 3 * S_PACKED}
B_ALG_SINGLE = 15 * 4 * D * D             # precision='single': 15 float passes
PROFILE = ROOT / "profiles" / "r2_stage_kernels.json"   # ncu --set full of the stage kernels
L2_STREAM_GBPS = 17242.0         # tools/micro/l2bw.cu: L2-resident 16-B streaming loads, all SMs
L2_GATHER_SECTOR_GBPS = 9270.0   # random 16-B gathers: one 32-B sector per SM cycle
REF_DIR = ROOT / "baseline" / "_ref"


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


def init_dist(world, local, backend, single=False):
    """torch.distributed for N > 1 (torchrun's env); with `single`, a one-rank
    group (the sharded code path at world size 1)."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        if not single:
            return None
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
        return dist
    if backend == "nccl":
        torch.cuda.set_device(local)
    dist.init_process_group(backend=backend)
    return dist


def barrier(dist, local=0):
    if dist is None:
        return
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


def host_info():
    model = platform.processor() or "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count() or 1}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
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


# --------------------------------------------------------------------------- CPU

class PortBaseline:
    """The C port of the reference path (oracle/heom_oracle.c, OpenMP) on this
    host's cores, timed on a bounded sample of the SAME workload (K = 1, N_max = 8
    whole-hierarchy RK4 steps) -- the reference itself cannot run K = 1."""

    def __init__(self, xf, system, bath, rates, threads):
        from oracle import oracle as orc
        self.orc, self.xf = orc, xf
        self.system, self.bath, self.rates = system, bath, rates
        self.threads = threads
        orc.set_threads(threads)
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
        return {"value": self.pb.n_tot * steps / wall, "unit": UNIT, "cores": self.threads,
                "kind": "port",
                "sample": f"{steps} RK4 steps of the full N_max=8 K=1 hierarchy "
                          f"({self.pb.n_tot} ADOs), {wall:.1f} s wall, oracle/heom_oracle.c "
                          f"OpenMP x{self.threads}"}


def ref_child(spec):
    """Runs in a subprocess (NUMBA_NUM_THREADS fixed before numba loads): the
    reference's own propagate() from baseline/_ref, timed like cli._bench_run
    (cli.py:374-381: enumeration and JIT warm-up outside the timer)."""
    sys.path.insert(0, str(REF_DIR))
    import excitonflow as ef
    from excitonflow.heom import _graph
    system = ef.build_fmo_system()
    out = {}
    for job in spec["jobs"]:
        bath = ef.BathParams.from_timescale(job["lam"], 166.0, job["T"])
        rates = ef.MarkovRates.from_inverse_ps(2.5, 250.0)
        nm, dt = job["n_max"], job["dt"]
        _graph(system.site_count, nm)
        warm = ef.PropagationConfig(dt_fs=dt, n_max=nm, t_end_fs=2 * dt, residual=None)
        ef.propagate(system, bath, rates, warm, 1)                  # JIT outside the timer
        cfg = ef.PropagationConfig(dt_fs=dt, n_max=nm, t_end_fs=job["steps"] * dt, residual=None,
                                   record_stride=max(1, job["steps"]))
        t0 = time.perf_counter()
        ef.propagate(system, bath, rates, cfg, 1)
        wall = time.perf_counter() - t0
        n_tot = ef.hierarchy_size(7, nm)
        out[job["name"]] = {"wall_s": wall, "steps": job["steps"], "n_tot": n_tot,
                            "value": n_tot * job["steps"] / wall}
    try:
        import numba
        out["threading_layer"] = numba.threading_layer()
        out["numba"] = numba.__version__
    except Exception as exc:  # threading_layer() raises before any parallel region ran
        out["threading_layer"] = f"unknown ({exc})"
    print(json.dumps(out), flush=True)


def run_ref_jobs(jobs, threads, timeout=600):
    env = dict(os.environ, NUMBA_NUM_THREADS=str(threads), OMP_NUM_THREADS=str(threads),
               NUMBA_CACHE_DIR=os.path.join(tempfile.gettempdir(), "hb_numba_cache"))
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--ref-child",
                        json.dumps({"jobs": jobs})], env=env, capture_output=True, text=True,
                       timeout=timeout)
    if p.returncode != 0:
        raise RuntimeError(p.stderr.strip().splitlines()[-1] if p.stderr.strip() else "ref child failed")
    return json.loads(p.stdout.strip().splitlines()[-1])


def reference_available():
    return (REF_DIR / "excitonflow" / "heom.py").exists()


def reference_numba(steps_main=20):
    """The real reference on this box: config-4's K = 0 analogue (N_max = 8,
    6,435 ADOs), config 2 (FMO 77 K, N_max = 4, 1 ps = 400 steps, full run) and a
    sample of the config-3 K = 0 eta twin (N_max = 6, dt 2.5 fs; the full run is
    23,519 steps, the wall is extrapolated from the sample), with 1 thread and
    with every core."""
    nproc = os.cpu_count() or 1
    jobs = [dict(name="n8_k0", n_max=8, dt=1.0, T=300.0, lam=35.0, steps=steps_main),
            dict(name="config2", n_max=4, dt=2.5, T=77.0, lam=35.0, steps=400),
            dict(name="eta_twin_sample", n_max=6, dt=2.5, T=300.0, lam=35.0, steps=300)]
    per = {}
    for th in sorted({1, nproc}):
        per[th] = run_ref_jobs(jobs, th)
    best = max(per, key=lambda th: per[th]["n8_k0"]["value"])
    r = per[best]
    eta = r["eta_twin_sample"]
    return {
        "kind": "reference", "impl": "excitonflow.propagate (numba, baseline/_ref, unmodified)",
        **host_info(), "threading_layer": r.get("threading_layer"), "numba": r.get("numba"),
        "value": r["n8_k0"]["value"], "unit": UNIT, "cores": best,
        "sample": f"{steps_main} RK4 steps of FMO 300 K N_max=8 K=0 (6435 ADOs; the reference "
                  f"has no Matsubara terms), NUMBA_NUM_THREADS={best}",
        "by_threads": {str(th): {k: v["value"] for k, v in per[th].items() if isinstance(v, dict)}
                       for th in per},
        "config2_wall_s": r["config2"]["wall_s"],
        "eta_twin_wall_s_extrapolated": eta["wall_s"] / eta["steps"] * 23519,
        "eta_twin_sample_steps": eta["steps"],
    }


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    line = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "none", "vs_baseline": None, "dtype": "f64", "data": "synthetic"}
    if reference_available():
        cb = reference_numba(max(1, args.steps))
        value = cb["value"]
        line.update(value=value, ms_per_step=1e3 * 6435 / value,
                    config={**config_dict(1), "workload": "FMO 300K N_max=8 K=0 (6435 ADOs), the "
                            "reference's largest analogue of config 4 (no Matsubara terms)",
                            "n_matsubara": 0, "n_ado": 6435,
                            "parallelism": f"CPU, NUMBA_NUM_THREADS={cb['cores']}"},
                    cpu_baseline=cb)
    else:
        xf, system, bath, rates = workload()
        base = PortBaseline(xf, system, bath, rates, os.cpu_count() or 1)
        cb = base.measure(float(os.environ.get("HB_REF_BUDGET_S", "20")))
        cb.update(host_info())
        cb["note"] = "baseline/_ref (the reference install) missing: C port timed instead"
        value = cb["value"]
        line.update(value=value, ms_per_step=1e3 * N_ADO / value, config=config_dict(1),
                    cpu_baseline=cb)
    line["e2e"] = {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU

def config_dict(world, sharded=False):
    par = "single GPU"
    if world > 1:
        par = f"sharded x{world} (NCCL halo of stage crosses)" if sharded else f"replicas x{world}"
    return {"workload": "FMO 300K N_max=8 K=1 (319770 ADOs), RK4 dt=1fs, one step = whole hierarchy",
            "n_max": N_MAX, "n_matsubara": K_MATS, "n_ado": N_ADO, "dt_fs": DT,
            "layout": "hermitian-packed AoSoA, tier-major ADO order (the reference's)",
            "l2": "inputs larger than L2 (4 x 125 MB state buffers, no flush needed)",
            "parallelism": par}


def ncu_traffic():
    """DRAM bytes per RK4 step of the four stage launches, from the committed
    ncu --set full capture (tools/gpu_profile.sh)."""
    if not PROFILE.exists():
        return None, "stage kernels", None, None
    try:
        launches = json.loads(PROFILE.read_text())["launches"]
        stages = [e for e in launches if "k_mm4" in e["kernel"]]
        traffic = sum(e["dram_total_MB"] for e in stages) * 1e6
        name = " | ".join(e["kernel"].split("(")[0].replace("void ", "") for e in stages)
        l2 = sum(e.get("l2_MB", 0.0) for e in stages) * 1e6 or None
        return traffic, name, [round(e["dram_total_MB"], 1) for e in stages], l2
    except (KeyError, ValueError, IndexError):
        return None, "stage kernels", None, None


def time_replica(xf, ops, device, args, dist, local, world):
    """Config 4 on this rank's GPU: K timed steps with the state resident."""
    from paper_1012_4382_b200.engine import DeviceRun
    run = DeviceRun(ops, N_MAX, DT, t_end_fs=1e15, record_stride=10 ** 12, device=device)
    rho0 = np.zeros((D, D), complex)
    rho0[0, 0] = 1.0
    run.set_rho0(rho0, [0.0, 0.0])
    run.time_steps(max(3, args.warmup))               # warm-up (untimed)
    launches0 = run.launch_count()
    barrier(dist, local)
    ms = run.time_steps(args.steps)                   # CUDA events on the handle's stream
    barrier(dist, local)
    launches = run.launch_count() - launches0
    ms_max = allmax(dist, ms, f"cuda:{device}")
    return run, ms_max, launches


def e2e_measure(xf, system, bath, rates, device, steps, dist, local):
    """propagate() through the public API with host inputs and a D2H record of
    the populations every step; host<->device bytes counted by the library."""
    import torch
    from paper_1012_4382_b200 import _native as N
    cfg = xf.PropagationConfig(dt_fs=DT, n_max=N_MAX, t_end_fs=steps * DT, residual=None,
                               n_matsubara=K_MATS, record_stride=1, device=device)
    xf.propagate(system, bath, rates, cfg, 1)         # warm (graph instantiate, pools)
    best, io = float("inf"), None
    for _ in range(3):
        barrier(dist, local)
        torch.cuda.synchronize()
        b0 = N.io_bytes()
        t0 = time.perf_counter()
        traj = xf.propagate(system, bath, rates, cfg, 1)
        el = time.perf_counter() - t0
        b1 = N.io_bytes()
        assert len(traj.times_fs) == steps + 1
        if el < best:
            best, io = el, (b1[0] - b0[0], b1[1] - b0[1])
    return best, io


def sweep_sample(xf, device, rank, world, n_points):
    """Config 5: the 8 x 8 temperature x lambda grid (N_max = 6, K = 1, residual
    1e-5, dt 1.25 fs), points dealt round-robin to the ranks, concurrent handles
    per GPU; at N = 1 a bounded share (n_points)."""
    from paper_1012_4382_b200 import sweep
    grid = sweep.temperature_lambda_grid()
    cfg = sweep.sweep_config(n_max=6, n_matsubara=1, dt_fs=1.25, residual=1e-5,
                             record_stride=100, device=device)
    worker = sweep.fmo_point_runner(cfg, xf.MarkovRates.from_inverse_ps(2.5, 250.0))
    mine = [p for i, p in sweep.shard_points(grid, rank, world)][:n_points]
    t0 = time.perf_counter()
    res = sweep.run_points(mine, worker, workers=min(8, len(mine)))
    wall = time.perf_counter() - t0
    steps = sum(r.steps for r in res)
    return {"points_timed": len(mine), "wall_s": wall, "steps": steps,
            "ado_steps_per_s": steps * 38760 / wall,
            "eta_first": res[0].efficiency if res else None,
            "grid": "T in {77..300} K x lambda in {10..120} cm^-1 (8 x 8), N_max=6, K=1, "
                    "residual 1e-5, dt 1.25 fs"}


def nccl_log_lines(limit=12):
    """The NCCL INIT log of this process (NCCL_DEBUG=INFO written to a file, so
    stdout keeps one JSON line): version, transports, communicator init."""
    path = Path(tempfile.gettempdir()) / f"hb_nccl_{os.getpid()}.log"
    if not path.exists():
        return None
    keep = [l.strip() for l in path.read_text(errors="replace").splitlines()
            if "NCCL INFO" in l and any(k in l for k in ("version", "Init", "NVLS", "P2P", "nranks",
                                                         "Channel 00", "NVLink", "Connected"))]
    maps = [l.split()[-1] for l in open("/proc/self/maps") if "libnccl" in l]
    return {"library": sorted(set(maps)), "lines": keep[:limit]}


def run_b200(args):
    world, rank, local = dist_env()
    if world > 1 or args.force_shard:  # NCCL communicator init visible, off stdout
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT,P2P,NVLS"
        os.environ["NCCL_DEBUG_FILE"] = str(Path(tempfile.gettempdir()) / f"hb_nccl_{os.getpid()}.log")
    import torch
    dist = init_dist(world, local, "nccl" if torch.cuda.is_available() else "gloo",
                     single=args.force_shard)
    device = local
    torch.cuda.set_device(device)
    xf, system, bath, rates = workload()
    from paper_1012_4382_b200.engine import BlockOperands, DeviceRun
    ops = BlockOperands(system, bath, rates, K_MATS)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)

    shard = None
    if (world > 1 and not args.replicas) or args.force_shard:
        try:
            shard = run_sharded(args, dist, world, rank, local, xf, ops)
        except Exception as exc:  # report it, keep the replica number
            shard = {"error": f"{type(exc).__name__}: {exc}"}

    clocks = ClockSampler(device)
    time.sleep(1.0)                                   # let nvidia-smi start sampling
    run, ms_max, launches = time_replica(xf, ops, device, args, dist, local, world)
    clk = clocks.stop()
    ms_step = ms_max / args.steps
    _, stage_ms = run.time_steps(1, per_stage=True)
    run.close()

    # the same workload in single precision (secondary, not the headline)
    single = None
    try:
        rs = DeviceRun(ops, N_MAX, DT, t_end_fs=1e15, record_stride=10 ** 12, device=device,
                       precision="single")
        rho0 = np.zeros((D, D), complex)
        rho0[0, 0] = 1.0
        rs.set_rho0(rho0, [0.0, 0.0])
        rs.time_steps(max(3, args.warmup))
        ms_s = rs.time_steps(args.steps) / args.steps
        rs.close()
        single = {"value": N_ADO / (ms_s / 1e3), "unit": UNIT, "ms_per_step": ms_s,
                  "dtype": "f32", "bytes_per_ado_step": B_ALG_SINGLE,
                  "achieved_GBps": N_ADO * B_ALG_SINGLE / (ms_s / 1e3) / 1e9}
    except Exception as exc:
        single = {"error": str(exc)}

    # device time of 1000 resident steps (same length as the longer e2e run: the
    # clock settles lower over a longer run than over the K timed steps)
    run_l = DeviceRun(ops, N_MAX, DT, t_end_fs=1e15, record_stride=10 ** 12, device=device)
    rho0_l = np.zeros((D, D), complex)
    rho0_l[0, 0] = 1.0
    run_l.set_rho0(rho0_l, [0.0, 0.0])
    run_l.time_steps(max(3, args.warmup))
    ms_1000 = run_l.time_steps(1000) / 1000
    run_l.close()
    e2e = {}
    for steps in (50, 1000):
        wall, (bi, bo) = e2e_measure(xf, system, bath, rates, device, steps, dist, local)
        wall = allmax(dist, wall, f"cuda:{device}")
        e2e[steps] = {"value": N_ADO * steps * world / wall, "wall_s": wall,
                      "h2d_bytes_per_step": bi / steps, "d2h_bytes_per_step": bo / steps}

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
            eta[tag] = {"eta": float(xf.efficiency(tr)), "trapping_time_ps": float(xf.trapping_time(tr)),
                        "wall_s": w, "steps": int(round(tr.times_fs[-1] / dtf)), "dt_fs": dtf,
                        "n_ado": xf.hierarchy_size(7 * (K + 1), nm)}
        eta["k0_nmax6"]["reference_eta"] = 0.9761164832557468   # tests/golden/traj_long.json

    sweep_res = None
    if not args.no_sweep:
        try:
            sweep_res = sweep_sample(xf, device, rank, world, 8 if world == 1 else 64)
            sweep_res["wall_s"] = allmax(dist, sweep_res["wall_s"], f"cuda:{device}")
        except Exception as exc:
            sweep_res = {"error": str(exc)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = PortBaseline(xf, system, bath, rates, os.cpu_count() or 1).measure(
                float(os.environ.get("HB_CPU_BUDGET_S", "15")))
            cpu.update(host_info())
        except Exception as exc:  # the baseline must never kill the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {exc}"}
        if reference_available() and not args.no_reference:
            try:
                cpu["reference"] = reference_numba()
            except Exception as exc:
                cpu["reference"] = {"error": str(exc)}

    if rank == 0:
        traffic, kname, traffic_stages, l2_bytes = ncu_traffic()
        achieved = N_ADO * B_ALG_STEP / (ms_step / 1e3) / 1e9
        stage_frac = [round(N_ADO * B_ALG_STAGE[s + 1] / (stage_ms[s] / 1e3) / 1e9 / peak, 3)
                      for s in range(4)]
        value_1 = N_ADO / (ms_step / 1e3)
        line = {
            "metric": METRIC, "value": value_1 * world, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per RK4 step (the 4 stage launches, ncu --set full)",
                         "traffic_by_stage_MB": traffic_stages,
                         "alg_bytes_per_step": B_ALG_STEP * N_ADO,
                         "kernel": f"{kname} (one launch per stage; achieved = 4,704 B x 319,770 "
                                   f"ADOs / timed ms_per_step)",
                         "bytes_per_ado_step": B_ALG_STEP,
                         "stage_us": [round(1e3 * x, 2) for x in stage_ms],
                         "stage_frac": stage_frac,
                         "stage_note": "stage_us from events around isolated launches (no PDL "
                                       "overlap), per-stage bytes 2S/4S/3S/3S, S = 392 B",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
                         # the ceiling the stage kernels actually press on: L2 sector traffic
                         # (own tile + link gathers + tables + stores), ncu lts__t_sectors
                         "l2": {"bytes_per_step": l2_bytes,
                                "achieved_GBps": l2_bytes / (ms_step / 1e3) / 1e9 if l2_bytes else None,
                                "stream_peak_GBps": L2_STREAM_GBPS,
                                "random_sector_peak_GBps": L2_GATHER_SECTOR_GBPS,
                                "source": "ncu lts__t_sectors.sum x 32 B (profiles/r2_stage_kernels.json); "
                                          "peaks: tools/micro/l2bw.cu on B200 (profiles/r2_l2bw.txt)"}},
            "e2e": {"value": e2e[50]["value"], "unit": UNIT,
                    "h2d_bytes_per_step": int(round(e2e[50]["h2d_bytes_per_step"])),
                    "d2h_bytes_per_step": int(round(e2e[50]["d2h_bytes_per_step"])),
                    "steps": 50, "frac_of_value": e2e[50]["value"] / (value_1 * world),
                    "bytes": "counted by the library (hb_io_bytes) around the call",
                    "api": "paper_1012_4382_b200.propagate (t_end run, a record every step)",
                    "steps_1000": {"value": e2e[1000]["value"],
                                   "frac_of_value": e2e[1000]["value"] / (value_1 * world),
                                   "device_ms_per_step_1000": ms_1000,
                                   "frac_of_device_1000": e2e[1000]["value"] / (N_ADO / (ms_1000 / 1e3) * world),
                                   "h2d_bytes_per_step": e2e[1000]["h2d_bytes_per_step"],
                                   "d2h_bytes_per_step": e2e[1000]["d2h_bytes_per_step"]}},
            "gpu_launches": int(launches),
            "single_precision": single,
            "eta_wall": eta or None,
            "sweep": sweep_res,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        if world > 1 or args.force_shard:
            line["replicas"] = {"value": value_1 * world, "ms_per_step": ms_step, "scaling": "weak"}
            line["nccl_init_log_rank0"] = nccl_log_lines()
            if shard is not None and "value" in shard:
                line.update(value=shard["value"], ms_per_step=shard["ms_per_step"],
                            scaling="strong", config=config_dict(world, sharded=True),
                            gpu_launches=shard["gpu_launches"])
                line["sharded"] = shard
            else:
                line["sharded"] = shard
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_sharded(args, dist, world, rank, local, xf, ops):
    """Config 4 split across the ranks: ONE hierarchy, contiguous tile ranges,
    NCCL exchange of the stage crosses (shard.py).  Device time of K steps,
    max over ranks."""
    import torch
    from paper_1012_4382_b200.shard import NcclShardedRun
    sr = NcclShardedRun(ops, N_MAX, DT, 1e15, rank, world, local, dist)
    rho0 = np.zeros((D, D), complex)
    rho0[0, 0] = 1.0
    sr.set_rho0(rho0, [0.0, 0.0])
    sr.time_steps(max(3, args.warmup))
    launches0 = sr.launch_count()
    barrier(dist, local)
    ms = sr.time_steps(args.steps)
    barrier(dist, local)
    launches = sr.launch_count() - launches0
    ms_max = allmax(dist, ms, f"cuda:{local}")
    info = sr.describe()
    sr.close()
    torch.cuda.synchronize()
    return {"value": N_ADO * args.steps / (ms_max / 1e3), "ms_per_step": ms_max / args.steps,
            "gpu_launches": int(launches), **info}


def spawn_ranks(args):
    """`python bench.py --gpus N` outside torchrun: start N ranks (one per GPU)."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible\n")
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas only (no sharded run)")
    ap.add_argument("--force-shard", action="store_true",
                    help="run the sharded path even at one rank (tests the NCCL code path)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-reference", action="store_true",
                    help="skip the numba reference inside the cpu_baseline")
    ap.add_argument("--no-eta", action="store_true", help="skip the config-3 eta wall-time runs")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-5 sweep sample")
    ap.add_argument("--ref-child", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ref_child is not None:
        ref_child(json.loads(args.ref_child))
        return 0
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
