"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

This script is the only place that executes the reference package
(`excitonflow`, /root/reference/pkg/src). It runs in the build container
(the reference does not exist on the GPU box) and writes small .npz/.json
fixtures that the test-suite, the C oracle pin and the GPU parity tests read.

Usage (from the repo root):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py            # fast fixtures (~1 min)
    ... make_golden.py --long                          # + the 300 K N_max=6 eta run (~5 min)
    ... make_golden.py --single                        # only the precision='single' runs

Every fixture records which reference call produced it (`source` key).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

import excitonflow as xf  # noqa: E402  (reference, read-only)
from excitonflow import _kernels  # noqa: E402
from excitonflow.heom import _BlockPropagator, _graph  # noqa: E402

OUT = Path(__file__).resolve().parent

# tables stored in full (small) and as hashes (large)
SMALL_TABLES = [(7, 0), (7, 2), (7, 3), (7, 4), (4, 5), (5, 3), (5, 4), (2, 4),
                (1, 20), (3, 6), (14, 2), (14, 3), (2, 6)]
HASH_TABLES = [(7, 6), (7, 8), (7, 10), (14, 4), (14, 6), (14, 8)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tables():
    arrays = {}
    for m, n in SMALL_TABLES:
        g = xf.enumerate_hierarchy(m, n)
        for name in ("indices", "tiers", "plus", "minus"):
            arrays[f"M{m}_N{n}_{name}"] = np.asarray(getattr(g, name))
    np.savez_compressed(OUT / "tables_small.npz", **arrays)
    hashes = {"source": "excitonflow.hierarchy.enumerate_hierarchy (hierarchy.py:59-105)"}
    for m, n in HASH_TABLES:
        t0 = time.time()
        g = xf.enumerate_hierarchy(m, n)
        hashes[f"M{m}_N{n}"] = {
            "n_tot": int(g.n_tot),
            "indices": sha(g.indices), "tiers": sha(g.tiers),
            "plus": sha(g.plus), "minus": sha(g.minus),
            # cheap spot values for debugging a mismatch
            "plus_row0": g.plus[0].tolist(), "minus_last": g.minus[-1].tolist(),
        }
        print(f"tables M={m} N={n}: {g.n_tot} ADOs in {time.time() - t0:.1f}s")
    (OUT / "tables_hash.json").write_text(json.dumps(hashes, indent=1))


def _operands(system, bath, rates, n_max):
    graph = _graph(system.site_count, n_max)
    ops = _BlockPropagator(system, bath, rates, graph, np.complex128)
    return graph, ops


def rhs_cases():
    """hierarchy_rhs_kernel (_kernels.py:23-58) on seeded random sigma."""
    fmo = xf.build_fmo_system()
    cases = {
        "fmo_n2": (fmo, xf.BathParams.from_timescale(35.0, 166.0, 300.0),
                   xf.MarkovRates.from_inverse_ps(2.5, 250.0), 2, 0),
        "fmo_n3_77k": (fmo, xf.BathParams.from_timescale(35.0, 166.0, 77.0),
                       xf.MarkovRates.from_inverse_ps(2.5, 250.0), 3, 1),
        "dimer_n4": (xf.ExcitonSystem(h_cm1=np.array([[100.0, 60.0], [60.0, 0.0]]),
                                      site_indices=(0, 1)),
                     xf.BathParams.from_timescale(20.0, 100.0, 77.0),
                     xf.MarkovRates.none(), 4, 2),
        "dephasing_n5": (xf.ExcitonSystem(h_cm1=np.array([[0.0, 0.0], [0.0, 200.0]]),
                                          site_indices=(1,)),
                         xf.BathParams.from_timescale(5.0, 100.0, 300.0),
                         xf.MarkovRates.none(), 5, 3),
    }
    arrays = {}
    for name, (system, bath, rates, n_max, seed) in cases.items():
        graph, ops = _operands(system, bath, rates, n_max)
        d = len(ops.block)
        rng = np.random.default_rng(seed)
        sig = (rng.standard_normal((graph.n_tot, d, d))
               + 1j * rng.standard_normal((graph.n_tot, d, d)))
        out = np.empty_like(sig)
        ops.rhs(out, sig)
        arrays.update({
            f"{name}_sig": sig, f"{name}_out": out,
            f"{name}_h": ops.h_block, f"{name}_site_of": ops.site_of,
            f"{name}_decay": ops.decay, f"{name}_a": np.float64(ops.a),
            f"{name}_b": np.float64(ops.b), f"{name}_gamma": np.float64(bath.gamma_fs1),
            f"{name}_n_sites": np.int64(system.site_count), f"{name}_n_max": np.int64(n_max),
        })
        # the other three kernels of the ABI on the same data
        x = sig.reshape(-1)
        y = out.reshape(-1)
        tmp = np.empty_like(x)
        _kernels.add_scaled(tmp, x, y, 0.37)
        arrays[f"{name}_add_scaled"] = tmp.copy()
        s2 = x.copy()
        _kernels.rk4_update(s2, x, y, tmp, x[::-1].copy(), 0.125)
        arrays[f"{name}_rk4_update"] = s2
        arrays[f"{name}_max_abs2"] = np.float64(_kernels.max_abs2(y))
    np.savez_compressed(OUT / "rhs_cases.npz", **arrays)


def dense_cases():
    """heom.heom_rhs / rk4_step (heom.py:175-219): the dense 9x9 definition."""
    fmo = xf.build_fmo_system()
    bath = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
    rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    graph = _graph(7, 2)
    rng = np.random.default_rng(5)
    sig = rng.standard_normal((graph.n_tot, 9, 9)) + 1j * rng.standard_normal((graph.n_tot, 9, 9))
    out = xf.heom_rhs(xf.HierarchyState(sig), graph, fmo, bath, rates)
    state = xf.HierarchyState.initial(graph, fmo, np.diag([0, 1.0] + [0] * 7).astype(complex))
    for _ in range(40):
        state = xf.rk4_step(state, graph, fmo, bath, rates, 2.5)
    np.savez_compressed(OUT / "dense_cases.npz", sig=sig, out=out, rk40_sigma=state.sigma,
                        rk40_time=np.float64(state.time_fs))


def _traj_arrays(prefix, traj, arrays, meta):
    arrays[f"{prefix}_times"] = traj.times_fs
    arrays[f"{prefix}_pops"] = traj.populations
    arrays[f"{prefix}_final_rho"] = traj.final_rho
    if traj.matrices is not None:
        arrays[f"{prefix}_matrices"] = traj.matrices
    meta[prefix] = {"stop_reason": traj.stop_reason, "n_records": int(len(traj.times_fs)),
                    "t_last": float(traj.times_fs[-1])}


def trajectories(long: bool):
    arrays, meta = {}, {"source": "excitonflow.heom.propagate / propagate_from (heom.py:286-419)"}
    fmo = xf.build_fmo_system()
    rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    bath300 = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
    bath77 = xf.BathParams.from_timescale(35.0, 166.0, 77.0)

    # config 1: dimer, N_max=4, K=0, 77 K, 1 ps
    dimer = xf.ExcitonSystem(h_cm1=np.array([[100.0, 60.0], [60.0, 0.0]]), site_indices=(0, 1))
    cfg = xf.PropagationConfig(dt_fs=0.5, n_max=4, t_end_fs=1000.0, residual=None, record_stride=20)
    rho0 = np.array([[1.0, 0.0], [0.0, 0.0]], dtype=complex)
    t0 = time.time()
    traj = xf.propagate_from(dimer, xf.BathParams.from_timescale(20.0, 100.0, 77.0),
                             xf.MarkovRates.none(), cfg, rho0)
    meta["dimer_n4_77k"] = {}
    _traj_arrays("dimer_n4_77k", traj, arrays, meta)
    meta["dimer_n4_77k"]["wall_s"] = time.time() - t0

    # config 2: FMO 77 K, N_max=4, 1 ps, every step
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=4, t_end_fs=1000.0, residual=None, record_stride=1)
    t0 = time.time()
    traj = xf.propagate(fmo, bath77, rates, cfg, 1)
    _traj_arrays("fmo_n4_77k", traj, arrays, meta)
    meta["fmo_n4_77k"]["wall_s"] = time.time() - t0

    # CLI default run, N_max=2, 1 ps (test_cli.py:110-129 frozen fixture source)
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=2, t_end_fs=1000.0, residual=None, record_stride=1)
    traj = xf.propagate(fmo, bath300, rates, cfg, 1)
    _traj_arrays("fmo_n2_300k", traj, arrays, meta)

    # matrices + Hermiticity over 1 ps (test_heom.py:245-251)
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=4, t_end_fs=1000.0, residual=None,
                               record_matrices=True, record_stride=40)
    traj = xf.propagate(fmo, bath300, rates, cfg, 1)
    _traj_arrays("fmo_n4_300k_mats", traj, arrays, meta)

    # residual policy, eta (test_observables.py:103-111)
    cfg = xf.PropagationConfig(dt_fs=5.0, n_max=2, residual=1e-5, record_stride=20)
    traj = xf.propagate(fmo, bath300, rates, cfg, 1)
    _traj_arrays("fmo_n2_eta", traj, arrays, meta)
    meta["fmo_n2_eta"]["eta"] = float(xf.efficiency(traj))
    meta["fmo_n2_eta"]["trapping_time_ps"] = float(xf.trapping_time(traj))

    # residual policy with a stride that does not divide the stop step (final partial record)
    cfg = xf.PropagationConfig(dt_fs=5.0, n_max=1, residual=1e-5, record_stride=7)
    traj = xf.propagate(fmo, bath300, rates, cfg, 6)
    _traj_arrays("fmo_n1_eta_site6", traj, arrays, meta)
    meta["fmo_n1_eta_site6"]["eta"] = float(xf.efficiency(traj))

    # pure dephasing, one-site 2-level system, N_max=20, matrices (test_heom.py:184-200)
    system = xf.ExcitonSystem(h_cm1=np.array([[0.0, 0.0], [0.0, 200.0]]), site_indices=(1,))
    cfg = xf.PropagationConfig(dt_fs=0.25, n_max=20, t_end_fs=500.0, residual=None,
                               record_stride=20, record_matrices=True)
    traj = xf.propagate_from(system, xf.BathParams.from_timescale(5.0, 100.0, 300.0),
                             xf.MarkovRates.none(), cfg,
                             np.array([[0.5, 0.5], [0.5, 0.5]], dtype=complex))
    _traj_arrays("dephasing_n20", traj, arrays, meta)

    # N_max = 0 (Markov only)
    cfg = xf.PropagationConfig(dt_fs=1.0, n_max=0, t_end_fs=200.0, residual=None)
    traj = xf.propagate(fmo, bath300, rates, cfg, 1)
    _traj_arrays("fmo_n0", traj, arrays, meta)

    # divergence guard (test_heom.py:166-170)
    cfg = xf.PropagationConfig(dt_fs=150.0, n_max=2, t_end_fs=30000.0, residual=None)
    try:
        xf.propagate(fmo, bath300, rates, cfg, 1)
        meta["diverge"] = {"raised": None}
    except xf.PropagationDiverged as exc:
        meta["diverge"] = {"raised": "PropagationDiverged", "message": str(exc)}

    # hard cap (test_heom.py:261-265)
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=0, residual=1e-5, hard_cap_fs=500.0)
    try:
        xf.propagate(fmo, bath300, xf.MarkovRates.none(), cfg, 1)
        meta["hardcap"] = {"raised": None}
    except xf.ConvergenceFailure as exc:
        meta["hardcap"] = {"raised": "ConvergenceFailure", "message": str(exc)}

    # non-exactly-Hermitian rho0 (allowed by the 1e-12 check at heom.py:297)
    rho0 = np.zeros((9, 9), dtype=complex)
    rho0[1, 1] = 0.6
    rho0[2, 2] = 0.4
    rho0[1, 2] = 0.3 + 1e-13j
    rho0[2, 1] = 0.3
    cfg = xf.PropagationConfig(dt_fs=2.5, n_max=2, t_end_fs=250.0, residual=None,
                               record_matrices=True, record_stride=10)
    traj = xf.propagate_from(fmo, bath300, rates, cfg, rho0)
    _traj_arrays("fmo_n2_nonherm", traj, arrays, meta)
    arrays["fmo_n2_nonherm_rho0"] = rho0

    if long:
        # config 3, K=0 twin: 300 K, N_max=6, residual 1e-5 -> eta
        cfg = xf.PropagationConfig(dt_fs=2.5, n_max=6, residual=1e-5, record_stride=100)
        t0 = time.time()
        traj = xf.propagate(fmo, bath300, rates, cfg, 1)
        _traj_arrays("fmo_n6_eta", traj, arrays, meta)
        meta["fmo_n6_eta"].update({"eta": float(xf.efficiency(traj)),
                                   "trapping_time_ps": float(xf.trapping_time(traj)),
                                   "wall_s": time.time() - t0})
        np.savez_compressed(OUT / "traj_long.npz",
                            **{k: v for k, v in arrays.items() if k.startswith("fmo_n6_eta")})
        (OUT / "traj_long.json").write_text(json.dumps({"fmo_n6_eta": meta["fmo_n6_eta"]}, indent=1))
        return
    np.savez_compressed(OUT / "traj.npz", **arrays)
    (OUT / "traj.json").write_text(json.dumps(meta, indent=1))


def single_precision():
    """precision='single' (complex64 state, heom.py:93-94): the reference's own
    smoke case (test_heom.py:353-360), config 2 and a residual/eta run, each with
    its double twin, so the suite can check single vs reference-single and the
    reference's single-vs-double bound (5e-7, test_acceptance.py:231-238)."""
    arrays, meta = {}, {"source": "excitonflow.heom.propagate, precision='single' (heom.py:74, 93-94)"}
    fmo = xf.build_fmo_system()
    rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    bath300 = xf.BathParams.from_timescale(35.0, 166.0, 300.0)
    bath77 = xf.BathParams.from_timescale(35.0, 166.0, 77.0)
    cases = {
        "smoke_n4": (bath300, dict(dt_fs=10.0, n_max=4, t_end_fs=1000.0, residual=None,
                                   record_stride=10)),
        "fmo_n4_77k": (bath77, dict(dt_fs=2.5, n_max=4, t_end_fs=1000.0, residual=None,
                                    record_stride=20)),
        "fmo_n2_eta": (bath300, dict(dt_fs=5.0, n_max=2, residual=1e-3, record_stride=20)),
    }
    for name, (bath, kw) in cases.items():
        for prec in ("single", "double"):
            traj = xf.propagate(fmo, bath, rates, xf.PropagationConfig(precision=prec, **kw), 1)
            key = f"{name}_{prec}"
            arrays[key + "_times"] = traj.times_fs
            arrays[key + "_pops"] = traj.populations
            meta[key] = {"stop_reason": traj.stop_reason, "eta": float(xf.efficiency(traj))}
    np.savez_compressed(OUT / "traj_single.npz", **arrays)
    (OUT / "traj_single.json").write_text(json.dumps(meta, indent=1))


def auto_truncate_cases():
    """heom.auto_truncate (heom.py:422-446) on the reference's own cases
    (test_heom.py:299-324): the returned tier, its trajectory and the trapping
    times of every tier the search visited."""
    fmo = xf.build_fmo_system()
    rates = xf.MarkovRates.from_inverse_ps(2.5, 250.0)
    arrays, meta = {}, {"source": "excitonflow.heom.auto_truncate (heom.py:422-446), "
                                  "cases of test_heom.py:299-324"}
    import warnings
    cases = {
        "pairwise": (xf.BathParams.from_timescale(5.0, 166.0, 300.0),
                     dict(dt_fs=10.0, n_max=0, residual=1e-5, hard_cap_fs=500000.0, record_stride=5),
                     dict(start_n=1, tol_ps=0.5)),
        "zero_coupling": (xf.BathParams.from_timescale(0.0, 166.0, 300.0),
                          dict(dt_fs=5.0, n_max=0, t_end_fs=20000.0, residual=None, record_stride=10),
                          dict()),
        "fmo35_tol": (xf.BathParams.from_timescale(35.0, 166.0, 300.0),
                      dict(dt_fs=10.0, n_max=0, residual=1e-5, hard_cap_fs=500000.0, record_stride=5),
                      dict(start_n=1, tol_ps=0.2)),
    }
    for name, (bath, ckw, akw) in cases.items():
        cfg = xf.PropagationConfig(**ckw)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            n, traj = xf.auto_truncate(fmo, bath, rates, cfg, 1, **akw)
            visited = {}
            lo = 0 if bath.lam_cm1 == 0 else akw.get("start_n", 2)
            for k in range(lo, n + 2):
                visited[str(k)] = float(xf.trapping_time(
                    xf.propagate(fmo, bath, rates, xf.PropagationConfig(**{**ckw, "n_max": k}), 1)))
        _traj_arrays(f"at_{name}", traj, arrays, meta)
        meta[f"at_{name}"].update(n=int(n), trapping_times=visited, config=ckw, kwargs=akw,
                                  bath=[bath.lam_cm1, 1.0 / bath.gamma_fs1, bath.temperature_k])
    try:  # the cap failure message (test_heom.py:319-324)
        xf.auto_truncate(fmo, xf.BathParams.from_timescale(35.0, 166.0, 300.0), rates,
                         xf.PropagationConfig(dt_fs=5.0, n_max=0, t_end_fs=500.0, residual=None),
                         1, tol_ps=1e-12, start_n=0, n_cap=2)
    except xf.ConvergenceFailure as exc:
        meta["cap_failure_message"] = str(exc)
    np.savez_compressed(OUT / "auto_truncate.npz", **arrays)
    (OUT / "auto_truncate.json").write_text(json.dumps(meta, indent=1))


def cli_artifacts():
    """The `excitonflow propagate` CSV (cli.py:287-293, 396-415) for two runs, and
    the emitted config header (cli.py:210-219) of a few configurations."""
    from dataclasses import replace as dc_replace
    from excitonflow import cli
    out = {"source": "excitonflow.cli.main propagate / cli.emit_config (cli.py:210-219, 396-415)",
           "runs": {}, "headers": {}}
    runs = {"n2_t200": ["propagate", "--n-max", "2", "--t-end-fs", "200", "--residual", "none"],
            "site6_lam55": ["propagate", "--n-max", "3", "--t-end-fs", "100", "--residual", "none",
                            "--site", "6", "--lambda-cm1", "55", "--record-stride", "4"]}
    for name, argv in runs.items():
        path = Path("/tmp") / f"golden_cli_{name}.csv"
        assert cli.main(argv + ["--out", str(path)]) == 0
        out["runs"][name] = {"argv": argv, "csv": path.read_text()}
    base = cli.RunConfig()
    cfgs = {"default": base,
            "auto": dc_replace(base, n_max=None, t_end_fs=1000.0, residual=None, workers=4),
            "sweep": dc_replace(base, lambdas=(10.0, 35.5), sites=(1, 6), n_max_list=(2, 4),
                                add_reorg_to_diagonal=True, precision="single")}
    for name, c in cfgs.items():
        out["headers"][name] = {"fields": {k: (list(v) if isinstance(v, tuple) else v)
                                           for k, v in c.__dict__.items()},
                                "lines": cli.emit_config(c)}
    (OUT / "cli_artifacts.json").write_text(json.dumps(out, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cli", action="store_true", help="only the CLI artifact fixtures")
    ap.add_argument("--auto-truncate", action="store_true", help="only the auto_truncate cases")
    ap.add_argument("--single", action="store_true", help="only the precision='single' runs")
    ap.add_argument("--long", action="store_true", help="only the N_max=6 eta run")
    ap.add_argument("--dense", action="store_true", help="only the dense heom_rhs fixtures")
    args = ap.parse_args()
    if args.cli:
        cli_artifacts()
        return
    if args.auto_truncate:
        auto_truncate_cases()
        return
    if args.single:
        single_precision()
        return
    if args.dense:
        dense_cases()
        return
    if args.long:
        trajectories(long=True)
        return
    tables()
    rhs_cases()
    dense_cases()
    trajectories(long=False)
    single_precision()
    auto_truncate_cases()
    cli_artifacts()


if __name__ == "__main__":
    main()
