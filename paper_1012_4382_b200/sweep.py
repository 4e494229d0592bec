"""Parameter sweeps: many independent propagations.

The reference evaluates sweep points with a ThreadPoolExecutor over nogil numba
kernels and merges results in point order (cli.py:279-284).
Here every point is an independent device run with its own handle and CUDA
stream; worker threads release the GIL inside the ctypes calls, so several
small hierarchies occupy one GPU concurrently.  Across GPUs the points are
dealt round-robin to the ranks (one process per GPU, replicas -- no
data-path collective) and gathered on rank 0 in point order.

Results are independent of the worker count and of the number of ranks: each
point runs the same deterministic kernels on its own state.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, replace
from typing import Callable, Optional, Sequence

from .heom import PropagationConfig, propagate
from .model import BathParams, MarkovRates, build_fmo_system
from .observables import Trajectory, efficiency, trapping_time


@dataclass(frozen=True)
class SweepPoint:
    temperature_k: float
    lam_cm1: float
    gamma_inv_fs: float = 166.0
    delta_e_cm1: float = 0.0
    initial_site: int = 1


@dataclass
class SweepResult:
    point: SweepPoint
    efficiency: float
    trapping_time_ps: float
    steps: int
    stop_reason: Optional[str]


def fmo_point_runner(config: PropagationConfig, rates: MarkovRates) -> Callable:
    """Default worker: FMO propagation of one (T, lambda) point -> eta, <t>."""
    def run(point: SweepPoint) -> SweepResult:
        system = build_fmo_system(delta_e_cm1=point.delta_e_cm1)
        bath = BathParams.from_timescale(point.lam_cm1, point.gamma_inv_fs, point.temperature_k)
        traj: Trajectory = propagate(system, bath, rates, config, point.initial_site)
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            eta = efficiency(traj)
            tt = trapping_time(traj) if len(traj.times_fs) >= 3 else float("nan")
        steps = int(round(traj.times_fs[-1] / config.dt_fs))
        return SweepResult(point, eta, tt, steps, traj.stop_reason)
    return run


def run_points(points: Sequence, worker: Callable, workers: int = 4) -> list:
    """worker(point) for every point, concurrently, results in point order."""
    if workers <= 1:
        return [worker(p) for p in points]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(worker, points))


def shard_points(points: Sequence, rank: int, world: int) -> list:
    """Round-robin deal of the points to the ranks: [(index, point)]."""
    return [(i, p) for i, p in enumerate(points) if i % world == rank]


def run_sweep(points: Sequence, worker: Callable, workers: int = 4, dist=None) -> Optional[list]:
    """Sweep over one process (dist None) or all ranks of torch.distributed.

    Every rank evaluates its share with `workers` threads on its own GPU; rank 0
    returns the full result list in point order, the other ranks return None.
    """
    if dist is None:
        return run_points(points, worker, workers)
    rank, world = dist.get_rank(), dist.get_world_size()
    mine = shard_points(points, rank, world)
    local = run_points([p for _, p in mine], worker, workers)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(list(zip([i for i, _ in mine], local)), gathered, dst=0)
    if rank != 0:
        return None
    out = [None] * len(points)
    for part in gathered:
        for i, r in part:
            out[i] = r
    return out


def temperature_lambda_grid(temperatures=(77.0, 100.0, 125.0, 150.0, 175.0, 200.0, 250.0, 300.0),
                            lambdas=(10.0, 20.0, 35.0, 55.0, 70.0, 85.0, 100.0, 120.0)):
    """Config 5's grid: 8 temperatures x 8 reorganisation energies."""
    return [SweepPoint(temperature_k=t, lam_cm1=lam) for t in temperatures for lam in lambdas]


def sweep_config(n_max: int = 6, n_matsubara: int = 1, dt_fs: float = 1.0, **kw) -> PropagationConfig:
    return replace(PropagationConfig(dt_fs=dt_fs, n_max=n_max, n_matsubara=n_matsubara), **kw)
