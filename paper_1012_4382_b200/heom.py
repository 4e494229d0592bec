"""HEOM propagation API (drop-in for the reference heom.py).

The hierarchy of auxiliary density operators (ADOs) sigma^(n) evolves as
(heom.py:7-20, generalised to K Matsubara terms per site, modes m = (j, k))

    d/dt sigma^n = -i[H, sigma^n] + L_markov(sigma^n) - (sum_m n_m nu_m) sigma^n
                   + sum_m i [P_j(m), sigma^(n+e_m)] + sum_m n_m theta_m(sigma^(n-e_m))
    theta_m = i a_k [P_j, .] + b_k {P_j, .}

and is integrated with classical RK4.  Everything inside the time loop runs on
the GPU (csrc/hb_stage.cu); this module validates inputs exactly like the
reference, prepares operands (engine.BlockOperands), starts the device run and
assembles the Trajectory.  Reference line numbers: PropagationConfig :57-94,
propagate_from :286-406, propagate :409-419, auto_truncate :422-446.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import _native as N
from .engine import (BlockOperands, DeviceRun, bath_coefficients, bath_modes,  # noqa: F401
                     loss_channels)
from .hierarchy import HierarchyGraph, hierarchy_size
from .model import BathParams, ExcitonSystem, MarkovRates
from .observables import Trajectory, trapping_time
from .units import ANGFREQ_RAD_FS


class PropagationDiverged(RuntimeError):
    """A matrix norm exceeded the blow-up bound during time stepping."""


class ConvergenceFailure(RuntimeError):
    """A stop policy or truncation search did not converge within its cap."""


@dataclass(frozen=True)
class PropagationConfig:
    """Time stepping and stop policy (reference fields and defaults) plus the
    B200 options.

    New fields (defaults reproduce the reference):
      n_matsubara  K, Matsubara terms per site (0 = the reference's bath);
      device       CUDA ordinal;
      layout       'auto' (Hermitian-packed when rho0 is exactly Hermitian),
                   'hermitian' or 'general';
      ordering     device ADO order: 'reference' (tier-major, default: whole
                   top-tier tiles take the paired-site rounds), 'lex' (locality)
                   or 'lex-split' (lex tiles, top tier last inside a tile);
      chunk_steps  RK4 steps per CUDA-graph launch (0 = library default);
      kernel       'auto' (unrolled thread-per-ADO kernel when the shape allows)
                   or 'generic' (runtime-shaped tile kernel).
    ``precision='single'`` (reference field, heom.py:74) runs a float32 state with
    float32 right-hand sides on the device; sinks, records and the stop policy
    stay float64.  It needs the production shape: an exactly Hermitian rho0,
    every block level a site, d <= 8, n_matsubara <= 1, kernel='auto'
    (otherwise ValueError).
    """

    dt_fs: float = 2.5
    n_max: int = 8
    t_end_fs: Optional[float] = None
    residual: Optional[float] = 1e-5
    hard_cap_fs: float = 200_000.0
    record_stride: int = 1
    precision: str = "double"
    record_matrices: bool = False
    blowup_norm: float = 1e6
    n_matsubara: int = 0
    device: int = 0
    layout: str = "auto"
    ordering: str = "reference"
    chunk_steps: int = 0
    kernel: str = "auto"

    def __post_init__(self):
        if self.dt_fs <= 0:
            raise ValueError("dt must be > 0")
        if self.n_max < 0:
            raise ValueError("n_max must be >= 0")
        if self.record_stride < 1:
            raise ValueError("record stride must be >= 1")
        if self.precision not in ("double", "single"):
            raise ValueError("precision must be 'double' or 'single'")
        if self.t_end_fs is None and self.residual is None:
            raise ValueError("need a stop policy: t_end_fs or residual")
        if self.t_end_fs is not None and self.t_end_fs < 0:
            raise ValueError("t_end_fs must be >= 0")
        if self.n_matsubara < 0:
            raise ValueError("n_matsubara must be >= 0")
        if self.layout not in N.HB_LAYOUT:
            raise ValueError("layout must be 'auto', 'hermitian' or 'general'")
        if self.ordering not in N.HB_ORDER:
            raise ValueError("ordering must be 'lex', 'lex-split' or 'reference'")
        if self.kernel not in N.HB_KERNEL:
            raise ValueError("kernel must be 'auto' or 'generic'")

    @property
    def dtype(self):
        return np.complex128 if self.precision == "double" else np.complex64


@dataclass
class HierarchyState:
    """Full hierarchy state on the host (reference order): sigma[0] is rho."""

    sigma: np.ndarray
    time_fs: float = 0.0

    @classmethod
    def initial(cls, graph: HierarchyGraph, system: ExcitonSystem, rho0: np.ndarray,
                dtype=np.complex128) -> "HierarchyState":
        d = system.dimension
        sigma = np.zeros((graph.n_tot, d, d), dtype=dtype)
        sigma[0] = np.asarray(rho0, dtype=dtype)
        return cls(sigma=sigma, time_fs=0.0)

    @property
    def rho(self) -> np.ndarray:
        return self.sigma[0]


def lindblad_markov(rho: np.ndarray, system: ExcitonSystem, rates: MarkovRates) -> np.ndarray:
    """Sum over loss channels of D(V) rho = V rho V+ - {V+V, rho}/2 (heom.py:137-150)."""
    out = np.zeros_like(rho, dtype=complex)
    for rate, src, dst in loss_channels(system, rates):
        out[dst, dst] += rate * rho[src, src]
        out[src, :] -= 0.5 * rate * rho[src, :]
        out[:, src] -= 0.5 * rate * rho[:, src]
    return out


def bath_backaction(system: ExcitonSystem, site_label: int, sigma: np.ndarray,
                    bath: BathParams) -> np.ndarray:
    """theta(sigma) = i a [P, sigma] + b {P, sigma} for one site (heom.py:153-165)."""
    a, b = bath_coefficients(bath)
    idx = system.site_basis_index(site_label)
    out = np.zeros_like(sigma, dtype=complex)
    out[idx, :] += (b + 1j * a) * sigma[idx, :]
    out[:, idx] += (b - 1j * a) * sigma[:, idx]
    return out


def heom_rhs(state: HierarchyState, graph: HierarchyGraph, system: ExcitonSystem,
             bath: BathParams, rates: MarkovRates) -> np.ndarray:
    """d sigma / dt of the full hierarchy on the FULL basis, sinks included
    (the dense semantic definition, heom.py:175-204), evaluated on the GPU by the
    generic stage kernel with the Lindblad sink refill (hb_heom_rhs)."""
    N.require_device(0)
    sigma = np.ascontiguousarray(state.sigma, dtype=np.complex128)
    n_tot, d, _ = sigma.shape
    h = np.ascontiguousarray(system.h_cm1 * ANGFREQ_RAD_FS)
    site_of = np.full(d, -1, np.int32)
    for slot, idx in enumerate(system.site_indices):
        site_of[idx] = slot
    decay = np.zeros(d)
    dst, src, rate = [], [], []
    for r, b_, a_ in loss_channels(system, rates):
        decay[b_] += r
        dst.append(a_)
        src.append(b_)
        rate.append(r)
    a, b = bath_coefficients(bath)
    plus = np.ascontiguousarray(graph.plus, dtype=np.int32)
    minus = np.ascontiguousarray(graph.minus, dtype=np.int32)
    nvec = np.ascontiguousarray(graph.indices, dtype=np.float64)
    tier_damp = np.ascontiguousarray(graph.tiers * bath.gamma_fs1, dtype=np.float64)
    dst = np.array(dst or [0], np.int32)
    src = np.array(src or [0], np.int32)
    rate = np.array(rate or [0.0])
    out = np.empty_like(sigma)
    rc = N.lib().hb_heom_rhs(N.ptr(out), N.ptr(sigma), n_tot, d, N.ptr(h), N.ptr(site_of),
                             N.ptr(plus), N.ptr(minus), plus.shape[1], N.ptr(nvec),
                             N.ptr(tier_damp), float(a), float(b), N.ptr(decay),
                             len(loss_channels(system, rates)),
                             N.ptr(dst), N.ptr(src), N.ptr(rate), 0)
    N.check(rc, "hb_heom_rhs")
    return out


def rk4_step(state: HierarchyState, graph: HierarchyGraph, system: ExcitonSystem,
             bath: BathParams, rates: MarkovRates, dt_fs: float,
             blowup_norm: float = 1e6) -> HierarchyState:
    """One classical RK4 step of the dense definition (heom.py:207-219); the
    stage combinations run on the device through the Level-2 kernel shims."""
    from . import kernels
    s = np.ascontiguousarray(state.sigma, dtype=np.complex128)
    flat = s.reshape(-1)
    k1 = heom_rhs(state, graph, system, bath, rates)
    tmp = np.empty_like(s)
    kernels.add_scaled(tmp.reshape(-1), flat, k1.reshape(-1), 0.5 * dt_fs)
    k2 = heom_rhs(HierarchyState(tmp.copy()), graph, system, bath, rates)
    kernels.add_scaled(tmp.reshape(-1), flat, k2.reshape(-1), 0.5 * dt_fs)
    k3 = heom_rhs(HierarchyState(tmp.copy()), graph, system, bath, rates)
    kernels.add_scaled(tmp.reshape(-1), flat, k3.reshape(-1), dt_fs)
    k4 = heom_rhs(HierarchyState(tmp.copy()), graph, system, bath, rates)
    new = s.copy()
    kernels.rk4_update(new.reshape(-1), k1.reshape(-1), k2.reshape(-1), k3.reshape(-1),
                       k4.reshape(-1), dt_fs / 6.0)
    if kernels.max_abs2(new.reshape(-1)) > blowup_norm * blowup_norm:
        raise PropagationDiverged(
            f"matrix norm exceeded {blowup_norm:g} at t = {state.time_fs + dt_fs} fs")
    return HierarchyState(sigma=new, time_fs=state.time_fs + dt_fs)


def _check_rho0(system: ExcitonSystem, rho0) -> np.ndarray:
    rho0 = np.asarray(rho0, dtype=complex)
    d = system.dimension
    if rho0.shape != (d, d):
        raise ValueError(f"initial state must be {d}x{d}")
    if not np.allclose(rho0, rho0.conj().T, atol=1e-12):
        raise ValueError("initial state must be Hermitian")
    return rho0


def _graph_checks(n_sites: int, n_max: int) -> None:
    # enumerate_hierarchy's validation (hierarchy.py:61-69), raised in the same order
    if n_sites < 1:
        raise ValueError("need at least one site")
    if n_max < 0:
        raise ValueError("truncation tier must be >= 0")
    n_tot = hierarchy_size(n_sites, n_max)
    if n_tot > np.iinfo(np.int32).max:
        raise ValueError(f"hierarchy with {n_tot} indices exceeds the supported index range")


def _trajectory(system, ops, config, run, steps, pops, mats, stop_reason) -> Trajectory:
    sig0, sinks = run.sigma0()
    d = system.dimension
    final = np.zeros((d, d), dtype=complex)
    final[np.ix_(ops.block, ops.block)] = sig0
    for k, s in enumerate(ops.sinks):
        final[s, s] = sinks[k]
    return Trajectory(
        times_fs=np.array([int(s) * config.dt_fs for s in steps]),
        populations=pops,
        site_indices=system.site_indices,
        ground_index=system.ground_index,
        rc_index=system.rc_index,
        stop_reason=stop_reason,
        final_rho=final,
        residual_threshold=config.residual,
        matrices=mats,
    )


def propagate_from(system: ExcitonSystem, bath: BathParams, rates: MarkovRates,
                   config: PropagationConfig, rho0: np.ndarray) -> Trajectory:
    """Propagate an arbitrary block-supported initial density matrix on the GPU."""
    rho0 = _check_rho0(system, rho0)
    K = config.n_matsubara
    _graph_checks(system.site_count * (K + 1), config.n_max)
    ops = BlockOperands(system, bath, rates, K)
    d = system.dimension
    for s in ops.sinks:
        if any(rho0[s, j] != 0 for j in range(d) if j != s):  # row only, as heom.py:303-305
            raise ValueError("initial state must not carry sink coherences")
    block = rho0[np.ix_(ops.block, ops.block)]
    if config.layout == "hermitian" and not np.array_equal(block, block.conj().T):
        raise ValueError("layout='hermitian' needs an exactly Hermitian rho0")
    run = DeviceRun(ops, config.n_max, config.dt_fs, t_end_fs=config.t_end_fs,
                    residual=config.residual, hard_cap_fs=config.hard_cap_fs,
                    record_stride=config.record_stride, record_matrices=config.record_matrices,
                    blowup_norm=config.blowup_norm, device=config.device, layout=config.layout,
                    ordering=config.ordering, chunk_steps=config.chunk_steps,
                    kernel=config.kernel, precision=config.precision)
    with run:
        run.set_rho0(block, [float(rho0[s, s].real) for s in ops.sinks])
        rc = run.run()
        if rc == N.HB_DIVERGED:
            step = int(run.result.steps)
            raise PropagationDiverged(
                f"matrix norm exceeded {config.blowup_norm:g} at t = {step * config.dt_fs} fs")
        if rc == N.HB_HARDCAP:
            raise ConvergenceFailure(
                f"residual policy not reached within the {config.hard_cap_fs} fs cap")
        reason = {N.HB_STOP_T_END: "t_end", N.HB_STOP_RESIDUAL: "residual"}.get(
            run.result.stop_reason)
        steps, pops, mats = run.records()
        return _trajectory(system, ops, config, run, steps, pops, mats, reason)


def propagate(system: ExcitonSystem, bath: BathParams, rates: MarkovRates,
              config: PropagationConfig, initial_site: int = 1) -> Trajectory:
    """Propagate from |site><site| with all auxiliaries zero."""
    idx = system.site_basis_index(initial_site)
    rho0 = np.zeros((system.dimension, system.dimension), dtype=complex)
    rho0[idx, idx] = 1.0
    return propagate_from(system, bath, rates, config, rho0)


def auto_truncate(system: ExcitonSystem, bath: BathParams, rates: MarkovRates,
                  config: PropagationConfig, initial_site: int = 1, tol_ps: float = 0.02,
                  start_n: int = 2, n_cap: int = 20, speculate: bool = True) -> tuple:
    """Raise n_max until consecutive trapping times agree within tol_ps
    (heom.py:422-446; same return value, same ConvergenceFailure message).

    With ``speculate`` the run of tier n + 2 starts on the GPU while tiers n and
    n + 1 are compared (each run is its own handle and stream; small hierarchies
    leave most SMs idle, so the two overlap).  The result is the same as the
    serial search: the speculative run is only used when the search reaches it,
    and an error it raised surfaces only then.  A speculative run still in
    flight when the search stops is waited for (a device run is not cancelled).
    """
    if tol_ps <= 0:
        raise ValueError("tolerance must be > 0")
    n = 0 if bath.lam_cm1 == 0 else max(0, start_n)

    def run(k):
        return propagate(system, bath, rates, replace(config, n_max=k), initial_site)

    if not speculate:
        prev = run(n)
        prev_t = trapping_time(prev)
        while n < n_cap:
            cur = run(n + 1)
            cur_t = trapping_time(cur)
            if abs(cur_t - prev_t) <= tol_ps:
                return n, prev
            n += 1
            prev, prev_t = cur, cur_t
        raise ConvergenceFailure(f"trapping time not converged to {tol_ps} ps by n_max = {n_cap}")

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=2) as pool:
        fut = {n: pool.submit(run, n)}
        if n < n_cap:
            fut[n + 1] = pool.submit(run, n + 1)
        prev = fut.pop(n).result()
        prev_t = trapping_time(prev)
        while n < n_cap:
            if n + 2 <= n_cap and n + 2 not in fut:
                fut[n + 2] = pool.submit(run, n + 2)  # speculative
            cur = fut.pop(n + 1).result()
            cur_t = trapping_time(cur)
            if abs(cur_t - prev_t) <= tol_ps:
                return n, prev
            n += 1
            prev, prev_t = cur, cur_t
    raise ConvergenceFailure(f"trapping time not converged to {tol_ps} ps by n_max = {n_cap}")
