"""Host mirror of the reference's _BlockPropagator + the device run handle.

``BlockOperands`` restates the operand preparation of heom.py:235-275
(sink detection, block Hamiltonian shifted by its mean diagonal and converted
to rad/fs, site slots, summed decay rates, sink integration terms in
``_loss_channels`` order heom.py:121-134) and adds the bath mode table
(``bath_modes``) that generalises heom.py:168-172 to K Matsubara terms.

``DeviceRun`` owns one ``hb_handle`` (csrc/hb_api.cu): device tables, state
buffers, control block, stream and CUDA graph.  All RK4 work happens on the GPU;
Python only packs operands, starts the run and unpacks records.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .units import ANGFREQ_RAD_FS, KB_CM1_PER_K


def loss_channels(system, rates):
    """(rate_fs1, src, dst) collapse channels, radiative first then trapping."""
    out = []
    if rates.gamma_phot_fs1 > 0:
        if system.ground_index is None:
            raise ValueError("radiative decay requires a ground state in the basis")
        out += [(rates.gamma_phot_fs1, i, system.ground_index) for i in system.site_indices]
    if rates.gamma_rc_fs1 > 0:
        if system.rc_index is None or not system.trap_sites:
            raise ValueError("trapping requires an RC state and trap sites")
        out += [(rates.gamma_rc_fs1, system.site_basis_index(lbl), system.rc_index)
                for lbl in system.trap_sites]
    return out


def bath_coefficients(bath):
    """(a, b) in fs^-2 of the high-temperature single exponential (heom.py:168-172)."""
    a = 2.0 * bath.lam_cm1 * KB_CM1_PER_K * bath.temperature_k * ANGFREQ_RAD_FS ** 2
    b = bath.lam_cm1 * ANGFREQ_RAD_FS * bath.gamma_fs1
    return a, b


def bath_modes(bath, n_matsubara: int = 0):
    """(nu_k, a_k, b_k), k = 0..K, of the Drude-Lorentz correlation function.

    theta_k = i a_k [P, .] + b_k {P, .}, damping n_k nu_k, raise +i[P, .].
    K = 0 reproduces the reference exactly (a = 2 lam kT, b = lam gamma, in rad/fs
    units).  K >= 1 (new; no reference counterpart):
    c_0 = lam gamma (cot(gamma/2kT) - i) -> a_0 = Re c_0, b_0 = lam gamma;
    nu_k = 2 pi k kT, c_k = 4 lam gamma kT nu_k / (nu_k^2 - gamma^2) -> a_k = c_k, b_k = 0.
    """
    if n_matsubara < 0:
        raise ValueError("n_matsubara must be >= 0")
    g = bath.gamma_fs1
    if n_matsubara == 0:
        a, b = bath_coefficients(bath)
        return np.array([g]), np.array([a]), np.array([b])
    lam = bath.lam_cm1 * ANGFREQ_RAD_FS
    kt = KB_CM1_PER_K * bath.temperature_k * ANGFREQ_RAD_FS
    nu, a, b = [g], [lam * g / math.tan(g / (2.0 * kt))], [lam * g]
    for k in range(1, n_matsubara + 1):
        vk = 2.0 * math.pi * k * kt
        nu.append(vk)
        a.append(4.0 * lam * g * kt * vk / (vk * vk - g * g))
        b.append(0.0)
    return np.array(nu), np.array(a), np.array(b)


class BlockOperands:
    """Operands of the block propagation (heom.py:235-275)."""

    def __init__(self, system, bath, rates, n_matsubara: int = 0, modes=None):
        h = system.h_cm1
        sinks = [i for i in (system.ground_index, system.rc_index) if i is not None]
        for s in sinks:
            if np.any(np.delete(h[s, :], s) != 0.0):
                raise ValueError("sink states must be decoupled in the Hamiltonian")
        self.sinks = sinks
        self.block = [i for i in range(system.dimension) if i not in sinks]
        pos = {full: k for k, full in enumerate(self.block)}
        hb = h[np.ix_(self.block, self.block)].astype(float)
        # uniform diagonal shift: invisible to the commutator (heom.py:252-254)
        hb -= np.mean(np.diag(hb)) * np.eye(len(self.block))
        self.h_block = np.ascontiguousarray(hb * ANGFREQ_RAD_FS)
        self.site_pos = np.array([pos[i] for i in system.site_indices], np.int32)
        self.site_of = np.full(len(self.block), -1, np.int32)
        self.site_of[self.site_pos] = np.arange(len(self.site_pos), dtype=np.int32)
        self.decay = np.zeros(len(self.block))
        terms = {s: [] for s in sinks}
        for rate, src, dst in loss_channels(system, rates):
            self.decay[pos[src]] += rate
            terms[dst].append((rate, pos[src]))
        self.sink_terms = [terms[s] for s in sinks]
        self.n_matsubara = n_matsubara
        self.nu, self.a, self.b = modes if modes is not None else bath_modes(bath, n_matsubara)
        self.d = len(self.block)
        self.n_sites = system.site_count
        self.d_full = system.dimension

    @property
    def modes(self) -> int:
        return self.n_sites * (self.n_matsubara + 1)


class DeviceRun:
    """One propagation on the GPU (wraps hb_create / hb_set_rho0 / hb_run)."""

    def __init__(self, ops: BlockOperands, n_max: int, dt_fs: float, t_end_fs=None,
                 residual=None, hard_cap_fs: float = 200_000.0, record_stride: int = 1,
                 record_matrices: bool = False, blowup_norm: float = 1e6, device: int = 0,
                 layout: str = "auto", ordering: str = "reference", chunk_steps: int = 0,
                 kernel: str = "auto", precision: str = "double", shard=None):
        N.require_device(device)
        if ops.d > 9:
            raise ValueError("block dimension above 9 is not supported by the device kernels")
        self.ops = ops
        self.dt = dt_fs
        self.record_matrices = record_matrices
        kp1 = ops.n_matsubara + 1
        f64 = lambda x: np.ascontiguousarray(x, dtype=np.float64)
        i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)
        keep = dict(
            h=f64(ops.h_block), site_of=i32(ops.site_of), decay=f64(ops.decay),
            nu=f64(ops.nu), a=f64(ops.a), b=f64(ops.b),
            sink_nterms=i32([len(t) for t in ops.sink_terms] or [0]),
            sink_rate=f64([r for t in ops.sink_terms for r, _ in t] or [0.0]),
            sink_pos=i32([p for t in ops.sink_terms for _, p in t] or [0]),
            site_pos=i32(ops.site_pos), block_full=i32(ops.block),
            sink_full=i32(ops.sinks or [0]))
        self._keep = keep
        p = N.HbParams()
        p.d, p.n_sites, p.kp1, p.n_max = ops.d, ops.n_sites, kp1, int(n_max)
        for k in ("h", "site_of", "decay", "nu", "a", "b", "sink_nterms", "sink_rate",
                  "sink_pos", "site_pos", "block_full", "sink_full"):
            setattr(p, k, keep[k].ctypes.data)
        p.n_sinks = len(ops.sinks)
        p.n_site_pos = len(ops.site_pos)
        p.d_full = ops.d_full
        p.dt = float(dt_fs)
        p.has_t_end = int(t_end_fs is not None)
        p.t_end = float(t_end_fs) if t_end_fs is not None else 0.0
        p.has_residual = int(residual is not None)
        p.residual = float(residual) if residual is not None else 0.0
        p.hard_cap = float(hard_cap_fs)
        p.record_stride = int(record_stride)
        p.record_matrices = int(bool(record_matrices))
        p.blowup_norm = float(blowup_norm)
        p.device = int(device)
        p.layout = N.HB_LAYOUT[layout]
        p.ordering = N.HB_ORDER[ordering]
        p.chunk_steps = int(chunk_steps)
        p.kernel_variant = N.HB_KERNEL[kernel]
        p.precision = N.HB_PREC[precision]
        self._params = p
        handle = C.c_void_p()
        if shard is None:
            N.check(N.lib().hb_create(C.byref(p), C.byref(handle)), "hb_create")
        else:  # one shard of a sharded run (shard.py ShardLayout): local tables
            groups = np.ascontiguousarray(np.concatenate(shard.groups) if len(shard.groups) else
                                          np.zeros(0), np.int32)
            t = N.HbShardTables()
            t.n_local, t.own_tiles, t.top_tile = shard.n_local, shard.own_tiles, shard.top_tile
            t.root = int(shard.root)
            keep.update(sp=np.ascontiguousarray(shard.plus, np.int32),
                        sm=np.ascontiguousarray(shard.minus, np.int32),
                        sn=np.ascontiguousarray(shard.nvec, np.uint8), sg=groups)
            t.plus, t.minus = keep["sp"].ctypes.data, keep["sm"].ctypes.data
            t.nvec, t.groups = keep["sn"].ctypes.data, keep["sg"].ctypes.data
            for g in range(4):
                t.group_count[g] = len(shard.groups[g])
            N.check(N.lib().hb_create_shard(C.byref(p), C.byref(t), C.byref(handle)),
                    "hb_create_shard")
        self._h = handle
        self.result = None

    def close(self):
        if getattr(self, "_h", None):
            N.lib().hb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_rho0(self, rho0_block: np.ndarray, sink_pops) -> None:
        r = np.ascontiguousarray(rho0_block, dtype=np.complex128)
        s = np.ascontiguousarray(list(sink_pops) or [0.0], dtype=np.float64)
        N.check(N.lib().hb_set_rho0(self._h, N.ptr(r), N.ptr(s)), "hb_set_rho0")

    def set_state(self, sig: np.ndarray, sink_pops) -> None:
        """Whole hierarchy state (n_tot, d, d) in the reference order (hb_set_state)."""
        r = np.ascontiguousarray(sig, dtype=np.complex128)
        s = np.ascontiguousarray(list(sink_pops) or [0.0], dtype=np.float64)
        N.check(N.lib().hb_set_state(self._h, N.ptr(r), N.ptr(s)), "hb_set_state")

    def run(self) -> int:
        """Returns the C status (HB_OK / HB_DIVERGED / HB_HARDCAP); others raise."""
        res = N.HbResult()
        rc = N.lib().hb_run(self._h, C.byref(res))
        self.result = res
        if rc not in (N.HB_OK, N.HB_DIVERGED, N.HB_HARDCAP):
            N.check(rc, "hb_run")
        return rc

    def records(self):
        n = int(N.lib().hb_record_count(self._h))
        df = self.ops.d_full
        steps = np.zeros(n, np.int64)
        pops = np.zeros((n, df))
        mats = np.zeros((n, df, df), np.complex128) if self.record_matrices else None
        N.check(N.lib().hb_get_records(self._h, N.ptr(steps), N.ptr(pops),
                                       N.ptr(mats) if mats is not None else None, n),
                "hb_get_records")
        return steps, pops, mats

    def sigma0(self):
        d = self.ops.d
        sig0 = np.zeros((d, d), np.complex128)
        sinks = np.zeros(max(1, len(self.ops.sinks)))
        N.check(N.lib().hb_get_sigma0(self._h, N.ptr(sig0), N.ptr(sinks)), "hb_get_sigma0")
        return sig0, sinks[: len(self.ops.sinks)]

    def state(self, n_tot: int):
        d = self.ops.d
        sig = np.zeros((n_tot, d, d), np.complex128)
        sinks = np.zeros(max(1, len(self.ops.sinks)))
        N.check(N.lib().hb_get_state(self._h, N.ptr(sig), N.ptr(sinks)), "hb_get_state")
        return sig, sinks[: len(self.ops.sinks)]

    def time_steps(self, n_steps: int, per_stage: bool = False):
        ms = C.c_double()
        stages = np.zeros(4) if per_stage else None
        N.check(N.lib().hb_time_steps(self._h, int(n_steps), C.byref(ms),
                                      N.ptr(stages) if per_stage else None), "hb_time_steps")
        return (ms.value, stages) if per_stage else ms.value

    def launch_count(self) -> int:
        return int(N.lib().hb_launch_count(self._h))
