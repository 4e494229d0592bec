"""ctypes front-end of the CPU oracle (oracle/heom_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py as the checker or the timed
CPU baseline; the product package never imports it.

Besides loading the C restatement this module restates, in numpy, the host-side
operand preparation of the reference so the oracle is independent of the
product's own host code:

* ``block_operands``   heom.py:235-275 (_BlockPropagator.__init__) and
                       heom.py:121-134 (_loss_channels)
* ``bath_modes``       heom.py:168-172 (bath_coefficients) for K=0; for K>=1 the
                       Drude-Lorentz Matsubara expansion documented in DESIGN.md
                       (not in the reference: parity for K>=1 is unpinned)
* ``propagate_from``   heom.py:286-406 driving ``or_propagate``
Objects passed in only need the reference's attribute names (duck typing), so
either the reference's or the product's ExcitonSystem/BathParams/MarkovRates work.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libheom_oracle.so"

# units.py:13-19 (restated)
C_CM_PER_FS = 2.99792458e-5
ANGFREQ = 2.0 * math.pi * C_CM_PER_FS
KB = 0.695035

T_END, RESIDUAL, DIVERGED, HARDCAP, CAPACITY = 1, 2, 3, 4, 5
STOP_NAMES = {T_END: "t_end", RESIDUAL: "residual"}

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class _Ops(C.Structure):
    _fields_ = [("n_tot", C.c_int64), ("d", C.c_int), ("n_sites", C.c_int), ("kp1", C.c_int),
                ("h", C.c_void_p), ("site_of", C.c_void_p), ("decay", C.c_void_p),
                ("plus", C.c_void_p), ("minus", C.c_void_p), ("indices", C.c_void_p),
                ("nu", C.c_void_p), ("a", C.c_void_p), ("b", C.c_void_p)]


class _Run(C.Structure):
    _fields_ = [("dt", C.c_double), ("has_t_end", C.c_int), ("t_end", C.c_double),
                ("has_residual", C.c_int), ("residual", C.c_double), ("hard_cap", C.c_double),
                ("stride", C.c_int64), ("blowup_norm", C.c_double), ("n_sinks", C.c_int),
                ("sink_nterms", C.c_void_p), ("sink_rate", C.c_void_p), ("sink_pos", C.c_void_p),
                ("n_site_pos", C.c_int), ("site_pos", C.c_void_p), ("max_steps", C.c_int64)]


_lib = None


def build() -> Path:
    """Compile the oracle with its Makefile (gcc)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.or_hierarchy_size.restype = C.c_int64
        L.or_hierarchy_size.argtypes = [C.c_int, C.c_int]
        L.or_enumerate.restype = C.c_int
        L.or_enumerate.argtypes = [C.c_int, C.c_int, _i32p, _i32p, _i32p, _i32p]
        L.or_rhs.restype = None
        L.or_rhs.argtypes = [C.POINTER(_Ops), _f64p, _f64p]
        L.or_add_scaled.argtypes = [C.c_int64, _f64p, _f64p, _f64p, C.c_double]
        L.or_rk4_update.argtypes = [C.c_int64, _f64p, _f64p, _f64p, _f64p, _f64p, C.c_double]
        L.or_max_abs2.restype = C.c_double
        L.or_max_abs2.argtypes = [C.c_int64, _f64p]
        L.or_np_sum.restype = C.c_double
        L.or_np_sum.argtypes = [_f64p, C.c_int]
        L.or_propagate.restype = C.c_int
        L.or_propagate.argtypes = [C.POINTER(_Ops), C.POINTER(_Run), _f64p, _f64p, C.c_int64,
                                   _i64p, _f64p, _f64p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """OpenMP thread count of the oracle (the reference's prange analogue)."""
    os.environ["OMP_NUM_THREADS"] = str(n)
    try:
        C.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


# ---------------------------------------------------------------------------
# hierarchy (hierarchy.py:59-105)

def hierarchy_size(modes: int, n_max: int) -> int:
    return math.comb(modes + n_max, modes)


def enumerate_hierarchy(modes: int, n_max: int):
    """(indices, tiers, plus, minus) int32 in the reference order."""
    n_tot = hierarchy_size(modes, n_max)
    if modes < 1 or n_max < 0:
        raise ValueError("bad hierarchy parameters")
    if n_tot > np.iinfo(np.int32).max:
        raise ValueError(f"hierarchy with {n_tot} indices exceeds the supported index range")
    indices = np.zeros((n_tot, modes), np.int32)
    tiers = np.zeros(n_tot, np.int32)
    plus = np.zeros((n_tot, modes), np.int32)
    minus = np.zeros((n_tot, modes), np.int32)
    rc = lib().or_enumerate(modes, n_max, indices, tiers, plus, minus)
    if rc != 0:
        raise ValueError(f"or_enumerate failed ({rc})")
    return indices, tiers, plus, minus


# ---------------------------------------------------------------------------
# operands (heom.py:121-134, 168-172, 235-275)

def loss_channels(system, rates):
    ch = []
    if rates.gamma_phot_fs1 > 0:
        for idx in system.site_indices:
            ch.append((rates.gamma_phot_fs1, idx, system.ground_index))
    if rates.gamma_rc_fs1 > 0:
        for label in system.trap_sites:
            ch.append((rates.gamma_rc_fs1, system.site_indices[label - 1], system.rc_index))
    return ch


def block_operands(system, rates):
    h = np.asarray(system.h_cm1, dtype=float)
    sinks = [i for i in (system.ground_index, system.rc_index) if i is not None]
    block = [i for i in range(h.shape[0]) if i not in sinks]
    pos_of = {full: blk for blk, full in enumerate(block)}
    hb = h[np.ix_(block, block)].astype(float)
    hb -= np.mean(np.diag(hb)) * np.eye(len(block))
    hb = np.ascontiguousarray(hb * ANGFREQ)
    site_pos = np.array([pos_of[i] for i in system.site_indices], np.int32)
    site_of = np.full(len(block), -1, np.int32)
    for slot, p in enumerate(site_pos):
        site_of[p] = slot
    decay = np.zeros(len(block))
    terms = {s: [] for s in sinks}
    for rate, src, dst in loss_channels(system, rates):
        decay[pos_of[src]] += rate
        terms[dst].append((rate, pos_of[src]))
    return dict(block=block, sinks=sinks, h=hb, site_pos=site_pos, site_of=site_of,
                decay=decay, sink_terms=[terms[s] for s in sinks])


def bath_modes(bath, n_matsubara: int = 0):
    """Per Matsubara index k: (nu_k, a_k, b_k) in fs^-1 / fs^-2.

    K=0 is heom.py:168-172 verbatim (high-temperature a, b).  K>=1 uses the exact
    Drude-Lorentz expansion C(t) = sum_k c_k exp(-nu_k t) (all in rad/fs):
    nu_0 = gamma, c_0 = lam*gamma*(cot(gamma/(2 kT)) - i);
    nu_k = 2 pi k kT, c_k = 4 lam gamma kT nu_k / (nu_k^2 - gamma^2);
    theta_0 = i Re(c_0)[V,.] - Im(c_0){V,.};  theta_k = i c_k [V,.].
    """
    gamma = bath.gamma_fs1
    if n_matsubara == 0:
        a = 2.0 * bath.lam_cm1 * KB * bath.temperature_k * ANGFREQ ** 2
        b = bath.lam_cm1 * ANGFREQ * gamma
        return np.array([gamma]), np.array([a]), np.array([b])
    lam = bath.lam_cm1 * ANGFREQ
    kt = KB * bath.temperature_k * ANGFREQ
    nu = [gamma]
    a = [lam * gamma / math.tan(gamma / (2.0 * kt))]
    b = [lam * gamma]
    for k in range(1, n_matsubara + 1):
        nk = 2.0 * math.pi * k * kt
        nu.append(nk)
        a.append(4.0 * lam * gamma * kt * nk / (nk * nk - gamma * gamma))
        b.append(0.0)
    return np.array(nu), np.array(a), np.array(b)


class Problem:
    """All arrays the C oracle needs for one system/bath/rates/n_max/K."""

    def __init__(self, system, bath, rates, n_max, n_matsubara=0, modes_override=None):
        self.system = system
        ops = block_operands(system, rates)
        self.__dict__.update(ops)
        self.d = len(self.block)
        self.n_sites = len(system.site_indices)
        self.kp1 = n_matsubara + 1
        nu, a, b = modes_override if modes_override is not None else bath_modes(bath, n_matsubara)
        self.nu, self.a, self.b = (np.ascontiguousarray(x, dtype=np.float64) for x in (nu, a, b))
        self.modes = self.n_sites * self.kp1
        self.indices, self.tiers, self.plus, self.minus = enumerate_hierarchy(self.modes, n_max)
        self.n_tot = self.indices.shape[0]
        self.n_max = n_max
        self._ops = _Ops(self.n_tot, self.d, self.n_sites, self.kp1,
                         self.h.ctypes.data, self.site_of.ctypes.data, self.decay.ctypes.data,
                         self.plus.ctypes.data, self.minus.ctypes.data, self.indices.ctypes.data,
                         self.nu.ctypes.data, self.a.ctypes.data, self.b.ctypes.data)

    def rhs(self, sig: np.ndarray) -> np.ndarray:
        sig = np.ascontiguousarray(sig, dtype=np.complex128)
        assert sig.shape == (self.n_tot, self.d, self.d)
        out = np.empty_like(sig)
        lib().or_rhs(C.byref(self._ops), sig.view(np.float64).reshape(-1),
                     out.view(np.float64).reshape(-1))
        return out


def rhs_from_arrays(sig, h, site_of, plus, minus, nvec, n_sites, kp1, nu, a, b, decay):
    """hierarchy_rhs_kernel signature (_kernels.py:24-25) on explicit operands."""
    sig = np.ascontiguousarray(sig, dtype=np.complex128)
    n_tot, d, _ = sig.shape
    keep = [np.ascontiguousarray(x, dtype=t) for x, t in
            ((h, np.float64), (site_of, np.int32), (decay, np.float64), (plus, np.int32),
             (minus, np.int32), (nvec, np.int32), (nu, np.float64), (a, np.float64),
             (b, np.float64))]
    ops = _Ops(n_tot, d, n_sites, kp1, *[k.ctypes.data for k in keep])
    out = np.empty_like(sig)
    lib().or_rhs(C.byref(ops), sig.view(np.float64).reshape(-1), out.view(np.float64).reshape(-1))
    return out


def propagate_from(system, bath, rates, config, rho0, n_matsubara=None, problem=None,
                   max_records=None, init_state=None):
    """heom.py:286-406 on the C oracle.  Returns a dict shaped like Trajectory
    (times_fs, populations, final_rho, matrices, stop_reason) or raises
    RuntimeError('diverged' / 'hardcap' ...) carrying the reference message."""
    K = getattr(config, "n_matsubara", 0) if n_matsubara is None else n_matsubara
    pb = problem or Problem(system, bath, rates, config.n_max, K)
    d_full = system.h_cm1.shape[0]
    rho0 = np.asarray(rho0, dtype=complex)
    sig = np.zeros((pb.n_tot, pb.d, pb.d), np.complex128)
    sig[0] = rho0[np.ix_(pb.block, pb.block)]
    if init_state is not None:  # the whole hierarchy (reference order), auxiliaries included
        sig[...] = init_state
    sink_pops = np.array([float(rho0[s, s].real) for s in pb.sinks] or [0.0])
    nterms = np.array([len(t) for t in pb.sink_terms] or [0], np.int32)
    rate = np.array([r for t in pb.sink_terms for r, _ in t] or [0.0])
    pos = np.array([p for t in pb.sink_terms for _, p in t] or [0], np.int32)
    dt = config.dt_fs
    if config.t_end_fs is not None:
        max_steps = int(math.ceil(config.t_end_fs / dt)) + 2
    else:
        max_steps = int(math.ceil(config.hard_cap_fs / dt)) + 2
    cap = max_records or (max_steps // config.record_stride + 3)
    rec_step = np.zeros(cap, np.int64)
    rec_sig0 = np.zeros(cap * pb.d * pb.d * 2)
    rec_sinks = np.zeros(cap * max(1, len(pb.sinks)))
    run = _Run(dt, int(config.t_end_fs is not None), float(config.t_end_fs or 0.0),
               int(config.residual is not None), float(config.residual or 0.0),
               float(config.hard_cap_fs), int(config.record_stride), float(config.blowup_norm),
               len(pb.sinks), nterms.ctypes.data, rate.ctypes.data, pos.ctypes.data,
               len(pb.site_pos), pb.site_pos.ctypes.data, max_steps)
    n_rec = C.c_int64()
    n_steps = C.c_int64()
    code = lib().or_propagate(C.byref(pb._ops), C.byref(run), sig.view(np.float64).reshape(-1),
                              sink_pops, cap, rec_step, rec_sig0, rec_sinks,
                              C.byref(n_rec), C.byref(n_steps))
    if code == DIVERGED:
        raise RuntimeError(f"diverged: matrix norm exceeded {config.blowup_norm:g} at t = "
                           f"{n_steps.value * dt} fs")
    if code == HARDCAP:
        raise RuntimeError(f"hardcap: residual policy not reached within the "
                           f"{config.hard_cap_fs} fs cap")
    if code == CAPACITY:
        raise RuntimeError("oracle buffer capacity exceeded")
    nr = n_rec.value
    sig0 = rec_sig0[: nr * pb.d * pb.d * 2].view(np.complex128).reshape(nr, pb.d, pb.d)
    sinks = rec_sinks[: nr * max(1, len(pb.sinks))].reshape(nr, -1)
    times = np.array([int(s) * dt for s in rec_step[:nr]])
    pops = np.zeros((nr, d_full))
    mats = np.zeros((nr, d_full, d_full), complex)
    for blk, full in enumerate(pb.block):
        pops[:, full] = np.real(sig0[:, blk, blk])
    for si, s in enumerate(pb.sinks):
        pops[:, s] = sinks[:, si]
        mats[:, s, s] = sinks[:, si]
    mats[:, np.ix_(pb.block, pb.block)[0], np.ix_(pb.block, pb.block)[1]] = sig0
    return dict(times_fs=times, populations=pops, final_rho=mats[-1], matrices=mats,
                stop_reason=STOP_NAMES[code], n_steps=n_steps.value, n_tot=pb.n_tot,
                final_state=sig)
