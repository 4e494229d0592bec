"""Level-2 kernel ABI: the reference's compiled kernels (_kernels.py:23-84) with
the same signatures, executed on the GPU through libheomb200.so.

These exist so code written against ``excitonflow._kernels`` (including the
reference's own tests, by monkeypatching) runs on the B200 kernels.  Each call
copies its host arrays to the device and back; the propagator itself never uses
this path (it keeps the state resident, heom.py -> engine.DeviceRun).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

DEVICE = 0


def _c128(a, name):
    if a.dtype != np.complex128 or not a.flags.c_contiguous:
        raise ValueError(f"{name} must be a C-contiguous complex128 array")
    return a


def hierarchy_rhs_kernel(out, sig, h, site_of, plus, minus, nvec, tier_damp, a_comm, b_anti,
                         decay):
    """out[k] = d sigma_k / dt for every ADO (_kernels.py:23-58)."""
    N.require_device(DEVICE)
    _c128(out, "out")
    _c128(sig, "sig")
    n_tot, d, _ = sig.shape
    modes = plus.shape[1]
    h = np.ascontiguousarray(h, dtype=np.float64)
    site_of = np.ascontiguousarray(site_of, dtype=np.int32)
    plus = np.ascontiguousarray(plus, dtype=np.int32)
    minus = np.ascontiguousarray(minus, dtype=np.int32)
    nvec = np.ascontiguousarray(nvec, dtype=np.float64)
    tier_damp = np.ascontiguousarray(tier_damp, dtype=np.float64)
    decay = np.ascontiguousarray(decay, dtype=np.float64)
    rc = N.lib().hb_rhs(N.ptr(out), N.ptr(sig), n_tot, d, N.ptr(h), N.ptr(site_of), N.ptr(plus),
                        N.ptr(minus), modes, N.ptr(nvec), N.ptr(tier_damp), float(a_comm),
                        float(b_anti), N.ptr(decay), DEVICE)
    N.check(rc, "hb_rhs")


def add_scaled(out, x, y, c):
    """out = x + c*y over flat complex arrays (_kernels.py:61-65)."""
    N.require_device(DEVICE)
    for a, nm in ((out, "out"), (x, "x"), (y, "y")):
        _c128(a, nm)
    N.check(N.lib().hb_add_scaled(N.ptr(out), N.ptr(x), N.ptr(y), float(c), out.size, DEVICE),
            "hb_add_scaled")


def rk4_update(sig, k1, k2, k3, k4, w):
    """sig += w*(k1 + 2*(k2 + k3) + k4) (_kernels.py:68-72)."""
    N.require_device(DEVICE)
    for a, nm in ((sig, "sig"), (k1, "k1"), (k2, "k2"), (k3, "k3"), (k4, "k4")):
        _c128(a, nm)
    N.check(N.lib().hb_rk4_update(N.ptr(sig), N.ptr(k1), N.ptr(k2), N.ptr(k3), N.ptr(k4),
                                  float(w), sig.size, DEVICE), "hb_rk4_update")


def max_abs2(x) -> float:
    """max |x_i|^2 over a flat complex array (_kernels.py:75-84)."""
    N.require_device(DEVICE)
    x = _c128(np.ascontiguousarray(x), "x")
    r = C.c_double()
    N.check(N.lib().hb_max_abs2(N.ptr(x), x.size, C.byref(r), DEVICE), "hb_max_abs2")
    return r.value
