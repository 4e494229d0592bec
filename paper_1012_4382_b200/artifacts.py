"""Run artifacts of the propagation path: the `#`-headed
CSV the reference CLI writes (cli.py:396-415) with the effective configuration
as `key = value` lines (cli.py:210-219), and the trajectory table of its
`propagate` command (cli.py:287-293).

The CLI itself (argument parsing, config files, the sweep commands) stays out
of scope; what is kept is the artifact contract: the same header schema
(``RunHeader`` mirrors the fields, defaults and value formatting of
cli.RunConfig, cli.py:44-100 and :146-155), the same column layout and the same
cell formatting (repr of floats, cli.py:399-402), so files written here read like
the reference's and reruns are byte-stable (test_cli.py:89-94).
"""

from __future__ import annotations

import io
from dataclasses import dataclass, fields
from typing import Optional

import numpy as np

from . import __version__
from .heom import PropagationConfig, auto_truncate, propagate
from .model import BathParams, MarkovRates, build_fmo_system


@dataclass(frozen=True)
class RunHeader:
    """The effective configuration recorded in an artifact (cli.py:44-73)."""

    solver: str = "heom"
    lambda_cm1: float = 35.0
    gamma_inv_fs: float = 166.0
    temperature_k: float = 300.0
    gamma_rc_inv_ps: float = 2.5
    gamma_phot_inv_ps: float = 250.0
    site: int = 1
    delta_e_cm1: float = 0.0
    e_rc_cm1: float = 0.0
    add_reorg_to_diagonal: bool = False
    dt_fs: float = 2.5
    n_max: Optional[int] = 8
    auto_tol_ps: float = 0.02
    n_cap: int = 20
    t_end_fs: Optional[float] = None
    residual: Optional[float] = 1e-5
    hard_cap_ps: float = 200.0
    record_stride: int = 1
    precision: str = "double"
    therm_t_end_ps: float = 30.0
    workers: int = 1
    lambdas: Optional[tuple] = None
    sites: Optional[tuple] = None
    delta_e_list: Optional[tuple] = None
    temperatures: Optional[tuple] = None
    n_max_list: Optional[tuple] = None
    steps: int = 1000


_FLOAT, _INT, _BOOL, _STR = "float", "int", "bool", "str"
_OPT_FLOAT, _N_MAX = "opt_float", "n_max"
_FLOATS, _INTS = "float_list", "int_list"
_KINDS = {
    "solver": _STR, "lambda_cm1": _FLOAT, "gamma_inv_fs": _FLOAT, "temperature_k": _FLOAT,
    "gamma_rc_inv_ps": _FLOAT, "gamma_phot_inv_ps": _FLOAT, "site": _INT, "delta_e_cm1": _FLOAT,
    "e_rc_cm1": _FLOAT, "add_reorg_to_diagonal": _BOOL, "dt_fs": _FLOAT, "n_max": _N_MAX,
    "auto_tol_ps": _FLOAT, "n_cap": _INT, "t_end_fs": _OPT_FLOAT, "residual": _OPT_FLOAT,
    "hard_cap_ps": _FLOAT, "record_stride": _INT, "precision": _STR, "therm_t_end_ps": _FLOAT,
    "workers": _INT, "lambdas": _FLOATS, "sites": _INTS, "delta_e_list": _FLOATS,
    "temperatures": _FLOATS, "n_max_list": _INTS, "steps": _INT,
}


def _format_value(kind: str, value) -> str:
    """cli.py:146-155"""
    if value is None:
        return "auto" if kind == _N_MAX else "none"
    if kind == _BOOL:
        return "true" if value else "false"
    if kind in (_FLOATS, _INTS):
        return ",".join(repr(v) if kind == _FLOATS else str(v) for v in value)
    if kind in (_FLOAT, _OPT_FLOAT):
        return repr(float(value))
    return str(value)


def emit_config(cfg: RunHeader) -> list:
    """Canonical ``key = value`` lines, unset sweep lists omitted (cli.py:210-219)."""
    lines = [f"version = {__version__}"]
    for f in fields(RunHeader):
        kind = _KINDS[f.name]
        value = getattr(cfg, f.name)
        if value is None and kind in (_FLOATS, _INTS):
            continue
        lines.append(f"{f.name} = {_format_value(kind, value)}")
    return lines


def _format_cell(x) -> str:
    """cli.py:399-402"""
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    return repr(float(x))


def write_csv(command: str, cfg: RunHeader, cols, rows, stream) -> None:
    """cli.py:405-411"""
    stream.write(f"# excitonflow {command}\n")
    for line in emit_config(cfg):
        stream.write(f"# {line}\n")
    stream.write(",".join(cols) + "\n")
    for row in rows:
        stream.write(",".join(_format_cell(x) for x in row) + "\n")


PROPAGATE_COLS = ["t_fs", "p_ground"] + [f"p_site{m}" for m in range(1, 8)] + ["p_RC", "trace"]


def propagate_rows(traj):
    """The `propagate` table of a trajectory (cli.py:287-293)."""
    rows = []
    for i, t in enumerate(traj.times_fs):
        p = traj.populations[i]
        rows.append([t, p[0], *p[1:8], p[8], p.sum()])
    return PROPAGATE_COLS, rows


def run_propagate(cfg: RunHeader, device: int = 0):
    """The `propagate` command's run (cli.py:225-276 _objects/_run_point for the
    HEOM solver) on the device; returns (n_max used, trajectory)."""
    if cfg.solver not in ("heom", "both"):
        raise ValueError("only the HEOM solver is part of this propagator")
    system = build_fmo_system(delta_e_cm1=cfg.delta_e_cm1, e_rc_cm1=cfg.e_rc_cm1,
                              reorg_shift_cm1=cfg.lambda_cm1 if cfg.add_reorg_to_diagonal else 0.0)
    bath = BathParams.from_timescale(cfg.lambda_cm1, cfg.gamma_inv_fs, cfg.temperature_k)
    rates = MarkovRates.from_inverse_ps(cfg.gamma_rc_inv_ps, cfg.gamma_phot_inv_ps)
    pconf = PropagationConfig(dt_fs=cfg.dt_fs, n_max=cfg.n_max if cfg.n_max is not None else 0,
                              t_end_fs=cfg.t_end_fs, residual=cfg.residual,
                              hard_cap_fs=1000.0 * cfg.hard_cap_ps, record_stride=cfg.record_stride,
                              precision=cfg.precision, device=device)
    if cfg.n_max is None:
        return auto_truncate(system, bath, rates, pconf, cfg.site, tol_ps=cfg.auto_tol_ps,
                             n_cap=cfg.n_cap)
    return cfg.n_max, propagate(system, bath, rates, pconf, cfg.site)


def propagate_csv(cfg: RunHeader, device: int = 0) -> str:
    """The CSV text `excitonflow propagate` writes for this configuration."""
    _, traj = run_propagate(cfg, device)
    cols, rows = propagate_rows(traj)
    out = io.StringIO()
    write_csv("propagate", cfg, cols, rows, out)
    return out.getvalue()


def read_csv(text: str):
    """(header lines without '# ', columns, rows as float array)."""
    header, cols, rows = [], None, []
    for line in text.splitlines():
        if line.startswith("#"):
            header.append(line[2:] if line.startswith("# ") else line[1:])
        elif cols is None:
            cols = line.split(",")
        elif line:
            rows.append([float(x) for x in line.split(",")])
    return header, cols, np.array(rows)
