"""Run artifacts: the `#`-headed CSV of the reference CLI
(cli.py:396-415) with the effective config (cli.py:210-219) and the `propagate`
table (cli.py:287-293), against fixtures written by the reference itself
(tests/golden/cli_artifacts.json, make_golden.py --cli)."""
import io
import json

import numpy as np
import pytest

from paper_1012_4382_b200 import artifacts as A
from tests.conftest import GOLDEN


@pytest.fixture(scope="module")
def golden_cli():
    return json.loads((GOLDEN / "cli_artifacts.json").read_text())


@pytest.mark.parametrize("name", ["default", "auto", "sweep"])
def test_header_lines_match_reference(golden_cli, name):
    g = golden_cli["headers"][name]
    f = {k: (tuple(v) if isinstance(v, list) else v) for k, v in g["fields"].items()}
    assert A.emit_config(A.RunHeader(**f)) == g["lines"]


def _header_for(argv):
    """RunHeader of the golden runs' command lines (flags -> fields)."""
    kw = {}
    it = iter(argv[1:])
    for flag in it:
        val = next(it)
        key = flag[2:].replace("-", "_")
        kw[key] = None if val == "none" else (int(val) if key in ("n_max", "site", "record_stride")
                                              else float(val))
    return A.RunHeader(**kw)


def test_csv_writer_reproduces_reference_bytes(golden_cli):
    """the writer alone: the reference's own rows re-emitted byte for byte"""
    for name, g in golden_cli["runs"].items():
        header, cols, rows = A.read_csv(g["csv"])
        out = io.StringIO()
        A.write_csv("propagate", _header_for(g["argv"]), cols,
                    [[r[0], *r[1:]] for r in rows.tolist()], out)
        assert out.getvalue() == g["csv"], name


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["n2_t200", "site6_lam55"])
def test_propagate_csv_matches_reference(golden_cli, name):
    """the same run on the device: identical header and columns, every cell
    within 1e-10 of the reference, byte-stable reruns (test_cli.py:89-94)"""
    g = golden_cli["runs"][name]
    cfg = _header_for(g["argv"])
    text = A.propagate_csv(cfg)
    assert text == A.propagate_csv(cfg)                # byte-stable rerun
    h, cols, rows = A.read_csv(text)
    h_ref, cols_ref, rows_ref = A.read_csv(g["csv"])
    assert h == h_ref and cols == cols_ref
    assert rows.shape == rows_ref.shape
    assert np.max(np.abs(rows - rows_ref)) < 1e-10
