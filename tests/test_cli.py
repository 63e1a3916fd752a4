"""The CLI mirror of the reference's cli.py:
exit codes, CSV schema, suites.  CPU: parsing and usage errors, the control
suite; GPU: every suite, a bench row and a sweep file."""
from __future__ import annotations

import csv
import io
import json
from contextlib import redirect_stdout

import pytest

from paper_2604_07311_b200 import cli


def _run(argv):
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


def test_header_is_the_reference_schema():
    assert cli.CSV_HEADER == "op,n,tree,mc,kc,nc,mr,nr,ways,time_s,gflops,max_rel_err"


@pytest.mark.parametrize("argv", [
    ["bench", "--op", "cholesky", "--n", "64", "--repeats", "2"],
    ["sweep", "--op", "cholesky", "--n", "64", "--bs", ",", "--out", "/tmp/x.csv"],
    ["check", "nosuch"],
])
def test_usage_errors_exit_2(argv):
    rc, _ = _run(argv)
    assert rc == 2


def test_bad_tree_file_exits_2(tmp_path):
    bad = tmp_path / "t.json"
    bad.write_text(json.dumps({"op": "cholesky", "variant": "unblocked1", "bs": 8}))
    rc, _ = _run(["bench", "--op", "cholesky", "--n", "64", "--tree", str(bad)])
    assert rc == 2


def test_control_suite_passes_on_cpu():
    rc, out = _run(["check", "control"])
    assert rc == 0 and out.strip() == "PASS control"


def test_forced_failure_knob(monkeypatch):
    monkeypatch.setenv(cli.FAIL_KNOB, "control")
    rc, out = _run(["check", "control"])
    assert rc == 1 and out.startswith("FAIL control")


@pytest.mark.gpu
def test_all_suites_pass(cuda):
    rc, out = _run(["check"])
    assert rc == 0, out
    assert [ln.split()[0] for ln in out.strip().splitlines()] == ["PASS"] * len(cli._SUITES)


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["cholesky", "gemm", "lu", "qr", "ltlt"])
def test_bench_row(cuda, op):
    rc, out = _run(["bench", "--op", op, "--n", "300"])
    assert rc == 0
    rows = list(csv.reader(io.StringIO(out)))
    assert rows[0] == cli.CSV_HEADER.split(",")
    row = dict(zip(rows[0], rows[1]))
    assert row["op"] == op and row["n"] == "300" and float(row["gflops"]) > 0
    assert 0 <= float(row["max_rel_err"]) < 1e-13


@pytest.mark.gpu
def test_sweep_writes_every_tree(cuda, tmp_path):
    out = tmp_path / "s.csv"
    rc, msg = _run(["sweep", "--op", "cholesky", "--n", "200", "--variants", "1,3", "--bs", "32,64", "--out", str(out)])
    assert rc == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == cli.CSV_HEADER.split(",") and len(rows) == 1 + 2 * 2 * 3  # variants x bs x leaves
    assert all(float(r[-1]) < 1e-13 for r in rows[1:])
