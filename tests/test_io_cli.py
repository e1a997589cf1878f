"""Scenario I/O and the `swflood` CLI (SPEC.md [MODULE] scenario_io,
SPEC.md:436-466) on the CPU: ESRI ASCII parsing rules, error messages with
line numbers, exit codes.  Everything that steps runs in test_gpu_cli.py."""
import os
import subprocess

import pytest

from conftest import ROOT

CLI = os.path.join(ROOT, "paper_1705_00614_b200", "swflood")


@pytest.fixture(scope="module")
def cli():
    from paper_1705_00614_b200 import build
    build.build()
    assert os.path.exists(CLI)
    return CLI


def run(cli, *args):
    p = subprocess.run([cli, *args], capture_output=True, text=True, timeout=120)
    return p.returncode, p.stdout, p.stderr


def write(path, text):
    with open(path, "w") as f:
        f.write(text)
    return str(path)


def test_info_parses_the_spec_2x2_example(cli, tmp_path):
    # 2x2 grid 0 1 2 3, cellsize 50 -> nx=ny=2, h=50
    f = write(tmp_path / "t.asc", "ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 50\n0 1\n2 3\n")
    rc, out, err = run(cli, "info", f)
    assert rc == 0, err
    assert "2 x 2 cells, h = 50 m" in out
    assert "min 0 m, max 3 m, mean 1.5 m" in out


def test_ragged_row_is_an_error_naming_the_row(cli, tmp_path):
    # SPEC.md:442
    f = write(tmp_path / "t.asc", "ncols 3\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 5\n1 2 3\n4 5\n")
    rc, out, err = run(cli, "info", f)
    assert rc == 1
    assert "t.asc:7: data row 2 has 2 values, ncols=3" in err


def test_malformed_header_and_nodata(cli, tmp_path):
    f = write(tmp_path / "h.asc", "ncols 2\nnrows\nxllcorner 0\n")
    rc, _, err = run(cli, "info", f)
    assert rc == 1 and "h.asc:2: malformed header" in err
    # SPEC.md:443 NODATA -> impermeable high ground at +1e4 m
    f = write(tmp_path / "n.asc",
              "ncols 2\nnrows 1\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n-9999 2\n")
    rc, out, err = run(cli, "info", f)
    assert rc == 0, err
    assert "max 10000 m" in out and "NODATA cells 1" in out


def test_usage_errors_exit_1(cli, tmp_path):
    assert run(cli, "frobnicate", "x")[0] == 1
    assert run(cli, "validate", "no-such-case")[0] == 1
    rc, _, err = run(cli, "info", "x.asc", "--bogus")
    assert rc == 1 and "unknown flag --bogus" in err


def test_scenario_validation_errors(cli, tmp_path):
    # SPEC.md:450 hydrograph with decreasing timestamps -> rejected
    f = write(tmp_path / "s.cfg", "synthetic = dam 64 1\nduration = 10\n[source gate]\n"
                                  "cells = 1 1 2 2\nhydrograph = 0:1, 5:2, 3:4\n")
    rc, _, err = run(cli, "run", f)
    assert rc == 1 and "s.cfg:5: source.hydrograph: hydrograph times must be strictly increasing" in err
    f = write(tmp_path / "m.cfg", "duration = 10\n")
    rc, _, err = run(cli, "run", f)
    assert rc == 1 and "needs 'terrain" in err
    f = write(tmp_path / "k.cfg", "synthetic = dam 64 1\nduration = 10\n[params]\nwat = 1\n")
    rc, _, err = run(cli, "run", f)
    assert rc == 1 and "k.cfg:4: unknown key 'params.wat'" in err
